"""Summaries of an ncu launch list (--csv --log-file, metrics gpu__time_duration.sum, dram__bytes_read.sum,
dram__bytes_write.sum, lts__t_bytes.sum, optional sm__pipe_tensor_cycles_active...).

    python tools/r2/ncu_summary.py LAUNCHES.csv STEP_LAUNCHES [--traffic CONFIG]

Takes the last STEP_LAUNCHES launches (one bench step), prints a markdown table per kernel (launches,
total ms, share, DRAM / L2 GB per launch, achieved DRAM GB/s) and per bench bucket (the kernels one
engine call launches: spmm_fwd = [k_to_bf16 | k_split_bf16 + k_spmm_tc] + k_spmm_fwd*, spmm_bwd likewise
with k_spmm_bwd*).  --traffic CONFIG merges the buckets' DRAM bytes per call into profiles/traffic.json
under CONFIG (the bench's roofline "traffic")."""
import collections
import csv
import json
import os
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launch = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launch.setdefault(r[ii], {"k": r[ki]})
        try:
            d[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    return list(launch.values())


def short(k):
    k = k.split("(")[0].replace("void ", "")
    for p in ("pgcn::<unnamed>::", "pgcn::", "tcs::", "tc::"):
        k = k.replace(p, "")
    return k


def main():
    L = load(sys.argv[1])
    n = int(sys.argv[2])
    L = L[-n:]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    dram = collections.defaultdict(float)
    l2 = collections.defaultdict(float)
    tens = collections.defaultdict(list)
    for d in L:
        k = short(d["k"])
        tot[k] += d.get("gpu__time_duration.sum", 0.0)
        cnt[k] += 1
        dram[k] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        l2[k] += d.get("lts__t_bytes.sum", 0)
        t = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
        if t is not None:
            tens[k].append(t)
    T = sum(tot.values())
    print("| kernel | launches | ms | share | DRAM GB/launch | L2 GB/launch | DRAM GB/s | tensor pipe % |")
    print("|---|---|---|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        c = cnt[k]
        tp = ("%.1f" % (sum(tens[k]) / len(tens[k]))) if tens[k] else ""
        print("| %s | %d | %.3f | %.1f%% | %.3f | %.3f | %.0f | %s |" % (
            k[:48], c, v / 1e6, 100 * v / T, dram[k] / c / 1e9, l2[k] / c / 1e9, dram[k] / (v / 1e9) / 1e9 if v else 0, tp))
    # buckets: consecutive launches ending in a gather SpMM
    buckets = collections.defaultdict(lambda: [0, 0.0, 0.0])
    pend = []
    for d in L:
        k = short(d["k"])
        if k.startswith(("k_to_bf16", "k_split_bf16", "k_spmm_tc")):
            pend.append(d)
            continue
        if k.startswith(("k_spmm_fwd", "k_spmm_bwd")):
            name = "spmm_fwd" if k.startswith("k_spmm_fwd") else "spmm_bwd"
            grp = pend + [d]
            b = buckets[name]
            b[0] += 1
            b[1] += sum(x.get("gpu__time_duration.sum", 0) for x in grp)
            b[2] += sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0) for x in grp)
        pend = []
    print()
    print("| bucket (one engine call) | calls | ms/call | DRAM GB/call | DRAM GB/s |")
    print("|---|---|---|---|---|")
    for name, (c, ms, by) in sorted(buckets.items()):
        print("| %s | %d | %.3f | %.3f | %.0f |" % (name, c, ms / c / 1e6, by / c / 1e9, by / (ms / 1e9) / 1e9))
    if "--traffic" in sys.argv:
        cfg = sys.argv[sys.argv.index("--traffic") + 1]
        path = os.path.join(os.path.dirname(__file__), "..", "..", "profiles", "traffic.json")
        try:
            tr = json.load(open(path))
        except Exception:
            tr = {}
        if not isinstance(tr.get(cfg), dict):
            tr = {k: v for k, v in tr.items() if isinstance(v, dict)}
        tr[cfg] = {name: by / c for name, (c, ms, by) in buckets.items()}
        tr["_source"] = ("ncu launch lists (dram__bytes_read.sum + dram__bytes_write.sum), DRAM bytes per engine "
                         "call summed over the kernels of the call, one bench step (tools/r2/ncu_summary.py)")
        json.dump(tr, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
