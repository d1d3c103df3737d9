"""Distils gpurun_out/ ncu outputs into committed summaries under profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py <tag> <launches.csv> <report.ncu-rep> [<report.ncu-rep> ...]

Writes profiles/<tag>_launches.md (per-kernel share of one step from the launch list),
profiles/<tag>_kernels.md (selected full-set metrics per captured launch) and updates
profiles/traffic.json (DRAM bytes per launch per kernel kind, consumed by bench.py).
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = [("k_spmm_tc", "spmm_tc"), ("k_split_bf16", "split_bf16"), ("k_to_bf16", "to_bf16"), ("k_spmm_fwd", "spmm_fwd"), ("k_spmm_bwd", "spmm_bwd"), ("k_umma_gemm", "gemm_tc"), ("k_gemm_fwd", "gemm_fwd"),
        ("k_gemm_dw", "gemm_dw"), ("k_gemm_da", "gemm_da"), ("k_dropout", "dropout"), ("k_gather", "gather"),
        ("k_grad_reduce", "grad_reduce"), ("k_loss", "loss"), ("k_opt", "update"), ("k_sum_grads", "update"),
        ("k_wprep", "wprep"), ("k_colsum", "colsum"), ("k_split_reduce", "split_reduce"), ("k_reduce_sum", "reduce_sum")]
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "s": 1e3}


def kind_of(name):
    for k, v in KIND:
        if k in name:
            return v
    return name[:40]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = kind_of(d["Kernel Name"])
        try:
            val = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        except ValueError:
            continue
        agg[k][d["Metric Name"]] += val
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
    return agg, cnt


def scope_traffic(path):
    """DRAM bytes per aggregation *scope* (what bench.py times as spmm_fwd / spmm_bwd): the table
    rounding / split and tensor-core tile launches that precede a gather launch belong to it."""
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        e = per.setdefault(d["ID"], [kind_of(d["Kernel Name"]), 0.0])
        try:
            e[1] += float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        except ValueError:
            pass
    pending, tot, n = 0.0, collections.defaultdict(float), collections.Counter()
    for kind, b in per.values():
        if kind in ("spmm_tc", "split_bf16", "to_bf16"):
            pending += b
        elif kind in ("spmm_fwd", "spmm_bwd"):
            tot[kind] += b + pending
            n[kind] += 1
            pending = 0.0
    return {k: tot[k] / n[k] for k in tot}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[m] = float(r[i].replace(",", "")) * (SCALE.get(units[i], 1.0) if "bytes" in m or "duration" in m else 1.0)
                except ValueError:
                    d[m] = r[i]
        res.append(d)
    return res


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    if not reps:
        reps = []
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    agg, cnt = launches(lcsv)
    # one step = launches of the last (timed) step; ncu saw warm-up + timed steps: report shares
    tot = sum(v.get("gpu__time_duration.sum", 0.0) for v in agg.values())
    lines = ["# %s: launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_*; --clock-control none)" % tag, "",
             "Cold-cache, serialised per-launch times of every kernel in the command (warm-up + timed steps):",
             "compare SHARES with bench.py's live breakdown, not absolutes.", "",
             "| kernel | launches | total ms | share | DRAM GB/launch |", "|---|---|---|---|---|"]
    traffic = {}
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", 0)):
        ms = v.get("gpu__time_duration.sum", 0.0)
        dram = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / max(cnt[k], 1)
        traffic[k] = dram
        lines.append("| %s | %d | %.3f | %.1f%% | %.3f |" % (k, cnt[k], ms, 100 * ms / tot, dram / 1e9))
    open(os.path.join(ROOT, "profiles", "%s_launches.md" % tag), "w").write("\n".join(lines) + "\n")
    klines = ["# %s: ncu --set full (selected metrics per captured launch)" % tag, ""]
    for rep in reps:
        res = raw(rep)
        klines.append("## %s" % os.path.basename(rep))
        klines.append("")
        for d in res:
            name = re.sub(r"\(.*", "", d.pop("kernel"))[-60:]
            klines.append("- `%s`: " % name + ", ".join(
                "%s=%s" % (m.split(".")[0].replace("__", ":"), ("%.4g" % d[m]) if isinstance(d[m], float) else d[m])
                for m in METRICS if m in d))
        klines.append("")
    open(os.path.join(ROOT, "profiles", "%s_kernels.md" % tag), "w").write("\n".join(klines) + "\n")
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    cur = json.load(open(tpath)) if os.path.exists(tpath) else {}
    cur.update({k: v for k, v in traffic.items()})
    cur.update(scope_traffic(lcsv))  # spmm_fwd / spmm_bwd: whole aggregation scope (tile path incl.)
    cur["_source"] = "%s: ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over launches)" % tag
    json.dump(cur, open(tpath, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
