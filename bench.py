"""bench.py -- full-graph PipeGCN training epochs/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config reddit]

One "step" = one full-graph iteration t of Alg. 1: forward of all L layers on
every partition with the boundary exchange, loss, backward with stale-gradient accumulation,
gradient all-reduce and the Adam update (Table 3) -- every row of SURVEY.md section 8(a).
Workload at N=1: BASELINE configs[1], the synthetic Reddit-shaped graph (232,965 nodes,
~114.6M CSR non-zeros, 602 features, 41 classes), 4-layer GraphSAGE hidden 256, 2 partitions
hosted on the one GPU exchanging through the LOOPBACK transport (the NCCL path's posted exchange:
pack -> comm stream -> one device copy per peer segment -> events), PIPE mode, dropout 0.5, Adam,
fp32 tier.  N > 1: one partition per GPU over NCCL; run outside torchrun, `--gpus N` launches the N
ranks itself and refuses (exit 3) when fewer than N GPUs are visible.
Timing: W untimed warm-up iterations, then K iterations bracketed by CUDA events on the context
stream (barrier + synchronize on both sides, max over ranks), no per-kernel instrumentation; a
second, instrumented pass gives the per-kernel breakdown and the roofline; inputs are far larger
than L2 (X alone 563 MB).
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full-graph epochs/s (max over ranks)"
EXIT_NOT_ENOUGH_GPUS = 3
UNIT = "epochs/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="reddit")
    ap.add_argument("--parts", type=int, default=0, help="partitions (default max(2, N))")
    ap.add_argument("--mode", default="pipe", choices=["pipe", "vanilla"])
    ap.add_argument("--smooth", default="", help="'', 'f', 'g' or 'gf'")
    ap.add_argument("--gemm", default="tc", choices=["tc", "simt", "bf16"])
    ap.add_argument("--gather", default="f32", choices=["f32", "bf16"],
                    help="bf16: the bf16 gather tier (SpMM tables rounded to bf16, 2e-2 tier; beyond SURVEY 8, not N1(iv))")
    ap.add_argument("--model", default="sage", choices=["sage", "gcn"],
                    help="GraphSAGE-mean (the paper's benchmark model) or GCN-sym (App. A.1, SURVEY N3)")
    ap.add_argument("--no-tiles", action="store_true",
                    help="gather-only aggregation (default: dense 128x64 tiles of P_i / P_i^T on the tensor cores "
                         "where they hold >= 25 %% of the edges; DESIGN.md 'Tensor-core tiles')")
    ap.add_argument("--tile-min", type=int, default=0, help="heavy-tile threshold in edges per 128x64 tile (0: library default)")
    ap.add_argument("--no-train-sparse", action="store_true",
                    help="compute the last layer on every row (default: only on train rows, SURVEY N1(ii); exact)")
    ap.add_argument("--transport", default="loopback", choices=["loopback", "local", "push"],
                    help="single-GPU runs: 'loopback' = the posted exchange of the NCCL path (pack -> comm stream "
                         "-> one device copy per peer segment -> events; App. F), 'local' = direct gathers, "
                         "'push' = producers store the exchanged rows into the receivers from their epilogues (N2); "
                         "N > 1 GPUs: NCCL, or with 'push' (PIPE, fp32 payloads) the epilogue stores go into the "
                         "peers' workspaces over NVLink (CUDA IPC)")
    ap.add_argument("--halo-payload", default="f32", choices=["f32", "bf16"],
                    help="bf16: exchange payloads rounded to bf16 (SURVEY N1(iv), 2e-2 tier)")
    ap.add_argument("--depth", type=int, default=1, help="pipeline depth s (R27)")
    ap.add_argument("--lean", action="store_true",
                    help="lean-memory mode (SURVEY N1(iii)): Z recomputed in the backward, shared Z / T scratches, "
                         "one slot for J and the feature messages; bit-identical results")
    ap.add_argument("--no-ablation", action="store_true", help="skip the no-communication timing ablation")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.path = os.path.join("/tmp", "pgcn_clocks_%d.csv" % os.getpid())

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        rows = []
        for line in open(self.path):
            c = [x.strip() for x in line.split(",")]
            if len(c) < 9:
                continue
            try:
                rows.append(dict(sm=float(c[1]), smax=float(c[2]), hw=c[5], hwt=c[6], swt=c[7], pcap=c[8]))
            except ValueError:
                pass
        if not rows:
            return None
        sms = sorted(r["sm"] for r in rows)
        reasons = set()
        for r in rows:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"), ("swt", "sw_thermal_slowdown"),
                            ("pcap", "sw_power_cap")):
                if r[k].lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": rows[0]["smax"], "reasons": sorted(reasons),
                "samples": len(rows)}


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
                "_fallback": True}


def max_over_ranks(x, dist):
    """Device-timed milliseconds -> the max over ranks (the slowest rank sets the epoch time)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def exchange_microbench(dist, view, widths, reps=10):
    """SURVEY 8(d) all-to-all evidence for N > 1: the halo exchange of this partition at each distinct
    layer-input width, as the grouped point-to-point send/recv the library posts (every peer j gets the
    rows S_{rank,j}; this rank receives its boundary segments), fp32 rows padded to ld = round_up(F, 4).
    Timed with CUDA events (NCCL) or the wall clock (gloo), max over ranks.  busBW = bytes sent per rank
    / time x (n - 1) / n, the all-to-all convention, against 900 GB/s per direction of NVLink 5."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    nccl = dist.get_backend() == "nccl"
    dev = "cuda" if nccl else "cpu"
    out = []
    for F in sorted(set(widths[:-1])):
        ld = (F + 3) // 4 * 4
        sends, recvs = {}, {}
        for j in range(world):
            if j == rank:
                continue
            ns = int(view["send_off"][j + 1] - view["send_off"][j])
            nr = int(view["halo_off"][j + 1] - view["halo_off"][j])
            sends[j] = torch.ones((ns, ld), device=dev)
            recvs[j] = torch.empty((nr, ld), device=dev)

        def once():
            ops = [dist.P2POp(dist.isend, sends[j], j) for j in sends] + [dist.P2POp(dist.irecv, recvs[j], j)
                                                                           for j in recvs]
            for r in dist.batch_isend_irecv(ops) if ops else []:
                r.wait()
        once()
        if nccl:
            torch.cuda.synchronize()
        dist.barrier()
        if nccl:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                once()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
        else:
            t0 = time.perf_counter()
            for _ in range(reps):
                once()
            ms = 1000.0 * (time.perf_counter() - t0) / reps
        ms = max_over_ranks(ms, dist)
        sent = sum(x.numel() * 4 for x in sends.values())
        sent_max = max_over_ranks(float(sent), dist)
        alg = sent_max / (ms / 1e3) / 1e9 if ms > 0 else None
        out.append({"F": F, "bytes_sent_max_rank": int(sent_max), "ms": ms, "algbw_GBps": alg,
                    "busbw_GBps": alg * (world - 1) / world if alg else None, "nvlink_GBps_per_dir": 900.0})
    return out


def build_workload(name, n_parts, model="sage"):
    import dataclasses

    from synth.graphs import CONFIGS, gen_graph, glorot_params, model_for
    t0 = time.time()
    g = gen_graph(name, seed=1)
    m = dataclasses.replace(model_for(name), model=model)
    params0 = glorot_params(m.widths, 3, model=model)
    return g, m, params0, time.time() - t0


class RankGraph:
    """The slice of a huge synthetic graph one rank materialises (papers100M-shaped multi-GPU runs): the
    full CSR structure is generated (and partitioned) on every rank, but X, labels and the train mask only
    for the rank's own rows (synth.graphs.rows_inputs, counter-based per row); n_train is the global count
    (all-reduced)."""

    def __init__(self, n, nnz, X, labels, train_mask, n_train):
        self.n, self.nnz, self.X, self.labels, self.train_mask, self._n_train = n, nnz, X, labels, train_mask, n_train

    @property
    def n_train(self):
        return self._n_train


def build_rank_workload(name, parts, rank, dist, pgcn, model="sage", n=None, nnz=None):
    """Per-rank workload of a huge config: structure + partition on every rank, inputs of the rank's rows
    only.  Returns (RankGraph, model cfg, params0, partitioning, seconds).  Host memory per rank: the CSR
    (7.3 GB at papers100M) + the partition arrays + this rank's X rows."""
    import dataclasses

    import numpy as np
    from synth.graphs import CONFIGS, gen_structure, glorot_params, model_for, rows_inputs
    t0 = time.time()
    row_ptr, col = gen_structure(name, seed=1, n=n, nnz=nnz)
    n, nnz = len(row_ptr) - 1, int(row_ptr[-1])
    part = pgcn.partition(n, row_ptr, col, parts)
    del row_ptr, col
    gid = part.view(rank)["inner_gid"]
    X, lab, tm = rows_inputs(name, gid, n=n)
    cnt = np.array([int(tm.sum())], dtype=np.int64)
    if dist is not None:
        import torch
        tt = torch.from_numpy(cnt).to("cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt)
        cnt = tt.cpu().numpy()
    m = dataclasses.replace(model_for(name), model=model)
    params0 = glorot_params(m.widths, 3, model=model)
    return RankGraph(n, nnz, X, lab, tm, int(cnt[0])), m, params0, part, time.time() - t0


SHARDED_N = 50_000_000  # configs above this many nodes build per-rank inputs (build_rank_workload)


def cpu_baseline(name, parts, mode, smooth, sample_n=16000, iters=5, model="sage"):
    """The oracle (oracle/, numpy/scipy fp64) as it stands, on a bounded sample of the same workload:
    the same generator recipe, degree, widths, dropout and partition count at N = sample_n, timed
    for `iters` PipeGCN iterations; per-epoch time extrapolated linearly in N (every term of the
    epoch -- SpMM nnz*F and GEMM N*F*F' -- is linear in N at fixed degree)."""
    from oracle import pipegcn
    from oracle.partition import partition as opart
    from synth.graphs import CONFIGS, gen_graph, glorot_params, model_for
    c = CONFIGS[name]
    deg = c["nnz"] / c["n"]
    g = gen_graph(name, seed=1, n=sample_n, nnz=int(sample_n * deg))
    import dataclasses
    m = dataclasses.replace(model_for(name), model=model)
    params0 = glorot_params(m.widths, 3, model=model)
    parts_o = opart(g.n, g.row_ptr, g.col_idx, parts)
    t0 = time.time()
    pipegcn.run(g, parts_o, params0, m, iters, mode=mode, smooth_f="f" in smooth, smooth_g="g" in smooth)
    dt = (time.time() - t0) / iters
    scale = c["n"] / sample_n
    epoch_s = dt * scale
    cores = len(os.sched_getaffinity(0))
    return {"value": 1.0 / epoch_s, "unit": UNIT, "cores": cores, "kind": "oracle", "extrapolated": True,
            "extrapolation": "measured s/iteration on the N=%d sample x N_full/N_sample = %.1f (every epoch term is "
                             "linear in N at fixed degree and widths)" % (sample_n, c["n"] / sample_n),
            "sample": "oracle PipeGCN (%s, %s) %d iterations on a %s-recipe graph with N=%d (nnz=%d, same degree, "
                      "widths, dropout, %d partitions); %.2f s/iteration x N_full/N_sample=%.1f" % (
                          mode, model, iters, name, sample_n, g.nnz, parts, dt, scale)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    parts = args.parts or max(2, args.gpus)
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(args.config, parts, args.mode, args.smooth, iters=1, model=args.model)
    info = None
    t0 = time.time()
    for _ in range(args.steps):
        info = cpu_baseline(args.config, parts, args.mode, args.smooth, iters=1, model=args.model)
        vals.append(1.0 / info["value"])
    wall = time.time() - t0
    ms = 1000.0 * sum(vals) / len(vals)
    v = 1000.0 / ms
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "%s-synthetic, %d partitions, %s%s" % (
               args.config, parts, args.mode, "" if args.model == "sage" else ", GCN-sym")},
           "cpu_baseline": dict(info, value=v),
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "wall_s": wall}
    print(json.dumps(out))


def spawn_ranks(args):
    """`--gpus N` (N > 1) outside torchrun: launch N ranks (one partition per GPU, NCCL) with
    torch.distributed.run on 127.0.0.1.  Refuses (exit 3, one JSON line) when fewer than N GPUs are
    visible -- a multi-GPU number is never produced by a single GPU."""
    import socket

    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(json.dumps({"metric": METRIC, "error": "--gpus %d needs %d visible GPUs, found %d" % (args.gpus, args.gpus, n),
                          "n_gpus": args.gpus, "n_gpus_visible": n}))
        sys.exit(EXIT_NOT_ENOUGH_GPUS)
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % args.gpus,
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def roofline(name, kd, pk, args, l2_peak):
    """Roofline object of the dominant kernel.  Per launch: achieved = algorithmic
    bytes (or flops) / mean launch duration, both measured live with CUDA events on the context
    stream during the instrumented pass.
      spmm_*  bound hbm: B_min (gathered table read once -- the compulsory traffic) over the measured
              HBM copy peak; beside it the per-edge B_gather model over the live L2 read peak.
      gemm_*  bound tensor: tensor-pipe flops executed (3xTF32 = 3 tf32 MMAs per fp32 product; bf16:
              1) over the dense peak of that dtype (MEASURED bf16 x nominal tf32/bf16 ratio 1/2).
      other   bound hbm: algorithmic bytes over the HBM copy peak."""
    n = max(kd["launches"], 1)
    sec = kd["ms"] / 1e3 / n
    roof = {"kernel": name, "launches_timed": kd["launches"], "ms_per_launch": kd["ms"] / n}
    tr = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(args.config, {}).get(name)
    except Exception:
        pass
    if name.startswith("gemm"):
        mult = 1.0 if args.gemm == "bf16" else 3.0
        peak = pk["bf16_tflops"] * (1.0 if args.gemm == "bf16" else 0.5)
        ach = mult * kd["flops"] / n / sec / 1e12
        roof.update(bound="tensor", achieved=ach, peak=peak, unit="TFLOP/s", frac=ach / peak,
                    peak_source="MEASURED_PEAKS.json bf16_tflops%s" % ("" if args.gemm == "bf16" else " x 1/2 (tf32)"),
                    traffic=tr, flops_per_launch=kd["flops"] / n, tensor_flop_multiplier=mult)
        return roof
    ach = kd["bytes"] / n / sec / 1e9
    roof.update(bound="hbm", achieved=ach, peak=pk["hbm_gbs"], unit="GB/s", frac=ach / pk["hbm_gbs"],
                peak_source="MEASURED_PEAKS.json hbm_gbs", traffic=tr, bytes_per_launch=kd["bytes"] / n)
    if name.startswith("spmm"):
        g = kd["gather_bytes"] / n / sec / 1e9
        roof["B_min_per_launch"] = kd["bytes"] / n
        roof["B_gather_per_launch"] = kd["gather_bytes"] / n
        roof["gather_view"] = {"achieved": g, "unit": "GB/s", "hbm_frac": g / pk["hbm_gbs"],
                               "l2_peak": l2_peak, "l2_frac": (g / l2_peak) if l2_peak else None,
                               "note": "per-edge model B_gather (a table row per edge); > HBM means L2/L1-served "
                                       "or on-chip reuse (tensor-core tiles)"}
        if tr:
            roof["dram_view"] = {"achieved": tr / sec / 1e9, "frac": tr / sec / 1e9 / pk["hbm_gbs"],
                                 "note": "ncu DRAM bytes per launch (profiles/) over this run's launch time"}
    return roof


def kernel_functions(kern):
    """Engine timing buckets -> the kernel functions that run in them (the contract's roofline is for the
    dominant *kernel*; a bucket can hold several):
      k_umma_gemm   the three node-update GEMM buckets (fwd / dW / dA; plus their tiny operand-prep and
                    column-sum launches), flops = fp32 products x 2;
      k_spmm_tc     the tile sub-intervals of both aggregation directions (bf16 split + tcgen05 tile MMA),
                    flops = MMA flops executed (0/1 tiles x 64 table rows, zeros included);
      k_spmm_fwd / k_spmm_bwd  the aggregation buckets minus their tile sub-intervals (the gather kernels:
                    light edges + epilogue on the tile path, the whole aggregation off it);
      the other buckets are one kernel each."""
    z = {"ms": 0.0, "launches": 0, "bytes": 0.0, "flops": 0.0, "gather_bytes": 0.0}
    g = lambda k: kern.get(k, z)  # noqa: E731
    out = {}
    gem = [g("gemm_fwd"), g("gemm_dw"), g("gemm_da")]
    out["k_umma_gemm"] = {k: sum(x[k] for x in gem) for k in z}
    tf, tb = g("spmm_tile_fwd"), g("spmm_tile_bwd")
    out["k_spmm_tc"] = {k: tf[k] + tb[k] for k in z}
    for d, t in (("spmm_fwd", tf), ("spmm_bwd", tb)):
        b = g(d)
        out["k_" + d] = dict(b, ms=b["ms"] - t["ms"], tile_path=t["launches"] > 0)
    for k in ("dropout", "gather", "grad_reduce", "loss", "update"):
        out["k_" + k] = dict(g(k))
    return {k: v for k, v in out.items() if v["launches"]}


def kernel_roofline(name, kd, pk, args, kern, l2p):
    """Roofline object of a kernel function (kernel_functions), per launch: achieved = algorithmic flops
    (tensor kernels) or bytes (the rest) / mean launch duration, measured live with CUDA events."""
    n = max(kd["launches"], 1)
    sec = kd["ms"] / 1e3 / n
    if name == "k_umma_gemm":
        # the binding roof at these GEMMs' arithmetic intensity (narrow layers sit below the
        # ridge): tensor if AI x HBM >= the dtype's tensor peak, else HBM with the algorithmic operand bytes
        mult = 1.0 if args.gemm == "bf16" else 3.0
        peak = pk["bf16_tflops"] * (1.0 if args.gemm == "bf16" else 0.5)
        ach = mult * kd["flops"] / n / sec / 1e12
        ai = mult * kd["flops"] / kd["bytes"] if kd["bytes"] > 0 else float("inf")
        common = {"kernel": name, "launches_timed": kd["launches"], "ms_per_launch": kd["ms"] / n, "traffic": None,
                  "flops_per_launch": kd["flops"] / n, "bytes_per_launch": kd["bytes"] / n,
                  "tensor_flop_multiplier": mult, "ai_flop_per_byte": ai,
                  "ridge_flop_per_byte": peak * 1e12 / (pk["hbm_gbs"] * 1e9),
                  "tensor": {"achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                             "peak_source": "MEASURED_PEAKS.json bf16_tflops%s" % (
                                 "" if args.gemm == "bf16" else " x 1/2 (tf32)")},
                  "note": "all node-update GEMM launches (fwd, dW, dA); flops = fp32 products x 2 x the tensor MMAs "
                          "per product; bytes = operand reads + output writes (algorithmic)"}
        if ai * pk["hbm_gbs"] * 1e9 >= peak * 1e12:
            return dict(common, bound="tensor", achieved=ach, peak=peak, unit="TFLOP/s", frac=ach / peak,
                        peak_source=common["tensor"]["peak_source"])
        gbs = kd["bytes"] / n / sec / 1e9
        return dict(common, bound="hbm", achieved=gbs, peak=pk["hbm_gbs"], unit="GB/s", frac=gbs / pk["hbm_gbs"],
                    peak_source="MEASURED_PEAKS.json hbm_gbs (AI below the tensor ridge)")
    if name == "k_spmm_tc":
        peak = pk["bf16_tflops"]
        ach = kd["flops"] / n / sec / 1e12
        return {"kernel": name, "launches_timed": kd["launches"], "ms_per_launch": kd["ms"] / n, "bound": "tensor",
                "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (kind::f16)", "traffic": None,
                "flops_per_launch": kd["flops"] / n, "tma_bytes_per_launch": kd["bytes"] / n,
                "note": "tile part of the aggregation (bf16 split + tcgen05 0/1-tile MMA, hi and lo tables in the "
                        "fp32 tier); flops = MMAs executed, zeros of the 0/1 tiles included"}
    bucket = name[2:]
    r = roofline(bucket, kern[bucket] if bucket in kern else kd, pk, args, l2p)
    r.update(kernel=name, launches_timed=kd["launches"], ms_per_launch=kd["ms"] / n)
    if bucket in kern and kd["ms"] > 0:  # achieved over this kernel's own time (the tile part is subtracted)
        r["achieved"] = kern[bucket]["bytes"] / n / sec / 1e9
        r["frac"] = r["achieved"] / r["peak"]
    return r


def l2_read_peak(pgcn, torch, stream):
    """Live L2 streaming-read bandwidth (64 MB buffer, resident in the 126 MB L2): the ceiling of
    L2-served gathers, reported beside the HBM roofline."""
    L = pgcn.lib()
    s = stream.cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nbytes = 64 << 20
    buf = torch.ones(nbytes // 4, device="cuda")
    out = torch.empty(148 * 8, device="cuda")
    reps, best = 50, 0.0
    for variant in (0, 1, 2):
        with torch.cuda.stream(stream):
            L.pgcn_dev_l2_read(buf.data_ptr(), nbytes, (variant << 24) | 2, out.data_ptr(), s)
            e0.record(stream)
            L.pgcn_dev_l2_read(buf.data_ptr(), nbytes, (variant << 24) | reps, out.data_ptr(), s)
            e1.record(stream)
        torch.cuda.synchronize()
        best = max(best, nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    import numpy as np
    import torch

    from paper_2203_10428_b200 import pgcn

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit("WORLD_SIZE=%d but --gpus %d" % (world, args.gpus))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = local_rank
    torch.cuda.set_device(dev)
    # N = 1: the configuration's partitions hosted on one GPU (loopback or local transport); N > 1: one
    # partition per GPU (NCCL transport), n_parts = N.
    parts = args.parts or (max(2, args.gpus) if world == 1 else world)
    if world > 1 and parts != world:
        raise SystemExit("multi-GPU runs host one partition per rank (--parts must equal WORLD_SIZE)")
    from synth.graphs import CONFIGS
    sharded = world > 1 and CONFIGS[args.config]["n"] > SHARDED_N
    if sharded:  # papers100M-shaped: every rank materialises only its own rows' inputs
        g, m, params0, part, t_gen = build_rank_workload(args.config, parts, rank, dist, pgcn, args.model)
        t_part = 0.0
    else:
        g, m, params0, t_gen = build_workload(args.config, parts, args.model)
        t0 = time.time()
        part = pgcn.partition(g.n, g.row_ptr, g.col_idx, parts)
        t_part = time.time() - t0
    transport = args.transport if world == 1 else ("nccl+push" if args.transport == "push" else "nccl")
    cfg = pgcn.make_config(m.widths, mode=args.mode, smooth_f="f" in args.smooth, smooth_g="g" in args.smooth,
                           gamma=m.gamma, dropout=m.dropout, loss=m.loss, opt="adam", lr=m.lr, n_global=g.n,
                           n_train_global=g.n_train, gemm=args.gemm, model=args.model, gather=args.gather,
                           train_sparse=not args.no_train_sparse, spmm_tiles=not args.no_tiles,
                           tile_min=args.tile_min, depth=args.depth,
                           transport=transport if transport in ("loopback", "push") else
                           ("push" if transport == "nccl+push" else "local"),
                           halo_payload=args.halo_payload, lean=args.lean)
    local_parts = list(range(parts)) if world == 1 else [rank]
    transport_note = None
    # Fit the workspace to this GPU: the posted exchange's message buffers must fit next to the activations,
    # else the local transport (no message buffers) hosts the partitions; a layout that still does not fit
    # runs in the lean-memory mode (N1(iii): same results, needs a posted transport -- NCCL, or loopback on
    # one GPU).  The line says which (config.transport_note).
    def fits(c):
        return pgcn.workspace_bytes(part, c, local_parts) <= torch.cuda.mem_get_info()[0] - (2 << 30)
    if not fits(cfg):
        need = pgcn.workspace_bytes(part, cfg, local_parts)
        if args.lean:
            raise SystemExit("bench: lean layout needs %.1f GB of workspace, %.1f GB free" % (
                need / 1e9, torch.cuda.mem_get_info()[0] / 1e9))
        if transport in ("loopback", "push"):
            cfg.transport = 0
            if fits(cfg):
                transport_note = "%s needs %.1f GB of workspace: local transport" % (transport, need / 1e9)
                transport = "local"
            else:
                cfg.transport = 1 if transport == "loopback" else 2
        if transport != "local":
            cfg.lean = 1
            if not fits(cfg):
                raise SystemExit("bench: even the lean layout needs %.1f GB of workspace" % (
                    pgcn.workspace_bytes(part, cfg, local_parts) / 1e9))
            args.lean = True
            transport_note = "default layout needs %.1f GB of workspace: lean-memory mode" % (need / 1e9)
    stream = torch.cuda.Stream()
    comm = pgcn.nccl_comm(rank, world) if world > 1 else None
    with torch.cuda.stream(stream):
        ctx = pgcn.Context(part, cfg, local_parts=local_parts, comm=comm, stream=stream)
    if transport == "nccl+push" and args.mode == "pipe" and args.halo_payload == "f32":
        ctx.ipc_connect()  # N2 over NVLink: producers store exchanged rows into the peers' workspaces
    views = [part.view(i) for i in local_parts]
    host = []
    for i, v in enumerate(views):
        gid = v["inner_gid"]
        if sharded:  # the rank's rows, already in V_i order
            X, lab, tm = (torch.from_numpy(a).pin_memory() for a in (g.X, g.labels, g.train_mask))
        else:
            X = torch.from_numpy(np.ascontiguousarray(g.X[gid])).pin_memory()
            lab = torch.from_numpy(np.ascontiguousarray(g.labels[gid])).pin_memory()
            tm = torch.from_numpy(np.ascontiguousarray(g.train_mask[gid])).pin_memory()
        host.append((X, lab, tm))
    nloc = len(local_parts)
    for i in range(nloc):  # one partition at a time: the device staging copy is freed right after
        d_in = tuple(a.cuda(non_blocking=True) for a in host[i])
        torch.cuda.synchronize()  # the H2D copies (current stream) land before the context stream reads them
        ctx.set_inputs(i, *d_in)
        torch.cuda.synchronize()
        del d_in
    torch.cuda.empty_cache()
    theta = torch.tensor(pgcn.flatten_params(params0), device="cuda")
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    t = 0
    W, K = max(args.warmup, 3), args.steps
    with torch.cuda.stream(stream):
        for _ in range(W):
            t += 1
            ctx.step(t, theta, grads, opt, loss)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(K)]

    def timed(k_steps, per_step_ms=None):
        """k_steps iterations bracketed by CUDA events on the context stream (barrier + synchronize on
        both sides); returns the max over ranks of the elapsed milliseconds.  per_step_ms (optional
        list) receives this rank's per-iteration durations (an event after every step)."""
        nonlocal t
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()
        ev0.record(stream)
        for k in range(k_steps):
            t += 1
            ctx.step(t, theta, grads, opt, loss)
            if per_step_ms is not None:
                step_ev[k].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        if per_step_ms is not None:
            prev = ev0
            for k in range(k_steps):
                per_step_ms.append(prev.elapsed_time(step_ev[k]))
                prev = step_ev[k]
        return max_over_ranks(ev0.elapsed_time(ev1), dist)

    # (1) headline: K iterations, no instrumentation
    clocks = Clocks(dev)
    clocks.start()
    launches0 = ctx.launch_count()
    xb0 = ctx.exchange_bytes()
    step_ms = []
    ms_total = timed(K, step_ms)
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    xb1 = ctx.exchange_bytes()
    ms = ms_total / K
    value = 1000.0 / ms
    loss_v = float(loss.item())
    if not (loss_v > 0.0 and loss_v == loss_v):  # every partition has train rows: the loss is positive
        raise SystemExit("bench: loss %r after the timed steps -- inputs not installed?" % loss_v)
    # (2) instrumented pass: per-kernel CUDA events on the context stream (roofline, breakdown)
    ctx.timing_enable(True)
    ms_instr = timed(K) / K
    kern = {name: ctx.timing_read(k) for k, name in enumerate(pgcn.KERNELS)}
    ctx.timing_enable(False)

    # (3) end to end through the C ABI with HOST buffers: every iteration's X, labels and train mask
    # are copied from pinned host memory by pgcn_stage_inputs (library copy stream, overlapped with the
    # iteration in flight), and each iteration's loss is read back to the host.
    e2e = None
    if args.config.startswith("papers"):
        args.no_e2e = True  # 14 GB of inputs per step over PCIe: no end-to-end leg for the papers shape
    if not args.no_e2e:
        loss_h = torch.zeros(1).pin_memory()
        ld0 = (m.widths[0] + 3) // 4 * 4  # host X kept in the library's padded row layout: one copy per step
        host = [(torch.nn.functional.pad(X, (0, ld0 - X.shape[1])).pin_memory(), lab, tm) for X, lab, tm in host]
        h2d = sum(sum(a.numel() * a.element_size() for a in h) for h in host)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0 = time.perf_counter()
        ev0.record(stream)
        for i in range(nloc):
            ctx.stage_inputs(i, *host[i])
        for k in range(K):
            t += 1
            ctx.step(t, theta, grads, opt, loss)
            if k + 1 < K:
                for i in range(nloc):
                    ctx.stage_inputs(i, *host[i])
            with torch.cuda.stream(stream):
                loss_h.copy_(loss, non_blocking=True)
            stream.synchronize()
            _ = float(loss_h.item())
        ev1.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(ev0.elapsed_time(ev1), dist) / K
        e2e = {"value": 1000.0 / e_ms, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4,
               "ms_per_step": e_ms, "host_wall_ms_per_step": 1000.0 * (time.perf_counter() - e0) / K,
               "note": "pgcn_stage_inputs(host pinned X, labels, train mask) every iteration (library copy "
                       "stream, overlapped with the iteration in flight) + pgcn_step + loss read back each step"}

    # (3b) N > 1: the exchange alone at each layer width (grouped send / recv, busBW)
    comm_bench = exchange_microbench(dist, views[0], m.widths) if dist is not None else None

    # (4) exposed communication: the same iterations with the transfers skipped (PGCN_XH_NOCOMM;
    # timing only -- the halo state is stale afterwards).  exposed = T - T_nocomm.
    comm_info = None
    if transport != "local":
        comm_info = {"transport": transport, "payload": args.halo_payload,
                     "bytes_per_step": {"fwd": (xb1[0] - xb0[0]) / K, "bwd": (xb1[1] - xb0[1]) / K}}
        if not args.no_ablation:
            ctx.exchange_hook(0, pgcn.XH_NOCOMM)
            ms_nc = timed(K) / K
            ctx.exchange_hook(0, 0)
            comm_info.update(ms_per_step_nocomm=ms_nc, exposed_ms_per_step=ms - ms_nc)

    pk = peaks()
    kf = kernel_functions(kern)
    buckets = {k: v for k, v in kern.items() if v["launches"] and not k.startswith("spmm_tile")}
    agg = [k for k in ("spmm_fwd", "spmm_bwd") if k in buckets]
    l2p = l2_read_peak(pgcn, torch, stream) if agg else None
    # (a) the dominant kernel function (contract: the roofline of the dominant kernel)
    name, kd = max(kf.items(), key=lambda kv: kv[1]["ms"])
    roof = kernel_roofline(name, kd, pk, args, kern, l2p)
    roof["share_of_step"] = kd["ms"] / (ms_instr * K)
    # (b) the aggregation as a whole (the method's SpMM): the larger bucket, B_min over HBM with
    # the per-edge (L2) and ncu-DRAM views
    roof_agg = None
    if agg:
        an = max(agg, key=lambda k: kern[k]["ms"])
        roof_agg = roofline(an, kern[an], pk, args, l2p)
        roof_agg["share_of_step"] = kern[an]["ms"] / (ms_instr * K)
    breakdown = {k: {"ms_per_step": v["ms"] / K, "share": v["ms"] / (ms_instr * K),
                     "GBps": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None,
                     "TFLOPs": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] > 0 and v["flops"] else None}
                 for k, v in buckets.items()}
    kernels = {k: {"ms_per_step": v["ms"] / K, "share": v["ms"] / (ms_instr * K), "launches_per_step": v["launches"] / K,
                   "TFLOPs": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] > 0 and v["flops"] else None}
               for k, v in kf.items()}
    cpu = None
    if not args.no_cpu and world == 1:
        try:
            cpu = cpu_baseline(args.config, parts, args.mode, args.smooth, model=args.model)
        except Exception as e:  # noqa: BLE001
            cpu = {"error": str(e)}
    if rank != 0:
        return
    tier = {("f32", "tc"): "fp32 tier: 3xTF32 tensor-core GEMMs, fp32 gathers, 2xbf16-split tile aggregation"
                           if not args.no_tiles else "fp32 tier: 3xTF32 tensor-core GEMMs, IEEE fp32 gathers",
            ("f32", "simt"): "IEEE fp32 (SIMT GEMMs, fp32 gathers)%s" % ("" if args.no_tiles else ", 2xbf16 tiles"),
            ("f32", "bf16"): "bf16 tensor-core GEMMs, fp32 gathers (2e-2 tier)",
            ("bf16", "tc"): "3xTF32 GEMMs, bf16 gathers (2e-2 tier)",
            ("bf16", "bf16"): "bf16 tensor-core GEMMs and gathers (2e-2 tier)",
            ("bf16", "simt"): "SIMT GEMMs, bf16 gathers (2e-2 tier)"}[(args.gather, args.gemm)]
    dtype = "f32" if (args.gather, args.gemm, args.halo_payload) == ("f32", "tc", "f32") or args.gemm == "simt" else "bf16"
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
           "precision": tier + ("" if args.halo_payload == "f32" else "; bf16 exchange payloads"),
           "data": "synthetic",
           "config": {"workload": "%s-synthetic N=%d nnz=%d F=%s, %d partitions on %d GPU(s), %s%s, "
                                  "dropout %.1f, Adam%s" % (args.config, g.n, g.nnz, m.widths, parts, world, args.mode,
                                                            ("-" + args.smooth.upper()) if args.smooth else "",
                                                            m.dropout, "" if args.model == "sage" else ", GCN-sym"),
                      "global_batch": g.n,
                      "parallelism": ("partition x%d on one GPU (%s transport)" % (parts, transport)) if world == 1 else
                      ("partition x%d, one per GPU: %s + all-reduce" % (
                          world, "halo rows stored into the peers' workspaces by the producing epilogues (N2, NVLink)"
                          if transport == "nccl+push" else "NCCL p2p halo exchange on a comm stream")),
                      "gemm": args.gemm, "gather": args.gather, "depth": args.depth, "transport": transport,
                      "lean": bool(args.lean),
                      "transport_note": transport_note,
                      "train_sparse_last_layer": not args.no_train_sparse, "spmm_tiles": not args.no_tiles,
                      "l2": "inputs larger than L2 (X %.0f MB, CSR %.0f MB)" % (g.X.nbytes / 1e6, g.nnz * 8 / 1e6)},
           "roofline": roof, "roofline_aggregation": roof_agg, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
           "comm": comm_info, "comm_bench": comm_bench, "step_ms": [round(x, 3) for x in step_ms], "breakdown": breakdown, "ms_per_step_instrumented": ms_instr, "loss": loss_v,
           "setup_s": {"generate": t_gen, "partition": t_part, "per_rank_inputs": sharded},
           "workspace_GB": ctx.ws.numel() / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
