"""SpMM design lab (diagnostics): times tools/spmm_lab.cu variants on the Reddit-shaped partition and
on synthetic gathers that isolate the L2 (table fits in L2) and DRAM (uniform over a large table)
ceilings.  Prints algorithmic gather GB/s = 4 * ld * nnz / time.

    python tools/spmm_lab.py
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

SO = os.path.join(ROOT, "tools", "libspmm_lab.so")


def build():
    src = os.path.join(ROOT, "tools", "spmm_lab.cu")
    if not os.path.exists(SO) or os.path.getmtime(SO) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                               "-Xcompiler", "-fPIC", src, "-o", SO])
    lib = ctypes.CDLL(SO)
    lib.lab_spmm.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 4 + [ctypes.c_int64, ctypes.c_int64,
                                                                      ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    return lib


def timeit(fn, reps=5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    lib = build()
    from paper_2203_10428_b200 import pgcn
    from synth.graphs import gen_graph
    g = gen_graph("reddit", seed=1)
    part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 2)
    v = part.view(0)
    n_in, n_all = v["n_inner"], v["n_inner"] + v["n_halo"]
    cases = {"reddit-p0": (v["row_ptr"], v["col_idx"], n_all)}
    rng = np.random.default_rng(0)
    nnz = v["nnz"]
    deg = np.diff(v["row_ptr"])
    cases["L2-table(30k rows)"] = (v["row_ptr"], rng.integers(0, 30000, nnz).astype(np.int32), 30000)
    cases["uniform(n_all)"] = (v["row_ptr"], rng.integers(0, n_all, nnz).astype(np.int32), n_all)
    st = torch.cuda.current_stream().cuda_stream
    inv = torch.tensor((1.0 / np.maximum(deg, 1)).astype(np.float32)).cuda()
    for ld in (604, 256, 44):
        D = torch.randn(n_all, ld, device="cuda")
        Z = torch.empty(n_in, ld, device="cuda")
        ref = None
        for name, (rp, col, nrows_tab) in cases.items():
            rp_t = torch.tensor(rp).cuda()
            col_t = torch.tensor(col).cuda()
            res = []
            for var in range(14):
                for gm in (64,):
                    fn = lambda: lib.lab_spmm(var, rp_t.data_ptr(), col_t.data_ptr(), inv.data_ptr(), D.data_ptr(), ld,
                                              n_in, Z.data_ptr(), gm, st)
                    if fn() != 0:
                        continue
                    ms = timeit(fn)
                    if var == 0:
                        ref = Z.clone()
                    else:
                        assert torch.equal(ref, Z), ("variant result differs", var)
                    res.append((var, gm, ms, 4.0 * ld * nnz / ms / 1e6))
            best = max(res, key=lambda r: r[3])
            print(f"ld={ld:4d} {name:20s} " + " ".join(f"v{r[0]}:{r[3]:6.0f}" for r in res) +
                  f"   best v{best[0]} {best[2]:.2f} ms {best[3]:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
