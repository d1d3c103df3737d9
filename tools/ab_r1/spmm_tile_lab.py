"""Tile-reuse SpMM lab (diagnostics): builds the 128-row x 64-column heavy-tile split of the
Reddit-shaped partition in numpy and times tools/spmm_tile_lab.cu (L1 vs shared-memory staging)
against the product kernel (pgcn_dev_spmm) at width 256; checks the results agree."""
import ctypes
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

R, C = 128, 64


def build_lib():
    src = os.path.join(ROOT, "tools", "spmm_tile_lab.cu")
    so = os.path.join(ROOT, "tools", "libspmm_tile_lab.so")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-shared",
                               "-Xcompiler", "-fPIC", src, "-o", so])
    L = ctypes.CDLL(so)
    L.lab_tiled.argtypes = [ctypes.c_int] + [ctypes.c_void_p] * 8 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                                                      ctypes.c_void_p, ctypes.c_void_p]
    return L


def tiles(rp, col, n_rows, tau):
    deg = np.diff(rp)
    rows = np.repeat(np.arange(n_rows, dtype=np.int64), deg)
    blk = rows // R
    ct = col.astype(np.int64) // C
    key = blk * (1 << 24) + ct
    uk, inv_k, cnt = np.unique(key, return_inverse=True, return_counts=True)
    heavy_e = cnt[inv_k] >= tau
    # heavy edges ordered by (block, tile, row); stable keeps CSR order inside a row
    hidx = np.nonzero(heavy_e)[0]
    order = hidx[np.lexsort((rows[hidx], key[hidx]))]
    hk = key[order]
    tk, tstart = np.unique(hk, return_index=True)
    n_t = tk.size
    tile_blk = tk >> 24
    tile_col0 = ((tk & ((1 << 24) - 1)) * C).astype(np.int32)
    blk_tile_ptr = np.searchsorted(tile_blk, np.arange((n_rows + R - 1) // R + 1)).astype(np.int32)
    tend = np.append(tstart[1:], order.size)
    tile_off = np.zeros((n_t, R + 1), np.int32)
    hrows = rows[order] % R
    for i in range(n_t):  # per-tile row offsets
        r = hrows[tstart[i]:tend[i]]
        tile_off[i, 1:] = np.cumsum(np.bincount(r, minlength=R))
        tile_off[i] += tstart[i]
    tile_colv = (col[order] - tile_col0[np.repeat(np.arange(n_t), tend - tstart)]).astype(np.uint8)
    lidx = np.nonzero(~heavy_e)[0]
    light_col = col[lidx].astype(np.int32)
    light_ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(rows[lidx], minlength=n_rows), out=light_ptr[1:])
    return blk_tile_ptr, tile_col0, tile_off.ravel(), tile_colv, light_ptr, light_col, heavy_e.mean(), n_t


def main():
    L = build_lib()
    from paper_2203_10428_b200 import pgcn
    from synth.graphs import gen_graph
    g = gen_graph("reddit", seed=1)
    part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 2)
    for which in ("fwd P_i", "bwd P_i^T"):
        v = part.view(0)
        if which.startswith("fwd"):
            rp, col, n_rows, n_cols = v["row_ptr"], v["col_idx"], v["n_inner"], v["n_inner"] + v["n_halo"]
        else:
            rp, col, n_rows, n_cols = v["t_row_ptr"], v["t_col_idx"], v["n_inner"] + v["n_halo"], v["n_inner"]
        t0 = time.time()
        tb = tiles(rp, col, n_rows, 32)
        print("%s: tiling %.1fs, heavy-edge fraction %.3f, %d tiles" % (which, time.time() - t0, tb[6], tb[7]),
              flush=True)
        dev = [torch.tensor(x).cuda() for x in tb[:6]]
        D = torch.randn(n_cols, 256, device="cuda")
        inv = torch.rand(n_rows, device="cuda")
        Z = torch.zeros(n_rows, 256, device="cuda")
        Zr = torch.zeros(n_rows, 256, device="cuda")
        work = torch.zeros(1, dtype=torch.int64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        rp_t, col_t = torch.tensor(rp).cuda(), torch.tensor(col).cuda()
        ref = lambda: pgcn.lib().pgcn_dev_spmm(rp_t.data_ptr(), col_t.data_ptr(), inv.data_ptr(), D.data_ptr(), 256,
                                               n_rows, n_cols, Zr.data_ptr(), st)
        nnz = int(rp[-1])
        for name, fn in [("product", ref)] + [("tiled-mode%d" % m, (lambda m=m: L.lab_tiled(
                m, *[x.data_ptr() for x in dev], inv.data_ptr(), D.data_ptr(), n_rows, n_cols, Z.data_ptr(),
                work.data_ptr(), st))) for m in (0, 1)]:
            for _ in range(2):
                assert fn() == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            err = (Z - Zr).abs().max().item() / Zr.abs().max().item() if name != "product" else 0.0
            print("  %-12s %7.3f ms  %6.0f GB/s algorithmic  rel.err %.1e" % (name, ms, 1024.0 * nnz / ms / 1e6, err),
                  flush=True)


if __name__ == "__main__":
    main()
