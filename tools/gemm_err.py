"""Prints the relative error of each node-update GEMM variant against float64 (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2203_10428_b200 import pgcn as P

def ld(f): return (f + 3) // 4 * 4
def rel(a, b): return np.abs(a - b).max() / np.abs(b).max()
for (M, F, N) in [(2000, 300, 512), (100000, 256, 256), (100000, 602, 256)]:
    rng = np.random.default_rng(0)
    A0 = np.zeros((M, ld(F)), np.float32); A0[:, :F] = rng.standard_normal((M, F))
    A1 = np.zeros((M, ld(F)), np.float32); A1[:, :F] = np.maximum(rng.standard_normal((M, F)), 0)
    W = (rng.standard_normal((2 * F + 1, N)) * 0.05).astype(np.float32)
    Mg = np.zeros((M, ld(N)), np.float32); Mg[:, :N] = rng.standard_normal((M, N)) * 1e-3
    inv = (1.0 / rng.integers(1, 50, M)).astype(np.float32)
    t = {k: torch.tensor(v).cuda() for k, v in dict(A0=A0, A1=A1, W=W, Mg=Mg, inv=inv).items()}
    A = np.hstack([A0[:, :F], A1[:, :F], np.ones((M, 1))]).astype(np.float64)
    refs = {0: A @ W.astype(np.float64), 1: A.T @ Mg[:, :N].astype(np.float64),
            2: Mg[:, :N].astype(np.float64) @ W[:2 * F].astype(np.float64).T}
    for v in ("tc", "bf16", "simt"):
        out = torch.zeros((M, ld(N)), device="cuda"); P.dev_gemm(0, v, t["A0"], t["A1"], M, F, t["W"], N, out, ld(N))
        e0 = rel(out.cpu().numpy()[:, :N], refs[0])
        out = torch.zeros((2 * F + 1, N), device="cuda"); P.dev_gemm(1, v, t["A0"], t["A1"], M, F, t["W"], N, out, N, Mg=t["Mg"])
        e1 = rel(out.cpu().numpy(), refs[1])
        L = ld(F); out = torch.zeros((M, 2 * L), device="cuda")
        P.dev_gemm(2, v, None, None, M, F, t["W"], N, out, 2 * L, Mg=t["Mg"], inv_deg=t["inv"])
        g = out.cpu().numpy(); e2 = max(rel(g[:, :F], refs[2][:, :F] * inv[:, None]), rel(g[:, L:L + F], refs[2][:, F:]))
        torch.cuda.synchronize()
        print(f"M={M} F={F} N={N} {v:5s} fwd {e0:.2e} dW {e1:.2e} dA {e2:.2e}", flush=True)
