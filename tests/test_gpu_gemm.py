"""GPU unit tests of the node-update GEMMs (include/pgcn_dev.h) against float64 numpy matmul of the
same fp32 inputs.  Tolerance: max|gpu - ref| <= tol * max|ref| with tol = 1e-4 for the fp32 tier
(3xTF32 tensor cores, SIMT fp32) and 2e-2 for the bf16 tensor-core variant (north_star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SHAPES = [(300, 37, 16), (1000, 602, 256), (513, 256, 41), (700, 300, 512), (129, 16, 7), (4096, 128, 48)]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def ld(f):
    return (f + 3) // 4 * 4


def mk(M, F, N, seed):
    rng = np.random.default_rng(seed)
    A0 = np.zeros((M, ld(F)), np.float32)
    A1 = np.zeros((M, ld(F)), np.float32)
    A0[:, :F] = rng.standard_normal((M, F))
    A1[:, :F] = rng.standard_normal((M, F))
    W = rng.standard_normal((2 * F + 1, N)).astype(np.float32) * 0.1
    Mg = np.zeros((M, ld(N)), np.float32)
    Mg[:, :N] = rng.standard_normal((M, N))
    inv = (1.0 / rng.integers(1, 50, M)).astype(np.float32)
    return A0, A1, W, Mg, inv


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


TOLS = {"tc": 1e-4, "simt": 1e-4, "bf16": 2e-2}
VARIANTS = ["tc", "simt", "bf16"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("M,F,N", SHAPES)
def test_forward(P, variant, M, F, N):
    import torch
    A0, A1, W, _, _ = mk(M, F, N, 1)
    out = torch.full((M, ld(N)), 7.0, device="cuda")
    t = [torch.tensor(x).cuda() for x in (A0, A1, W)]
    P.dev_gemm(0, variant, t[0], t[1], M, F, t[2], N, out, ld(N), relu=True)
    torch.cuda.synchronize()
    A = np.hstack([A0[:, :F], A1[:, :F], np.ones((M, 1), np.float32)]).astype(np.float64)
    ref = np.maximum(A @ W.astype(np.float64), 0)
    got = out.cpu().numpy()
    assert rel(got[:, :N], ref) <= TOLS[variant]
    assert (got[:, N:] == 0).all()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("M,F,N", SHAPES)
def test_weight_gradient(P, variant, M, F, N):
    import torch
    A0, A1, W, Mg, _ = mk(M, F, N, 2)
    out = torch.zeros((2 * F + 1, N), device="cuda")
    t = [torch.tensor(x).cuda() for x in (A0, A1, W, Mg)]
    P.dev_gemm(1, variant, t[0], t[1], M, F, t[2], N, out, N, Mg=t[3])
    torch.cuda.synchronize()
    A = np.hstack([A0[:, :F], A1[:, :F], np.ones((M, 1), np.float32)]).astype(np.float64)
    ref = A.T @ Mg[:, :N].astype(np.float64)
    assert rel(out.cpu().numpy(), ref) <= TOLS[variant]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("M,F,N", SHAPES)
def test_input_gradient(P, variant, M, F, N):
    import torch
    A0, A1, W, Mg, inv = mk(M, F, N, 3)
    L = ld(F)
    out = torch.full((M, 2 * L), 7.0, device="cuda")
    t = [torch.tensor(x).cuda() for x in (W, Mg, inv)]
    P.dev_gemm(2, variant, None, None, M, F, t[0], N, out, 2 * L, Mg=t[1], inv_deg=t[2])
    torch.cuda.synchronize()
    dA = Mg[:, :N].astype(np.float64) @ W[:2 * F].astype(np.float64).T
    got = out.cpu().numpy()
    assert rel(got[:, :F], dA[:, :F] * inv[:, None]) <= TOLS[variant]
    assert rel(got[:, L:L + F], dA[:, F:]) <= TOLS[variant]
    assert (got[:, F:L] == 0).all() and (got[:, L + F:] == 0).all()


# The dW GEMM at the row counts the bench reduces over: a Reddit-shaped partition (116,483 rows; the
# split-K plan with many splits) and a papers100M-shaped 8-way partition (13.9M rows; the colsum bias
# row's chunked second pass).  Inputs are drawn on the device (seeded); the reference is the same
# contraction in float64 (cuBLAS DGEMM through torch: a library primitive, the plain definition A^T M).
BIG = [(116483, 256, 256), (116483, 602, 256), (13_900_000, 48, 48), (13_900_000, 128, 48)]


@pytest.mark.parametrize("variant", ["tc", "bf16"])
@pytest.mark.parametrize("M,F,N", BIG)
def test_weight_gradient_full_size(P, variant, M, F, N):
    import torch
    gen = torch.Generator(device="cuda").manual_seed(M + F + N)
    A0 = torch.zeros((M, ld(F)), device="cuda")
    A1 = torch.zeros((M, ld(F)), device="cuda")
    A0[:, :F] = torch.randn((M, F), device="cuda", generator=gen)
    A1[:, :F] = torch.randn((M, F), device="cuda", generator=gen)
    Mg = torch.zeros((M, ld(N)), device="cuda")
    Mg[:, :N] = torch.randn((M, N), device="cuda", generator=gen) * 1e-3
    W = torch.zeros((2 * F + 1, N), device="cuda")
    out = torch.zeros((2 * F + 1, N), device="cuda")
    P.dev_gemm(1, variant, A0, A1, M, F, W, N, out, N, Mg=Mg)
    torch.cuda.synchronize()
    ref = torch.zeros((2 * F + 1, N), dtype=torch.float64, device="cuda")
    step = 1 << 21
    for r0 in range(0, M, step):  # fp64 A^T M in row chunks (bounded scratch)
        r1 = min(M, r0 + step)
        m = Mg[r0:r1, :N].double()
        ref[:F] += A0[r0:r1, :F].double().T @ m
        ref[F:2 * F] += A1[r0:r1, :F].double().T @ m
        ref[2 * F] += m.sum(0)
    got, ref = out.double(), ref
    err = float((got - ref).abs().max() / ref.abs().max())
    assert err <= TOLS[variant], (M, F, N, variant, err)
