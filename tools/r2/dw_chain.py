"""dW accumulation-chain study: relative error against float64 (per row block of G: Z rows, D rows, bias
row) and time of the tcgen05 dW GEMM at the bench's row counts, for the chain cap PGCN_DW_KMAX given
in the environment (k-blocks of 32 rows per tile; 0 = uncapped).  One JSON line per shape."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402

for M, F, N in ((13_900_000, 48, 48), (1_224_515, 128, 128), (116_483, 256, 256), (358_424, 512, 512)):
    g = torch.Generator(device="cuda").manual_seed(M)
    ld = (F + 3) // 4 * 4
    A0 = torch.zeros((M, ld), device="cuda")
    A1 = torch.zeros((M, ld), device="cuda")
    A0[:, :F] = torch.randn((M, F), device="cuda", generator=g)
    A1[:, :F] = torch.randn((M, F), device="cuda", generator=g)
    ldn = (N + 3) // 4 * 4
    Mg = torch.zeros((M, ldn), device="cuda")
    Mg[:, :N] = torch.randn((M, N), device="cuda", generator=g) * 1e-3
    W = torch.zeros((2 * F + 1, N), device="cuda")
    out = torch.zeros((2 * F + 1, N), device="cuda")
    res = {}
    for variant in ("tc", "bf16"):
        scratch = pgcn.dev_gemm(1, variant, A0, A1, M, F, W, N, out, N, Mg=Mg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            pgcn.dev_gemm(1, variant, A0, A1, M, F, W, N, out, N, Mg=Mg)
        e1.record()
        torch.cuda.synchronize()
        ref = torch.zeros((2 * F + 1, N), dtype=torch.float64, device="cuda")
        step = 1 << 21
        for r0 in range(0, M, step):
            r1 = min(M, r0 + step)
            m = Mg[r0:r1, :N].double()
            ref[:F] += A0[r0:r1, :F].double().T @ m
            ref[F:2 * F] += A1[r0:r1, :F].double().T @ m
            ref[2 * F] += m.sum(0)
        d = (out.double() - ref).abs()
        scale = float(ref.abs().max())
        res[variant] = {"ms": e0.elapsed_time(e1) / 3, "rel": float(d.max()) / scale,
                        "rel_Z": float(d[:F].max()) / scale, "rel_D": float(d[F:2 * F].max()) / scale,
                        "rel_bias": float(d[2 * F].max()) / scale}
    print(json.dumps({"kmax": os.environ.get("PGCN_DW_KMAX", "default"), "M": M, "F": F, "N": N, **res}), flush=True)
    del A0, A1, Mg
    torch.cuda.empty_cache()
