"""Host logic of bench.py (no GPU): the roll-up of the engine's timing buckets into kernel functions, the
roofline of the dominant kernel (binding roof by arithmetic intensity for the GEMMs), and the reference
arm's oracle timing on a small sample."""
import types

import bench

Z = {"ms": 0.0, "launches": 0, "bytes": 0.0, "flops": 0.0, "gather_bytes": 0.0}


def k(ms, n, b=0.0, f=0.0):
    return {"ms": ms, "launches": n, "bytes": b, "flops": f, "gather_bytes": 10 * b}


def test_kernel_functions_rollup():
    kern = {"spmm_fwd": k(10.0, 4, 1e9), "spmm_bwd": k(8.0, 4, 1e9), "gemm_fwd": k(3.0, 6, 1e9, 1e12),
            "gemm_dw": k(2.0, 3, 1e9, 2e12), "gemm_da": k(1.0, 2, 1e9, 5e11), "dropout": k(1.0, 4, 1e9),
            "gather": dict(Z), "grad_reduce": k(0.5, 2, 1e8), "loss": k(0.1, 1, 1e6), "update": k(0.01, 1, 1e5),
            "spmm_tile_fwd": k(4.0, 3, 2e9, 3e12), "spmm_tile_bwd": k(3.0, 3, 2e9, 2e12)}
    kf = bench.kernel_functions(kern)
    assert kf["k_umma_gemm"]["ms"] == 6.0 and kf["k_umma_gemm"]["flops"] == 3.5e12 and kf["k_umma_gemm"]["launches"] == 11
    assert kf["k_spmm_tc"]["ms"] == 7.0 and kf["k_spmm_tc"]["flops"] == 5e12
    assert kf["k_spmm_fwd"]["ms"] == 6.0 and kf["k_spmm_bwd"]["ms"] == 5.0     # bucket minus its tile part
    assert kf["k_spmm_fwd"]["tile_path"]
    assert "k_gather" not in kf                                                  # no launches
    total = sum(v["ms"] for v in kf.values())
    assert abs(total - sum(v["ms"] for n, v in kern.items() if not n.startswith("spmm_tile"))) < 1e-12


def test_gemm_roofline_binding_roof():
    pk = {"hbm_gbs": 6000.0, "bf16_tflops": 1600.0}
    args = types.SimpleNamespace(gemm="tc", config="x")
    # AI = 3 * flops / bytes: 3 * 1e12 / 1e9 = 3000 flop/B > ridge 800e12 / 6e12 = 133 -> tensor
    r = bench.kernel_roofline("k_umma_gemm", k(10.0, 10, 1e9, 1e12), pk, args, {}, None)
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and abs(r["achieved"] - 300.0) < 1e-9
    assert abs(r["frac"] - 300.0 / 800.0) < 1e-12
    # AI = 3 * 1e10 / 1e9 = 30 flop/B < 133 -> HBM-bound: algorithmic bytes over the copy peak
    r = bench.kernel_roofline("k_umma_gemm", k(10.0, 10, 1e9, 1e10), pk, args, {}, None)
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["achieved"] - 100.0) < 1e-9
    assert abs(r["frac"] - 100.0 / 6000.0) < 1e-12
    # the tile aggregation: executed MMA flops over the bf16 peak
    r = bench.kernel_roofline("k_spmm_tc", k(2.0, 4, 1e9, 8e11), pk, args, {}, None)
    assert r["bound"] == "tensor" and abs(r["achieved"] - 400.0) < 1e-9 and abs(r["frac"] - 0.25) < 1e-12


def test_reference_arm_sample_runs():
    out = bench.cpu_baseline("cora", 2, "pipe", "", sample_n=400, iters=1)
    assert out["kind"] == "oracle" and out["value"] > 0 and out["cores"] >= 1 and out["extrapolated"]
