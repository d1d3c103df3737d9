"""GPU parity of the GCN-sym path (N3; App. A.1, reading R26) against the fp64
oracle: same harness and tolerance as tests/test_gpu_parity.py (1e-4 relative per tensor for the
3xTF32 path, 2e-2 for the bf16 tensor-core variant)."""
import numpy as np
import pytest

from oracle.partition import contiguous_map
from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import TOL, check_against_oracle, oracle_run, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def mcfg(widths, p, lr, loss, gamma=0.95):
    return ModelCfg(widths=widths, dropout=p, lr=lr, opt="sgd", loss=loss, gamma=gamma, model="gcn")


MODES = [("vanilla", False, False), ("pipe", False, False), ("pipe", True, True)]


@pytest.mark.parametrize("mode,sf,sg", MODES)
@pytest.mark.parametrize("p", [0.0, 0.5])
@pytest.mark.parametrize("tf", [True, False])
def test_gcn_cora(P, mode, sf, sg, p, tf):
    g = gen_graph("cora", seed=1)
    widths = [1433, 16, 7]
    params0 = glorot_params(widths, 3, model="gcn")
    gpu, _ = run_gpu(P, g, widths, 2, 4, params0, mode=mode, smooth_f=sf, smooth_g=sg, dropout=p, loss="ce",
                     opt="sgd", lr=0.5, transform_first=tf, model="gcn")
    ora = oracle_run(gpu, g, 2, params0, mcfg(widths, p, 0.5, "ce"), 4, mode=mode, smooth_f=sf, smooth_g=sg)
    check_against_oracle(gpu, ora, 2, 2, what=f"gcn cora {mode} p{p} tf{tf}")


@pytest.mark.parametrize("tf", [True, False])
@pytest.mark.parametrize("gemm,tol", [("tc", TOL), ("bf16", 2e-2)])
def test_gcn_multi_tile_ragged(P, tf, gemm, tol):
    """3 layers with ragged widths (103 -> 70 -> 45 -> 13), 3 partitions, BCE, dropout 0.3; both
    transform-first (layers 2, 3) and aggregate-first."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5, model="gcn")
    gpu, _ = run_gpu(P, g, widths, 3, 3, params0, mode="pipe", smooth_f=True, smooth_g=True, gamma=0.7,
                     dropout=0.3, loss="bce", opt="sgd", lr=2.0, transform_first=tf, model="gcn", gemm=gemm)
    ora = oracle_run(gpu, g, 3, params0, mcfg(widths, 0.3, 2.0, "bce", 0.7), 3, tol=tol, mode="pipe",
                     smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, 3, 3, tol=tol, what=f"gcn ragged tf{tf} {gemm}")


def test_gcn_wide_and_empty_partition(P):
    """Reddit-like widths (602 -> 256 -> 41) and a partition map with an empty partition."""
    g = gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=602, classes=41)
    widths = [602, 256, 41]
    params0 = glorot_params(widths, 7, model="gcn")
    part_of = contiguous_map(g.n, 3)
    part_of[part_of == 1] = 2                                     # partition 1 owns nothing
    gpu, _ = run_gpu(P, g, widths, 3, 3, params0, part_of=part_of, mode="pipe", dropout=0.5, loss="ce",
                     opt="sgd", lr=0.1, model="gcn")
    from oracle import pipegcn
    from oracle.partition import partition as op
    from test_gpu_parity import kernel_relu_decision
    ora = pipegcn.run(g, op(g.n, g.row_ptr, g.col_idx, 3, part_of), params0, mcfg(widths, 0.5, 0.1, "ce"), 3,
                      mode="pipe", relu_decision=kernel_relu_decision(gpu))
    check_against_oracle(gpu, ora, 2, 3, what="gcn wide")


def test_gcn_rejects_simt(P):
    g = gen_graph("cora", seed=1, n=100, nnz=400, f0=8, classes=3)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config([8, 4, 3], n_global=g.n, n_train_global=g.n_train, model="gcn", gemm="simt")
    with pytest.raises(P.PgcnError) as e:
        P.Context(part, cfg)
    assert e.value.code == P.EUNSUPPORTED


def test_gcn_param_count(P):
    cfg = P.make_config([10, 7, 3], n_global=5, model="gcn")
    assert P.param_count(cfg) == (10 + 1) * 7 + (7 + 1) * 3
    assert np.isclose(P.param_count(P.make_config([10, 7, 3], n_global=5)), (20 + 1) * 7 + (14 + 1) * 3)
