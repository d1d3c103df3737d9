"""GPU parity of the bf16 gather tier (pgcn_config.gather = 1) against the fp64
oracle at the north_star's bf16 tier (2e-2 relative per tensor): every table an SpMM gathers is
rounded to bf16 (fp32 accumulation), with fp32-grade (3xTF32) or bf16 tensor-core GEMMs.

Cases: GraphSAGE and GCN-sym; both aggregation orders (transform-first exercises the narrow
transposed SpMM on inv_deg o M, aggregate-first the SpMM on dZ'); widths whose bf16 rows need a
padded vector (41, 45, 13 columns) and several 16-byte vectors per lane (602, 1433 columns);
3 partitions with ragged tails; dropout and EMA smoothing on."""
import pytest

from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import check_against_oracle, oracle_run, run_gpu

pytestmark = pytest.mark.gpu
TOL16 = 2e-2


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def case(name):
    if name == "cora":
        return gen_graph("cora", seed=1), [1433, 16, 7], "ce", 2
    if name == "wide":
        return gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=602, classes=41), [602, 256, 41], "ce", 2
    if name == "ragged3":
        return gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13), [103, 70, 45, 13], "bce", 3
    raise KeyError(name)


@pytest.mark.parametrize("name", ["cora", "wide", "ragged3"])
@pytest.mark.parametrize("tf", [True, False])
@pytest.mark.parametrize("gemm", ["tc", "bf16"])
@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_bf16_gather(P, name, tf, gemm, model):
    g, widths, loss, n_parts = case(name)
    L = len(widths) - 1
    params0 = glorot_params(widths, 3, model=model)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.3, loss=loss, opt="sgd", lr=0.5, gemm=gemm,
              transform_first=tf, model=model, gather="bf16")
    T = 3
    gpu, _ = run_gpu(P, g, widths, n_parts, T, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss, model=model)
    ora = oracle_run(gpu, g, n_parts, params0, cfg, T, tol=TOL16, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, L, n_parts, tol=TOL16, what=f"bf16-gather {name} tf{tf} {gemm} {model}")


def test_bf16_gather_vanilla_first_iteration_rows(P):
    """VANILLA at t = 1 and PIPE at t = 1 (boundary rows not valid yet: the checked kernel variant
    that skips neighbours >= n_valid) on the wide case, aggregate-first."""
    g, widths, loss, n_parts = case("wide")
    params0 = glorot_params(widths, 3)
    for mode in ("vanilla", "pipe"):
        kw = dict(mode=mode, dropout=0.5, loss=loss, opt="sgd", lr=0.5, transform_first=False, gather="bf16")
        gpu, _ = run_gpu(P, g, widths, n_parts, 2, params0, **kw)
        cfg = ModelCfg(widths=widths, dropout=0.5, lr=0.5, opt="sgd", loss=loss)
        ora = oracle_run(gpu, g, n_parts, params0, cfg, 2, tol=TOL16, mode=mode)
        check_against_oracle(gpu, ora, 2, n_parts, tol=TOL16, what=f"bf16-gather {mode}")
