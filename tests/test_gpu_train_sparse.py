"""GPU parity of the train-row-sparse last layer (pgcn_config.train_sparse) against the
fp64 oracle, which computes the last layer on every row (Alg. 1 as written).  The optimisation is
exact: loss, every G_i and G, the updated parameters, every hidden layer's H and J must match at the
tier's tolerance; the logits Y^(L) are compared on train rows only (elsewhere they are not computed).

Cases: products-shaped (8 % train) and Cora-shaped (5 %) graphs, GraphSAGE and GCN-sym, both
aggregation orders of the last layer, 2-3 partitions, VANILLA and PIPE-GF, fp32 (1e-4) and the bf16
gather tier (2e-2); a partition without train rows; several steps so the stale messages of the
sparse backward feed later iterations."""
import numpy as np
import pytest

from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import TOL, flat, oracle_run, rel, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def check_sparse(gpu, ora, g, part_views, L, n_parts, tol, what):
    for t, (a, b) in enumerate(zip(gpu, ora), start=1):
        assert abs(a["loss"] - b["loss"]) <= tol * abs(b["loss"]), (what, t, a["loss"], b["loss"])
        for l in range(1, L + 1):
            for i in range(n_parts):
                ga, ob = a["H"][l][i], b["H"][l][i]
                if l == L:  # logits: train rows only
                    tr = g.train_mask[part_views[i]["inner_gid"]].astype(bool)
                    ga, ob = ga[tr], ob[tr]
                e = rel(ga, ob)
                assert e <= tol, (what, "H", t, l, i, e)
        for l in range(1, L):
            for i in range(n_parts):
                e = rel(a["J"][l][i], b["J"][l][i])
                assert e <= tol, (what, "J", t, l, i, e)
        assert rel(a["G"], flat(b["G"])) <= tol, (what, "G", t)
        for i in range(n_parts):
            assert rel(a["G_parts"][i], flat(b["G_parts"][i])) <= tol, (what, "G_i", t, i)
        assert rel(a["params"], flat(b["params"])) <= tol, (what, "params", t)


def run_case(P, g, widths, n_parts, T, model, tf, mode, sm, gather, loss="ce", part_of=None):
    tol = TOL if gather == "f32" else 2e-2
    params0 = glorot_params(widths, 3, model=model)
    kw = dict(mode=mode, smooth_f=sm, smooth_g=sm, dropout=0.3, loss=loss, opt="sgd", lr=0.5, transform_first=tf,
              model=model, gather=gather, train_sparse=True)
    gpu, _ = run_gpu(P, g, widths, n_parts, T, params0, part_of=part_of, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss, model=model)
    ora = oracle_run(gpu, g, n_parts, params0, cfg, T, tol=tol, mode=mode, smooth_f=sm, smooth_g=sm)
    part = P.partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    views = [part.view(i) for i in range(n_parts)]
    check_sparse(gpu, ora, g, views, len(widths) - 1, n_parts, tol, f"sparse {model} tf{tf} {mode} {gather}")


@pytest.mark.parametrize("model", ["sage", "gcn"])
@pytest.mark.parametrize("tf", [True, False])
@pytest.mark.parametrize("mode,sm", [("vanilla", False), ("pipe", True)])
@pytest.mark.parametrize("gather", ["f32", "bf16"])
def test_train_sparse_products_shaped(P, model, tf, mode, sm, gather):
    g = gen_graph("products", seed=4, n=4000, nnz=60000, f0=100, classes=47)
    run_case(P, g, [100, 64, 48, 47], 3, 3, model, tf, mode, sm, gather)


@pytest.mark.parametrize("tf", [True, False])
def test_train_sparse_cora(P, tf):
    g = gen_graph("cora", seed=1)
    run_case(P, g, [1433, 16, 7], 2, 4, "sage", tf, "pipe", True, "f32")


def test_train_sparse_partition_without_train_rows(P):
    """Partition 1 owns no train rows (its last-layer SpMMs get an empty row list / empty P^T|train)."""
    g = gen_graph("products", seed=6, n=3000, nnz=40000, f0=100, classes=47)
    n = g.n
    part_of = np.zeros(n, np.int32)
    part_of[n // 2:] = 1
    g.train_mask[n // 2:] = 0
    run_case(P, g, [100, 32, 47], 2, 3, "sage", True, "pipe", True, "f32", part_of=part_of)
