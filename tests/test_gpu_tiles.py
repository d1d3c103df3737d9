"""GPU parity of the tensor-core dense-tile aggregation (pgcn_config.spmm_tiles; DESIGN.md "Tensor-core
tiles") against the fp64 oracle.  Heavy 128 x 64 tiles of P_i / P_i^T are summed as 0/1 blocks times
the gathered rows on tcgen05 (fp32 tier: 2-term tf32 split, 1e-4; bf16 gather tier: bf16 rows, 2e-2),
the light edges by the gather SpMM on top.  tile_min = 1 puts every edge in a tile (the light CSR is
empty), tile_min = 24 mixes both; widths cover one n-tile (41, 96 -> BN 64/128 after padding), a full
256-column tile, and a 602-wide table (3 n-tiles); both aggregation orders, GraphSAGE and GCN-sym,
dropout and EMA smoothing on, 2 and 3 partitions.  t = 1 runs the gather-only variant (boundary rows
not valid yet), t >= 2 the tile path."""
import numpy as np
import pytest

from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import check_against_oracle, oracle_run, rel, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def case(name):
    if name == "dense":   # dense communities (Reddit-like), 3 layers, 2 partitions
        return gen_graph("reddit", seed=3, n=3000, nnz=150000, f0=200, classes=41), [200, 256, 96, 41], "ce", 2
    if name == "wide":    # 602-wide input table (aggregate-first layer 1: 3 n-tiles of the tile kernel)
        return gen_graph("reddit", seed=4, n=1500, nnz=60000, f0=602, classes=41), [602, 256, 41], "ce", 2
    if name == "ragged3":
        return gen_graph("yelp", seed=5, n=2001, nnz=50000, f0=70, classes=13), [70, 100, 33, 13], "bce", 3
    raise KeyError(name)


@pytest.mark.parametrize("name", ["dense", "wide", "ragged3"])
@pytest.mark.parametrize("tmin", [1, 24])
@pytest.mark.parametrize("tf", [True, False])
@pytest.mark.parametrize("gather", ["f32", "bf16"])
def test_tiles_vs_oracle(P, name, tmin, tf, gather):
    g, widths, loss, n_parts = case(name)
    L = len(widths) - 1
    tol = 1e-4 if gather == "f32" else 2e-2
    params0 = glorot_params(widths, 3)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.3, loss=loss, opt="sgd", lr=0.5,
              transform_first=tf, gather=gather, spmm_tiles=True, tile_min=tmin)
    T = 3
    gpu, _ = run_gpu(P, g, widths, n_parts, T, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss)
    ora = oracle_run(gpu, g, n_parts, params0, cfg, T, tol=tol, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, L, n_parts, tol=tol, what=f"tiles {name} t{tmin} tf{tf} {gather}")


@pytest.mark.parametrize("gather", ["f32", "bf16"])
@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_tiles_light_mix(P, gather, model):
    """A quarter of the edges light (tile_min 200): the gather pass adds the light edges to the tile
    sums and applies the epilogues (self loop and row scale of GCN-sym, dropout mask of the
    transposed pass); both tiers, GraphSAGE and GCN-sym, both aggregation orders."""
    g, widths, loss, n_parts = case("dense")
    tol = 1e-4 if gather == "f32" else 2e-2
    params0 = glorot_params(widths, 3, model=model)
    for tf in (True, False):
        kw = dict(mode="pipe", smooth_f=True, dropout=0.3, loss=loss, opt="sgd", lr=0.5, transform_first=tf,
                  gather=gather, model=model, spmm_tiles=True, tile_min=200)
        gpu, _ = run_gpu(P, g, widths, n_parts, 3, params0, **kw)
        cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss, model=model)
        ora = oracle_run(gpu, g, n_parts, params0, cfg, 3, tol=tol, mode="pipe", smooth_f=True)
        check_against_oracle(gpu, ora, 3, n_parts, tol=tol, what=f"light-mix {gather} {model} tf{tf}")


@pytest.mark.parametrize("tf", [True, False])
@pytest.mark.parametrize("mode", ["pipe", "vanilla"])
def test_tiles_gcn(P, tf, mode):
    """GCN-sym (R26): self loop and d~^-1/2 row scale in the gather epilogue on top of the tile sums."""
    g, widths, loss, n_parts = case("dense")
    params0 = glorot_params(widths, 3, model="gcn")
    kw = dict(mode=mode, dropout=0.3, loss=loss, opt="sgd", lr=0.5, transform_first=tf, model="gcn",
              spmm_tiles=True, tile_min=8)
    gpu, _ = run_gpu(P, g, widths, n_parts, 3, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss, model="gcn")
    ora = oracle_run(gpu, g, n_parts, params0, cfg, 3, mode=mode)
    check_against_oracle(gpu, ora, 3, n_parts, what=f"tiles gcn tf{tf} {mode}")


def test_tiles_on_off_agree(P):
    """Same run with and without the tile path: the sums are only reassociated (fp32 tier), so the loss
    and every layer output agree to fp32 rounding (1e-5 relative) at t = 1 (gather only) and t = 2 (tile
    path, same weights).  Later iterations are compared with the oracle above only: a ReLU' decision
    at |Y| ~ 1e-7 may legitimately differ between two fp32 summation orders and moves G by a whole J
    entry (reading R25), so the weights of t >= 3 differ slightly.)"""
    g, widths, loss, n_parts = case("dense")
    params0 = glorot_params(widths, 3)
    kw = dict(mode="pipe", smooth_g=True, dropout=0.3, loss=loss, opt="sgd", lr=0.5)
    a, _ = run_gpu(P, g, widths, n_parts, 2, params0, spmm_tiles=True, tile_min=16, **kw)
    b, _ = run_gpu(P, g, widths, n_parts, 2, params0, spmm_tiles=False, **kw)
    for t, (x, y) in enumerate(zip(a, b), start=1):
        assert abs(x["loss"] - y["loss"]) <= 1e-5 * abs(y["loss"]), t
        for l in x["H"]:
            for i in range(n_parts):
                assert rel(x["H"][l][i], y["H"][l][i]) <= 1e-5, (t, l, i)


def test_tiles_used(P):
    """The dense case really takes the tile path (heavy edges >= 25 % at the default threshold)."""
    g, widths, loss, n_parts = case("dense")
    part = P.partition(g.n, g.row_ptr, g.col_idx, n_parts)
    for i in range(n_parts):
        for which in (0, 1):
            t = part.tiles(i, which, 96)
            assert t["nnz_heavy"] >= 0.25 * (t["nnz_heavy"] + t["nnz_light"])
    assert np.isfinite(t["n_tiles"])
