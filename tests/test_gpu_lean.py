"""Lean-memory mode (pgcn_config.lean): Z recomputed in the backward from one shared
scratch, one T scratch, one slot for J^(l) and for the packed feature messages, and the compact last
layer's rows bounded by the global train count.  The mode only drops buffers: every result must be bit
for bit the one of the default layout (loss, theta, G, every kept H^(l), every J^(l)) -- for
transform-first and aggregate-first layers, the compact last layer, the tensor-core tile aggregation,
GCN-sym, VANILLA / PIPE / PIPE-GF / depth 2, bf16 payloads, the LOOPBACK and PUSH transports -- also
with a 3 ms delay injected before every transfer on the comm stream (the single slots are only safe
because of the added waits), and the workspace must shrink.  One case against the fp64 oracle.
"""
import numpy as np
import pytest

from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import check_against_oracle, oracle_run, run_gpu

pytestmark = pytest.mark.gpu
DELAY_NS = 3_000_000


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def run(P, g, widths, n_parts, T, params0, hook=None, **kw):
    import torch
    part = P.partition(g.n, g.row_ptr, g.col_idx, n_parts)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, **kw)
    ctx = P.Context(part, cfg)
    if hook is not None:
        ctx.exchange_hook(*hook)
    for i in range(n_parts):
        gid = part.view(i)["inner_gid"]
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    L = len(widths) - 1
    recs = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, opt, loss)
        H = {}
        for l in range(1, L + 1):
            try:
                H[l] = [ctx.tensor(i, P.T_H, l, t)[:, :widths[l]].clone() for i in range(n_parts)]
            except P.PgcnError:  # lean + compact last layer: logits of non-train rows are not kept
                assert kw.get("lean") and l == L
        J = {l: [ctx.tensor(i, P.T_J, l, t)[:, :widths[l]].clone() for i in range(n_parts)] for l in range(1, L)}
        recs.append((loss.clone(), theta.clone(), grads.clone(), H, J))
    torch.cuda.synchronize()
    out = [dict(loss=float(lo.item()), params=th.cpu().numpy(), G=gr.cpu().numpy(),
                H={l: [x.cpu().numpy() for x in v] for l, v in H.items()},
                J={l: [x.cpu().numpy() for x in v] for l, v in J.items()}) for lo, th, gr, H, J in recs]
    return out, ctx


def same(a, b):
    """Bit-identical records over the tensors both runs kept."""
    for x, y in zip(a, b):
        assert x["loss"] == y["loss"]
        assert np.array_equal(x["params"], y["params"]) and np.array_equal(x["G"], y["G"])
        for l in set(x["H"]) & set(y["H"]):
            assert all(np.array_equal(u, v) for u, v in zip(x["H"][l], y["H"][l])), "H^(%d)" % l
        for l in x["J"]:
            assert all(np.array_equal(u, v) for u, v in zip(x["J"][l], y["J"][l])), "J^(%d)" % l


# papers-like: layer 1 transform-first (2 F_1 < F_0), layer 2 aggregate-first, layer 3 the compact
# last layer (aggregate-first GraphSAGE, few train rows)
PAPERS = dict(name="papers", seed=3, n=4001, nnz=36000, f0=40, classes=17)
PAPERS_W = [40, 12, 12, 17]


@pytest.mark.parametrize("transport", ["loopback", "push"])
@pytest.mark.parametrize("mode,sf,sg,depth,payload", [
    ("pipe", False, False, 1, "f32"), ("vanilla", False, False, 1, "f32"), ("pipe", True, True, 1, "f32"),
    ("pipe", False, False, 2, "f32"), ("pipe", True, True, 1, "bf16")])
@pytest.mark.parametrize("dropout", [0.0, 0.3])
def test_lean_bit_identical_papers_like(P, transport, mode, sf, sg, depth, payload, dropout):
    if payload == "bf16" and transport == "push":
        pytest.skip("PUSH moves fp32 payloads")
    c = dict(PAPERS)
    g = gen_graph(c.pop("name"), **c)
    params0 = glorot_params(PAPERS_W, 5)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, dropout=dropout, loss="ce", opt="adam", lr=0.01,
              depth=depth, transport=transport, halo_payload=payload, train_sparse=True)
    T = 2 * depth + 3
    ref, c0 = run(P, g, PAPERS_W, 3, T, params0, **kw)
    lean, c1 = run(P, g, PAPERS_W, 3, T, params0, lean=True, **kw)
    same(ref, lean)
    assert c1.ws.numel() < c0.ws.numel()


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_lean_bit_identical_tiles(P, model):
    """Reddit-like dense communities (tensor-core tiles on, tile_min 8): aggregate-first layers 1-2
    recompute Z on the tile path, layer 3 transform-first."""
    g = gen_graph("reddit", seed=3, n=800, nnz=24000, f0=32, classes=5)
    widths = [32, 64, 64, 5]
    params0 = glorot_params(widths, 3, model=model)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.5, loss="ce", opt="sgd", lr=0.5, model=model,
              spmm_tiles=True, tile_min=8, transport="loopback", train_sparse=True)
    ref, _ = run(P, g, widths, 2, 5, params0, **kw)
    lean, _ = run(P, g, widths, 2, 5, params0, lean=True, **kw)
    same(ref, lean)


@pytest.mark.parametrize("mode,depth", [("pipe", 1), ("pipe", 2), ("vanilla", 1)])
def test_lean_delay_injection(P, mode, depth):
    """A 3 ms spin before every transfer on the comm stream: the single J / message slots are rewritten
    only after the delayed transfer read them (the lean waits), so nothing changes."""
    c = dict(PAPERS)
    g = gen_graph(c.pop("name"), **c)
    params0 = glorot_params(PAPERS_W, 5)
    kw = dict(mode=mode, dropout=0.3, loss="ce", opt="sgd", lr=1.0, depth=depth, transport="loopback",
              train_sparse=True, lean=True)
    T = 2 * depth + 3
    ref, _ = run(P, g, PAPERS_W, 3, T, params0, **kw)
    slow, _ = run(P, g, PAPERS_W, 3, T, params0, hook=(DELAY_NS, 0), **kw)
    same(ref, slow)


def test_lean_against_oracle(P):
    """Yelp-like (BCE, ragged widths, layer 1 aggregate-first): lean PIPE-GF through the loopback
    exchange against the fp64 oracle at 1e-4."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    T = 4
    gpu, _ = run_gpu(P, g, widths, 3, T, params0, mode="pipe", smooth_f=True, smooth_g=True, gamma=0.7,
                     dropout=0.3, loss="bce", opt="sgd", lr=2.0, transport="loopback", lean=True)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=2.0, opt="sgd", loss="bce", gamma=0.7)
    ora = oracle_run(gpu, g, 3, params0, cfg, T, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, 3, 3, what="lean PIPE-GF")


def test_lean_train_bound_enforced(P):
    """lean + compact last layer sizes the train-row buffers by n_train_global: a partition holding more
    train rows than that is rejected by pgcn_set_inputs (PGCN_EINVAL), not overrun."""
    import torch
    c = dict(PAPERS)
    g = gen_graph(c.pop("name"), **c)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config(PAPERS_W, n_global=g.n, n_train_global=3, train_sparse=True, lean=True,
                        transport="loopback")
    ctx = P.Context(part, cfg)
    gid = part.view(0)["inner_gid"]
    tm = np.ones(len(gid), dtype=np.uint8)
    with pytest.raises(P.PgcnError):
        ctx.set_inputs(0, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(), torch.tensor(tm).cuda())
