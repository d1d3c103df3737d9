"""Parity at BASELINE.json's full size in bench.py's launch configuration (Reddit-shaped graph,
232,965 nodes, ~114M CSR non-zeros, 4 layers 602-256-256-256-41, 2 partitions on one GPU, PIPE,
dropout 0.5, Adam, tensor-core GEMMs):

* every partition array bit-exact against the oracle partitioner (Alg. 1 l.1-5);
* sampled rows of the layer-1 aggregation Z and output H^(1) at t = 1 (boundary rows still 0, l.6)
  and t = 2 (stale X boundary installed, dropout mask of t = 2, weights after step 1), recomputed
  one row at a time by the oracle's definitions in float64 (Eq. 3, App. F masks);
* properties that hold at any size: finite loss, loss ~ log(41) at t = 1, finite gradients.
Tolerance: the fp32 tier, 1e-4 of the sampled tensor's max magnitude."""
import numpy as np
import pytest

from oracle.hashmask import keep_mask
from oracle.partition import partition as oracle_partition
from synth.graphs import gen_graph, glorot_params, model_for

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def setup():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    g = gen_graph("reddit", seed=1)
    m = model_for("reddit")
    return pgcn, g, m


def test_partition_bit_exact_full_size(setup):
    P, g, m = setup
    pp = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    op = oracle_partition(g.n, g.row_ptr, g.col_idx, 2)
    for i in range(2):
        a, b = pp.view(i), op[i]
        for k in ("inner_gid", "halo_gid", "halo_off", "send_off", "send_idx", "row_ptr", "col_idx", "t_row_ptr",
                  "t_col_idx", "inv_ptr", "inv_pos"):
            assert np.array_equal(a[k].astype(np.int64), np.asarray(b[k]).astype(np.int64)), k
        assert np.array_equal(a["inv_deg"], np.asarray(b["inv_deg"]).astype(np.float32))


def row_oracle(g, P, v_local, t, W, b, p, seed, L, halo_zero):
    """Z and H^(1) of local inner row v of partition P at iteration t, one row, float64:
    Z_v = (1/d_v) sum_{u in N(v)} dropout_t(X)_u (Eq. 3; boundary rows 0 at t = 1, Alg. 1 l.6)."""
    N = g.n
    gv = int(P["inner_gid"][v_local])
    nb = g.col_idx[g.row_ptr[gv]:g.row_ptr[gv + 1]].astype(np.int64)
    F = g.X.shape[1]
    use = nb
    if halo_zero:
        lo, hi = P["inner_gid"][0], P["inner_gid"][-1]
        use = nb[(nb >= lo) & (nb <= hi)]          # contiguous partitions (R19): owned iff in range
    keep = keep_mask(t, 1, L, N, use, F, seed, p)
    acc = (g.X[use].astype(np.float64) * keep / (1.0 - p)).sum(0) if use.size else np.zeros(F)
    deg = nb.size
    Z = acc / deg if deg else acc
    Dv = g.X[gv].astype(np.float64) * keep_mask(t, 1, L, N, [gv], F, seed, p)[0] / (1.0 - p)
    Y = np.concatenate([Z, Dv]) @ W.astype(np.float64) + b.astype(np.float64)
    return Z, np.maximum(Y, 0.0)


@pytest.mark.parametrize("tf", [True, False])
def test_sampled_layer1_rows_full_size(setup, tf):
    """tf: bench's default transform-before-aggregate on layer 1 (the Z view then holds
    S = inv_deg P (D W_neigh), checked as Z_v W_neigh) or aggregate-first (Z itself)."""
    import torch
    P, g, m = setup
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config(m.widths, mode="pipe", dropout=m.dropout, loss=m.loss, opt="adam", lr=m.lr, n_global=g.n,
                        n_train_global=g.n_train, seed=4, transform_first=tf)
    ctx = P.Context(part, cfg)
    views = [part.view(i) for i in range(2)]
    keep = []
    for i, v in enumerate(views):
        gid = v["inner_gid"]
        a = tuple(torch.tensor(x).cuda() for x in (g.X[gid], g.labels[gid], g.train_mask[gid]))
        keep.append(a)
        ctx.set_inputs(i, *a)
    params0 = glorot_params(m.widths, 3)
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    L = len(m.widths) - 1
    F0, F1 = m.widths[0], m.widths[1]
    rng = np.random.default_rng(11)
    W_by_t = {}
    for t in (1, 2):
        W_by_t[t] = P.unflatten_params(theta.cpu().numpy().copy(), m.widths)[0]
        ctx.step(t, theta, grads, opt, loss)
        torch.cuda.synchronize()
        lv = float(loss.item())
        assert np.isfinite(lv)
        if t == 1:
            assert abs(lv - np.log(41) * g.n_train / g.n_train) < 1.0     # ~ log C at init
        assert torch.isfinite(grads).all()
        for i, v in enumerate(views):
            zt = ctx.tensor(i, P.T_Z, 1, t)
            Zg = zt[:, :zt.shape[1]].cpu().numpy()
            Hg = ctx.tensor(i, P.T_H, 1, t)[:, :F1].cpu().numpy()
            rows = rng.choice(v["n_inner"], 24, replace=False)
            W, b = W_by_t[t]
            Zr, Hr = zip(*[row_oracle(g, v, r, t, W, b, m.dropout, 4, L, halo_zero=(t == 1)) for r in rows])
            Zr, Hr = np.array(Zr), np.array(Hr)
            if Zg.shape[1] == F1:                     # transform-first: S_v = Z_v W_neigh
                Zr = Zr @ W[:F0].astype(np.float64)
            ez = np.abs(Zg[rows] - Zr).max() / max(np.abs(Zr).max(), 1e-30)
            eh = np.abs(Hg[rows] - Hr).max() / max(np.abs(Hr).max(), 1e-30)
            assert ez <= 1e-4, (t, i, ez)
            assert eh <= 1e-4, (t, i, eh)


def row_oracle_gcn(g, P, v_local, t, W, b, p, seed, L, halo_zero):
    """H^(1) of local inner row v under GCN-sym (App. A.1, R26), one row, float64:
    H_v = ReLU(s_v (s_v D_v + sum_{u in N(v)} s_u D_u) W + b), s_u = (d_u + 1)^-1/2 with full-graph
    degrees; boundary neighbours contribute 0 at t = 1 (Alg. 1 l.6)."""
    N = g.n
    gv = int(P["inner_gid"][v_local])
    nb = g.col_idx[g.row_ptr[gv]:g.row_ptr[gv + 1]].astype(np.int64)
    F = g.X.shape[1]
    use = nb
    if halo_zero:
        lo, hi = P["inner_gid"][0], P["inner_gid"][-1]
        use = nb[(nb >= lo) & (nb <= hi)]
    s_of = lambda u: 1.0 / np.sqrt(np.diff(g.row_ptr)[u].astype(np.float64) + 1.0)  # noqa: E731
    Du = g.X[use].astype(np.float64) * keep_mask(t, 1, L, N, use, F, seed, p) / (1.0 - p)
    Dv = g.X[gv].astype(np.float64) * keep_mask(t, 1, L, N, [gv], F, seed, p)[0] / (1.0 - p)
    sv = s_of(np.array([gv]))[0]
    Z = sv * (sv * Dv + (s_of(use)[:, None] * Du).sum(0))
    return np.maximum(Z @ W.astype(np.float64) + b.astype(np.float64), 0.0)


def test_sampled_layer1_rows_full_size_gcn(setup):
    """GCN-sym (N3) at the full Reddit size in bench.py --model gcn's configuration (layer 1
    transform-first): sampled H^(1) rows at t = 1, 2 against the one-row oracle."""
    import torch
    P, g, m = setup
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config(m.widths, mode="pipe", dropout=m.dropout, loss=m.loss, opt="adam", lr=m.lr, n_global=g.n,
                        n_train_global=g.n_train, seed=4, model="gcn")
    ctx = P.Context(part, cfg)
    views = [part.view(i) for i in range(2)]
    keep = []
    for i, v in enumerate(views):
        gid = v["inner_gid"]
        a = tuple(torch.tensor(x).cuda() for x in (g.X[gid], g.labels[gid], g.train_mask[gid]))
        keep.append(a)
        ctx.set_inputs(i, *a)
    params0 = glorot_params(m.widths, 3, model="gcn")
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    L = len(m.widths) - 1
    F1 = m.widths[1]
    rng = np.random.default_rng(12)
    for t in (1, 2):
        W, b = P.unflatten_params(theta.cpu().numpy().copy(), m.widths, model="gcn")[0]
        ctx.step(t, theta, grads, opt, loss)
        torch.cuda.synchronize()
        assert np.isfinite(float(loss.item())) and torch.isfinite(grads).all()
        for i, v in enumerate(views):
            Hg = ctx.tensor(i, P.T_H, 1, t)[:, :F1].cpu().numpy()
            rows = rng.choice(v["n_inner"], 24, replace=False)
            Hr = np.array([row_oracle_gcn(g, v, r, t, W, b, m.dropout, 4, L, halo_zero=(t == 1)) for r in rows])
            eh = np.abs(Hg[rows] - Hr).max() / max(np.abs(Hr).max(), 1e-30)
            assert eh <= 1e-4, (t, i, eh)
