"""Pins for oracle/pipegcn.py: O2 (vanilla) and O3 (PipeGCN, Alg. 1).

Each pin checks the oracle against something other than itself:
* O2 == O1 (vanilla partition-parallel training is full-graph training; P = P_in + P_bd)
* O3 with one partition == O1
* O3 at t = 1 == O1 on P_in only, degrees unchanged (Alg. 1 l.6: boundary features 0)
* O3 forward/backward == the App. A.1 matrix form with P_in / P_bd and stale H, M, W
  (PAPER.md:661-675), assembled over the whole graph
* eta = 0, p = 0: O3's G equals O2's for t >= 2L (Cor. A.10's eta -> 0 limit)
* EMA with gamma = 0 is the identity; with eta = 0 smoothed O3 converges geometrically to O2
* layer-1 output is exact for t >= 2 (X is constant)
* golden hand-derived t = 1 values (tests/golden/tiny4.json)
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pipegcn, sage
from oracle.partition import contiguous_map, partition
from synth.graphs import ModelCfg, gen_graph, glorot_params, random_graph


def small_graph(seed=1, n=120, ml=False):
    g = gen_graph("cora", seed=seed, n=n, nnz=n * 6, f0=9, classes=4, comm=4)
    if ml:
        g.labels = (np.random.default_rng(seed).random((n, 4)) < 0.3).astype(np.uint8)
        g.multilabel = True
    return g


def cfg(widths, p=0.0, lr=0.05, opt="sgd", loss="ce", gamma=0.95):
    return ModelCfg(widths=widths, dropout=p, lr=lr, opt=opt, loss=loss, gamma=gamma)


def assemble(parts, per_part, n, width):
    out = np.full((n, width), np.nan)
    for P, a in zip(parts, per_part):
        out[P["inner_gid"]] = a
    return out


def close(a, b, rtol=1e-10):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(np.abs(b).max(), 1e-300)
    return np.abs(a - b).max() <= rtol * scale


@pytest.mark.parametrize("n_parts", [1, 2, 3, 4])
@pytest.mark.parametrize("p,loss,opt", [(0.0, "ce", "sgd"), (0.5, "ce", "sgd"), (0.3, "bce", "adam")])
def test_vanilla_equals_full_graph(n_parts, p, loss, opt):
    g = small_graph(ml=(loss == "bce"))
    c = cfg([9, 8, 6, 4], p=p, loss=loss, opt=opt)
    params = glorot_params(c.widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts)
    T = 4
    full = sage.train_full(g, params, c, T)
    van = pipegcn.run(g, parts, params, c, T, mode="vanilla")
    for t in range(T):
        assert np.isclose(van[t]["loss"], full[t]["loss"], rtol=1e-12)
        for l in range(1, 4):
            assert close(assemble(parts, van[t]["H"][l], g.n, c.widths[l]), full[t]["H"][l])
        for l in range(1, 3):
            assert close(assemble(parts, van[t]["J"][l], g.n, c.widths[l]), full[t]["J"][l])
        for (a, b), (x, y) in zip(van[t]["G"], full[t]["grads"]):
            assert close(a, x) and close(b, y)
        for (a, b), (x, y) in zip(van[t]["params"], full[t]["params"]):
            assert close(a, x) and close(b, y)


def test_pipe_one_partition_is_full_graph():
    g = small_graph()
    c = cfg([9, 8, 4], p=0.5)
    params = glorot_params(c.widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 1)
    full = sage.train_full(g, params, c, 3)
    pipe = pipegcn.run(g, parts, params, c, 3, mode="pipe", smooth_f=True, smooth_g=True)
    for t in range(3):
        assert np.isclose(pipe[t]["loss"], full[t]["loss"], rtol=1e-13)
        for (a, b), (x, y) in zip(pipe[t]["G"], full[t]["grads"]):
            assert close(a, x, 1e-12) and close(b, y, 1e-12)


@pytest.mark.parametrize("n_parts,p", [(2, 0.0), (3, 0.5), (4, 0.3)])
def test_pipe_t1_is_P_in_only(n_parts, p):
    g = small_graph(seed=2)
    c = cfg([9, 8, 7, 4], p=p)
    params = glorot_params(c.widths, 3)
    part_of = contiguous_map(g.n, n_parts)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    rec = pipegcn.run(g, parts, params, c, 1, mode="pipe")[0]
    # O1 on the graph with cross-partition edges removed, full-graph degrees kept
    deg = np.diff(g.row_ptr)
    rows = np.repeat(np.arange(g.n), deg)
    keep = part_of[rows] == part_of[g.col_idx]

    class G:
        pass
    gi = G()
    gi.n, gi.X, gi.labels, gi.train_mask = g.n, g.X, g.labels, g.train_mask
    gi.row_ptr = np.zeros(g.n + 1, np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=g.n), out=gi.row_ptr[1:])
    gi.col_idx = g.col_idx[keep]
    inv_full = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
    ref = sage.forward_backward(gi, params, 1, c, inv_deg=inv_full)
    assert np.isclose(rec["loss"], ref["loss"], rtol=1e-12)
    for l in range(1, 4):
        assert close(assemble(parts, rec["H"][l], g.n, c.widths[l]), ref["H"][l])
    for (a, b), (x, y) in zip(rec["G"], ref["grads"]):
        assert close(a, x) and close(b, y)


def test_golden_tiny4_pipe_t1(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "tiny4.json")))

    class G:
        pass
    g = G()
    g.n = 4
    g.row_ptr, g.col_idx = np.array(gd["row_ptr"]), np.array(gd["col_idx"])
    g.X = np.array(gd["X"])
    g.labels = np.zeros(4, np.int32)
    g.train_mask = np.ones(4, np.uint8)
    c = cfg([1, 1])
    parts = partition(4, g.row_ptr, g.col_idx, 2)
    recs = pipegcn.run(g, parts, [(np.array(gd["W"]), np.array(gd["b"]))], c, 2, mode="pipe")
    np.testing.assert_allclose(recs[0]["H"][1][0][:, 0], gd["pipe_t1"]["Y_part0"], rtol=1e-15)
    np.testing.assert_allclose(recs[0]["H"][1][1][:, 0], gd["pipe_t1"]["Y_part1"], rtol=1e-15)
    # t = 2: the X boundary rows have arrived -> full-graph values (layer 1 is exact)
    np.testing.assert_allclose(np.concatenate([recs[1]["H"][1][0][:, 0], recs[1]["H"][1][1][:, 0]]),
                               gd["full"]["Y"], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("n_parts", [2, 3])
def test_matrix_form_app_a1(n_parts):
    """App. A.1, GraphSAGE form, p = 0, eta > 0 (weights change):
    Z^(t) = P_in H^(t) + P_bd H^(t-1);  J^(t,l-1) = P_in^T dZ^(t) + P_bd^T dZ^(t-1) + dD_self^(t)
    with dZ^(t) = M^(t) W_neigh^(t)T and dZ^(t-1) = M^(t-1) W_neigh^(t-1)T (stale weights, l.675)."""
    g = small_graph(seed=3, n=150)
    widths = [9, 8, 7, 4]
    c = cfg(widths, p=0.0, lr=0.3)
    params0 = glorot_params(widths, 5)
    part_of = contiguous_map(g.n, n_parts)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    T = 5
    recs = pipegcn.run(g, parts, params0, c, T, mode="pipe")
    deg = np.diff(g.row_ptr)
    rows = np.repeat(np.arange(g.n), deg)
    inv = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
    same = part_of[rows] == part_of[g.col_idx]
    P_in = sp.csr_matrix((inv[rows] * same, (rows, g.col_idx)), shape=(g.n, g.n))
    P_bd = sp.csr_matrix((inv[rows] * ~same, (rows, g.col_idx)), shape=(g.n, g.n))
    L = 3
    Ws = [[(np.asarray(W, float), np.asarray(b, float)) for W, b in params0]] + [r["params"] for r in recs]
    X = g.X.astype(np.float64)

    def Hfull(t, l):          # H^(t,l) over all nodes (l = 0 -> X)
        return X if l == 0 else assemble(parts, recs[t - 1]["H"][l], g.n, widths[l])

    def Mfull(t, l):
        J = assemble(parts, recs[t - 1]["J"][l], g.n, widths[l])
        Y = assemble(parts, recs[t - 1]["Y"][l], g.n, widths[l])
        return J * (Y > 0) if l < L else J

    for t in range(2, T + 1):
        W_t = Ws[t - 1]
        for l in range(1, L + 1):
            W, b = W_t[l - 1]
            Z = P_in @ Hfull(t, l - 1) + P_bd @ Hfull(t - 1, l - 1)
            Y = np.hstack([Z, Hfull(t, l - 1)]) @ W + b
            H = np.maximum(Y, 0) if l < L else Y
            assert close(Hfull(t, l), H, 1e-11), (t, l)
        for l in range(L, 1, -1):
            F = widths[l - 1]
            Wn, Ws_ = W_t[l - 1][0][:F], W_t[l - 1][0][F:]
            Wn_old = Ws[t - 2][l - 1][0][:F]
            Mt, Mo = Mfull(t, l), Mfull(t - 1, l)
            J = P_in.T @ (Mt @ Wn.T) + P_bd.T @ (Mo @ Wn_old.T) + Mt @ Ws_.T
            assert close(assemble(parts, recs[t - 1]["J"][l - 1], g.n, F), J, 1e-11), (t, l)


@pytest.mark.parametrize("L", [2, 3, 4])
def test_eta0_pipe_gradients_equal_vanilla_after_2L(L):
    g = small_graph(seed=4)
    widths = [9] + [8] * (L - 1) + [4]
    c = cfg(widths, p=0.0, lr=0.0)
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    T = 2 * L + 2
    van = pipegcn.run(g, parts, params, c, T, mode="vanilla")
    pip = pipegcn.run(g, parts, params, c, T, mode="pipe")

    def gerr(t):
        return max(np.abs(a - x).max() for (a, _), (x, _) in zip(pip[t - 1]["G"], van[t - 1]["G"]))
    assert gerr(1) > 1e-6                     # staleness is real at t = 1
    for t in range(2 * L, T + 1):
        assert gerr(t) <= 1e-13 * max(np.abs(x).max() for x, _ in van[t - 1]["G"]), t


@pytest.mark.parametrize("sf,sg", [(True, False), (False, True), (True, True)])
def test_ema_gamma0_is_identity(sf, sg):
    g = small_graph(seed=5)
    c = cfg([9, 8, 7, 4], p=0.5, lr=0.1)
    params = glorot_params(c.widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    a = pipegcn.run(g, parts, params, c, 4, mode="pipe")
    b = pipegcn.run(g, parts, params, c, 4, mode="pipe", smooth_f=sf, smooth_g=sg, gamma=0.0)
    for ra, rb in zip(a, b):
        assert ra["loss"] == rb["loss"]
        for (x, y), (u, v) in zip(ra["G"], rb["G"]):
            assert np.array_equal(x, u) and np.array_equal(y, v)


def test_ema_converges_geometrically_eta0():
    g = small_graph(seed=6)
    gamma = 0.9
    widths = [9, 8, 7, 4]
    c = cfg(widths, p=0.0, lr=0.0, gamma=gamma)
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 2)
    T = 40
    van = pipegcn.run(g, parts, params, c, 2, mode="vanilla")
    pip = pipegcn.run(g, parts, params, c, T, mode="pipe", smooth_f=True, smooth_g=True)
    err = [max(np.abs(a - x).max() for (a, _), (x, _) in zip(r["G"], van[-1]["G"])) for r in pip]
    tail = err[8:]
    assert all(b <= a * 1.0000001 for a, b in zip(tail, tail[1:]))           # monotone
    for t in range(8, T - 6):
        assert err[t + 6] <= (gamma + 0.03) ** 6 * err[t]


def test_layer1_exact_for_t_ge_2():
    g = small_graph(seed=7)
    c = cfg([9, 8, 7, 4], p=0.5, lr=0.2)
    params = glorot_params(c.widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    recs = pipegcn.run(g, parts, params, c, 5, mode="pipe", smooth_f=True)
    Ws = [params] + [r["params"] for r in recs]
    for t in range(2, 6):
        ref = sage.forward_backward(g, Ws[t - 1], t, c)
        assert close(assemble(parts, recs[t - 1]["H"][1], g.n, 8), ref["H"][1], 1e-12)


def test_staleness_error_definition():
    """Fig. 5/7: err = ||used - fresh||_F.  Vanilla uses fresh values (0); at t = 1
    PIPE uses zero boundary rows, so err_f equals the norm of the owners' fresh rows (recomputed
    here from the recorded layer outputs by gid); with eta = 0, p = 0 both errors vanish once the
    pipeline has filled (t >= 2L); gamma = 0 smoothing gives the unsmoothed errors exactly."""
    g = small_graph(seed=8)
    widths = [9, 8, 7, 4]
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    c = cfg(widths, p=0.0, lr=0.2)
    van = pipegcn.run(g, parts, params, c, 3, mode="vanilla")
    assert all(v == 0.0 for r in van for v in list(r["err_f"].values()) + list(r["err_g"].values()))
    pip = pipegcn.run(g, parts, params, c, 3, mode="pipe")
    H1 = assemble(parts, pip[0]["H"][1], g.n, widths[1])
    fresh = np.concatenate([H1[P["halo_gid"]] for P in parts])
    assert np.isclose(pip[0]["err_f"][2], np.linalg.norm(fresh), rtol=1e-13)
    c0 = cfg(widths, p=0.0, lr=0.0)
    L = 3
    z = pipegcn.run(g, parts, params, c0, 2 * L + 1, mode="pipe")
    assert z[0]["err_f"][2] > 0 and z[0]["err_g"][2] > 0
    for t in range(2 * L, 2 * L + 1):
        for l in range(1, L + 1):
            assert z[t - 1]["err_f"][l] <= 1e-12 * max(1.0, z[0]["err_f"][2])
        for l in range(2, L + 1):
            assert z[t - 1]["err_g"][l] <= 1e-12 * max(1.0, z[0]["err_g"][2])
    s0 = pipegcn.run(g, parts, params, c, 3, mode="pipe", smooth_f=True, smooth_g=True, gamma=0.0)
    for a, b in zip(pip, s0):
        assert a["err_f"] == b["err_f"] and a["err_g"] == b["err_g"]


# ---------------------------------------------------------------- pipeline depth s (reading R27)
@pytest.mark.parametrize("n_parts,depth", [(2, 2), (3, 3)])
def test_depth_matrix_form(n_parts, depth):
    """App. A.1's matrix form with the one-iteration delay replaced by s:
    Z^(t) = P_in H^(t) + P_bd H^(t-s) for t > s;  J^(t,l-1) = P_in^T M^(t) W^(t)T_neigh +
    P_bd^T M^(t-s) W^(t-s)T_neigh + M^(t) W^(t)T_self (sender's weights of iteration t - s)."""
    g = small_graph(seed=9, n=150)
    widths = [9, 8, 7, 4]
    c = cfg(widths, p=0.0, lr=0.3)
    params0 = glorot_params(widths, 5)
    part_of = contiguous_map(g.n, n_parts)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    T = depth + 4
    recs = pipegcn.run(g, parts, params0, c, T, mode="pipe", depth=depth)
    deg = np.diff(g.row_ptr)
    rows = np.repeat(np.arange(g.n), deg)
    inv = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
    same = part_of[rows] == part_of[g.col_idx]
    P_in = sp.csr_matrix((inv[rows] * same, (rows, g.col_idx)), shape=(g.n, g.n))
    P_bd = sp.csr_matrix((inv[rows] * ~same, (rows, g.col_idx)), shape=(g.n, g.n))
    L = 3
    Ws = [[(np.asarray(W, float), np.asarray(b, float)) for W, b in params0]] + [r["params"] for r in recs]
    X = g.X.astype(np.float64)

    def Hf(t, l):
        return X if l == 0 else assemble(parts, recs[t - 1]["H"][l], g.n, widths[l])

    def Mf(t, l):
        J = assemble(parts, recs[t - 1]["J"][l], g.n, widths[l])
        Y = assemble(parts, recs[t - 1]["Y"][l], g.n, widths[l])
        return J * (Y > 0) if l < L else J

    for t in range(1, T + 1):
        for l in range(1, L + 1):
            W, b = Ws[t - 1][l - 1]
            Hold = Hf(t - depth, l - 1) if t > depth else np.zeros_like(Hf(t, l - 1))
            Y = np.hstack([P_in @ Hf(t, l - 1) + P_bd @ Hold, Hf(t, l - 1)]) @ W + b
            assert close(Hf(t, l), np.maximum(Y, 0) if l < L else Y, 1e-11), (t, l)
        for l in range(L, 1, -1):
            F = widths[l - 1]
            Wt = Ws[t - 1][l - 1][0]
            J = P_in.T @ (Mf(t, l) @ Wt[:F].T) + Mf(t, l) @ Wt[F:].T
            if t > depth:
                J = J + P_bd.T @ (Mf(t - depth, l) @ Ws[t - 1 - depth][l - 1][0][:F].T)
            assert close(assemble(parts, recs[t - 1]["J"][l - 1], g.n, F), J, 1e-11), (t, l)


@pytest.mark.parametrize("depth", [2, 3])
def test_depth_eta0_converges_to_vanilla(depth):
    """eta = 0, p = 0: with an s-deep pipeline every stale value is exact once the pipeline has
    filled (t >= 2 s L), and not before (t = s + 1 still sees stale gradients)."""
    L = 3
    g = small_graph(seed=10)
    widths = [9, 8, 7, 4]
    c = cfg(widths, p=0.0, lr=0.0)
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    T = 2 * depth * L + 1
    van = pipegcn.run(g, parts, params, c, 1, mode="vanilla")
    pip = pipegcn.run(g, parts, params, c, T, mode="pipe", depth=depth)

    def gerr(t):
        return max(np.abs(a - x).max() for (a, _), (x, _) in zip(pip[t - 1]["G"], van[0]["G"]))
    scale = max(np.abs(x).max() for x, _ in van[0]["G"])
    assert gerr(depth + 1) > 1e-6 * scale
    for t in range(2 * depth * L, T + 1):
        assert gerr(t) <= 1e-13 * scale, t
    # depth s at t <= s is the t = 1 computation with the weights of t (here unchanged): identical
    for t in range(2, depth + 1):
        assert pip[t - 1]["loss"] == pip[0]["loss"]


def test_depth_ema_gamma0_is_identity():
    g = small_graph(seed=11)
    c = cfg([9, 8, 7, 4], p=0.5, lr=0.1)
    params = glorot_params(c.widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    a = pipegcn.run(g, parts, params, c, 5, mode="pipe", depth=2)
    b = pipegcn.run(g, parts, params, c, 5, mode="pipe", depth=2, smooth_f=True, smooth_g=True, gamma=0.0)
    for ra, rb in zip(a, b):
        assert ra["loss"] == rb["loss"]


@pytest.mark.parametrize("ema_init", ["first", "zero"])
@pytest.mark.parametrize("depth", [1, 2])
def test_ema_f_transient_closed_form(ema_init, depth):
    """EMA-F transient values (Sec. 3.4; readings R12, R14, R27), pinned by the EMA
    recursion's closed form.  With eta = 0 and p = 0 the owners' layer-1 rows take two values only:
    a = H1 computed with zero X boundary rows (t <= s, Alg. 1 l.6) and b = the full-graph H1 once X's
    boundary rows are installed (t > s; O1, oracle/sage.py).  The layer-2 boundary rows consumed at t carry
    the rows sent at t - s, so the messages are a for t in [s+1, 2s] and b afterwards, and the smoothed
    rows are
      t in [s+1, 2s]: first-receipt init a;  zero init (1 - gamma^(t-s)) a
      t >= 2s:        gamma^(t-2s) c + (1 - gamma^(t-2s)) b,  c = a (first) or (1 - gamma^s) a (zero).
    A swapped gamma / 1 - gamma, a late or early first receipt, or smoothing the fresh instead of the
    stale rows fails it."""
    g = small_graph(seed=11)
    widths = [9, 8, 4]
    gamma = 0.7
    c = cfg(widths, p=0.0, lr=0.0, gamma=gamma)
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    T = 2 * depth + 5
    recs = pipegcn.run(g, parts, params, c, T, mode="pipe", smooth_f=True, ema_init=ema_init, depth=depth)
    a = assemble(parts, recs[0]["H"][1], g.n, widths[1])      # t = 1: zero X boundary rows
    b = sage.forward_backward(g, params, 1, c)["H"][1]        # full graph (p = 0: no mask)
    assert np.abs(a - b).max() > 1e-3                         # the transient is not trivial
    s = depth
    for t in range(s + 1, T + 1):
        if t <= 2 * s:
            exp = a if ema_init == "first" else (1.0 - gamma ** (t - s)) * a
        else:
            c0 = a if ema_init == "first" else (1.0 - gamma ** s) * a
            k = t - 2 * s
            exp = gamma ** k * c0 + (1.0 - gamma ** k) * b
        for i, P in enumerate(parts):
            got = recs[t - 1]["halo"][2][i]
            assert close(got, exp[P["halo_gid"]], 1e-12), (t, i)


def test_ema_g_transient_closed_form():
    """EMA-G transient (Sec. 3.4; readings R12, R13), first-receipt init, eta = 0, p = 0,
    L = 2, no feature smoothing.  The forward is constant from t = 3 on (layer-2 halos = the full-graph H1
    sent at t >= 2), so the raw gradient messages consumed at t are m1 (t = 2), m2 (t = 3) and m* (t >= 4),
    and the smoothed run differs from the plain one only through C_hat - C summed per row (S):
      t = 2: 0;   t = 3: gamma S(m1 - m2);   t >= 4: gamma^(t-3) (gamma S(m1 - m2) + S(m2 - m*)),
    where S(m2 - m*) = J_plain(3) - J_plain(4) (same local term from t = 3 on).  So the accumulated J^(1)
    must satisfy J_g(t) - J_p(t) = gamma^(t-3) [(J_g(3) - J_p(3)) + (J_p(3) - J_p(4))] for t >= 4."""
    g = small_graph(seed=12)
    widths = [9, 8, 4]
    gamma = 0.6
    c = cfg(widths, p=0.0, lr=0.0, gamma=gamma)
    params = glorot_params(widths, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3)
    T = 8
    plain = pipegcn.run(g, parts, params, c, T, mode="pipe")
    smooth = pipegcn.run(g, parts, params, c, T, mode="pipe", smooth_g=True)
    Jp = [assemble(parts, r["J"][1], g.n, widths[1]) for r in plain]
    Jg = [assemble(parts, r["J"][1], g.n, widths[1]) for r in smooth]
    assert close(Jg[1], Jp[1], 1e-13)                      # t = 2: the first receipt is the message itself
    d3 = Jg[2] - Jp[2]
    assert np.abs(d3).max() > 1e-6 * np.abs(Jp[2]).max()     # the transient is not trivial
    base = d3 + (Jp[2] - Jp[3])
    for t in range(4, T + 1):
        assert np.allclose(Jg[t - 1] - Jp[t - 1], gamma ** (t - 3) * base, rtol=0, atol=1e-12 * np.abs(Jp[2]).max()), t
