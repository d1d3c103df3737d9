"""Pins for the GCN-sym model of the oracle (N3; App. A.1, reading R26).

P = D~^-1/2 (A + I) D~^-1/2 with D~ = diag(d + 1); layer Y = P D W + b.  Checked against things
other than the oracle's own formula:
* closed-form spectral facts of the normalised adjacency: P symmetric, P D~^1/2 1 = D~^1/2 1
  (eigenvalue 1), spectrum in (-1, 1]
* on a k-regular graph P = (A + I)/(k + 1), so GCN training equals the (already pinned)
  GraphSAGE-mean training with W_neigh = k/(k+1) W, W_self = W/(k+1): losses, J and the gradient
  G_gcn = k/(k+1) G_neigh + 1/(k+1) G_self agree over several SGD steps
* an isolated node keeps its own row (P_vv = 1)
* float64 finite differences of the loss
* O2 (vanilla) == O1, O3 at t = 1 == O1 on P_in with full-graph degrees (Alg. 1 l.6), and O3 ==
  the App. A.1 matrix form Z = P_in H^(t) W + P_bd H^(t-1) W, J = P_in^T M W^T + P_bd^T M' W'^T
"""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import pipegcn, sage
from oracle.partition import contiguous_map, partition
from synth.graphs import ModelCfg, gen_graph, glorot_params, random_graph


class G:
    pass


def circulant(n, k, f0, classes, seed):
    """k-regular ring lattice: v ~ v +- 1..k/2 (mod n), neighbours in ascending order."""
    rng = np.random.default_rng(seed)
    g = G()
    g.n = n
    nb = [sorted({(v + s) % n for s in range(1, k // 2 + 1)} | {(v - s) % n for s in range(1, k // 2 + 1)})
          for v in range(n)]
    g.row_ptr = np.concatenate([[0], np.cumsum([len(x) for x in nb])]).astype(np.int64)
    g.col_idx = np.concatenate(nb).astype(np.int64)
    g.X = rng.normal(size=(n, f0)).astype(np.float32)
    g.labels = rng.integers(0, classes, n).astype(np.int32)
    g.train_mask = (rng.random(n) < 0.6).astype(np.uint8)
    return g


def cfg(widths, p=0.0, lr=0.1, loss="ce", model="gcn", opt="sgd"):
    return ModelCfg(widths=widths, dropout=p, lr=lr, opt=opt, loss=loss, model=model)


def close(a, b, rtol=1e-10):
    a, b = np.asarray(a), np.asarray(b)
    return np.abs(a - b).max() <= rtol * max(np.abs(b).max(), 1e-300)


def assemble(parts, per_part, n, width):
    out = np.full((n, width), np.nan)
    for P, a in zip(parts, per_part):
        out[P["inner_gid"]] = a
    return out


@pytest.mark.parametrize("seed", range(4))
def test_normalised_adjacency_spectral_facts(seed):
    g = random_graph(40, 0.12, seed, f0=3, isolated=2)
    P = sage.prop_matrix(g.n, g.row_ptr, g.col_idx, model="gcn").toarray()
    assert np.allclose(P, P.T, atol=1e-15)
    d = np.diff(g.row_ptr) + 1.0
    x = np.sqrt(d)
    assert np.allclose(P @ x, x, rtol=1e-13)                     # D~^1/2 1 is an eigenvector, lambda = 1
    ev = np.linalg.eigvalsh(P)
    assert ev.max() <= 1 + 1e-12 and ev.min() > -1 - 1e-12
    iso = np.nonzero(np.diff(g.row_ptr) == 0)[0]
    assert iso.size and all(P[v, v] == 1.0 and P[v].sum() == 1.0 for v in iso)


@pytest.mark.parametrize("k,L,p", [(2, 2, 0.0), (4, 3, 0.0), (6, 3, 0.4)])
def test_regular_graph_equals_sage_training(k, L, p):
    g = circulant(36, k, 5, 3, seed=k)
    widths = [5] + [6] * (L - 1) + [3]
    gp = glorot_params(widths, 2, model="gcn")
    a, c = k / (k + 1.0), 1.0 / (k + 1.0)
    sp_ = [(np.vstack([a * W.astype(np.float64), c * W.astype(np.float64)]), b) for W, b in gp]
    T = 4
    rg = sage.train_full(g, gp, cfg(widths, p=p, lr=0.3), T)
    rs = sage.train_full(g, sp_, cfg(widths, p=p, lr=0.3, model="sage"), 1)
    assert np.isclose(rg[0]["loss"], rs[0]["loss"], rtol=1e-13)
    for l in range(1, L):
        assert close(rg[0]["J"][l], rs[0]["J"][l], 1e-12)
    for (gW, gb), (sW, sb) in zip(rg[0]["grads"], rs[0]["grads"]):
        F = gW.shape[0]
        assert close(gW, a * sW[:F] + c * sW[F:], 1e-12) and close(gb, sb, 1e-12)
    # later iterations: map the GCN trajectory's weights to SAGE and compare the next step
    for t in range(2, T + 1):
        pw = rg[t - 2]["params"]
        ps = [(np.vstack([a * W, c * W]), b) for W, b in pw]
        r = sage.forward_backward(g, ps, t, cfg(widths, p=p, model="sage"))
        assert np.isclose(rg[t - 1]["loss"], r["loss"], rtol=1e-12)


@pytest.mark.parametrize("loss,p,L", [("ce", 0.0, 2), ("ce", 0.5, 3), ("bce", 0.3, 2)])
def test_finite_differences(loss, p, L):
    ml = loss == "bce"
    g = random_graph(14, 0.3, 5, f0=3, classes=3, multilabel=ml, isolated=1)
    widths = [3] + [4] * (L - 1) + [3]
    c = cfg(widths, p=p, loss=loss)
    params = [(W.astype(np.float64) * 2.0, np.random.default_rng(9).normal(size=b.shape) * 0.1)
              for W, b in glorot_params(widths, 7, model="gcn")]
    t = 2
    out = sage.forward_backward(g, params, t, c)
    rng = np.random.default_rng(0)
    eps = 1e-6
    checked = 0
    for l in range(L):
        for which in (0, 1):
            arr = params[l][which]
            for _ in range(6):
                idx = tuple(rng.integers(0, s) for s in arr.shape)

                def f(delta):
                    pp = [(W.copy(), b.copy()) for W, b in params]
                    pp[l][which][idx] += delta
                    return sage.forward_backward(g, pp, t, c)["loss"]
                fd = (f(eps) - f(-eps)) / (2 * eps)
                fd2 = (f(2 * eps) - f(-2 * eps)) / (4 * eps)
                if abs(fd - fd2) > 1e-7 * max(1.0, abs(fd)):
                    continue                                          # ReLU kink inside the stencil
                an = out["grads"][l][which][idx]
                assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)), (l, which, idx, fd, an)
                checked += 1
    assert checked >= 4 * L


def small_graph(seed=1, n=120):
    return gen_graph("cora", seed=seed, n=n, nnz=n * 6, f0=9, classes=4, comm=4)


@pytest.mark.parametrize("n_parts", [1, 2, 4])
@pytest.mark.parametrize("p", [0.0, 0.5])
def test_vanilla_equals_full_graph(n_parts, p):
    g = small_graph()
    c = cfg([9, 8, 6, 4], p=p, lr=0.2)
    params = glorot_params(c.widths, 3, model="gcn")
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts)
    T = 3
    full = sage.train_full(g, params, c, T)
    van = pipegcn.run(g, parts, params, c, T, mode="vanilla")
    for t in range(T):
        assert np.isclose(van[t]["loss"], full[t]["loss"], rtol=1e-12)
        for l in range(1, 3):
            assert close(assemble(parts, van[t]["J"][l], g.n, c.widths[l]), full[t]["J"][l])
        for (a, b), (x, y) in zip(van[t]["G"], full[t]["grads"]):
            assert close(a, x) and close(b, y)


def test_pipe_t1_is_P_in_only_with_full_degrees():
    g = small_graph(seed=2)
    c = cfg([9, 8, 7, 4], p=0.3)
    params = glorot_params(c.widths, 3, model="gcn")
    part_of = contiguous_map(g.n, 3)
    parts = partition(g.n, g.row_ptr, g.col_idx, 3, part_of)
    rec = pipegcn.run(g, parts, params, c, 1, mode="pipe")[0]
    deg = np.diff(g.row_ptr)
    rows = np.repeat(np.arange(g.n), deg)
    keep = part_of[rows] == part_of[g.col_idx]
    gi = G()
    gi.n, gi.X, gi.labels, gi.train_mask = g.n, g.X, g.labels, g.train_mask
    gi.row_ptr = np.zeros(g.n + 1, np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=g.n), out=gi.row_ptr[1:])
    gi.col_idx = g.col_idx[keep]
    ref = sage.forward_backward(gi, params, 1, c, deg_full=deg)
    assert np.isclose(rec["loss"], ref["loss"], rtol=1e-12)
    for (a, b), (x, y) in zip(rec["G"], ref["grads"]):
        assert close(a, x) and close(b, y)


@pytest.mark.parametrize("n_parts", [2, 3])
def test_matrix_form_app_a1(n_parts):
    """App. A.1 verbatim (GCN form): Z^(t,l) = P_in H^(t,l-1) W^(t) + P_bd
    H^(t-1,l-1) W^(t) + b; J^(t,l-1) = P_in^T M^(t,l) W^(t)T + P_bd^T M^(t-1,l) W^(t-1)T."""
    g = small_graph(seed=3, n=150)
    widths = [9, 8, 7, 4]
    c = cfg(widths, lr=0.3)
    params0 = glorot_params(widths, 5, model="gcn")
    part_of = contiguous_map(g.n, n_parts)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    T = 5
    recs = pipegcn.run(g, parts, params0, c, T, mode="pipe")
    Pfull = sage.prop_matrix(g.n, g.row_ptr, g.col_idx, model="gcn").tocoo()
    same = part_of[Pfull.row] == part_of[Pfull.col]
    P_in = sp.csr_matrix((Pfull.data * same, (Pfull.row, Pfull.col)), shape=(g.n, g.n))
    P_bd = sp.csr_matrix((Pfull.data * ~same, (Pfull.row, Pfull.col)), shape=(g.n, g.n))
    L = 3
    Ws = [[(np.asarray(W, float), np.asarray(b, float)) for W, b in params0]] + [r["params"] for r in recs]
    X = g.X.astype(np.float64)

    def Hf(t, l):
        return X if l == 0 else assemble(parts, recs[t - 1]["H"][l], g.n, widths[l])

    def Mf(t, l):
        J = assemble(parts, recs[t - 1]["J"][l], g.n, widths[l])
        Y = assemble(parts, recs[t - 1]["Y"][l], g.n, widths[l])
        return J * (Y > 0) if l < L else J

    for t in range(2, T + 1):
        for l in range(1, L + 1):
            W, b = Ws[t - 1][l - 1]
            Y = P_in @ Hf(t, l - 1) @ W + P_bd @ Hf(t - 1, l - 1) @ W + b
            assert close(Hf(t, l), np.maximum(Y, 0) if l < L else Y, 1e-11), (t, l)
        for l in range(L, 1, -1):
            W, W_old = Ws[t - 1][l - 1][0], Ws[t - 2][l - 1][0]
            J = P_in.T @ (Mf(t, l) @ W.T) + P_bd.T @ (Mf(t - 1, l) @ W_old.T)
            assert close(assemble(parts, recs[t - 1]["J"][l - 1], g.n, widths[l - 1]), J, 1e-11), (t, l)
