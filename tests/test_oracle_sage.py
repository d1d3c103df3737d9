"""Pins for oracle/sage.py (O1 full-graph GraphSAGE-mean; Eq. 1-3, App. A.1)."""
import json
import os

import numpy as np
import pytest

from oracle.sage import Adam, forward_backward, loss_and_grad, sgd_update
from synth.graphs import ModelCfg, glorot_params, random_graph


def dense_P(g):
    """P[v, u] = 1/d_v for u in N(v), built entry by entry from Eq. 3's definition."""
    n = g.n
    P = np.zeros((n, n))
    for v in range(n):
        nb = g.col_idx[g.row_ptr[v]:g.row_ptr[v + 1]]
        for u in nb:
            P[v, u] += 1.0 / len(nb)
    return P


def cfg_for(widths, p=0.0, loss="ce"):
    return ModelCfg(widths=widths, dropout=p, lr=0.1, opt="sgd", loss=loss)


@pytest.mark.parametrize("seed", range(6))
def test_aggregation_matches_dense_bruteforce(seed):
    g = random_graph(30 + seed, 0.15, seed, f0=4, isolated=seed % 2)
    cfg = cfg_for([4, 3], p=0.0)
    params = glorot_params(cfg.widths, seed)
    out = forward_backward(g, params, 1, cfg)
    Z = out["A"][0][:, :4]
    np.testing.assert_allclose(Z, dense_P(g) @ g.X.astype(np.float64), rtol=1e-13, atol=1e-14)
    # isolated nodes aggregate to 0 (reading R1)
    deg = np.diff(g.row_ptr)
    assert (Z[deg == 0] == 0).all()


def test_golden_tiny4_forward(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "tiny4.json")))

    class G:
        pass
    g = G()
    g.n = gd["n"]
    g.row_ptr = np.array(gd["row_ptr"])
    g.col_idx = np.array(gd["col_idx"])
    g.X = np.array(gd["X"])
    g.labels = np.zeros(4, np.int32)
    g.train_mask = np.ones(4, np.uint8)
    cfg = cfg_for([1, 1], p=0.0)
    out = forward_backward(g, [(np.array(gd["W"]), np.array(gd["b"]))], 1, cfg)
    np.testing.assert_allclose(out["A"][0][:, 0], gd["full"]["Z"], rtol=1e-15)
    np.testing.assert_allclose(out["Y"][0][:, 0], gd["full"]["Y"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(np.maximum(out["Y"][0][:, 0], 0), gd["full"]["ReLU_Y"])


def _loss_of(g, params, cfg, t):
    return forward_backward(g, params, t, cfg)["loss"]


@pytest.mark.parametrize("loss,p,L", [("ce", 0.0, 2), ("ce", 0.5, 2), ("bce", 0.3, 3), ("ce", 0.0, 3)])
def test_finite_differences(loss, p, L):
    """Float64 central differences of the O1 loss w.r.t. every W and b entry (sampled)."""
    ml = loss == "bce"
    g = random_graph(14, 0.3, 5, f0=3, classes=3, multilabel=ml, isolated=1)
    widths = [3] + [4] * (L - 1) + [3]
    cfg = cfg_for(widths, p=p, loss=loss)
    params = [(W.astype(np.float64) * 2.0, np.random.default_rng(9).normal(size=b.shape) * 0.1)
              for W, b in glorot_params(widths, 7)]
    t = 3
    out = forward_backward(g, params, t, cfg)
    rng = np.random.default_rng(0)
    eps = 1e-6
    for l in range(L):
        for which in (0, 1):
            arr = params[l][which]
            idxs = [tuple(rng.integers(0, s) for s in arr.shape) for _ in range(6)]
            for idx in idxs:
                def f(delta):
                    pp = [(W.copy(), b.copy()) for W, b in params]
                    pp[l][which][idx] += delta
                    return _loss_of(g, pp, cfg, t)
                # skip ReLU kinks inside the FD stencil
                fd = (f(eps) - f(-eps)) / (2 * eps)
                an = out["grads"][l][which][idx]
                fd2 = (f(2 * eps) - f(-2 * eps)) / (4 * eps)
                if abs(fd - fd2) > 1e-7 * max(1.0, abs(fd)):
                    continue
                assert abs(fd - an) <= 1e-6 * max(1e-3, abs(an)), (l, which, idx, fd, an)


def test_ce_closed_form_properties():
    rng = np.random.default_rng(1)
    Y = rng.normal(size=(7, 5))
    lab = rng.integers(0, 5, 7)
    m = np.array([1, 1, 0, 1, 0, 1, 1], np.uint8)
    loss, J = loss_and_grad(Y, lab, m, 10, "ce")
    assert np.allclose(J.sum(1), 0.0, atol=1e-16)               # softmax grad rows sum to 0
    assert (J[m == 0] == 0).all()
    # uniform logits: loss = log C per train row / n_train
    l0, _ = loss_and_grad(np.zeros((7, 5)), lab, m, 10, "ce")
    assert np.isclose(l0, m.sum() * np.log(5) / 10, rtol=1e-15)
    # BCE at zero logits: log 2 per label
    l1, J1 = loss_and_grad(np.zeros((7, 5)), (rng.random((7, 5)) < .5).astype(np.uint8), m, 10, "bce")
    assert np.isclose(l1, m.sum() * 5 * np.log(2) / 50, rtol=1e-15)


def test_sgd_is_alg1_update():
    W = np.ones((2, 2))
    b = np.zeros(2)
    out = sgd_update([(W, b)], [(np.full((2, 2), 3.0), np.ones(2))], 0.5)
    assert np.array_equal(out[0][0], np.full((2, 2), -0.5)) and np.array_equal(out[0][1], -0.5 * np.ones(2))


def test_adam_matches_torch():
    import torch
    rng = np.random.default_rng(2)
    W = rng.normal(size=(4, 3))
    b = rng.normal(size=3)
    tw = torch.tensor(W.copy(), requires_grad=True)
    tb = torch.tensor(b.copy(), requires_grad=True)
    opt = torch.optim.Adam([tw, tb], lr=0.01)
    adam = Adam(0.01)
    params = [(W, b)]
    for k in range(5):
        gW, gb = rng.normal(size=(4, 3)), rng.normal(size=3) * 1e-3
        tw.grad = torch.tensor(gW)
        tb.grad = torch.tensor(gb)
        opt.step()
        params = adam.update(params, [(gW, gb)])
        np.testing.assert_allclose(params[0][0], tw.detach().numpy(), rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(params[0][1], tb.detach().numpy(), rtol=1e-12, atol=1e-14)
