"""O1: full-graph GraphSAGE-mean training -- test infrastructure only (see oracle/__init__.py).

Layer l (Eq. 1-2; GraphSAGE update PAPER.md:44; mean aggregator Eq. 3
PAPER.md:456 without partitions; dropout after communication PAPER.md:983):

    D^(l)  = dropout_{t,l}(H^(l-1))                      (reading R5)
    Z^(l)  = P D^(l),   P[v,u] = 1/d_v for u in N(v)      (Eq. 3; R1)
    A^(l)  = [Z^(l) | D^(l)]                             (CONCAT(z_v, h_v); R3)
    Y^(l)  = A^(l) W^(l) + b^(l)                         (R4: bias on every layer)
    H^(l)  = ReLU(Y^(l)) for l < L, Y^(L) for l = L      (R4)

Backward (App. A.1 PAPER.md:651-657 with sigma' = 1[Y > 0], and Alg. 1 l.18-20):

    M^(l)    = J^(l) o sigma'(Y^(l))   (M^(L) = J^(L))
    G^(l)    = A^(l)T M^(l),  g_b^(l) = sum_v M^(l)_v
    dA       = M^(l) W^(l)T = [dZ | dD_self]
    J^(l-1)  = (P^T dZ + dD_self) o keep / (1 - p)

Loss (reading R6): mean over the global train set -- softmax cross-entropy over N_train,
or sigmoid BCE over N_train * C.  `inv_deg` may be overridden to pin Alg. 1 l.6 (zero
boundary features at t = 1: O1 on the graph without cross edges, degrees unchanged).
"""
import numpy as np
import scipy.sparse as sp

from .hashmask import dropout


def prop_matrix(n, row_ptr, col_idx, inv_deg=None, model="sage", deg_full=None):
    """sage: P[v, u] = inv_deg[v] for u in N(v) (Eq. 3).
    gcn:  P = D~^-1/2 (A + I) D~^-1/2 (App. A.1) with D~ = deg_full + 1 (deg_full
          defaults to the row lengths; overridden to pin Alg. 1 l.6 with full-graph degrees)."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    deg = np.diff(row_ptr)
    if model == "gcn":
        d = deg if deg_full is None else np.asarray(deg_full)
        s = 1.0 / np.sqrt(d.astype(np.float64) + 1.0)
        rows = np.repeat(np.arange(n), deg)
        cols = np.asarray(col_idx, dtype=np.int64)
        r = np.concatenate([rows, np.arange(n)])
        c = np.concatenate([cols, np.arange(n)])
        return sp.csr_matrix((s[r] * s[c], (r, c)), shape=(n, n))
    if inv_deg is None:
        inv_deg = np.where(deg > 0, 1.0 / np.maximum(deg, 1), 0.0)
    vals = np.repeat(np.asarray(inv_deg, dtype=np.float64), deg)
    return sp.csr_matrix((vals, np.asarray(col_idx, dtype=np.int64), row_ptr), shape=(n, n))


def loss_and_grad(Y, labels, train_mask, n_train, kind):
    """(loss, J = dLoss/dY) for the rows of Y.  Rows outside the train mask get J = 0.
    CE:  loss = sum_train -log softmax(Y_v)[y_v] / n_train
    BCE: loss = sum_train sum_c [log(1 + e^{Y}) - y Y] / (n_train * C)."""
    Y = np.asarray(Y, dtype=np.float64)
    m = np.asarray(train_mask).astype(bool)
    J = np.zeros_like(Y)
    if kind == "ce":
        Ym = Y[m]
        mx = Ym.max(1, keepdims=True)
        e = np.exp(Ym - mx)
        s = e.sum(1, keepdims=True)
        prob = e / s
        y = np.asarray(labels)[m].astype(np.int64)
        logp = (Ym - mx - np.log(s))[np.arange(y.size), y]
        loss = -logp.sum() / n_train
        g = prob.copy()
        g[np.arange(y.size), y] -= 1.0
        J[m] = g / n_train
    elif kind == "bce":
        C = Y.shape[1]
        Ym = Y[m]
        y = np.asarray(labels)[m].astype(np.float64)
        sp_ = np.logaddexp(0.0, Ym)
        loss = (sp_ - y * Ym).sum() / (n_train * C)
        J[m] = (1.0 / (1.0 + np.exp(-Ym)) - y) / (n_train * C)
    else:
        raise ValueError(kind)
    return float(loss), J


def forward_backward(g, params, t, cfg, seed=4, inv_deg=None, n_train=None, deg_full=None):
    """One full-graph iteration t: returns dict(H, A, Y, loss, J, grads).
    g: synth.Graph-like (n, row_ptr, col_idx, X, labels, train_mask); params: [(W, b)].
    cfg.model "sage" (default, A = [PD | D], W = [W_neigh; W_self]) or "gcn" (A = P D, App. A.1
    PAPER.md:637-647 with the bias of reading R26)."""
    n = g.n
    L = len(params)
    model = getattr(cfg, "model", "sage")
    P = prop_matrix(n, g.row_ptr, g.col_idx, inv_deg, model, deg_full)
    gids = np.arange(n)
    p = cfg.dropout
    H = np.asarray(g.X, dtype=np.float64)
    out = dict(H=[H], A=[], Y=[], keep=[])
    for l in range(1, L + 1):
        W, b = (np.asarray(a, dtype=np.float64) for a in params[l - 1])
        D, keep = dropout(H, t, l, L, n, gids, seed, p)
        Z = P @ D
        A = np.hstack([Z, D]) if model == "sage" else Z
        Y = A @ W + b
        H = np.maximum(Y, 0.0) if l < L else Y
        out["A"].append(A)
        out["Y"].append(Y)
        out["keep"].append(keep)
        out["H"].append(H)
    nt = int(np.asarray(g.train_mask).astype(bool).sum()) if n_train is None else n_train
    loss, J = loss_and_grad(out["Y"][-1], g.labels, g.train_mask, nt, cfg.loss)
    out["loss"] = loss
    Js = {L: J}
    grads = [None] * L
    for l in range(L, 0, -1):
        W = np.asarray(params[l - 1][0], dtype=np.float64)
        M = J * (out["Y"][l - 1] > 0) if l < L else J
        grads[l - 1] = (out["A"][l - 1].T @ M, M.sum(0))
        if l > 1:
            dA = M @ W.T
            s = 1.0 / (1.0 - p) if p > 0 else 1.0
            if model == "sage":
                F = W.shape[0] // 2
                J = (P.T @ dA[:, :F] + dA[:, F:]) * out["keep"][l - 1] * s
            else:
                J = (P.T @ dA) * out["keep"][l - 1] * s
            Js[l - 1] = J
    out["J"] = Js
    out["grads"] = grads
    return out


def sgd_update(params, grads, lr):
    """Alg. 1 l.32: W_t = W_{t-1} - eta * G."""
    return [(W - lr * gW, b - lr * gb) for (W, b), (gW, gb) in zip(params, grads)]


class Adam:
    """Adam (Kingma & Ba 2015) with PyTorch's defaults, the optimiser of Table 3:
    m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;  w -= lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)."""

    def __init__(self, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, beta1, beta2, eps
        self.m = None
        self.v = None
        self.k = 0

    def update(self, params, grads):
        flat_g = [a for gW, gb in grads for a in (gW, gb)]
        if self.m is None:
            self.m = [np.zeros_like(a, dtype=np.float64) for a in flat_g]
            self.v = [np.zeros_like(a, dtype=np.float64) for a in flat_g]
        self.k += 1
        out, it = [], iter(range(len(flat_g)))
        flat_p = [np.asarray(a, dtype=np.float64) for W, b in params for a in (W, b)]
        new = []
        for i in it:
            g = flat_g[i]
            self.m[i] = self.b1 * self.m[i] + (1 - self.b1) * g
            self.v[i] = self.b2 * self.v[i] + (1 - self.b2) * g * g
            mh = self.m[i] / (1 - self.b1 ** self.k)
            vh = self.v[i] / (1 - self.b2 ** self.k)
            new.append(flat_p[i] - self.lr * mh / (np.sqrt(vh) + self.eps))
        for j in range(0, len(new), 2):
            out.append((new[j], new[j + 1]))
        return out


def train_full(g, params0, cfg, T, seed=4, opt=None):
    """Full-graph training for T iterations (t = 1..T); returns list of per-iteration dicts."""
    params = [(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in params0]
    opt = opt or cfg.opt
    adam = Adam(cfg.lr) if opt == "adam" else None
    recs = []
    for t in range(1, T + 1):
        r = forward_backward(g, params, t, cfg, seed)
        params = adam.update(params, r["grads"]) if adam else sgd_update(params, r["grads"], cfg.lr)
        r["params"] = params
        recs.append(r)
    return recs
