"""O2 (vanilla partition-parallel) and O3 (PipeGCN) -- test infrastructure only.

Follows Alg. 1 (PAPER.md:104 lines 1-7 and PAPER.md:450 lines 8-35) per partition i,
simulating all n partitions in one process, in the paper's order:

  forward, l = 1..L                                                  (Alg. 1 l.8-15)
    l.9-11  if t > 1: wait thread_f^(l); install the received B^(l) as the
            boundary rows H^(l-1)_{S_{j,i}}  (optionally smoothed, Sec. 3.4)
    l.12-13 send H^(l-1)_{S_{i,j}} to every j (consumed at t + 1)
    l.14    H^(l)_{V_i} = sigma(P_i H^(l-1) W_{t-1}^(l))   -- GraphSAGE form, oracle/sage.py
  l.16    J^(L)_{V_i} = dLoss/dH^(L)
  backward, l = L..1                                                 (Alg. 1 l.17-30)
    l.18    G_i^(l)   = [P_i H^(l-1)]^T (J^(l) o sigma')
    l.20    J^(l-1)   = P_i^T (J^(l) o sigma') W^T     (all rows: inner + boundary)
    l.22-25 wait thread_b^(l); J^(l-1)_{S_{i,j}} += C_j^(l)   (C = gradients sent at t - 1)
    l.27    send J^(l-1)_{S_{j,i}} (the boundary rows) to their owners j
  l.31-32 G = AllReduce(G_i) (sum, ascending i; reading R6);  W_t = W_{t-1} - eta G  (or Adam)

Mode "vanilla" (O2, Fig. 1(a)): each exchange is consumed in the
same iteration (no staleness) -- equal to full-graph training (P = P_in + P_bd).
Mode "pipe" (O3): exchanges are consumed one iteration later (Eq. 3-4, PAPER.md:456-458;
matrix form PAPER.md:661-677).  t = 1: boundary rows are 0 for every layer (l.6, reading
R8) and no gradient is accumulated (reading R9).
Smoothing (Sec. 3.4): `smooth_f` -- EMA of installed boundary features for layers l >= 2
(reading R14); `smooth_g` -- EMA of each received gradient message before the sum
(reading R13).  `ema_init` "first" (reading R12) or "zero".
Dropout is applied after install (App. F) with the gid-keyed mask.
Pipeline depth (`depth` = s, reading R27; the future work of App. C: "using two
iterations of compute to hide one iteration of communication"): an exchange sent at t is consumed
at t + s (s = 1 is Alg. 1); for t <= s boundary rows are 0 and no gradient is accumulated.
"""
import numpy as np

from .hashmask import dropout
from .partition import local_P
from .sage import Adam, loss_and_grad, sgd_update


class _Sparse:
    """The sparse product P @ D of Eq. 3 / P^T @ dA of Alg. 1 l.20 as a library primitive: the same
    float64 matrix product as scipy's `P @ D`, executed by PyTorch's multithreaded CPU CSR kernel
    (scipy's is single-threaded: ~13 s per 256-wide product on a full-size Reddit partition).  No
    blocking or reordering beyond the library's own summation order."""

    def __init__(self, P):
        import warnings

        import torch
        P = P.tocsr()
        self.shape = P.shape
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            self.t = torch.sparse_csr_tensor(torch.from_numpy(P.indptr.astype(np.int64)),
                                             torch.from_numpy(P.indices.astype(np.int64)),
                                             torch.from_numpy(P.data.astype(np.float64)), size=P.shape)

    def __matmul__(self, D):
        import torch
        D = np.ascontiguousarray(D, dtype=np.float64)
        if self.shape[0] == 0 or D.shape[1] == 0 or self.shape[1] == 0:
            return np.zeros((self.shape[0], D.shape[1]))
        return (self.t @ torch.from_numpy(D)).numpy()


def run(g, parts, params0, cfg, T, mode="pipe", smooth_f=False, smooth_g=False, gamma=None,
        ema_init="first", seed=4, opt=None, keep_A=False, relu_decision=None, depth=1):
    """Train for t = 1..T.  Returns a list (one dict per t) with
    loss, H[l][i] (inner rows of layer l output), J[l][i] (inner J^(l) after accumulation),
    halo[l][i] (boundary rows used as input of layer l), G_parts[i], G, params (after update),
    err_f[l] / err_g[l] (Fig. 5/7: Frobenius norm of the boundary features /
    received feature-gradient messages actually used minus the fresh ones of the same iteration;
    0 when nothing is used, e.g. t = 1).

    relu_decision(t, l, i, Y) -> bool mask, optional: the sigma'(Y) = 1[Y > 0] decision used in
    the backward (App. A.1).  Default Y > 0.  Parity tests pass a hook that adopts
    the kernel's decision where |Y| is within the comparison tolerance of 0 (DESIGN.md reading
    R25: a float-decided discrete choice is taken in the kernel's precision on both sides)."""
    assert mode in ("pipe", "vanilla") and depth >= 1
    gamma = cfg.gamma if gamma is None else gamma
    n = len(parts)
    L = len(params0)
    N = g.n
    p = cfg.dropout
    s = 1.0 / (1.0 - p) if p > 0 else 1.0
    model = getattr(cfg, "model", "sage")
    Ps = [_Sparse(local_P(P, model)) for P in parts]
    PTs = [_Sparse(local_P(P, model).T) for P in parts]
    gids = [np.concatenate([P["inner_gid"], P["halo_gid"]]) for P in parts]
    X = np.asarray(g.X, dtype=np.float64)
    labels = np.asarray(g.labels)
    tmask = np.asarray(g.train_mask).astype(bool)
    n_train = int(tmask.sum())
    params = [(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in params0]
    opt = opt or cfg.opt
    adam = Adam(cfg.lr) if opt == "adam" else None

    recv_f = {l: {} for l in range(1, L + 1)}      # recv_f[l][t'] = B^(l) sent at t', per receiver
    ema_f = {l: [None] * n for l in range(1, L + 1)}
    recv_b = {l: {} for l in range(1, L + 1)}      # recv_b[l][t'][owner] = C^(l) sent at t', list per peer
    ema_b = {l: [None] * n for l in range(1, L + 1)}
    recs = []
    for t in range(1, T + 1):
        rec = dict(t=t, H={}, J={}, halo={}, A={}, Y={}, err_f={}, err_g={})
        H_in = [X[P["inner_gid"]] for P in parts]
        saved = {}
        # ---------------- forward (Alg. 1 l.8-15)
        for l in range(1, L + 1):
            W, b = params[l - 1]
            F = H_in[0].shape[1]
            # l.12-13: what i sends to j this iteration = H^(l-1)_{S_{i,j}}
            sent = [[H_in[i][parts[i]["send_idx"][parts[i]["send_off"][j]:parts[i]["send_off"][j + 1]]]
                     for j in range(n)] for i in range(n)]
            # receiver j's boundary block in (owner, gid) order = concat over owners i of sent[i][j]
            arrived = [np.vstack([sent[i][j] for i in range(n)]) if parts[j]["n_halo"] else
                       np.zeros((0, F)) for j in range(n)]
            halos = []
            for i in range(n):
                if mode == "vanilla":
                    halo = arrived[i]
                elif t <= depth:
                    halo = np.zeros((parts[i]["n_halo"], F))                 # l.6 / R8 (R27)
                else:
                    halo = recv_f[l][t - depth][i]                           # l.9-11
                    if smooth_f and l >= 2:
                        if ema_f[l][i] is None:
                            ema_f[l][i] = halo.copy() if ema_init == "first" else \
                                (1.0 - gamma) * halo
                        else:
                            ema_f[l][i] = gamma * ema_f[l][i] + (1.0 - gamma) * halo
                        halo = ema_f[l][i]
                halos.append(halo)
            if mode == "pipe":
                recv_f[l][t] = arrived                                       # consumed at t + depth
                recv_f[l].pop(t - depth, None)
            H_out = []
            for i in range(n):
                full = np.vstack([H_in[i], halos[i]])
                D, keep = dropout(full, t, l, L, N, gids[i], seed, p)
                Z = Ps[i] @ D
                A = np.hstack([Z, D[:parts[i]["n_inner"]]]) if model == "sage" else Z
                Y = A @ W + b
                H_out.append(np.maximum(Y, 0.0) if l < L else Y)
                saved[(l, i)] = (A, Y, keep)
            rec["halo"][l] = halos
            # Fig. 5/7: Frobenius norm of (boundary features used - fresh ones)
            rec["err_f"][l] = float(np.sqrt(sum(((h - a) ** 2).sum() for h, a in zip(halos, arrived))))
            rec["H"][l] = H_out
            if keep_A:
                rec["A"][l] = [saved[(l, i)][0] for i in range(n)]
            rec["Y"][l] = [saved[(l, i)][1] for i in range(n)]
            H_in = H_out
        # ---------------- loss (l.16)
        loss = 0.0
        J = []
        for i, P in enumerate(parts):
            li, Ji = loss_and_grad(H_in[i], labels[P["inner_gid"]], tmask[P["inner_gid"]], n_train,
                                   cfg.loss)
            loss += li
            J.append(Ji)
        rec["loss"] = loss
        rec["J"][L] = J
        # ---------------- backward (l.17-30)
        G_parts = [[None] * L for _ in range(n)]
        for l in range(L, 0, -1):
            W, b = params[l - 1]
            F = W.shape[0] // 2 if model == "sage" else W.shape[0]
            J_in, J_halo = [], []
            for i in range(n):
                A, Y, keep = saved[(l, i)]
                if l < L:
                    mask = (Y > 0) if relu_decision is None else relu_decision(t, l, i, Y)
                    M = J[i] * mask
                else:
                    M = J[i]
                G_parts[i][l - 1] = (A.T @ M, M.sum(0))                      # l.18
                if l > 1:                                                    # l.20
                    dA = M @ W.T
                    if model == "sage":
                        dD = PTs[i] @ dA[:, :F]
                        dD[:parts[i]["n_inner"]] += dA[:, F:]
                    else:
                        dD = PTs[i] @ dA
                    Jf = dD * keep * s
                    J_in.append(Jf[:parts[i]["n_inner"]].copy())
                    J_halo.append(Jf[parts[i]["n_inner"]:])
            if l == 1:
                break
            # message from i to owner j: i's boundary rows owned by j (aligned with S_{j,i})
            cur = [[J_halo[i][parts[i]["halo_off"][j]:parts[i]["halo_off"][j + 1]] for i in range(n)]
                   for j in range(n)]
            esq = 0.0
            for j in range(n):
                if mode == "vanilla":
                    contrib = cur[j]
                elif t <= depth:
                    contrib = None                                           # R9 (R27)
                else:
                    contrib = recv_b[l][t - depth][j]                        # l.22
                    if smooth_g:
                        if ema_b[l][j] is None:
                            ema_b[l][j] = [c.copy() if ema_init == "first" else (1.0 - gamma) * c
                                           for c in contrib]
                        else:
                            ema_b[l][j] = [gamma * e + (1.0 - gamma) * c
                                           for e, c in zip(ema_b[l][j], contrib)]
                        contrib = ema_b[l][j]
                # used minus fresh; nothing received (t = 1) means 0 was used (R9)
                esq += sum((((c if contrib is not None else 0.0) - f) ** 2).sum()
                           for c, f in zip(contrib if contrib is not None else cur[j], cur[j]))
                if contrib is not None:
                    P = parts[j]
                    for i in range(n):                                       # l.23-25
                        seg = P["send_idx"][P["send_off"][i]:P["send_off"][i + 1]]
                        np.add.at(J_in[j], seg, contrib[i])
                if mode == "pipe":
                    recv_b[l].setdefault(t, [None] * n)[j] = cur[j]          # l.27, used at t + depth
            recv_b[l].pop(t - depth, None)
            J = J_in
            rec["J"][l - 1] = J
            rec["err_g"][l] = float(np.sqrt(esq))  # gradient messages used vs fresh (Fig. 5/7)
        # ---------------- l.31-32
        G = []
        for l in range(L):
            gW = sum(G_parts[i][l][0] for i in range(n))
            gb = sum(G_parts[i][l][1] for i in range(n))
            G.append((gW, gb))
        rec["G_parts"] = G_parts
        rec["G"] = G
        params = adam.update(params, G) if adam else sgd_update(params, G, cfg.lr)
        rec["params"] = params
        recs.append(rec)
    return recs
