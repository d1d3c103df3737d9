"""Full-step parity at the bench's full sizes (App. A.1 PAPER.md:661-677 defines every step): the
Reddit-shaped graph (232,965 nodes, 113.6M non-zeros, 602-256-256-256-41) and the products-shaped
graph (2.45M nodes, 61.9M non-zeros, 100-128-128-47), 2 partitions on one GPU, in the bench's launch
configuration -- LOOPBACK exchange, tensor-core tile aggregation, transform-first layers, train-row-
sparse last layer, PIPE, dropout -- against the fp64 oracle for t = 1, 2 (t = 2 consumes the stale
exchange of t = 1): the loss, every H^(l) (inner rows; logits on train rows, the only rows the last
layer computes), every accumulated J^(l), every G_i, G and the updated parameters, at 1e-4.
SGD (Alg. 1 l.32): Adam's update is not a 1e-4 quantity of fp32 gradients."""
import dataclasses

import numpy as np
import pytest

from synth.graphs import gen_graph, glorot_params, model_for
from test_gpu_parity import flat, oracle_run, rel

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def run_full(P, g, m, params0, T):
    import torch
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config(m.widths, mode="pipe", dropout=m.dropout, loss=m.loss, opt="sgd", lr=m.lr, n_global=g.n,
                        n_train_global=g.n_train, dump_j=True, train_sparse=True, spmm_tiles=True,
                        transport="loopback")
    ctx = P.Context(part, cfg)
    views = [part.view(i) for i in range(2)]
    for i, v in enumerate(views):
        gid = v["inner_gid"]
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    loss = torch.zeros(1, device="cuda")
    L = len(m.widths) - 1
    recs = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, None, loss)
        torch.cuda.synchronize()
        rec = dict(loss=float(loss.item()), G=grads.cpu().numpy().copy(), params=theta.cpu().numpy().copy(),
                   H={}, J={}, G_parts=[ctx.tensor(i, P.T_G).cpu().numpy().ravel().copy() for i in range(2)])
        for l in range(1, L + 1):
            rec["H"][l] = [ctx.tensor(i, P.T_H, l, t)[:, :m.widths[l]].cpu().numpy().copy() for i in range(2)]
        for l in range(1, L):
            rec["J"][l] = [ctx.tensor(i, P.T_J, l, t)[:, :m.widths[l]].cpu().numpy().copy() for i in range(2)]
        recs.append(rec)
    train = [g.train_mask[v["inner_gid"]].astype(bool) for v in views]
    return recs, train


@pytest.mark.parametrize("name", ["reddit", "products"])
def test_full_size_two_iterations(P, name):
    g = gen_graph(name, seed=1)
    m = dataclasses.replace(model_for(name), opt="sgd", lr=0.05)
    params0 = glorot_params(m.widths, 3)
    T = 2
    gpu, train = run_full(P, g, m, params0, T)
    ora = oracle_run(gpu, g, 2, params0, m, T, mode="pipe")
    L = len(m.widths) - 1
    for t in range(T):
        a, b = gpu[t], ora[t]
        assert abs(a["loss"] - b["loss"]) <= TOL * abs(b["loss"]), (name, t, a["loss"], b["loss"])
        for l in range(1, L + 1):
            for i in range(2):
                ga, ob = a["H"][l][i], np.asarray(b["H"][l][i])
                if l == L:  # train-row-sparse last layer: logits exist on train rows only
                    ga, ob = ga[train[i]], ob[train[i]]
                e = rel(ga, ob)
                assert e <= TOL, (name, "H", t + 1, l, i, e)
        for l in range(1, L):
            for i in range(2):
                e = rel(a["J"][l][i], b["J"][l][i])
                assert e <= TOL, (name, "J", t + 1, l, i, e)
        for i in range(2):
            e = rel(a["G_parts"][i], flat(b["G_parts"][i]))
            assert e <= TOL, (name, "G_i", t + 1, i, e)
        assert rel(a["G"], flat(b["G"])) <= TOL, (name, "G", t + 1)
        assert rel(a["params"], flat(b["params"])) <= TOL, (name, "params", t + 1)
