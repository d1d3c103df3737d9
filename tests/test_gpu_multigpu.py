"""The NCCL transport with one partition per rank on separate GPUs (Alg. 1 l.12-13,
l.22-27, l.31; App. F comm stream).

Each of `world` processes hosts partition `rank` on GPU `rank` and exchanges boundary features and
gradients with ncclSend/ncclRecv on the library's comm stream and all-reduces G on the compute stream.
Every per-iteration record (partition loss, theta, G, H^(l), J^(l)) must match the single-process run of
the same partitions through the LOOPBACK transport -- the same control flow with device copies as the
transfer -- to 1e-5 relative (bit-identical is expected for two ranks: the all-reduce of two addends is
one fp32 add either way).  Modes: VANILLA, PIPE, PIPE-GF, depth 2; NCCL send/recv, and PUSH across ranks
(N2 over NVLink: the producing epilogues store the exchanged rows into the peers' workspaces, mapped with
CUDA IPC; include/pgcn.h pgcn_ipc_export).

Skipped when fewer than `world` GPUs are visible (the one-GPU boxes of this build); two ranks on one GPU
are never used (NCCL rejects them, and ranks whose kernels wait on one another must not share a GPU).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("vanilla", False, False, 1, "nccl"), ("pipe", False, False, 1, "nccl"), ("pipe", True, True, 1, "nccl"),
         ("pipe", False, False, 2, "nccl"),
         # N2 over NVLink: producers store the exchanged rows into the peers' workspaces (CUDA IPC)
         ("pipe", False, False, 1, "push"), ("pipe", True, True, 1, "push"), ("pipe", False, False, 2, "push")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from synth.graphs import gen_graph, glorot_params
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    return g, widths, glorot_params(widths, 5)


def _kw(mode, sf, sg, depth, transport="nccl"):
    return dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, dropout=0.3, loss="bce", opt="sgd", lr=2.0,
                depth=depth)


def _records(P, ctx, locals_, widths, T, theta, grads, loss_parts):
    import torch
    L = len(widths) - 1
    recs = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, None, loss_parts)
        recs.append(dict(params=theta.clone(), G=grads.clone(),
                         H={l: [ctx.tensor(i, P.T_H, l, t)[:, :widths[l]].clone() for i in range(len(locals_))]
                            for l in range(1, L + 1)},
                         J={l: [ctx.tensor(i, P.T_J, l, t)[:, :widths[l]].clone() for i in range(len(locals_))]
                            for l in range(1, L)}))
    torch.cuda.synchronize()
    out = []
    for r in recs:
        out.append(dict(params=r["params"].cpu().numpy(), G=r["G"].cpu().numpy(),
                        H={l: [x.cpu().numpy() for x in v] for l, v in r["H"].items()},
                        J={l: [x.cpu().numpy() for x in v] for l, v in r["J"].items()}))
    return out


def _worker(rank, world, port, case, T, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        from paper_2203_10428_b200 import pgcn as P
        g, widths, params0 = _problem()
        part = P.partition(g.n, g.row_ptr, g.col_idx, world)
        cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True,
                            transport="push" if case[4] == "push" else "local", **_kw(*case))
        comm = P.nccl_comm(rank, world)
        ctx = P.Context(part, cfg, local_parts=[rank], comm=comm)
        if case[4] == "push":
            ctx.ipc_connect()
        gid = part.view(rank)["inner_gid"]
        ctx.set_inputs(0, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
        theta = torch.tensor(P.flatten_params(params0)).cuda()
        grads = torch.zeros_like(theta)
        loss = torch.zeros(1, device="cuda")
        recs = _records(P, ctx, [rank], widths, T, theta, grads, loss)
        fb, bb = ctx.exchange_bytes()
        q.put((rank, recs, fb, bb, None))
        ctx.close()
    except Exception as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, None, 0, 0, repr(e)))
    finally:
        dist.destroy_process_group()


def _rel(a, b):
    den = max(float(np.max(np.abs(b))) if b.size else 0.0, 1e-30)
    return float(np.max(np.abs(a - b))) / den if a.size else 0.0


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("case", CASES)
def test_nccl_ranks_match_loopback(world, case):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    if torch.cuda.device_count() < world:
        pytest.skip("needs %d GPUs (found %d): one partition per GPU over NCCL" % (world, torch.cuda.device_count()))
    import torch.multiprocessing as mp

    from paper_2203_10428_b200 import build
    from paper_2203_10428_b200 import pgcn as P
    build.build()
    T = 2 * case[3] + 3
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, case, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, _, _, _, err in res:
        assert err is None, "rank %d: %s" % (rank, err)
    # the same partitions in one process through the LOOPBACK transport
    g, widths, params0 = _problem()
    part = P.partition(g.n, g.row_ptr, g.col_idx, world)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, transport="loopback",
                        **_kw(*case))
    ctx = P.Context(part, cfg)
    for i in range(world):
        gid = part.view(i)["inner_gid"]
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    ref = _records(P, ctx, list(range(world)), widths, T, theta, torch.zeros_like(theta), torch.zeros(1, device="cuda"))
    fb0, bb0 = ctx.exchange_bytes()
    if case[4] == "nccl":  # (PUSH counts the pushed rows, not the posted bytes)
        assert sum(r[2] for r in res) == fb0 and sum(r[3] for r in res) == bb0, "exchanged bytes differ"
    worst = 0.0
    for t in range(T):
        for rank, recs, _, _, _ in res:
            r, o = recs[t], ref[t]
            worst = max(worst, _rel(r["params"], o["params"]), _rel(r["G"], o["G"]))
            for l in r["H"]:
                worst = max(worst, _rel(r["H"][l][0], o["H"][l][rank]))
            for l in r["J"]:
                worst = max(worst, _rel(r["J"][l][0], o["J"][l][rank]))
    assert worst <= 1e-5, "NCCL ranks vs single-process loopback: max relative error %.3e" % worst
