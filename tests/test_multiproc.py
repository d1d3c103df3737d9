"""Multi-process host logic with world_size 2 on CPU (gloo): the NCCL-id bootstrap and the
partition index lists exchanged between ranks (an id round-trip: every owner sends its S_{i,j}
global ids and each receiver must get exactly its boundary segment B_j ∩ V_i, Alg. 1 l.2-5;
the backward direction returns the boundary ids to their owners in send order), plus the
bench's max-over-ranks reduction."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_10428_b200 import pgcn
        from synth.graphs import gen_graph
        import bench
        g = gen_graph("cora", seed=7, n=900, nnz=5000, f0=4, classes=3)
        part = pgcn.partition(g.n, g.row_ptr, g.col_idx, world)
        v = part.view(rank)
        # forward direction: send S_{rank,j} gids to j; receive my boundary segment owned by j
        reqs, bufs = [], {}
        for j in range(world):
            if j == rank:
                continue
            snd = torch.tensor(v["inner_gid"][v["send_idx"][v["send_off"][j]:v["send_off"][j + 1]]], dtype=torch.int64)
            n_recv = int(v["halo_off"][j + 1] - v["halo_off"][j])
            bufs[j] = torch.zeros(n_recv, dtype=torch.int64)
            reqs.append(dist.isend(snd, j))
            reqs.append(dist.irecv(bufs[j], j))
        for r in reqs:
            r.wait()
        ok_f = all(np.array_equal(bufs[j].numpy(), v["halo_gid"][v["halo_off"][j]:v["halo_off"][j + 1]])
                   for j in bufs)
        # backward direction: send my boundary rows' gids to their owners; owners receive in send order
        reqs, bufs = [], {}
        for j in range(world):
            if j == rank:
                continue
            snd = torch.tensor(v["halo_gid"][v["halo_off"][j]:v["halo_off"][j + 1]], dtype=torch.int64)
            bufs[j] = torch.zeros(int(v["send_off"][j + 1] - v["send_off"][j]), dtype=torch.int64)
            reqs.append(dist.isend(snd, j))
            reqs.append(dist.irecv(bufs[j], j))
        for r in reqs:
            r.wait()
        ok_b = all(np.array_equal(bufs[j].numpy(),
                                  v["inner_gid"][v["send_idx"][v["send_off"][j]:v["send_off"][j + 1]]]) for j in bufs)
        # NCCL unique ids broadcast by rank 0 (bytes identical on every rank)
        cm = pgcn.nccl_comm(rank, world)
        ids = bytes(cm._ids)
        allids = [None] * world
        dist.all_gather_object(allids, ids)
        ok_id = all(x == allids[0] for x in allids) and any(allids[0])
        mx = bench.max_over_ranks(float(rank + 1) * 10.0, dist)
        # the bench's exchange microbenchmark (gloo here, NCCL on GPUs): runs, sizes match the views
        cb = bench.exchange_microbench(dist, v, [4, 6, 3], reps=2)
        assert [c["F"] for c in cb] == [4, 6]
        assert all(c["bytes_sent_max_rank"] >= 0 and c["ms"] >= 0 for c in cb)
        q.put((rank, ok_f, ok_b, ok_id, mx, int(v["n_send"]), int(v["n_halo"])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_two_process_index_round_trip(world):
    from paper_2203_10428_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_f, ok_b, ok_id, mx, n_send, n_halo in res:
        assert ok_f and ok_b, rank
        assert ok_id
        assert mx == 10.0 * world
        assert n_send > 0 and n_halo > 0


def _rank_workload_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_10428_b200 import pgcn
        from synth.graphs import rows_inputs
        import bench
        g, m, params0, part, _ = bench.build_rank_workload("papers", world, rank, dist, pgcn, n=20000, nnz=180000)
        gid = part.view(rank)["inner_gid"]
        # the rank's rows are the rows of any larger request (per-row counter-based inputs)
        lo = max(int(gid[0]) - 100, 0)
        Xs, ls, ts = rows_inputs("papers", np.arange(lo, int(gid[-1]) + 1), n=g.n)
        ok_rows = (np.array_equal(g.X, Xs[gid - lo]) and np.array_equal(g.labels, ls[gid - lo]) and
                   np.array_equal(g.train_mask, ts[gid - lo]))
        q.put((rank, gid.tolist(), int(g.train_mask.sum()), g.n_train, ok_rows, m.widths, g.n))
    finally:
        dist.destroy_process_group()


def test_rank_sharded_workload():
    """papers100M-shaped multi-GPU runs build per-rank inputs (bench.build_rank_workload): the ranks'
    rows partition the node set, each rank's X / labels / train mask rows equal the per-row generator's
    rows of any request containing them, and n_train_global is the all-reduced train count."""
    from paper_2203_10428_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_workload_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = res[0][6]
    allg = sorted(x for r in res for x in r[1])
    assert allg == list(range(n))
    total = sum(r[2] for r in res)
    assert total > 0 and all(r[3] == total for r in res)
    assert all(r[4] for r in res)
    assert res[0][5] == [128, 48, 48, 172]
