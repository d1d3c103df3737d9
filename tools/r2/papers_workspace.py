"""Device workspace of the ogbn-papers100M-shaped run (111M nodes, 1.6B CSR non-zeros, 128-48-48-172,
SURVEY 8(a)) per rank, for p = 8 / 4 / 2 partitions (one per GPU, NCCL transport), with and without the
lean-memory mode (N1(iii)) -- from the host-only pgcn_workspace_bytes query, no GPU needed.

Only the graph structure is generated (the synth recipe's edge draw and nnz refit, no features: the
workspace does not depend on X's values).  n_train_global = 1.1 % of the nodes (the recipe's train
fraction).  Prints one JSON line per (p, mode): the largest rank's workspace in GB.

    python tools/r2/papers_workspace.py [--parts 8,4,2] [--config papers]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parts", default="8,4,2")
    ap.add_argument("--config", default="papers")
    a = ap.parse_args()
    from paper_2203_10428_b200 import pgcn
    from synth.graphs import CONFIGS, _draw_edges, model_for
    c = CONFIGS[a.config]
    n, nnz_t = c["n"], c["nnz"]
    t0 = time.time()
    scale = 1.0
    for _ in range(6):  # the generator's nnz refit (synth.graphs.gen_graph), structure only
        row_ptr, col = _draw_edges(n, min(c["comm"], n), nnz_t / (2.0 * n), scale, 0.10, 1)
        got = int(row_ptr[-1])
        if abs(got - nnz_t) <= 0.01 * nnz_t:
            break
        scale *= nnz_t / got
    t_gen = time.time() - t0
    m = model_for(a.config)
    n_train = int(round(c["train"] * n))
    for p in [int(x) for x in a.parts.split(",")]:
        t0 = time.time()
        part = pgcn.partition(n, row_ptr, col, p)
        t_part = time.time() - t0
        views = [part.view(r) for r in range(p)]
        for lean in (False, True):
            cfg = pgcn.make_config(m.widths, dropout=m.dropout, loss=m.loss, opt="adam", lr=m.lr, n_global=n,
                                   n_train_global=n_train, train_sparse=True, spmm_tiles=False, lean=lean)
            ws = [pgcn.workspace_bytes(part, cfg, [r]) for r in range(p)]
            print(json.dumps({"config": a.config, "n": n, "nnz": int(row_ptr[-1]), "parts": p, "lean": lean,
                              "transport": "nccl (one partition per rank)",
                              "workspace_GB_max_rank": max(ws) / 1e9, "workspace_GB_per_rank": [w / 1e9 for w in ws],
                              "n_inner_max": max(int(v["n_inner"]) for v in views),
                              "n_halo_max": max(int(v["n_halo"]) for v in views),
                              "n_send_max": max(int(v["n_send"]) for v in views),
                              "generate_s": t_gen, "partition_s": t_part}), flush=True)
        part.close()
        del views


if __name__ == "__main__":
    main()
