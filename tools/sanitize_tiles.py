"""compute-sanitizer run of the tensor-core tile aggregation (spmm_tiles): a small dense-community
graph, 2 partitions, PIPE with dropout, 3 iterations; fp32 (hi/lo, 2 CTAs/SM, A in TMEM) and bf16
(A in shared memory) tiers, GraphSAGE and GCN-sym, both aggregation orders, tile_min 1 (all edges in
tiles) and 24 (light edges too)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402
from synth.graphs import gen_graph, glorot_params  # noqa: E402

g = gen_graph("reddit", seed=3, n=1200, nnz=40000, f0=40, classes=7)
widths = [40, 130, 7]
for gather in ("f32", "bf16"):
    for model in ("sage", "gcn"):
        for tf in (True, False):
            for tmin in (1, 24):
                part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 2)
                cfg = pgcn.make_config(widths, mode="pipe", smooth_g=True, dropout=0.5, loss="ce", opt="adam",
                                       n_global=g.n, n_train_global=g.n_train, transform_first=tf, gather=gather,
                                       model=model, spmm_tiles=True, tile_min=tmin)
                ctx = pgcn.Context(part, cfg)
                keep = []
                for i in range(2):
                    gid = part.view(i)["inner_gid"]
                    a = (torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                         torch.tensor(g.train_mask[gid]).cuda())
                    keep.append(a)
                    ctx.set_inputs(i, *a)
                theta = torch.tensor(pgcn.flatten_params(glorot_params(widths, 3, model=model))).cuda()
                grads = torch.zeros_like(theta)
                opt = torch.zeros(2 * theta.numel(), device="cuda")
                loss = torch.zeros(1, device="cuda")
                for t in range(1, 4):
                    ctx.step(t, theta, grads, opt, loss)
                torch.cuda.synchronize()
                print(gather, model, tf, tmin, "loss", float(loss.item()))
