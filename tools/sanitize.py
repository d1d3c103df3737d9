"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): Cora-shaped,
2 partitions, PIPE-GF with dropout, 3 iterations: tensor-core and SIMT GEMMs, both aggregation
orders, fp32 and bf16 gathers (bf16 gathers with the tensor-core GEMMs), GraphSAGE and GCN-sym."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402
from synth.graphs import gen_graph, glorot_params  # noqa: E402

g = gen_graph("cora", seed=1, n=700, nnz=3000, f0=37, classes=5)
RUNS = [(gemm, tf, "f32", "sage") for gemm in ("tc", "simt") for tf in (True, False)]
RUNS += [("tc", tf, "bf16", model) for tf in (True, False) for model in ("sage", "gcn")]
RUNS += [("tc", tf, "f32", "gcn") for tf in (True, False)]
for gemm, tf, gather, model in RUNS:
    if True:
        widths = [37, 24, 5]
        part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 2)
        cfg = pgcn.make_config(widths, mode="pipe", smooth_f=True, smooth_g=True, dropout=0.5, loss="ce", opt="adam",
                               n_global=g.n, n_train_global=g.n_train, gemm=gemm, transform_first=tf,
                               gather=gather, model=model)
        ctx = pgcn.Context(part, cfg)
        keep = []
        for i in range(2):
            gid = part.view(i)["inner_gid"]
            a = (torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(), torch.tensor(g.train_mask[gid]).cuda())
            keep.append(a)
            ctx.set_inputs(i, *a)
        theta = torch.tensor(pgcn.flatten_params(glorot_params(widths, 3, model=model))).cuda()
        grads = torch.zeros_like(theta)
        opt = torch.zeros(2 * theta.numel(), device="cuda")
        loss = torch.zeros(1, device="cuda")
        for t in range(1, 4):
            ctx.step(t, theta, grads, opt, loss)
        torch.cuda.synchronize()
        print(gemm, tf, gather, model, "loss", float(loss.item()))
