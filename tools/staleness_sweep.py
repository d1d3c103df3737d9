"""N4: Fig. 4/5/7-style study on the Reddit-shaped graph (2 partitions on one GPU, Adam lr 0.01,
dropout 0.5, Table 3): training loss and per-layer staleness errors ||used - fresh||_F of boundary
features and gradient messages, for VANILLA, PIPE, PIPE-F/-G/-GF, a gamma sweep and the deeper
pipeline of App. C (depth 2, 3; reading R27).  Writes gpurun_out/r1_staleness.md (copied to
profiles/ by hand: gpurun only brings gpurun_out/ back)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402
from synth.graphs import gen_graph, glorot_params, model_for  # noqa: E402

T = int(os.environ.get("STALE_T", "60"))
g = gen_graph("reddit", seed=1)
m = model_for("reddit")
part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 2)
views = [part.view(i) for i in range(2)]
inputs = [tuple(torch.tensor(x).cuda() for x in (g.X[v["inner_gid"]], g.labels[v["inner_gid"]],
                                                 g.train_mask[v["inner_gid"]])) for v in views]
L = len(m.widths) - 1
runs = [("GCN (vanilla)", "vanilla", False, False, 0.95, 1), ("PipeGCN", "pipe", False, False, 0.95, 1),
        ("PipeGCN-F", "pipe", True, False, 0.95, 1), ("PipeGCN-G", "pipe", False, True, 0.95, 1),
        ("PipeGCN-GF", "pipe", True, True, 0.95, 1), ("PipeGCN-GF g=0.7", "pipe", True, True, 0.7, 1),
        ("PipeGCN-GF g=0.5", "pipe", True, True, 0.5, 1), ("PipeGCN-GF g=0", "pipe", True, True, 0.0, 1),
        ("PipeGCN depth 2", "pipe", False, False, 0.95, 2), ("PipeGCN-GF depth 2", "pipe", True, True, 0.95, 2),
        ("PipeGCN depth 3", "pipe", False, False, 0.95, 3)]
rows = []
for name, mode, sf, sg, gam, depth in runs:
    cfg = pgcn.make_config(m.widths, mode=mode, smooth_f=sf, smooth_g=sg, gamma=gam, dropout=m.dropout, loss=m.loss,
                           opt="adam", lr=m.lr, n_global=g.n, n_train_global=g.n_train, staleness_stats=True,
                           depth=depth)
    ctx = pgcn.Context(part, cfg)
    for i in range(2):
        ctx.set_inputs(i, *inputs[i])
    theta = torch.tensor(pgcn.flatten_params(glorot_params(m.widths, 3))).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    losses, ef, eg = [], [], []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, opt, loss)
        st = [ctx.staleness(l) for l in range(1, L + 1)]
        losses.append(float(loss.item()))
        ef.append([s[0] for s in st])
        eg.append([s[1] for s in st])
    ef, eg = np.array(ef), np.array(eg)
    tail = slice(T // 2, T)
    rows.append((name, losses[0], losses[T // 4], losses[T // 2], losses[-1], ef[tail].mean(0), eg[tail].mean(0)))
    print(name, "loss", ["%.4f" % x for x in losses[::10]], flush=True)
    del ctx
lines = ["# r1: staleness study (N4; paper Fig. 4, 5, 7 analogue)", "",
         "Reddit-shaped synthetic graph, 2 partitions on one B200 (local transport), GraphSAGE 602-256x3-41, Adam",
         "lr 0.01, dropout 0.5 (Table 3), %d iterations. Errors are ||used - fresh||_F summed over both" % T,
         "partitions (pgcn_staleness), averaged over iterations %d..%d; feature error of layer l = boundary rows of" %
         (T // 2 + 1, T), "the layer-l input, gradient error of layer l = messages accumulated into J^(l-1).", "",
         "| run | loss t=1 | t=%d | t=%d | t=%d | feature err l=2..%d | gradient err l=2..%d |" % (T // 4, T // 2, T, L, L),
         "|---|---|---|---|---|---|---|"]
for name, l0, l1, l2, l3, f, gg in rows:
    lines.append("| %s | %.4f | %.4f | %.4f | %.4f | %s | %s |" % (
        name, l0, l1, l2, l3, " / ".join("%.3g" % x for x in f[1:]), " / ".join("%.3g" % x for x in gg[1:])))
lines += ["", "Layer-1 feature errors are 0 for t > depth (X is constant, R10); VANILLA errors are 0 by construction.",
          "Depth s (R27): boundary values are s iterations old (compare the depth rows with PipeGCN / PipeGCN-GF)."]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
open(os.path.join(ROOT, "gpurun_out", "r1_staleness.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
