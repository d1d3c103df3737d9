"""compute-sanitizer driver for the posted exchange (LOOPBACK transport): 3 partitions, PIPE-GF at
depth 1 and 2, VANILLA, fp32 and bf16 payloads, tile aggregation on a dense-community graph, the delay
hook, the streaming input re-upload (pgcn_stage_inputs), the PUSH transport and the lean-memory mode
(one J / message slot guarded by waits), 4 iterations each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2203_10428_b200 import pgcn  # noqa: E402
from synth.graphs import gen_graph, glorot_params  # noqa: E402

RUNS = [dict(mode="pipe", smooth_f=True, smooth_g=True, depth=1), dict(mode="pipe", smooth_f=True, smooth_g=True, depth=2),
        dict(mode="vanilla"), dict(mode="pipe", smooth_g=True, halo_payload="bf16"),
        dict(mode="vanilla", halo_payload="bf16"), dict(mode="pipe", spmm_tiles=True, tile_min=8, hook=1),
        dict(mode="pipe", smooth_f=True, smooth_g=True, transport="push"), dict(mode="vanilla", transport="push"),
        dict(mode="pipe", depth=2, model="gcn", transport="push"),
        dict(mode="pipe", smooth_f=True, smooth_g=True, lean=True, train_sparse=True),
        dict(mode="pipe", depth=2, lean=True, hook=1), dict(mode="vanilla", lean=True, transport="push")]
for kw in RUNS:
    hook = kw.pop("hook", 0)
    dense = "tile_min" in kw
    g = gen_graph("reddit", seed=3, n=800, nnz=24000, f0=32, classes=5) if dense else \
        gen_graph("cora", seed=1, n=700, nnz=3000, f0=37, classes=5)
    widths = [g.X.shape[1], 24, 20, 5]
    part = pgcn.partition(g.n, g.row_ptr, g.col_idx, 3)
    kw.setdefault("transport", "loopback")
    cfg = pgcn.make_config(widths, dropout=0.5, loss="ce", opt="adam", n_global=g.n, n_train_global=g.n_train, **kw)
    ctx = pgcn.Context(part, cfg)
    if hook:
        ctx.exchange_hook(200000, 0)
    host = []
    for i in range(3):
        gid = part.view(i)["inner_gid"]
        h = (torch.tensor(g.X[gid]).pin_memory(), torch.tensor(g.labels[gid]).pin_memory(),
             torch.tensor(g.train_mask[gid]).pin_memory())
        host.append(h)
        ctx.set_inputs(i, *(a.cuda() for a in h))
    theta = torch.tensor(pgcn.flatten_params(glorot_params(widths, 3, model=kw.get("model", "sage")))).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    for t in range(1, 5):
        ctx.step(t, theta, grads, opt, loss)
        for i in range(3):
            ctx.stage_inputs(i, *host[i])
    torch.cuda.synchronize()
    print(kw, "hook" if hook else "", "loss", float(loss.item()), "exchanged", ctx.exchange_bytes())
