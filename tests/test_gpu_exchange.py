"""The posted exchange as a running data plane on one GPU (SURVEY 8(a) S2/S10 and its stream/event
contract; 8(e)): the LOOPBACK transport runs the NCCL transport's control flow -- pack on the compute
stream, event, one transfer per (sender, receiver) segment on the high-priority comm stream, event,
consumer waits for the iteration it consumes (Alg. 1 l.12-13, l.22-27; App. F
PAPER.md:981) -- with a device copy as the transfer.

Checks:
  * parity with the fp64 oracle (1e-4) for VANILLA, PIPE, PIPE-F/-G/-GF, both EMA inits, depth 2 and
    3, GraphSAGE and GCN-sym, the tensor-core tile aggregation;
  * bit-identity with the LOCAL transport (the exchange moves values, it never computes with them);
  * delay injection: a spin kernel before every transfer on the comm stream leaves every
    result bit-identical, and dropping the backward or forward wait (fault injection) changes them;
  * bf16 payloads (N1(iv)): 2e-2 parity, exactly half the exchanged bytes.
"""
import numpy as np
import pytest

from synth.graphs import ModelCfg, gen_graph, glorot_params
from test_gpu_parity import check_against_oracle, oracle_run, run_gpu

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


def run_ctx(P, g, widths, n_parts, T, params0, hook=None, **kw):
    """T iterations on a fresh context; returns (per-t records of loss / params / G / H / J, ctx)."""
    import torch
    part = P.partition(g.n, g.row_ptr, g.col_idx, n_parts)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, **kw)
    ctx = P.Context(part, cfg)
    if hook is not None:
        ctx.exchange_hook(*hook)
    for i in range(n_parts):
        gid = part.view(i)["inner_gid"]
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    L = len(widths) - 1
    recs = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, opt, loss)
        # no host sync between steps here: the comm stream may run behind (that is the point of the
        # delay tests); the records are read after the whole run
        recs.append((loss.clone(), theta.clone(), grads.clone(),
                     [[ctx.tensor(i, P.T_H, l, t)[:, :widths[l]].clone() for i in range(n_parts)]
                      for l in range(1, L + 1)],
                     [[ctx.tensor(i, P.T_J, l, t)[:, :widths[l]].clone() for i in range(n_parts)]
                      for l in range(1, L)]))
    torch.cuda.synchronize()
    out = []
    for lo, th, gr, H, J in recs:
        out.append(dict(loss=float(lo.item()), params=th.cpu().numpy(), G=gr.cpu().numpy(),
                        H={l + 1: [x.cpu().numpy() for x in H[l]] for l in range(L)},
                        J={l + 1: [x.cpu().numpy() for x in J[l]] for l in range(L - 1)}))
    return out, ctx


def identical(a, b):
    for x, y in zip(a, b):
        if x["loss"] != y["loss"] or not np.array_equal(x["params"], y["params"]) or not np.array_equal(x["G"], y["G"]):
            return False
        for l in x["H"]:
            if not all(np.array_equal(u, v) for u, v in zip(x["H"][l], y["H"][l])):
                return False
        for l in x["J"]:
            if not all(np.array_equal(u, v) for u, v in zip(x["J"][l], y["J"][l])):
                return False
    return True


MODES = [("vanilla", False, False, "first"), ("pipe", False, False, "first"), ("pipe", True, False, "first"),
         ("pipe", False, True, "first"), ("pipe", True, True, "first"), ("pipe", True, True, "zero")]


@pytest.mark.parametrize("mode,sf,sg,ema_init", MODES)
@pytest.mark.parametrize("depth", [1, 2])
def test_loopback_parity_and_bit_identity(P, mode, sf, sg, ema_init, depth):
    """3 layers, 3 partitions, ragged widths, dropout, BCE: the loopback exchange against the oracle
    (1e-4) and bit-identical to the LOCAL transport."""
    if mode == "vanilla" and depth > 1:
        pytest.skip("depth applies to PIPE")
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, ema_init=ema_init, dropout=0.3, loss="bce",
              opt="sgd", lr=2.0, depth=depth)
    T = 2 * depth + 2
    gpu, ctx = run_gpu(P, g, widths, 3, T, params0, transport="loopback", **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=2.0, opt="sgd", loss="bce", gamma=0.7)
    ora = oracle_run(gpu, g, 3, params0, cfg, T, mode=mode, smooth_f=sf, smooth_g=sg, ema_init=ema_init, depth=depth)
    check_against_oracle(gpu, ora, 3, 3, what=f"loopback {mode} F{sf} G{sg} {ema_init} s{depth}")
    fb, bb = ctx.exchange_bytes()
    assert fb > 0 and bb > 0
    a, _ = run_ctx(P, g, widths, 3, T, params0, transport="loopback", **kw)
    b, _ = run_ctx(P, g, widths, 3, T, params0, transport="local", **kw)
    assert identical(a, b), "loopback and local transports must agree bit for bit"
    c, ctxp = run_ctx(P, g, widths, 3, T, params0, transport="push", **kw)
    assert identical(c, b), "the fused push (N2) must agree bit for bit with the local transport"
    assert ctxp.exchange_bytes() == ctx.exchange_bytes()


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_loopback_gcn_and_tiles(P, model):
    """Reddit-like dense communities (tensor-core tile aggregation on, tile_min 8), 2 partitions,
    PIPE-GF; GraphSAGE and GCN-sym: oracle parity and bit-identity with LOCAL."""
    g = gen_graph("reddit", seed=3, n=800, nnz=24000, f0=32, classes=5)
    widths = [32, 64, 40, 5]
    params0 = glorot_params(widths, 3, model=model)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.5, loss="ce", opt="sgd", lr=0.5, model=model,
              spmm_tiles=True, tile_min=8)
    T = 4
    gpu, _ = run_gpu(P, g, widths, 2, T, params0, transport="loopback", **kw)
    cfg = ModelCfg(widths=widths, dropout=0.5, lr=0.5, opt="sgd", loss="ce", model=model)
    ora = oracle_run(gpu, g, 2, params0, cfg, T, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, 3, 2, what=f"loopback tiles {model}")
    a, _ = run_ctx(P, g, widths, 2, T, params0, transport="loopback", **kw)
    b, _ = run_ctx(P, g, widths, 2, T, params0, transport="local", **kw)
    assert identical(a, b)
    c, _ = run_ctx(P, g, widths, 2, T, params0, transport="push", **kw)  # GCN-sym tf layers: pack + copy
    assert identical(c, b)


DELAY_NS = 3_000_000  # 3 ms before every transfer: the comm stream falls far behind the compute


@pytest.mark.parametrize("mode,sf,sg,depth", [("pipe", True, True, 1), ("pipe", False, False, 2),
                                              ("vanilla", False, False, 1)])
def test_delay_injection_is_invisible(P, mode, sf, sg, depth):
    """a spin kernel on the comm stream before every transfer must not change any result
    bit (the consumers wait for the events of the iteration they consume)."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, dropout=0.3, loss="bce", opt="sgd", lr=2.0,
              depth=depth, transport="loopback")
    T = 2 * depth + 3
    ref, _ = run_ctx(P, g, widths, 3, T, params0, **kw)
    slow, _ = run_ctx(P, g, widths, 3, T, params0, hook=(DELAY_NS, 0), **kw)
    assert identical(ref, slow)


@pytest.mark.parametrize("flag", ["b", "f"])
def test_dropped_wait_is_detected(P, flag):
    """Fault injection: with the same delay, a context that skips the backward (ev_b_done) or forward
    (ev_f_done) wait must produce different results -- the delay test above has teeth."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, gamma=0.7, dropout=0.3, loss="bce", opt="sgd", lr=2.0,
              transport="loopback")
    T = 5
    ref, _ = run_ctx(P, g, widths, 3, T, params0, **kw)
    fl = P.XH_SKIP_B_WAIT if flag == "b" else P.XH_SKIP_F_WAIT
    bad, _ = run_ctx(P, g, widths, 3, T, params0, hook=(DELAY_NS, fl), **kw)
    assert not identical(ref, bad), "dropping the %s wait under delay went unnoticed" % flag


@pytest.mark.parametrize("mode,sf,sg", [("pipe", True, True), ("vanilla", False, False), ("pipe", False, False)])
@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_bf16_payloads(P, mode, sf, sg, model):
    """N1(iv): bf16 exchange payloads (features and gradients rounded to bf16 for the transfer, fp32
    everywhere else) at the 2e-2 tier against the fp64 oracle, and exactly half the payload bytes of
    the fp32 exchange."""
    tol = 2e-2
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5, model=model)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, dropout=0.3, loss="bce", opt="sgd", lr=2.0,
              model=model, transport="loopback")
    T = 4
    gpu, ctx16 = run_gpu(P, g, widths, 3, T, params0, halo_payload="bf16", **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=2.0, opt="sgd", loss="bce", gamma=0.7, model=model)
    ora = oracle_run(gpu, g, 3, params0, cfg, T, tol=tol, mode=mode, smooth_f=sf, smooth_g=sg)
    check_against_oracle(gpu, ora, 3, 3, tol=tol, what=f"bf16 payload {mode} {model}")
    _, ctx32 = run_gpu(P, g, widths, 3, T, params0, **kw)
    f16, b16 = ctx16.exchange_bytes()
    f32, b32 = ctx32.exchange_bytes()
    assert f16 > 0 and b16 > 0 and 2 * f16 == f32 and 2 * b16 == b32


def test_nocomm_ablation_runs(P):
    """PGCN_XH_NOCOMM (timing ablation): every kernel runs, no transfer is posted."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    out, ctx = run_ctx(P, g, widths, 3, 3, params0, hook=(0, P.XH_NOCOMM), mode="pipe", dropout=0.3, loss="bce",
                       opt="sgd", lr=2.0, transport="loopback")
    assert ctx.exchange_bytes() == (0, 0)
    assert np.isfinite(out[-1]["loss"])


def test_hook_rejected_on_local_transport(P):
    import torch  # noqa: F401
    g = gen_graph("cora", seed=1, n=200, nnz=800, f0=8, classes=3)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    ctx = P.Context(part, P.make_config([8, 4, 3], n_global=g.n, n_train_global=g.n_train))
    with pytest.raises(P.PgcnError) as e:
        ctx.exchange_hook(1000, 0)
    assert e.value.code == P.EUNSUPPORTED
    with pytest.raises(P.PgcnError) as e:
        P.Context(part, P.make_config([8, 4, 3], n_global=g.n, n_train_global=g.n_train, halo_payload="bf16"))
    assert e.value.code == P.EUNSUPPORTED


@pytest.mark.parametrize("p", [0.5, 0.0])
def test_stage_inputs_overlapped_reupload(P, p):
    """pgcn_stage_inputs (the end-to-end path): re-uploading the same inputs from pinned host memory on
    the library's copy stream every iteration, issued while the previous iteration is in flight, leaves
    every result bit-identical (the copy of X waits for that iteration's last read of X: layer 1's
    dropout, or with p = 0 layer 1's weight gradient)."""
    import torch
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    kw = dict(mode="pipe", smooth_g=True, dropout=p, loss="bce", opt="sgd", lr=2.0, transport="loopback")
    T = 4
    ref, _ = run_ctx(P, g, widths, 3, T, params0, **kw)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 3)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, **kw)
    ctx = P.Context(part, cfg)
    host = []
    for i in range(3):
        gid = part.view(i)["inner_gid"]
        X = torch.tensor(g.X[gid])
        if p == 0.0:  # the library's padded row layout (one contiguous copy) instead of F_0-wide rows
            X = torch.nn.functional.pad(X, (0, (X.shape[1] + 3) // 4 * 4 - X.shape[1]))
        h = (X.pin_memory(), torch.tensor(g.labels[gid]).pin_memory(), torch.tensor(g.train_mask[gid]).pin_memory())
        host.append(h)
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), h[1].cuda(), h[2].cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    loss = torch.zeros(1, device="cuda")
    for i in range(3):
        ctx.stage_inputs(i, *host[i])
    losses = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, None, loss)
        if t < T:
            for i in range(3):
                ctx.stage_inputs(i, *host[i])
        losses.append(loss.clone())
    torch.cuda.synchronize()
    assert [float(x.item()) for x in losses] == [r["loss"] for r in ref]
    assert np.array_equal(theta.cpu().numpy(), ref[-1]["params"])


@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_caller_buffer_layer_calls(P, model):
    """pgcn_layer_fwd_io / pgcn_layer_bwd_io (SURVEY 8(b) signatures): an iteration composed from the
    caller-buffer layer calls -- weights as separate W, b buffers, every H^(l) copied out and fed back
    in as the next layer's h_in, J^(l) fed back as j_out, dW/db and J^(l-1) copied out -- is bit-identical
    to pgcn_step, and its outputs equal the context's own tensors."""
    import torch
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    L = 3
    params0 = glorot_params(widths, 5, model=model)
    kw = dict(mode="pipe", smooth_g=True, dropout=0.3, loss="bce", opt="sgd", lr=2.0, transport="loopback", model=model)
    T = 3
    ref, _ = run_ctx(P, g, widths, 3, T, params0, **kw)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 3)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, **kw)
    ctx = P.Context(part, cfg)
    n_in = []
    for i in range(3):
        gid = part.view(i)["inner_gid"]
        n_in.append(len(gid))
        ctx.set_inputs(i, torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(),
                       torch.tensor(g.train_mask[gid]).cuda())
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    loss = torch.zeros(1, device="cuda")
    ns = 2 if model == "sage" else 1
    for t in range(1, T + 1):
        lay = P.unflatten_params(theta, widths, model)
        Ws = [W.contiguous().clone() for W, _ in lay]
        bs = [b.contiguous().clone() for _, b in lay]
        H = {}
        for l in range(1, L + 1):
            h_in = None if l == 1 else H[l - 1]
            H[l] = [torch.full((n, widths[l]), float("nan"), device="cuda") for n in n_in]
            ctx.layer_fwd_io(t, l, Ws[l - 1], bs[l - 1], h_in=h_in, h_out=H[l])
        ctx.loss(t, loss)
        Jnext = None
        dWs = {}
        for l in range(L, 0, -1):
            dW = torch.empty((ns * widths[l - 1], widths[l]), device="cuda")
            db = torch.empty(widths[l], device="cuda")
            j_in = [torch.empty((n, widths[l - 1]), device="cuda") for n in n_in] if l >= 2 else None
            ctx.layer_bwd_io(t, l, Ws[l - 1], bs[l - 1], j_out=Jnext, dW_local=dW, db_local=db, j_in=j_in)
            dWs[l] = (dW, db)
            if l >= 2:
                torch.cuda.synchronize()
                for i in range(3):  # the context's own accumulated J^(l-1) (dump_j) equals j_in
                    assert torch.equal(j_in[i], ctx.tensor(i, P.T_J, l - 1, t)[:, :widths[l - 1]])
            Jnext = j_in
        ctx.update(t, theta, grads)
        torch.cuda.synchronize()
        r = ref[t - 1]
        assert float(loss.item()) == r["loss"]
        assert np.array_equal(theta.cpu().numpy(), r["params"]), t
        assert np.array_equal(grads.cpu().numpy(), r["G"]), t
        for l in range(1, L):
            for i in range(3):
                assert np.array_equal(H[l][i].cpu().numpy(), r["H"][l][i]), (t, l, i)
        flatG = torch.cat([torch.cat([dWs[l][0].ravel(), dWs[l][1]]) for l in range(1, L + 1)])
        assert np.array_equal(flatG.cpu().numpy(), r["G"]), t  # one context: dW_local sums = G
