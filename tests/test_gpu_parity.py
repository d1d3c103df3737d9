"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded
inputs.  Tolerance (north_star): per tensor
max|gpu - oracle| <= 1e-4 * max|oracle| for the fp32 path.

Cases span several SpMM/GEMM tiles and ragged tails (widths not multiples of 4, 64, 128),
isolated nodes, empty partitions, every mode (VANILLA, PIPE, PIPE-F/-G/-GF), dropout on/off,
CE and BCE, SGD and Adam."""
import numpy as np
import pytest

from oracle import pipegcn
from oracle.partition import partition as oracle_partition
from synth.graphs import ModelCfg, gen_graph, glorot_params

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


def rel(g, r):
    g, r = np.asarray(g, np.float64), np.asarray(r, np.float64)
    return np.abs(g - r).max() / max(np.abs(r).max(), 1e-30) if r.size else 0.0


def flat(layers):
    return np.concatenate([np.concatenate([np.ravel(W), np.ravel(b)]) for W, b in layers])


def run_gpu(P, g, widths, n_parts, T, params0, part_of=None, **kw):
    import torch
    part = P.partition(g.n, g.row_ptr, g.col_idx, n_parts, part_of)
    cfg = P.make_config(widths, n_global=g.n, n_train_global=g.n_train, dump_j=True, **kw)
    ctx = P.Context(part, cfg)
    keep = []
    for i in range(n_parts):
        gid = part.view(i)["inner_gid"]
        X = torch.tensor(g.X[gid]).cuda()
        lab = torch.tensor(g.labels[gid]).cuda()
        tm = torch.tensor(g.train_mask[gid]).cuda()
        keep.append((X, lab, tm))
        ctx.set_inputs(i, X, lab, tm)
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    L = len(widths) - 1
    recs = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, opt, loss)
        torch.cuda.synchronize()
        rec = dict(loss=float(loss.item()), G=grads.cpu().numpy().copy(), params=theta.cpu().numpy().copy(), H={},
                   J={}, G_parts=[ctx.tensor(i, P.T_G).cpu().numpy().ravel().copy() for i in range(n_parts)])
        for l in range(1, L + 1):
            rec["H"][l] = [ctx.tensor(i, P.T_H, l, t)[:, :widths[l]].cpu().numpy().copy() for i in range(n_parts)]
        for l in range(1, L):
            rec["J"][l] = [ctx.tensor(i, P.T_J, l, t)[:, :widths[l]].cpu().numpy().copy() for i in range(n_parts)]
        recs.append(rec)
    return recs, ctx


def kernel_relu_decision(gpu, tol=TOL):  # noqa: D401
    """sigma' hook for the oracle (reading R25).  sigma' = 1[Y > 0] is a discrete decision taken on a
    float; where the oracle's Y lies within the GPU's measured error of 0 the sign is not resolved by
    the fp32 arithmetic, so the oracle takes the kernel's decision (H > 0) there and keeps its own
    everywhere else.  The band is measured per (t, layer, partition): 4 x max|H_gpu - Y| over the
    elements both sides find positive (where H_gpu = Y_gpu), capped at the tier tolerance tol*max|Y|.
    The overridden fraction is asserted by oracle_run (<= 1e-3 at the 1e-4 tier, <= 8e-2 at 2e-2)."""
    stats = {"overridden": 0, "differ": 0, "total": 0, "max_band_rel": 0.0}

    def decide(t, l, i, Y):
        own = Y > 0
        if Y.size == 0:
            return own
        Hg = gpu[t - 1]["H"][l][i]
        ymax = max(np.abs(Y).max(), 1e-30)
        both = (Hg > 0) & own
        err = float(np.abs(Hg[both] - Y[both]).max()) if both.any() else tol * ymax
        band = min(4.0 * err, tol * ymax)
        border = np.abs(Y) <= band
        k = Hg > 0
        stats["overridden"] += int(border.sum())
        stats["differ"] += int((border & (own != k)).sum())
        stats["total"] += int(Y.size)
        stats["max_band_rel"] = max(stats["max_band_rel"], band / ymax)
        return np.where(border, k, own)
    decide.stats = stats
    return decide


RELU_LOG = []  # (what, stats) of every oracle run with the hook, printed by -s / kept for reports


def oracle_run(gpu, g, n_parts, params0, cfg, T, tol=TOL, **kw):
    dec = kernel_relu_decision(gpu, tol)
    ora = pipegcn.run(g, oracle_partition(g.n, g.row_ptr, g.col_idx, n_parts), params0, cfg, T, relu_decision=dec,
                      **kw)
    st = dec.stats
    frac = st["overridden"] / max(st["total"], 1)
    RELU_LOG.append(dict(st, frac=frac))
    print("R25 hook: %d of %d sigma' decisions in the measured band (%.2e), %d taken from the kernel against "
          "the oracle's own, band <= %.1e max|Y|" % (st["overridden"], st["total"], frac, st["differ"],
                                                    st["max_band_rel"]))
    # fp32 tier: the band is a few ulps of the pre-activations -> a tiny fraction; 2e-2 tier: the band can
    # reach the 2 % cap, and for roughly Gaussian Y (max ~ 4 sigma) P(|Y| < 0.02 max) ~ 6 %
    assert frac <= (1e-3 if tol <= 1e-4 else 8e-2), st
    return ora


def check_against_oracle(gpu, ora, L, n_parts, tol=TOL, what=""):
    for t, (a, b) in enumerate(zip(gpu, ora), start=1):
        assert abs(a["loss"] - b["loss"]) <= tol * abs(b["loss"]), (what, t, a["loss"], b["loss"])
        for l in range(1, L + 1):
            for i in range(n_parts):
                e = rel(a["H"][l][i], b["H"][l][i])
                assert e <= tol, (what, "H", t, l, i, e)
        for l in range(1, L):
            for i in range(n_parts):
                e = rel(a["J"][l][i], b["J"][l][i])
                assert e <= tol, (what, "J", t, l, i, e)
        e = rel(a["G"], flat(b["G"]))
        assert e <= tol, (what, "G", t, e)
        for i in range(n_parts):
            e = rel(a["G_parts"][i], flat(b["G_parts"][i]))
            assert e <= tol, (what, "G_i", t, i, e)
        e = rel(a["params"], flat(b["params"]))
        assert e <= tol, (what, "params", t, e)


MODES = [("vanilla", False, False), ("pipe", False, False), ("pipe", True, False), ("pipe", False, True),
         ("pipe", True, True)]


@pytest.mark.parametrize("mode,sf,sg", MODES)
@pytest.mark.parametrize("p", [0.0, 0.5])
@pytest.mark.parametrize("tf", [True, False])
def test_cora_two_partitions(P, mode, sf, sg, p, tf):
    """BASELINE configs[0]: Cora-shaped graph, 2-layer GraphSAGE hidden 16, 2 partitions on 1 GPU;
    tf = transform-before-aggregate on both layers (N1) or aggregate-first as written (Eq. 3)."""
    g = gen_graph("cora", seed=1)
    widths = [1433, 16, 7]
    params0 = glorot_params(widths, 3)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.95, dropout=p, loss="ce", opt="sgd", lr=0.5,
              transform_first=tf)
    T = 4
    gpu, _ = run_gpu(P, g, widths, 2, T, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=p, lr=0.5, opt="sgd", loss="ce", gamma=0.95)
    ora = oracle_run(gpu, g, 2, params0, cfg, T, mode=mode, smooth_f=sf, smooth_g=sg)
    check_against_oracle(gpu, ora, 2, 2, what=f"cora {mode} F{sf} G{sg} p{p}")


@pytest.mark.parametrize("mode,sf,sg,ema_init", [("pipe", True, True, "first"), ("pipe", True, True, "zero"),
                                                 ("vanilla", False, False, "first"), ("pipe", False, False, "first")])
def test_multi_tile_ragged_bce_three_parts(P, mode, sf, sg, ema_init):
    """Several tiles + ragged widths (103 -> 70 -> 45 -> 13, none a multiple of 4), 3 layers,
    3 partitions, multilabel BCE, dropout 0.3, SGD trajectory over 3 iterations."""
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    kw = dict(mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, ema_init=ema_init, dropout=0.3, loss="bce",
              opt="sgd", lr=2.0)
    T = 3
    gpu, _ = run_gpu(P, g, widths, 3, T, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=2.0, opt="sgd", loss="bce", gamma=0.7)
    ora = oracle_run(gpu, g, 3, params0, cfg, T, mode=mode, smooth_f=sf, smooth_g=sg, ema_init=ema_init)
    check_against_oracle(gpu, ora, 3, 3, what=f"bce {mode} {ema_init}")


def test_adam_teacher_forced(P):
    """Adam (Table 3) amplifies absolute gradient rounding near eps (dUpdate/dg <= lr/eps), so a
    free-running fp32-vs-fp64 Adam trajectory is not a 1e-4 quantity.  Instead,
    at every step the GPU update is checked against the oracle's Adam fed the GPU's own theta_{t-1}
    and G_t (teacher forcing); G_1 and the loss of step 1 are checked against the oracle outright."""
    import torch
    from oracle.sage import Adam
    g = gen_graph("yelp", seed=2, n=2000, nnz=30000, f0=33, classes=9)
    widths = [33, 24, 9]
    params0 = glorot_params(widths, 5)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config(widths, mode="pipe", smooth_g=True, dropout=0.1, loss="bce", opt="adam", lr=0.01,
                        n_global=g.n, n_train_global=g.n_train)
    ctx = P.Context(part, cfg)
    keep = []
    for i in range(2):
        gid = part.view(i)["inner_gid"]
        a = (torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(), torch.tensor(g.train_mask[gid]).cuda())
        keep.append(a)
        ctx.set_inputs(i, *a)
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    opt = torch.zeros(2 * theta.numel(), device="cuda")
    loss = torch.zeros(1, device="cuda")
    adam = Adam(0.01)
    cfgm = ModelCfg(widths=widths, dropout=0.1, lr=0.01, opt="adam", loss="bce")
    ora = pipegcn.run(g, oracle_partition(g.n, g.row_ptr, g.col_idx, 2), params0, cfgm, 1, mode="pipe", smooth_g=True)
    for t in range(1, 4):
        before = theta.cpu().numpy().astype(np.float64)
        ctx.step(t, theta, grads, opt, loss)
        torch.cuda.synchronize()
        G = grads.cpu().numpy().astype(np.float64)
        if t == 1:
            assert rel(G, flat(ora[0]["G"])) <= TOL
            assert abs(loss.item() - ora[0]["loss"]) <= TOL * abs(ora[0]["loss"])
        lay = P.unflatten_params(before, widths)
        glay = P.unflatten_params(G, widths)
        ref = flat(adam.update(lay, glay))
        got = theta.cpu().numpy()
        err = np.abs(got - ref).max()
        assert err <= 1e-7 * np.abs(ref).max() + 1e-5 * 0.01, (t, err)


@pytest.mark.parametrize("gemm", ["tc", "simt"])
def test_wide_rows_and_hidden_256(P, gemm):
    """Reddit-like widths at small N: 602 -> 256 -> 41 (SpMM: 5 chunks of 32 lanes; tensor-core
    GEMM: 2 K-segments of 19 k-blocks, N tiles of 256 and 48, dA halves of 3 tiles)."""
    g = gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=602, classes=41)
    widths = [602, 256, 41]
    params0 = glorot_params(widths, 7)
    kw = dict(mode="pipe", dropout=0.5, loss="ce", opt="sgd", lr=0.1, gemm=gemm)
    gpu, _ = run_gpu(P, g, widths, 2, 3, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.5, lr=0.1, opt="sgd", loss="ce")
    ora = oracle_run(gpu, g, 2, params0, cfg, 3, mode="pipe")
    check_against_oracle(gpu, ora, 2, 2, what="wide " + gemm)


def test_tc_gemm_large_widths(P):
    """Yelp-like hidden 512 (two N tiles of 256 in FWD, two F tiles in DW) and > 128-row M tiles."""
    g = gen_graph("yelp", seed=5, n=2500, nnz=30000, f0=300, classes=100)
    widths = [300, 512, 100]
    params0 = glorot_params(widths, 2)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.1, loss="bce", opt="sgd", lr=1.0)
    gpu, _ = run_gpu(P, g, widths, 2, 2, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.1, lr=1.0, opt="sgd", loss="bce")
    ora = oracle_run(gpu, g, 2, params0, cfg, 2, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, 2, 2, what="yelp-wide")


def test_empty_partitions_and_one_partition(P):
    """Degenerate cases: more partitions than nodes in some ranges (empty V_i), and n = 1."""
    g = gen_graph("cora", seed=4, n=6, nnz=10, f0=5, classes=3, comm=2)
    widths = [5, 4, 3]
    params0 = glorot_params(widths, 1)
    cfg = ModelCfg(widths=widths, dropout=0.0, lr=0.2, opt="sgd", loss="ce")
    for n_parts in (1, 8):
        gpu, _ = run_gpu(P, g, widths, n_parts, 3, params0, mode="pipe", loss="ce", opt="sgd", lr=0.2)
        ora = oracle_run(gpu, g, n_parts, params0, cfg, 3, mode="pipe")
        check_against_oracle(gpu, ora, 2, n_parts, what=f"degenerate n={n_parts}")


def test_order_violations_poison_nothing(P):
    import torch
    g = gen_graph("cora", seed=1, n=200, nnz=800, f0=8, classes=3)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    cfg = P.make_config([8, 4, 3], n_global=g.n, n_train_global=g.n_train)
    ctx = P.Context(part, cfg)
    theta = torch.zeros(P.param_count(cfg), device="cuda")
    with pytest.raises(P.PgcnError) as e:
        ctx.layer_fwd(2, 1, theta)            # t must start at 1
    assert e.value.code == P.ESTATE
    with pytest.raises(P.PgcnError) as e:
        ctx.layer_bwd(1, 2, theta)            # backward before forward
    assert e.value.code == P.ESTATE
    ctx.layer_fwd(1, 1, theta)                # the context is still usable
    with pytest.raises(P.PgcnError) as e:
        ctx.layer_fwd(1, 1, theta)            # layer 1 twice
    assert e.value.code == P.ESTATE
    ctx.layer_fwd(1, 2, theta)
    ctx.loss(1)


def test_launches_counted(P):
    import torch
    g = gen_graph("cora", seed=1, n=300, nnz=1200, f0=8, classes=3)
    gpu, ctx = run_gpu(P, g, [8, 6, 3], 2, 2, glorot_params([8, 6, 3], 1), mode="pipe")
    assert ctx.launch_count() > 20


@pytest.mark.parametrize("case", ["cora", "wide", "yelp"])
@pytest.mark.parametrize("tf", [True, False])
def test_bf16_tensor_core_variant(P, case, tf):
    """gemm = bf16 (kind::f16 tcgen05, fp32 accumulation) against the fp64 oracle at the north_star's
    2e-2 tier, PIPE with smoothing and dropout, both aggregation orders, 2 iterations (SGD)."""
    tol = 2e-2
    if case == "cora":
        g = gen_graph("cora", seed=1)
        widths = [1433, 16, 7]
        loss = "ce"
    elif case == "wide":
        g = gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=602, classes=41)
        widths = [602, 256, 41]
        loss = "ce"
    else:
        g = gen_graph("yelp", seed=5, n=2500, nnz=30000, f0=300, classes=100)
        widths = [300, 512, 100]
        loss = "bce"
    params0 = glorot_params(widths, 3)
    kw = dict(mode="pipe", smooth_f=True, smooth_g=True, dropout=0.3, loss=loss, opt="sgd", lr=0.5, gemm="bf16",
              transform_first=tf)
    gpu, _ = run_gpu(P, g, widths, 2, 2, params0, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.3, lr=0.5, opt="sgd", loss=loss)
    ora = oracle_run(gpu, g, 2, params0, cfg, 2, tol=tol, mode="pipe", smooth_f=True, smooth_g=True)
    check_against_oracle(gpu, ora, 2, 2, tol=tol, what="bf16 %s tf%s" % (case, tf))


@pytest.mark.parametrize("mode,sf,sg", [("pipe", False, False), ("pipe", True, True), ("vanilla", False, False)])
def test_staleness_errors_match_oracle(P, mode, sf, sg):
    """N4 / Fig. 5-7: per-layer ||used - fresh||_F of boundary features and gradient
    messages, GPU (pgcn_staleness) vs the oracle's err_f / err_g.  A norm of differences of fp32
    quantities: tolerance 1e-3 of the value plus 1e-6 of the fresh magnitude scale."""
    import torch
    g = gen_graph("yelp", seed=2, n=3001, nnz=40000, f0=103, classes=13)
    widths = [103, 70, 45, 13]
    params0 = glorot_params(widths, 5)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 3)
    cfg = P.make_config(widths, mode=mode, smooth_f=sf, smooth_g=sg, gamma=0.7, dropout=0.3, loss="bce",
                        opt="sgd", lr=2.0, n_global=g.n, n_train_global=g.n_train, staleness_stats=True)
    ctx = P.Context(part, cfg)
    keep = []
    for i in range(3):
        gid = part.view(i)["inner_gid"]
        a = (torch.tensor(g.X[gid]).cuda(), torch.tensor(g.labels[gid]).cuda(), torch.tensor(g.train_mask[gid]).cuda())
        keep.append(a)
        ctx.set_inputs(i, *a)
    theta = torch.tensor(P.flatten_params(params0)).cuda()
    grads = torch.zeros_like(theta)
    T = 3
    got = []
    for t in range(1, T + 1):
        ctx.step(t, theta, grads, None, None)
        got.append({l: ctx.staleness(l) for l in range(1, 4)})
    ora = pipegcn.run(g, oracle_partition(g.n, g.row_ptr, g.col_idx, 3), params0,
                      ModelCfg(widths=widths, dropout=0.3, lr=2.0, opt="sgd", loss="bce", gamma=0.7), T, mode=mode,
                      smooth_f=sf, smooth_g=sg)
    for t in range(T):
        for l in range(1, 4):
            f_gpu, g_gpu = got[t][l]
            f_ora = ora[t]["err_f"][l]
            g_ora = ora[t]["err_g"].get(l, 0.0)
            assert abs(f_gpu - f_ora) <= 1e-3 * f_ora + 1e-6, (t, l, f_gpu, f_ora)
            assert abs(g_gpu - g_ora) <= 1e-3 * g_ora + 1e-9, (t, l, g_gpu, g_ora)
    if mode == "vanilla":
        assert all(v == (0.0, 0.0) for d in got for v in d.values())


@pytest.mark.parametrize("depth", [2, 3])
@pytest.mark.parametrize("sf,sg", [(False, False), (True, True)])
@pytest.mark.parametrize("model", ["sage", "gcn"])
def test_pipeline_depth(P, depth, sf, sg, model):
    """Depth-s pipeline (R27, App. C future work PAPER.md:923): exchanges consumed s iterations
    later, s + 1 rotating buffers; 3 layers, 3 partitions, dropout, over 2 s + 2 iterations so the
    zero-halo start (t <= s), the first receipt (EMA init) and steady state are all covered."""
    g = gen_graph("reddit", seed=6, n=2500, nnz=30000, f0=37, classes=5)
    widths = [37, 30, 22, 5]
    params0 = glorot_params(widths, 4, model=model)
    T = 2 * depth + 2
    kw = dict(mode="pipe", smooth_f=sf, smooth_g=sg, gamma=0.8, dropout=0.2, loss="ce", opt="sgd", lr=0.5)
    gpu, _ = run_gpu(P, g, widths, 3, T, params0, depth=depth, model=model, **kw)
    cfg = ModelCfg(widths=widths, dropout=0.2, lr=0.5, opt="sgd", loss="ce", gamma=0.8, model=model)
    ora = oracle_run(gpu, g, 3, params0, cfg, T, mode="pipe", smooth_f=sf, smooth_g=sg, depth=depth)
    check_against_oracle(gpu, ora, 3, 3, what=f"depth {depth} {model} F{sf} G{sg}")
