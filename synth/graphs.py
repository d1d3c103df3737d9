"""Deterministic synthetic graphs shaped like the paper's datasets.

Recipe (SURVEY.md section 8(d) generator v1):

* N nodes split into C contiguous communities of floor(N/C) gids (the last one
  absorbs the remainder).
* Each node v draws k_v ~ round(s * nnz/(2N) * lambda_v) undirected edge stubs,
  lambda_v ~ LogNormal(-1/2, 1) clipped at 50 (heavy-tailed degrees, mean 1).
  Each stub's far end is uniform inside v's community with probability 1-c
  (c = 0.10), else uniform over all nodes.
* Symmetrise, drop self loops and duplicates, sort rows ascending.  The global
  scale s is re-fitted (same seed, fresh draw) until nnz is within 1% of the
  target.  "Edges" = CSR non-zeros (each undirected edge stored twice).
* Features: N(0,1) fp32 plus 1.0 at column (community mod F); Cora-like graphs
  use Bernoulli(0.0127) binary features, row-normalised.
* Labels: community mod n_classes with prob 0.8, else uniform; multilabel
  (Yelp-like): community-biased Bernoulli multi-hot.
* Train mask: uniform(0,1) < train_frac.
* Weights: Glorot-uniform W (2F_in x F_out), zero bias, numpy default_rng.

Nothing here computes any part of the PipeGCN method.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Graph:
    name: str
    n: int
    row_ptr: np.ndarray      # int64 [n+1]
    col_idx: np.ndarray      # int32 [nnz]  in-neighbours of each row, ascending
    X: np.ndarray            # float32 [n, F0]
    labels: np.ndarray       # int32 [n] (single label) or uint8 [n, C] (multilabel)
    train_mask: np.ndarray   # uint8 [n]
    n_classes: int
    multilabel: bool

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def n_train(self) -> int:
        return int(self.train_mask.sum())


@dataclasses.dataclass
class ModelCfg:
    """GraphSAGE sizes and training hyper-parameters (Table 3)."""
    widths: list            # [F0, F1, ..., FL]
    dropout: float
    lr: float
    opt: str                # "adam" | "sgd"
    loss: str               # "ce" | "bce"
    gamma: float = 0.95     # default smoothing decay
    model: str = "sage"     # "sage" (GraphSAGE-mean, CONCAT) or "gcn" (App. A.1 propagation)

    @property
    def n_layers(self) -> int:
        return len(self.widths) - 1


# name -> (N, nnz target, F0, n_classes, communities, train_frac, multilabel,
#          feature kind, hidden, layers, dropout, lr)
CONFIGS = {
    # Not in the paper; BASELINE.json configs[0] (parity / smoke size).
    "cora": dict(n=2708, nnz=10556, f0=1433, classes=7, comm=8, train=0.052, multilabel=False,
                 feat="binary", hidden=16, layers=2, dropout=0.5, lr=0.01),
    # Table 3 rows; papers hidden width 48 from Table 3.
    "reddit": dict(n=232965, nnz=114615892, f0=602, classes=41, comm=64, train=0.66, multilabel=False,
                   feat="gauss", hidden=256, layers=4, dropout=0.5, lr=0.01),
    "products": dict(n=2449029, nnz=61859140, f0=100, classes=47, comm=64, train=0.08, multilabel=False,
                     feat="gauss", hidden=128, layers=3, dropout=0.3, lr=0.003),
    "yelp": dict(n=716847, nnz=6977410, f0=300, classes=100, comm=64, train=0.75, multilabel=True,
                 feat="gauss", hidden=512, layers=4, dropout=0.1, lr=0.001),
    "papers": dict(n=111059956, nnz=1615685872, f0=128, classes=172, comm=512, train=0.011,
                   multilabel=False, feat="gauss", hidden=48, layers=3, dropout=0.0, lr=0.01),
    # papers100M recipe at a quarter of the nodes and edges (same degree, widths, train fraction and
    # community size): 2 partitions of it have the per-GPU shape of the 8-GPU papers100M run
    # (13.9M inner rows, ~200M local edges each) and fit one B200.
    "papers-q": dict(n=27764989, nnz=403921468, f0=128, classes=172, comm=128, train=0.011,
                     multilabel=False, feat="gauss", hidden=48, layers=3, dropout=0.0, lr=0.01),
    # one eighth of papers100M (same degree, widths, train fraction and community size): the shape the ncu
    # captures use -- papers-q's 170 GB workspace leaves no room for ncu's kernel replay buffers
    "papers-e": dict(n=13882494, nnz=201960734, f0=128, classes=172, comm=64, train=0.011,
                     multilabel=False, feat="gauss", hidden=48, layers=3, dropout=0.0, lr=0.01),
}


def model_for(name: str, **over) -> ModelCfg:
    c = dict(CONFIGS[name])
    c.update({k: v for k, v in over.items() if k in c})
    widths = [c["f0"]] + [c["hidden"]] * (c["layers"] - 1) + [c["classes"]]
    m = ModelCfg(widths=widths, dropout=c["dropout"], lr=c["lr"], opt="adam",
                 loss="bce" if c["multilabel"] else "ce")
    for k in ("opt", "loss", "gamma", "dropout", "lr"):
        if k in over:
            setattr(m, k, over[k])
    return m


_LIB = None


def _lib():
    """ctypes handle to synth/libsynth.so (built from synth/gen.cpp on first use)."""
    global _LIB
    if _LIB is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so, cpp = os.path.join(here, "libsynth.so"), os.path.join(here, "gen.cpp")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(cpp):
            tmp = so + ".%d.tmp" % os.getpid()
            subprocess.check_call(["g++", "-O3", "-std=c++17", "-shared", "-fPIC", "-pthread",
                                   cpp, "-o", tmp])
            os.replace(tmp, so)
        lib = ctypes.CDLL(so)
        lib.synth_edges.restype = ctypes.c_int64
        lib.synth_edges.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_uint64, ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        lib.synth_free.argtypes = [ctypes.c_void_p]
        lib.synth_rows.restype = None
        lib.synth_rows.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                   ctypes.c_double, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _LIB = lib
    return _LIB


def _draw_edges(n, n_comm, stubs_mean, scale, cross, seed):
    import ctypes
    lib = _lib()
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    colp = ctypes.c_void_p()
    nnz = lib.synth_edges(n, n_comm, stubs_mean, scale, cross, seed, 0,
                          row_ptr.ctypes.data, ctypes.byref(colp))
    if nnz < 0:
        raise RuntimeError("synth_edges failed (%d)" % nnz)
    col = np.empty(nnz, dtype=np.int32)
    if nnz:
        ctypes.memmove(col.ctypes.data, colp.value, 4 * nnz)
    lib.synth_free(colp)
    return row_ptr, col


def gen_structure(name: str, seed: int = 1, n: Optional[int] = None, nnz: Optional[int] = None,
                  comm: Optional[int] = None, cross: float = 0.10):
    """The CSR structure of gen_graph(name, ...) alone (same edge draw and nnz refit, no inputs):
    (row_ptr int64 [n+1], col_idx int32 [nnz])."""
    c = dict(CONFIGS[name])
    n = c["n"] if n is None else n
    nnz_t = c["nnz"] if nnz is None else nnz
    n_comm = min(c["comm"] if comm is None else comm, n)
    stubs_mean = nnz_t / (2.0 * n)
    scale = 1.0
    for _ in range(6):
        row_ptr, col = _draw_edges(n, n_comm, stubs_mean, scale, cross, seed)
        got = int(row_ptr[-1])
        if got == 0 or abs(got - nnz_t) <= 0.01 * nnz_t:
            break
        scale *= nnz_t / got
    return row_ptr, col


def rows_inputs(name: str, gids, seed: int = 1, n: Optional[int] = None, f0: Optional[int] = None,
                classes: Optional[int] = None, comm: Optional[int] = None):
    """Inputs of the rows `gids` only, for graphs too large to materialise X on every rank (the
    papers100M-shaped multi-GPU run: each rank builds its own partition's rows).  Counter-based per row
    (synth_rows in gen.cpp): any subset of rows is reproducible on its own.  Same distributions as
    gen_graph's single-label recipe (X ~ N(0,1) + 1 at column (community mod F), label = community mod C
    w.p. 0.8, train ~ U(0,1) < train_frac), different random values.  Returns (X float32 [m, f0],
    labels int32 [m], train_mask uint8 [m])."""
    import ctypes
    c = dict(CONFIGS[name])
    if c["multilabel"]:
        raise ValueError("rows_inputs: single-label configs only")
    n = c["n"] if n is None else n
    f0 = c["f0"] if f0 is None else f0
    classes = c["classes"] if classes is None else classes
    n_comm = min(c["comm"] if comm is None else comm, n)
    gids = np.ascontiguousarray(gids, dtype=np.int64)
    m = len(gids)
    X = np.empty((m, f0), dtype=np.float32)
    lab = np.empty(m, dtype=np.int32)
    tm = np.empty(m, dtype=np.uint8)
    _lib().synth_rows(ctypes.c_uint64(seed * 1000003 + 2), n, n_comm, f0, classes, float(c["train"]),
                      gids.ctypes.data, m, 0, X.ctypes.data, lab.ctypes.data, tm.ctypes.data)
    return X, lab, tm


def gen_graph(name: str, seed: int = 1, n: Optional[int] = None, nnz: Optional[int] = None,
              f0: Optional[int] = None, classes: Optional[int] = None, comm: Optional[int] = None,
              cross: float = 0.10) -> Graph:
    """Seeded graph of config `name`, optionally resized (tests use small n)."""
    c = dict(CONFIGS[name])
    n = c["n"] if n is None else n
    nnz_t = c["nnz"] if nnz is None else nnz
    f0 = c["f0"] if f0 is None else f0
    classes = c["classes"] if classes is None else classes
    n_comm = min(c["comm"] if comm is None else comm, n)
    stubs_mean = nnz_t / (2.0 * n)
    scale = 1.0
    for _ in range(6):
        row_ptr, col = _draw_edges(n, n_comm, stubs_mean, scale, cross, seed)
        got = int(row_ptr[-1])
        if got == 0 or abs(got - nnz_t) <= 0.01 * nnz_t:
            break
        scale *= nnz_t / got
    rng = np.random.default_rng([seed, 2])
    csize = max(n // n_comm, 1)
    community = np.minimum(np.arange(n) // csize, n_comm - 1)
    if c["feat"] == "binary":
        X = (rng.random((n, f0), dtype=np.float32) < 0.0127).astype(np.float32)
        X[np.arange(n), community % f0] = 1.0
        X /= X.sum(1, keepdims=True)
    else:
        X = rng.standard_normal((n, f0), dtype=np.float32)
        X[np.arange(n), community % f0] += 1.0
    rng = np.random.default_rng([seed, 5])
    if c["multilabel"]:
        base = rng.random((n, classes)) < 0.05
        pref = (np.arange(classes)[None, :] % n_comm) == (community[:, None] % classes % n_comm)
        labels = (base | (pref & (rng.random((n, classes)) < 0.7))).astype(np.uint8)
    else:
        rnd = rng.integers(0, classes, n)
        labels = np.where(rng.random(n) < 0.8, community % classes, rnd).astype(np.int32)
    train_mask = (rng.random(n) < c["train"]).astype(np.uint8)
    if train_mask.sum() == 0:
        train_mask[0] = 1
    return Graph(name=name, n=n, row_ptr=row_ptr, col_idx=col, X=np.ascontiguousarray(X),
                 labels=labels, train_mask=train_mask, n_classes=classes,
                 multilabel=bool(c["multilabel"]))


def glorot_params(widths, seed: int = 3, model: str = "sage"):
    """Per-layer (W, b float32).  sage: W [2F_in x F_out], rows 0..F_in-1 multiply the aggregated
    z, rows F_in..2F_in-1 the node's own h (CONCAT(z, h)).  gcn: W [F_in x F_out]."""
    rng = np.random.default_rng(seed)
    out = []
    k = 2 if model == "sage" else 1
    for fi, fo in zip(widths[:-1], widths[1:]):
        a = np.sqrt(6.0 / (k * fi + fo))
        W = rng.uniform(-a, a, (k * fi, fo)).astype(np.float32)
        out.append((W, np.zeros(fo, dtype=np.float32)))
    return out


def param_count(widths) -> int:
    return sum(2 * fi * fo + fo for fi, fo in zip(widths[:-1], widths[1:]))


def random_graph(n: int, p_edge: float, seed: int, f0: int = 5, classes: int = 3,
                 multilabel: bool = False, isolated: int = 0) -> Graph:
    """Erdos-Renyi symmetric graph for tiny-size pins (brute force / finite differences)."""
    rng = np.random.default_rng([seed, 77])
    A = rng.random((n, n)) < p_edge
    A = np.triu(A, 1)
    A = A | A.T
    if isolated:
        A[:isolated, :] = False
        A[:, :isolated] = False
    rows, cols = np.nonzero(A)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    X = rng.standard_normal((n, f0)).astype(np.float32)
    if multilabel:
        labels = (rng.random((n, classes)) < 0.4).astype(np.uint8)
    else:
        labels = rng.integers(0, classes, n).astype(np.int32)
    train_mask = (rng.random(n) < 0.6).astype(np.uint8)
    train_mask[0] = 1
    return Graph(name="random", n=n, row_ptr=row_ptr, col_idx=cols.astype(np.int32), X=X,
                 labels=labels, train_mask=train_mask, n_classes=classes, multilabel=multilabel)
