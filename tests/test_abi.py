"""C-ABI boundary (no GPU needed): the library loads, exports every symbol include/pgcn.h
declares, and pgcn_partition (host C++) is bit-exact with the oracle's Alg. 1 l.1-5."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle.partition import contiguous_map
from oracle.partition import partition as oracle_partition
from synth.graphs import gen_graph, random_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def header_functions():
    import glob
    src = "\n".join(open(f).read() for f in sorted(glob.glob(os.path.join(ROOT, "include", "*.h"))))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pgcn_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(P):
    lib = ctypes.CDLL(P.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert P.lib().pgcn_version() >= 100


ARRAYS = ["inner_gid", "halo_gid", "halo_off", "send_off", "send_idx", "row_ptr", "col_idx", "t_row_ptr",
          "t_col_idx", "inv_ptr", "inv_pos", "deg"]


def compare(pv, ov):
    for k in ARRAYS:
        np.testing.assert_array_equal(pv[k].astype(np.int64), np.asarray(ov[k]).astype(np.int64), err_msg=k)
    # fp32(1)/fp32(d) is the correctly rounded 1/d, i.e. the fp64 value rounded once to fp32
    np.testing.assert_array_equal(pv["inv_deg"], np.asarray(ov["inv_deg"]).astype(np.float32))
    for k in ("n_inner", "n_halo", "nnz", "n_send"):
        assert pv[k] == ov[k], k


@pytest.mark.parametrize("seed", range(50))
def test_partition_bit_exact_random(P, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    g = random_graph(n, float(rng.uniform(0.0, 0.4)), seed, isolated=int(rng.integers(0, 3)))
    for n_parts in (1, 2, 3, 4, 8):
        part_of = rng.integers(0, n_parts, n).astype(np.int32) if seed % 2 else None
        pp = P.partition(n, g.row_ptr, g.col_idx, n_parts, part_of, n_threads=1 + seed % 4)
        op = oracle_partition(n, g.row_ptr, g.col_idx, n_parts, part_of)
        for i in range(n_parts):
            compare(pp.view(i), op[i])


@pytest.mark.parametrize("n_parts", [2, 4, 8])
def test_partition_bit_exact_generator_graph(P, n_parts):
    g = gen_graph("yelp", seed=1, n=20000, nnz=200000, f0=4, classes=3)
    pp = P.partition(g.n, g.row_ptr, g.col_idx, n_parts)
    op = oracle_partition(g.n, g.row_ptr, g.col_idx, n_parts)
    for i in range(n_parts):
        compare(pp.view(i), op[i])


def test_partition_errors(P):
    rp = np.array([0, 1, 2], np.int64)
    col = np.array([1, 0], np.int32)
    with pytest.raises(P.PgcnError) as e:
        P.partition(2, rp, col, 0)
    assert e.value.code == P.EINVAL
    with pytest.raises(P.PgcnError) as e:
        P.partition(2, rp, np.array([1, 5], np.int32), 2)
    assert e.value.code == P.EINVAL and "col_idx" in str(e.value)
    with pytest.raises(P.PgcnError) as e:
        P.partition(2, np.array([0, 2, 1], np.int64), col, 2)
    assert e.value.code == P.EINVAL
    with pytest.raises(P.PgcnError) as e:
        P.partition(2, rp, col, 2, part_of=np.array([0, 3], np.int32))
    assert e.value.code == P.EINVAL


def test_partition_deterministic_across_threads(P):
    g = gen_graph("cora", seed=3)
    a = P.partition(g.n, g.row_ptr, g.col_idx, 4, n_threads=1)
    b = P.partition(g.n, g.row_ptr, g.col_idx, 4, n_threads=8)
    for i in range(4):
        va, vb = a.view(i), b.view(i)
        for k in ARRAYS + ["inv_deg"]:
            assert np.array_equal(va[k], vb[k])


def test_contiguous_map_matches_header_rule():
    # lo_p = floor(p * N / n) (include/pgcn.h, reading R19)
    m = contiguous_map(10, 3)
    assert m.tolist() == [0, 0, 0, 1, 1, 1, 2, 2, 2, 2]


def test_lean_workspace_host_query(P):
    """N1(iii) lean-memory mode through the host-only workspace query: a papers-shaped layer stack
    (transform-first layer 1, compact last layer) needs fewer bytes with lean = 1, exactly the dropped
    buffers' worth at least the shared Z / J slots; lean with the LOCAL transport and several
    partitions is rejected (PGCN_EUNSUPPORTED)."""
    g = gen_graph("papers", seed=3, n=20000, nnz=180000, f0=64, classes=40)
    widths = [64, 16, 16, 40]
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    kw = dict(n_global=g.n, n_train_global=g.n_train, train_sparse=True, transport="loopback")
    full = P.workspace_bytes(part, P.make_config(widths, **kw))
    lean = P.workspace_bytes(part, P.make_config(widths, lean=True, **kw))
    v = [part.view(i) for i in range(2)]
    n_in = [int(x["n_inner"]) for x in v]
    n_all = [int(x["n_inner"] + x["n_halo"]) for x in v]
    # at least: the last layer's logits (n_in x 40) and two of the three Z buffers (n_in x 16), one J slot
    # per hidden layer (n_all x 16) are gone; M shrinks from width 40 to 16
    dropped = sum(4 * (ni * 40 + 2 * ni * 16 + 2 * na * 16 + ni * 24) for ni, na in zip(n_in, n_all))
    assert full - lean >= 0.95 * dropped, (full, lean, dropped)
    with pytest.raises(P.PgcnError):
        P.workspace_bytes(part, P.make_config(widths, lean=True, **dict(kw, transport="local")))
    # one partition: nothing is exchanged, LOCAL is fine
    part1 = P.partition(g.n, g.row_ptr, g.col_idx, 1)
    assert P.workspace_bytes(part1, P.make_config(widths, lean=True, **dict(kw, transport="local"))) > 0
