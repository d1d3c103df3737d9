"""Dense-tile decomposition of the aggregation patterns (host C++, no GPU): pgcn_dev_tiles against a
brute-force rebuild.  The tensor-core aggregation sums heavy 128 x 64
tiles as 0/1 blocks and the light CSR by gathers, so bit-exact here means: heavy bits + light edges
reproduce every row of P_i / P_i^T as a multiset, heavy tiles are exactly the tiles with >= tile_min
edges, and the light CSR is sorted by column within each row."""
import numpy as np
import pytest

from synth.graphs import gen_graph, random_graph


@pytest.fixture(scope="module")
def P():
    from paper_2203_10428_b200 import build, pgcn
    build.build()
    return pgcn


def brute(rp, col, n_rows, tmin):
    """Per (row block, column tile) edge counts, heavy set, and the expected light edge lists."""
    counts = {}
    for r in range(n_rows):
        for e in range(rp[r], rp[r + 1]):
            k = (r // 128, int(col[e]) // 64)
            counts[k] = counts.get(k, 0) + 1
    heavy = {k for k, c in counts.items() if c >= tmin}
    light = []
    for r in range(n_rows):
        seen = set()
        row = []
        for e in range(rp[r], rp[r + 1]):
            c = int(col[e])
            if (r // 128, c // 64) in heavy and c not in seen:
                seen.add(c)
            else:
                row.append(c)
        light.append(row)
    return counts, heavy, light


def check(P, part, i, which, tmin):
    v = part.view(i)
    if which == 0:
        rp, col, n_rows, n_cols = v["row_ptr"], v["col_idx"], v["n_inner"], v["n_inner"] + v["n_halo"]
    else:
        rp, col, n_rows, n_cols = v["t_row_ptr"], v["t_col_idx"], v["n_inner"] + v["n_halo"], v["n_inner"]
    t = part.tiles(i, which, tmin)
    assert t["n_rows"] == n_rows and t["n_cols"] == n_cols
    assert t["n_rb"] == (n_rows + 127) // 128
    counts, heavy, light = brute(rp, col, n_rows, tmin)
    # heavy tiles: exactly the tiles with >= tmin edges, column tiles ascending within a block
    got = set()
    for b in range(t["n_rb"]):
        cols = t["tile_col"][t["rb_ptr"][b]:t["rb_ptr"][b + 1]]
        assert np.all(np.diff(cols) > 0)
        got |= {(b, int(j)) for j in cols}
    assert got == heavy
    # light CSR: exactly the non-heavy (or repeated) edges, columns ascending within a row
    assert t["nnz_light"] == sum(len(x) for x in light)
    for r in range(n_rows):
        np.testing.assert_array_equal(t["lcol"][t["lrp"][r]:t["lrp"][r + 1]], np.sort(np.asarray(light[r], np.int32)))
    # heavy bits + light edges = each row as a multiset
    rows = [[] for _ in range(n_rows)]
    for b in range(t["n_rb"]):
        for k in range(t["rb_ptr"][b], t["rb_ptr"][b + 1]):
            for r in range(128):
                w = int(t["mask"][128 * k + r])
                if w:
                    assert b * 128 + r < n_rows
                for c in range(64):
                    if (w >> c) & 1:
                        assert 64 * int(t["tile_col"][k]) + c < n_cols
                        rows[b * 128 + r].append(64 * int(t["tile_col"][k]) + c)
    assert t["nnz_heavy"] == sum(len(x) for x in rows)
    for r in range(n_rows):
        assert sorted(rows[r] + light[r]) == sorted(int(c) for c in col[rp[r]:rp[r + 1]]), r
    # work order: a permutation by descending tile count, stable
    cnt = np.diff(t["rb_ptr"])
    assert sorted(t["order"].tolist()) == list(range(t["n_rb"]))
    key = [(-int(cnt[b]), b) for b in t["order"]]
    assert key == sorted(key)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("tmin", [1, 3, 40])
def test_tiles_random(P, seed, tmin):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(100, 700))
    g = random_graph(n, float(rng.uniform(0.01, 0.2)), seed, isolated=int(rng.integers(0, 5)))
    part = P.partition(n, g.row_ptr, g.col_idx, 1 + seed % 3)
    for i in range(part.n_parts):
        for which in (0, 1):
            check(P, part, i, which, tmin)


def test_tiles_community_graph(P):
    """Reddit-like structure (dense communities): most edges land in heavy tiles."""
    g = gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=8, classes=4)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    for i in range(2):
        for which in (0, 1):
            check(P, part, i, which, 96)
            t = part.tiles(i, which, 96)
            assert t["nnz_heavy"] > 0.5 * (t["nnz_heavy"] + t["nnz_light"])


def test_tiles_repeated_edges(P):
    """A repeated (row, col) pair cannot be counted twice by a bitmask: the repeat goes light."""
    n = 200
    rows = [[(r * 7 + k) % n for k in range(5)] + [(r * 7) % n] for r in range(n)]  # first neighbour twice
    rp = np.zeros(n + 1, np.int64)
    rp[1:] = np.cumsum([len(x) for x in rows])
    col = np.concatenate([np.asarray(x, np.int32) for x in rows])
    part = P.partition(n, rp, col, 1)
    for which in (0, 1):
        for tmin in (1, 2):
            check(P, part, 0, which, tmin)
    t = part.tiles(0, 0, 1)
    assert t["nnz_light"] >= n  # every repeat is light


def test_tiles_empty(P):
    rp = np.zeros(11, np.int64)
    part = P.partition(10, rp, np.zeros(0, np.int32), 2)
    for i in range(2):
        for which in (0, 1):
            t = part.tiles(i, which, 1)
            assert t["n_tiles"] == 0 and t["nnz_light"] == 0


def test_config_fields_reach_the_library(P):
    """pgcn_config.spmm_tiles / tile_min / train_sparse cross the C ABI (ctypes layout = include/pgcn.h):
    the workspace grows by the tile sets exactly when the tile path is enabled on a dense graph, shrinks
    when a huge tile_min leaves no heavy tiles, and invalid values are rejected."""
    import ctypes
    import numpy as np
    g = gen_graph("reddit", seed=3, n=1500, nnz=60000, f0=16, classes=4)
    part = P.partition(g.n, g.row_ptr, g.col_idx, 2)
    local = np.arange(2, dtype=np.int32)

    def ws(**kw):
        cfg = P.make_config([16, 32, 4], n_global=g.n, n_train_global=g.n_train, **kw)
        nb = ctypes.c_size_t()
        rc = P.lib().pgcn_workspace_bytes(part.handle, local.ctypes.data, 2, ctypes.byref(cfg), ctypes.byref(nb))
        return rc, nb.value
    rc0, off = ws(spmm_tiles=False)
    rc1, on = ws(spmm_tiles=True, tile_min=1)
    rc2, none = ws(spmm_tiles=True, tile_min=128 * 64)
    assert rc0 == rc1 == rc2 == 0
    assert on > off and none == off
    assert ws(spmm_tiles=True, tile_min=-1)[0] == P.EINVAL
