"""Pins for oracle/partition.py (Alg. 1 l.1-5).

Brute force: the set definitions written out with Python sets on tiny graphs; hand-derived
golden arrays (tests/golden/tiny4.json); structural invariants on generator graphs."""
import json
import os

import numpy as np
import pytest

from oracle.partition import contiguous_map, partition
from synth.graphs import gen_graph, random_graph


def brute_sets(n, row_ptr, col_idx, part_of, n_parts):
    N = {v: [int(u) for u in col_idx[row_ptr[v]:row_ptr[v + 1]]] for v in range(n)}
    V = [sorted(v for v in range(n) if part_of[v] == i) for i in range(n_parts)]
    B = []
    for i in range(n_parts):
        s = set()
        for v in V[i]:
            for u in N[v]:
                if part_of[u] != i:
                    s.add(u)
        B.append(sorted(s, key=lambda u: (part_of[u], u)))
    S = {(i, j): sorted(set(B[j]) & set(V[i])) for i in range(n_parts) for j in range(n_parts)}
    return N, V, B, S


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("n_parts", [1, 2, 3, 4])
def test_partition_matches_set_definitions(seed, n_parts):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    g = random_graph(n, float(rng.uniform(0.02, 0.4)), seed, isolated=int(rng.integers(0, 3)))
    if seed % 3 == 0:
        part_of = rng.integers(0, n_parts, n).astype(np.int32)   # caller-supplied map
    else:
        part_of = contiguous_map(n, n_parts)
    parts = partition(n, g.row_ptr, g.col_idx, n_parts, part_of)
    N, V, B, S = brute_sets(n, g.row_ptr, g.col_idx, part_of, n_parts)
    deg = np.diff(g.row_ptr)
    for i, P in enumerate(parts):
        assert P["inner_gid"].tolist() == V[i]
        assert P["halo_gid"].tolist() == B[i]
        for j in range(n_parts):
            seg = P["halo_gid"][P["halo_off"][j]:P["halo_off"][j + 1]].tolist()
            assert seg == S[(j, i)]                                          # S_{j,i} = B_i ∩ V_j
            snd = P["send_idx"][P["send_off"][j]:P["send_off"][j + 1]]
            assert [V[i][k] for k in snd] == S[(i, j)]                      # S_{i,j} = B_j ∩ V_i
        loc_gid = V[i] + B[i]
        for r, v in enumerate(V[i]):
            cols = P["col_idx"][P["row_ptr"][r]:P["row_ptr"][r + 1]]
            assert [loc_gid[c] for c in cols] == N[v]                       # global order kept
            assert P["inv_deg"][r] == (1.0 / deg[v] if deg[v] else 0.0)
        for u in range(len(loc_gid)):
            tv = P["t_col_idx"][P["t_row_ptr"][u]:P["t_row_ptr"][u + 1]].tolist()
            assert tv == [r for r, v in enumerate(V[i]) for x in N[v] if x == loc_gid[u]]
        for r in range(len(V[i])):
            ks = P["inv_pos"][P["inv_ptr"][r]:P["inv_ptr"][r + 1]].tolist()
            assert ks == [k for k in range(P["n_send"]) if P["send_idx"][k] == r]


def test_golden_tiny4(golden_dir):
    gd = json.load(open(os.path.join(golden_dir, "tiny4.json")))
    parts = partition(gd["n"], np.array(gd["row_ptr"]), np.array(gd["col_idx"]), gd["n_parts"])
    for P, E in zip(parts, gd["parts"]):
        for k, v in E.items():
            if k.startswith("_"):
                continue
            np.testing.assert_array_equal(np.asarray(P[k]), np.asarray(v), err_msg=k)


@pytest.mark.parametrize("n_parts", [2, 4, 8])
def test_invariants_generator_graph(n_parts):
    g = gen_graph("cora", seed=1)
    parts = partition(g.n, g.row_ptr, g.col_idx, n_parts)
    allv = np.concatenate([P["inner_gid"] for P in parts])
    assert np.array_equal(np.sort(allv), np.arange(g.n))                     # ⋃V_i = V, disjoint
    for i, P in enumerate(parts):
        assert not np.intersect1d(P["inner_gid"], P["halo_gid"]).size        # B_i ∩ V_i = ∅
        assert P["send_off"][i + 1] == P["send_off"][i]                      # S_{i,i} = ∅
        for j, Q in enumerate(parts):
            a = P["send_off"][j + 1] - P["send_off"][j]
            b = Q["halo_off"][i + 1] - Q["halo_off"][i]
            assert a == b                                                    # |S_{i,j}| matches
            np.testing.assert_array_equal(
                P["inner_gid"][P["send_idx"][P["send_off"][j]:P["send_off"][j + 1]]],
                Q["halo_gid"][Q["halo_off"][i]:Q["halo_off"][i + 1]])
        # inverse map o send_idx = identity
        for r in range(P["n_inner"]):
            ks = P["inv_pos"][P["inv_ptr"][r]:P["inv_ptr"][r + 1]]
            assert (P["send_idx"][ks] == r).all()
        assert P["inv_ptr"][-1] == P["n_send"]
        # every cross edge's source is a boundary node
        assert P["t_row_ptr"][-1] == P["nnz"]
