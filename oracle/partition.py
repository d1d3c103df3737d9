"""Alg. 1 lines 1-5 -- test infrastructure only (see oracle/__init__.py).

For partition i of n (node -> partition map `part_of`):

  l.1   V_i     = { v in G_i : v not in B_i }  -- the nodes partition i owns
        B_i     = { u : u in N(v) for some v in V_i, part_of[u] != i }  (boundary / halo)
  l.2-3 S_{i,j} = B_j  intersect V_i   (rows i sends to j)
  l.4-5 S_{j,i} = B_i  intersect V_j   (rows i receives from j)
  P_i   = rows V_i of the propagation matrix, columns V_i + B_i, with the mean
          aggregator's weight 1/d_v (Eq. 3; d_v = full-graph degree,
          PAPER.md:462, reading R1).

Canonical orders (reading R20, needed for "bit-exact"): V_i ascending gid; B_i by
(owner, gid); S_{i,j} ascending gid; local CSR keeps each row's global neighbour
order; transposed rows list inner v ascending; inverse send map ascending k.
Default map (reading R19, METIS is out of scope): contiguous ranges
lo_p = floor(p * N / n).
"""
import numpy as np


def contiguous_map(n: int, n_parts: int) -> np.ndarray:
    lo = (np.arange(n_parts + 1, dtype=np.int64) * n) // n_parts
    part_of = np.empty(n, dtype=np.int32)
    for p in range(n_parts):
        part_of[lo[p]:lo[p + 1]] = p
    return part_of


def partition(n, row_ptr, col_idx, n_parts, part_of=None):
    """List of per-partition dicts with the arrays of include/pgcn.h `pgcn_part_view`."""
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    part_of = contiguous_map(n, n_parts) if part_of is None else np.asarray(part_of, dtype=np.int32)
    deg = np.diff(row_ptr)
    parts = []
    # l.1: inner and boundary sets
    for i in range(n_parts):
        inner = np.nonzero(part_of == i)[0].astype(np.int64)
        starts, ends = row_ptr[inner], row_ptr[inner + 1]
        nb = np.concatenate([col_idx[s:e] for s, e in zip(starts, ends)]) if inner.size else \
            np.zeros(0, np.int64)
        halo = np.unique(nb[part_of[nb] != i])
        halo = halo[np.lexsort((halo, part_of[halo]))]          # (owner, gid)
        halo_off = np.searchsorted(part_of[halo], np.arange(n_parts + 1), side="left").astype(np.int64)
        parts.append(dict(part=i, n_parts=n_parts, inner_gid=inner, halo_gid=halo.astype(np.int64),
                          halo_off=halo_off))
    # l.2-5: S_{i,j} = B_j ∩ V_i  (= j's halo segment owned by i, already ascending gid)
    for i, P in enumerate(parts):
        inner = P["inner_gid"]
        send_gid, send_off = [], [0]
        for j in range(n_parts):
            Q = parts[j]
            seg = Q["halo_gid"][Q["halo_off"][i]:Q["halo_off"][i + 1]] if j != i else np.zeros(0, np.int64)
            seg = seg[np.isin(seg, inner)]                      # B_j ∩ V_i
            send_gid.append(seg)
            send_off.append(send_off[-1] + seg.size)
        send_gid = np.concatenate(send_gid) if send_gid else np.zeros(0, np.int64)
        P["send_off"] = np.array(send_off, dtype=np.int64)
        P["send_idx"] = np.searchsorted(inner, send_gid).astype(np.int32)
        P["send_gid"] = send_gid
    # local P_i pattern, inv_deg, transposed pattern, inverse send map
    for i, P in enumerate(parts):
        inner, halo = P["inner_gid"], P["halo_gid"]
        n_in, n_bd = inner.size, halo.size
        loc = np.full(n, -1, dtype=np.int64)
        loc[inner] = np.arange(n_in)
        loc[halo] = n_in + np.arange(n_bd)
        starts, ends = row_ptr[inner], row_ptr[inner + 1]
        lens = ends - starts
        rp = np.zeros(n_in + 1, dtype=np.int64)
        np.cumsum(lens, out=rp[1:])
        cols = np.concatenate([col_idx[s:e] for s, e in zip(starts, ends)]) if n_in else np.zeros(0, np.int64)
        lc = loc[cols]
        assert (lc >= 0).all()
        d = deg[inner]
        inv = np.where(d > 0, 1.0 / np.maximum(d, 1), 0.0)
        # P_i^T: for local row u, the inner rows v (ascending) whose neighbour list holds u
        rows_of = np.repeat(np.arange(n_in, dtype=np.int64), lens)
        order = np.argsort(lc, kind="stable")
        t_rp = np.zeros(n_in + n_bd + 1, dtype=np.int64)
        np.cumsum(np.bincount(lc, minlength=n_in + n_bd), out=t_rp[1:])
        si = P["send_idx"].astype(np.int64)
        iorder = np.argsort(si, kind="stable")
        inv_ptr = np.zeros(n_in + 1, dtype=np.int64)
        np.cumsum(np.bincount(si, minlength=n_in), out=inv_ptr[1:])
        P.update(n_inner=n_in, n_halo=n_bd, nnz=int(rp[-1]), n_send=int(si.size),
                 deg=deg[np.concatenate([inner, halo])].astype(np.int64),
                 row_ptr=rp, col_idx=lc.astype(np.int32), inv_deg=inv,
                 t_row_ptr=t_rp, t_col_idx=rows_of[order].astype(np.int32),
                 inv_ptr=inv_ptr, inv_pos=iorder.astype(np.int32))
    return parts


def local_P(P, model="sage"):
    """scipy CSR of P_i (n_inner x (n_inner + n_halo)).
    sage: values inv_deg[v] (mean aggregator, Eq. 3).
    gcn:  P = D~^-1/2 (A + I) D~^-1/2 (App. A.1), D~ = d + 1 (full-graph degrees of
          both endpoints, incl. boundary nodes): P_i[v, u] = 1/sqrt((d_v+1)(d_u+1)) for u in N(v) and
          the self loop u = v."""
    import scipy.sparse as sp
    n_in, n_all = P["n_inner"], P["n_inner"] + P["n_halo"]
    if model == "sage":
        vals = np.repeat(P["inv_deg"], np.diff(P["row_ptr"]))
        return sp.csr_matrix((vals, P["col_idx"].astype(np.int64), P["row_ptr"]), shape=(n_in, n_all))
    s = 1.0 / np.sqrt(P["deg"].astype(np.float64) + 1.0)
    rows = np.repeat(np.arange(n_in), np.diff(P["row_ptr"]))
    cols = P["col_idx"].astype(np.int64)
    r = np.concatenate([rows, np.arange(n_in)])
    c = np.concatenate([cols, np.arange(n_in)])
    return sp.csr_matrix((s[r] * s[c], (r, c)), shape=(n_in, n_all))
