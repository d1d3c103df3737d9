// Host partitioner: Alg. 1 l.1-5 -- see include/pgcn.h for the contract.
//
//   V_i     = nodes owned by i                     (l.1)
//   B_i     = off-partition in-neighbours of V_i   (l.1)
//   S_{i,j} = B_j ∩ V_i, S_{j,i} = B_i ∩ V_j       (l.2-5)
//   P_i     = rows V_i of P with weight 1/d_v      (Eq. 3; d_v full degree)
//
// Design: one pass per partition over its own rows (partitions are independent after the
// boundary sets are known, so they run on separate threads); every output order is the
// canonical one of include/pgcn.h (reading R20), so the result does not depend on the
// thread count.  Global -> local lookups use one shared int32 array of size N
// (`pos_in_part`, a node's rank inside its owner); V_i comes from one counting pass over the
// nodes, and each partition's boundary scan marks seen nodes in an N-bit set (N/8 bytes per
// thread).  A worker that throws (std::bad_alloc) hands the exception to the calling thread,
// which returns PGCN_ENOMEM.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <new>
#include <thread>
#include <vector>

#include "common.h"
#include "pgcn.h"
#include "tiles.h"

struct PartArrays {
  std::vector<int64_t> inner_gid, halo_gid, halo_off, send_off, row_ptr, t_row_ptr, inv_ptr;
  std::vector<int32_t> send_idx, col_idx, t_col_idx, inv_pos;
  std::vector<float> inv_deg;
  std::vector<int64_t> deg;  // full-graph degree of inner then boundary rows (GCN-sym, R26)
};

struct pgcn_partitioning {
  int64_t n;
  int32_t n_parts;
  std::vector<int32_t> part_of;
  std::vector<PartArrays> parts;
  // dense-tile decompositions of P_i / P_i^T (tiles.h), built on first use
  std::mutex tile_mu;
  std::map<std::tuple<int32_t, int, int32_t>, std::unique_ptr<pgcn::TileSet>> tiles;
};

namespace {

// Runs f(0..n_items) on up to n_threads threads; the first exception thrown by any item is
// rethrown on the calling thread after every worker has joined.
template <class F>
void run_threads(int n_items, int n_threads, F f) {
  n_threads = std::max(1, std::min(n_threads, n_items));
  if (n_threads == 1) {
    for (int i = 0; i < n_items; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  std::atomic<int> next{0};
  std::mutex mu;
  std::exception_ptr err;
  for (int k = 0; k < n_threads; ++k)
    th.emplace_back([&] {
      try {
        for (int i = next++; i < n_items; i = next++) f(i);
      } catch (...) {
        std::lock_guard<std::mutex> g(mu);
        if (!err) err = std::current_exception();
        next = n_items;  // stop handing out items
      }
    });
  for (auto& x : th) x.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

extern "C" int pgcn_partition(int64_t n, const int64_t* row_ptr, const int32_t* col_idx,
                              int32_t n_parts, const int32_t* part_of_in, int32_t n_threads,
                              pgcn_partitioning** out) {
  using namespace pgcn;
  if (!out) return fail(PGCN_EINVAL, "pgcn_partition: out is NULL");
  *out = nullptr;
  if (n <= 0 || n >= (int64_t(1) << 31)) return fail(PGCN_EINVAL, "pgcn_partition: n_nodes out of range");
  if (!row_ptr || (!col_idx && row_ptr[n] > 0)) return fail(PGCN_EINVAL, "pgcn_partition: null CSR");
  if (n_parts < 1 || n_parts > PGCN_MAX_PARTS) return fail(PGCN_EINVAL, "pgcn_partition: n_parts out of range");
  if (row_ptr[0] != 0) return fail(PGCN_EINVAL, "pgcn_partition: row_ptr[0] != 0");
  for (int64_t v = 0; v < n; ++v)
    if (row_ptr[v + 1] < row_ptr[v]) return fail(PGCN_EINVAL, "pgcn_partition: row_ptr not monotone");
  const int64_t nnz = row_ptr[n];
  if (n_threads <= 0) n_threads = (int)std::max(1u, std::thread::hardware_concurrency());

  std::unique_ptr<pgcn_partitioning> P;
  try {
    P.reset(new pgcn_partitioning());
    P->n = n;
    P->n_parts = n_parts;
    P->part_of.resize(n);
    if (part_of_in) {
      for (int64_t v = 0; v < n; ++v) {
        if (part_of_in[v] < 0 || part_of_in[v] >= n_parts)
          return fail(PGCN_EINVAL, "pgcn_partition: part_of out of range");
        P->part_of[v] = part_of_in[v];
      }
    } else {
      for (int32_t p = 0; p < n_parts; ++p) {
        int64_t lo = (int64_t)p * n / n_parts, hi = (int64_t)(p + 1) * n / n_parts;
        for (int64_t v = lo; v < hi; ++v) P->part_of[v] = p;
      }
    }
    {  // column range check (parallel)
      std::atomic<bool> bad{false};
      const int chunks = 64;
      run_threads(chunks, n_threads, [&](int c) {
        int64_t lo = nnz * c / chunks, hi = nnz * (c + 1) / chunks;
        for (int64_t e = lo; e < hi; ++e)
          if (col_idx[e] < 0 || col_idx[e] >= n) { bad = true; return; }
      });
      if (bad) return fail(PGCN_EINVAL, "pgcn_partition: col_idx out of range");
    }
    const int32_t* part_of = P->part_of.data();
    // rank of each node inside its owner (V_i ascending gid -> local inner id)
    std::vector<int32_t> pos_in_part(n);
    std::vector<int64_t> count(n_parts, 0);
    for (int64_t v = 0; v < n; ++v) pos_in_part[v] = (int32_t)count[part_of[v]]++;
    P->parts.resize(n_parts);
    for (int32_t i = 0; i < n_parts; ++i) P->parts[i].inner_gid.resize(count[i]);
    for (int64_t v = 0; v < n; ++v) P->parts[part_of[v]].inner_gid[pos_in_part[v]] = v;  // V_i ascending

    // l.1: B_i (boundary sorted by (owner, gid))
    run_threads(n_parts, n_threads, [&](int i) {
      PartArrays& A = P->parts[i];
      std::vector<uint64_t> seen((size_t)(n + 63) / 64, 0);
      std::vector<int64_t> halo;
      for (int64_t v : A.inner_gid)
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
          const int32_t u = col_idx[e];
          const uint64_t bit = uint64_t(1) << (u & 63);
          if (part_of[u] != i && !(seen[u >> 6] & bit)) {
            seen[u >> 6] |= bit;
            halo.push_back(u);
          }
        }
      std::sort(halo.begin(), halo.end(), [&](int64_t a, int64_t b) {
        return part_of[a] != part_of[b] ? part_of[a] < part_of[b] : a < b;
      });
      A.halo_gid = std::move(halo);
      A.halo_off.assign(n_parts + 1, 0);
      for (int64_t u : A.halo_gid) A.halo_off[part_of[u] + 1]++;
      for (int j = 0; j < n_parts; ++j) A.halo_off[j + 1] += A.halo_off[j];
    });
    // l.2-5: S_{i,j} = B_j ∩ V_i = j's boundary segment owned by i (ascending gid)
    run_threads(n_parts, n_threads, [&](int i) {
      PartArrays& A = P->parts[i];
      A.send_off.assign(n_parts + 1, 0);
      for (int j = 0; j < n_parts; ++j) {
        const PartArrays& B = P->parts[j];
        int64_t len = (j == i) ? 0 : B.halo_off[i + 1] - B.halo_off[i];
        A.send_off[j + 1] = A.send_off[j] + len;
      }
      A.send_idx.resize(A.send_off[n_parts]);
      for (int j = 0; j < n_parts; ++j) {
        if (j == i) continue;
        const PartArrays& B = P->parts[j];
        for (int64_t k = 0; k < B.halo_off[i + 1] - B.halo_off[i]; ++k)
          A.send_idx[A.send_off[j] + k] = pos_in_part[B.halo_gid[B.halo_off[i] + k]];
      }
      // inverse send map: positions k with send_idx[k] == v, ascending k
      const int64_t n_in = (int64_t)A.inner_gid.size();
      A.inv_ptr.assign(n_in + 1, 0);
      for (int32_t v : A.send_idx) A.inv_ptr[v + 1]++;
      for (int64_t v = 0; v < n_in; ++v) A.inv_ptr[v + 1] += A.inv_ptr[v];
      A.inv_pos.resize(A.send_idx.size());
      std::vector<int64_t> cur(A.inv_ptr.begin(), A.inv_ptr.end() - 1);
      for (int64_t k = 0; k < (int64_t)A.send_idx.size(); ++k) A.inv_pos[cur[A.send_idx[k]]++] = (int32_t)k;
    });
    // P_i pattern (global neighbour order kept), inv_deg, P_i^T pattern
    run_threads(n_parts, n_threads, [&](int i) {
      PartArrays& A = P->parts[i];
      const int64_t n_in = (int64_t)A.inner_gid.size(), n_bd = (int64_t)A.halo_gid.size();
      std::vector<int32_t> hpos;  // gid -> boundary position, only for this partition's halo
      std::vector<std::pair<int32_t, int32_t>> hmap(A.halo_gid.size());
      for (int64_t k = 0; k < n_bd; ++k) hmap[k] = {(int32_t)A.halo_gid[k], (int32_t)k};
      std::sort(hmap.begin(), hmap.end());
      auto halo_pos = [&](int32_t u) -> int32_t {
        auto it = std::lower_bound(hmap.begin(), hmap.end(), std::make_pair(u, INT32_MIN));
        return it->second;
      };
      A.row_ptr.assign(n_in + 1, 0);
      A.inv_deg.resize(n_in);
      for (int64_t r = 0; r < n_in; ++r) {
        int64_t v = A.inner_gid[r];
        int64_t d = row_ptr[v + 1] - row_ptr[v];
        A.row_ptr[r + 1] = A.row_ptr[r] + d;
        A.inv_deg[r] = d > 0 ? 1.0f / (float)d : 0.0f;
      }
      A.deg.resize(n_in + n_bd);
      for (int64_t r = 0; r < n_in; ++r) A.deg[r] = A.row_ptr[r + 1] - A.row_ptr[r];
      for (int64_t k = 0; k < n_bd; ++k) A.deg[n_in + k] = row_ptr[A.halo_gid[k] + 1] - row_ptr[A.halo_gid[k]];
      A.col_idx.resize(A.row_ptr[n_in]);
      std::vector<int64_t> tcount(n_in + n_bd + 1, 0);
      for (int64_t r = 0; r < n_in; ++r) {
        int64_t v = A.inner_gid[r];
        int64_t o = A.row_ptr[r];
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; ++e) {
          int32_t u = col_idx[e];
          int32_t c = part_of[u] == i ? pos_in_part[u] : (int32_t)(n_in + halo_pos(u));
          A.col_idx[o + (e - row_ptr[v])] = c;
          tcount[c + 1]++;
        }
      }
      for (int64_t u = 0; u < n_in + n_bd; ++u) tcount[u + 1] += tcount[u];
      A.t_row_ptr = tcount;
      A.t_col_idx.resize(A.col_idx.size());
      std::vector<int64_t> cur(tcount.begin(), tcount.end() - 1);
      for (int64_t r = 0; r < n_in; ++r)
        for (int64_t e = A.row_ptr[r]; e < A.row_ptr[r + 1]; ++e) A.t_col_idx[cur[A.col_idx[e]]++] = (int32_t)r;
    });
  } catch (const std::bad_alloc&) {
    return fail(PGCN_ENOMEM, "pgcn_partition: host allocation failed");
  } catch (...) {
    return fail(PGCN_ENOMEM, "pgcn_partition: worker failed");
  }
  *out = P.release();
  return PGCN_OK;
}

extern "C" int pgcn_partition_view(const pgcn_partitioning* p, int32_t part, pgcn_part_view* o) {
  using namespace pgcn;
  if (!p || !o) return fail(PGCN_EINVAL, "pgcn_partition_view: null argument");
  if (part < 0 || part >= p->n_parts) return fail(PGCN_EINVAL, "pgcn_partition_view: part out of range");
  const PartArrays& A = p->parts[part];
  o->part = part;
  o->n_parts = p->n_parts;
  o->n_inner = (int64_t)A.inner_gid.size();
  o->n_halo = (int64_t)A.halo_gid.size();
  o->nnz = (int64_t)A.col_idx.size();
  o->n_send = (int64_t)A.send_idx.size();
  o->inner_gid = A.inner_gid.data();
  o->halo_gid = A.halo_gid.data();
  o->halo_off = A.halo_off.data();
  o->send_off = A.send_off.data();
  o->send_idx = A.send_idx.data();
  o->row_ptr = A.row_ptr.data();
  o->col_idx = A.col_idx.data();
  o->inv_deg = A.inv_deg.data();
  o->t_row_ptr = A.t_row_ptr.data();
  o->t_col_idx = A.t_col_idx.data();
  o->inv_ptr = A.inv_ptr.data();
  o->inv_pos = A.inv_pos.data();
  o->deg = A.deg.data();
  return PGCN_OK;
}

extern "C" int64_t pgcn_partition_n_nodes(const pgcn_partitioning* p) { return p ? p->n : -1; }

extern "C" void pgcn_partition_free(pgcn_partitioning* p) { delete p; }

namespace pgcn {

const TileSet* part_tiles(const pgcn_partitioning* p, int32_t part, int which, int32_t min_edges) {
  if (!p || part < 0 || part >= p->n_parts) return nullptr;
  auto* q = const_cast<pgcn_partitioning*>(p);
  std::lock_guard<std::mutex> g(q->tile_mu);
  auto key = std::make_tuple(part, which, min_edges);
  auto it = q->tiles.find(key);
  if (it != q->tiles.end()) return it->second.get();
  const PartArrays& a = p->parts[part];
  const int64_t n_in = (int64_t)a.inner_gid.size(), n_all = n_in + (int64_t)a.halo_gid.size();
  auto ts = std::make_unique<TileSet>();
  const int nt = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (which == 0) build_tiles(a.row_ptr.data(), a.col_idx.data(), n_in, n_all, min_edges, nt, *ts);
  else build_tiles(a.t_row_ptr.data(), a.t_col_idx.data(), n_all, n_in, min_edges, nt, *ts);
  const TileSet* r = ts.get();
  q->tiles.emplace(key, std::move(ts));
  return r;
}

}  // namespace pgcn
