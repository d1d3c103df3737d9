// sm_100a kernels of the PipeGCN hot path: aggregation SpMM (S3), transposed SpMM (S8),
// dropout (R5), boundary gather / EMA install (S1, S2, Sec. 3.4), stale-gradient accumulation
// (S9), loss (S5), SIMT fp32 GEMMs (S4, S6, S7; parity path) and the optimiser (S11, S12).
// Step numbers refer to SURVEY.md section 8(a); paper citations are in kernels.cuh / pgcn.h.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "kernels.cuh"
#include "pgcn_dev.h"

namespace pgcn {
namespace {

constexpr int kThreads = 256;
inline int grid_for(int64_t work, int per_block, int max_blocks = 0) {
  if (max_blocks <= 0) max_blocks = sm_count() * 16;
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// Bits 40..63 of SplitMix64(z) (reading R5 keeps an element iff they are >= thr).  The output
// xorshift z ^ (z >> 31) only changes bits 0..32, so it is skipped: same bits, fewer instructions.
__device__ __forceinline__ uint32_t smix_top24(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z >> 40);
}

// key = ((t(L+1)+l)N + gid) F + col: the row part kr = (key_base + gid) F is hoisted per row.
__device__ __forceinline__ uint64_t row_key(const DropSpec& d, int64_t gid) {
  return ((uint64_t)d.key_base + (uint64_t)gid) * (uint64_t)d.width;
}
__device__ __forceinline__ bool keep_at(const DropSpec& d, uint64_t kr, int64_t c) {
  return smix_top24((kr + (uint64_t)c) ^ d.seed) >= d.thr;
}
// Same decision as keep_at on the high word only: (z >> 40) >= thr  <=>  hi32(z) >= thr << 8 (thr < 2^24),
// and the last multiply only needs hi32 of the product.  k_dropout is ALU-bound on this hash (the
// branchy per-element form ran ~50 instructions per element, ~4.3 TB/s), so it is written out.
__device__ __forceinline__ bool keep_fast(uint64_t key, uint64_t seed, uint32_t thr8) {
  uint64_t z = (key ^ seed) + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  const uint32_t top = __umulhi(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu;
  return top >= thr8;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// bf16 packing (round to nearest even) and exact widening accumulate of a bf16 pair on FADD2.
__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ void bf16x2_acc(float& a0, float& a1, uint32_t w) {
  // mixed-precision adds (fp32 += bf16 half-word): one FHADD.BF16 per element, no unpacking
  asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
      "add.rn.f32.bf16 %0, l, %0;\n\tadd.rn.f32.bf16 %1, h, %1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "r"(w));
}
// Neighbour row c's float4 at lane base bq: one IMAD.WIDE.U32 with a 64-bit addend.
__device__ __forceinline__ const float4* nbr(const char* bq, uint32_t c, uint32_t row_bytes) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(c), "r"(row_bytes), "l"(reinterpret_cast<uint64_t>(bq)));
  return reinterpret_cast<const float4*>(r);
}
// Same sums as f4add (round-to-nearest per component) on the packed fp32x2 pipe (FADD2): half
// the add instructions of the SpMM inner loops.
__device__ __forceinline__ void f4acc(float4& a, const float4& b) {
  asm("{\n\t.reg .b64 p, q;\n\t"
      "mov.b64 p, {%0, %1};\n\tmov.b64 q, {%4, %5};\n\tadd.rn.f32x2 p, p, q;\n\tmov.b64 {%0, %1}, p;\n\t"
      "mov.b64 p, {%2, %3};\n\tmov.b64 q, {%6, %7};\n\tadd.rn.f32x2 p, p, q;\n\tmov.b64 {%2, %3}, p;\n\t}"
      : "+f"(a.x), "+f"(a.y), "+f"(a.z), "+f"(a.w)
      : "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w));
}
__device__ __forceinline__ float4 f4scale(float4 a, float s) {
  return make_float4(a.x * s, a.y * s, a.z * s, a.w * s);
}
__device__ __forceinline__ float comp(const float4& v, int j) {
  return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set_comp(float4& v, int j, float x) {
  if (j == 0) v.x = x; else if (j == 1) v.y = x; else if (j == 2) v.z = x; else v.w = x;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
  }
}

__device__ __forceinline__ int find_seg(const SegTable& t, int64_t r) {
  int lo = 0, hi = t.n_seg - 1;  // largest s with off[s] <= r
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (t.off[mid] <= r) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Division-free grid-stride walk over the float4 elements (r, x) of an n_rows x ld4 array: one
// 64-bit division per thread at the start, then (r, x) advances by the grid size with a carry.
struct RowCursor {
  int64_t r;
  int x, dx;
  int64_t dr;
  __device__ __forceinline__ RowCursor(int64_t ld4) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T = (int64_t)gridDim.x * blockDim.x;
    r = g / ld4;
    x = (int)(g - r * ld4);
    dr = T / ld4;
    dx = (int)(T - dr * ld4);
  }
  __device__ __forceinline__ void next(int ld4) {
    r += dr;
    x += dx;
    if (x >= ld4) { x -= ld4; ++r; }
  }
};

// ---------------------------------------------------------------- dropout (S3 prologue, R5)
// d.scale is applied only when d.on (the transposed SpMMs pass a zero-initialised "no dropout" spec).
__device__ __forceinline__ float4 drop4(const float4 h, int64_t x, uint64_t kr, float sr, const DropSpec& d) {
  float4 out;
  if (d.on && d.thr < (1u << 24) && 4 * x + 4 <= d.width) {  // whole float4 in the row: branch-free mask
    const uint64_t k0 = kr + (uint64_t)(4 * x);
    const uint32_t thr8 = d.thr << 8;
    out.x = keep_fast(k0, d.seed, thr8) ? h.x * d.scale * sr : 0.f;
    out.y = keep_fast(k0 + 1, d.seed, thr8) ? h.y * d.scale * sr : 0.f;
    out.z = keep_fast(k0 + 2, d.seed, thr8) ? h.z * d.scale * sr : 0.f;
    out.w = keep_fast(k0 + 3, d.seed, thr8) ? h.w * d.scale * sr : 0.f;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = 4 * x + j;
      float v = 0.f;
      if (c < d.width && (!d.on || keep_at(d, kr, c))) v = (d.on ? comp(h, j) * d.scale : comp(h, j)) * sr;
      set_comp(out, j, v);
    }
  }
  return out;
}

// One float4 per thread per grid-stride step (two loads in flight per thread, hashed after both
// landed, measured no faster: r1n).
__global__ void k_dropout(const float4* __restrict__ H, float4* __restrict__ D, int64_t ld4, int64_t n_rows,
                          int64_t n_valid, const int64_t* __restrict__ gid, DropSpec d, const float* __restrict__ rs) {
  for (RowCursor rc(ld4); rc.r < n_rows; rc.next((int)ld4)) {
    const int64_t r = rc.r, x = rc.x, i = r * ld4 + x;
    float4 out = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < n_valid) out = drop4(H[i], x, row_key(d, gid[r]), rs ? rs[r] : 1.f, d);
    D[i] = out;
  }
}

// ---------------------------------------------------------------- SpMM forward (S3)
// Output rows, their in-place partial sums and dD_self are touched once per launch: streamed with
// evict-first hints (__ldcs / __stcs) so they do not displace the gathered table from L2.
// Work item = (row, chunk): a group of G lanes owns NC*G float4 columns of one output row (for
// every width used here one chunk covers the whole row) and keeps NC float4 accumulators; U
// neighbour rows are in flight per step, so each lane has NC*U 16-byte loads outstanding.  The
// (G, NC, U) table in spmm_shape() was measured with tools/ab_r1/spmm_lab.py on B200 (whole row per
// group, ~8 loads in flight).  Neighbour ids are loaded G at a time (coalesced)
// and broadcast with shuffles.  Sums run in CSR order, then the row is scaled by inv_deg (R16).
// Work distribution: static grid-stride, or (work != nullptr) dynamic -- each group takes the
// next K items from a per-launch atomic counter, so heavy-tailed degrees do not leave a tail of
// groups still busy with their statically assigned long rows.  K (launcher: ~128 edges per grab)
// keeps the single counter off the critical path on low-degree graphs (papers-shaped: 14.5 edges
// per row would otherwise mean one same-address atomic per 14.5 edges).
template <int G>
__device__ __forceinline__ int64_t next_item(unsigned long long* work, int lane, unsigned gm, int64_t cur,
                                             int64_t stride, int K, int64_t& cend) {
  if (!work) return cur + stride;
  if (cur + 1 < cend) return cur + 1;
  unsigned long long v = 0;
  if (lane == 0) v = atomicAdd(work, (unsigned long long)K);
  const int64_t b = (int64_t)__shfl_sync(gm, v, 0, G);
  cend = b + K;
  return b;
}

template <int G, int NC, int U, int MINB, bool CHK>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_fwd(const int64_t* __restrict__ rp,
                                                             const int32_t* __restrict__ col,
                                                             const float* __restrict__ inv_deg,
                                                             const float4* __restrict__ D, int64_t ld4, int64_t n_rows,
                                                             int64_t n_valid, int nchunk, float4* __restrict__ Z,
                                                             unsigned long long* work, int grabk, int self,
                                                             const float* __restrict__ bias, int64_t n_bias, int relu,
                                                             const int32_t* __restrict__ rows, int addend, int compact) {
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const int64_t n_items = n_rows * nchunk;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  // Hot-loop addressing is 32-bit: neighbour row c sits at lane_base + c * row_bytes (one
  // IMAD.WIDE per edge; the launcher guarantees ld4 * 16 < 2^32 and ids < 2^31).
  const uint32_t row_bytes = (uint32_t)ld4 * 16u;
  const uint32_t nv = (uint32_t)n_valid;
  int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
  int64_t cend = 0;
  if (work) first = next_item<G>(work, lane, gm, -1, 0, grabk, cend);
  for (int64_t it = first; it < n_items; it = next_item<G>(work, lane, gm, it, stride, grabk, cend)) {
    // item -> (chunk, row), chunk-major: with several column chunks every row's chunk 0 is gathered
    // before any chunk 1, so each phase's working set is 1/nchunk of the table (L2-resident when the
    // launcher picks nchunk for that); rows: optional row list
    const int64_t ch = nchunk > 1 ? it / n_rows : 0;
    const int64_t ri = it - ch * n_rows;
    const int64_t row = rows ? (int64_t)rows[ri] : ri;
    const int64_t x0 = ch * (NC * G) + lane;
    // Lanes past the row end gather a clamped in-row column (same sectors as their neighbours,
    // no extra traffic) and never store, so the loop carries no column predicates.
    int xq[NC];
    const char* bq[NC];  // lane column base per chunk: neighbour c's float4 is at bq + c * row_bytes
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      xq[q] = (int)(x0 + q * G < ld4 ? x0 + q * G : ld4 - 1);
      bq[q] = reinterpret_cast<const char*>(D + xq[q]);
    }
    float4 acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {  // GCN-sym self loop (A + I, R26): the row's own (inner) input
      acc[q] = self ? __ldg(D + row * ld4 + xq[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (addend) f4acc(acc[q], __ldcs(Z + row * ld4 + xq[q]));  // heavy-tile sums (spmm_tc) of this row, in place
    }
    const int64_t beg = rp[row], end = rp[row + 1];
    for (int64_t e0 = beg; e0 < end; e0 += G) {
      const int cnt = (int)((end - e0) < G ? (end - e0) : G);
      const int my = lane < cnt ? __ldg(col + e0 + lane) : 0;
      int j = 0;
      for (; j + U <= cnt; j += U) {
        float4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u, G);
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = (!CHK || c < nv) ? __ldg(nbr(bq[q], c, row_bytes))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NC; ++q) f4acc(acc[q], v[u][q]);
      }
      if (j < cnt) {  // remainder (< U edges): one predicated batch, every load in flight at once
        float4 v[U][NC];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u < cnt ? j + u : j, G);
          ok[u] = j + u < cnt && (!CHK || c < nv);
#pragma unroll
          for (int q = 0; q < NC; ++q) v[u][q] = ok[u] ? __ldg(nbr(bq[q], c, row_bytes)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u])
#pragma unroll
            for (int q = 0; q < NC; ++q) f4acc(acc[q], v[u][q]);
      }
    }
    const float s = inv_deg[row];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t x = x0 + q * G;
      if (x >= ld4) continue;
      float4 o = f4scale(acc[q], s);
      if (bias) {  // fused node-update epilogue (GCN-sym transform-first: H = act(P (D W) + b))
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v = comp(o, j) + (4 * x + j < n_bias ? bias[4 * x + j] : 0.f);
          set_comp(o, j, relu ? fmaxf(v, 0.f) : v);
        }
      }
      __stcs(Z + (compact ? ri : row) * ld4 + x, o);  // compact: output row = position in the row list
    }
  }
}

// ---------------------------------------------------------------- transposed SpMM (S8)
template <int G, int NC, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_bwd(const int64_t* __restrict__ trp,
                                                             const int32_t* __restrict__ tcol,
                                                             const float4* __restrict__ dZs,
                                                             const float4* __restrict__ dDs, int64_t ldA4, int64_t n_in,
                                                             int64_t n_all, int nchunk, float4* __restrict__ J,
                                                             int64_t ld4, const int64_t* __restrict__ gid, DropSpec d,
                                                             unsigned long long* work, int grabk, const float* __restrict__ rs,
                                                             int addend, const int32_t* __restrict__ dmap,
                                                             const __grid_constant__ PushSpec ps) {
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const int64_t n_items = n_all * nchunk;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  const uint32_t row_bytes = (uint32_t)ldA4 * 16u;  // 32-bit hot-loop addressing (see k_spmm_fwd)
  const char* base = reinterpret_cast<const char*>(dZs);
  int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
  int64_t cend = 0;
  if (work) first = next_item<G>(work, lane, gm, -1, 0, grabk, cend);
  for (int64_t it = first; it < n_items; it = next_item<G>(work, lane, gm, it, stride, grabk, cend)) {
    const int64_t ch = nchunk > 1 ? it / n_all : 0;  // chunk-major, see k_spmm_fwd
    const int64_t u0 = it - ch * n_all;
    const int64_t x0 = ch * (NC * G) + lane;
    int xq[NC];
    const char* bq[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      xq[q] = (int)(x0 + q * G < ld4 ? x0 + q * G : ld4 - 1);
      bq[q] = base + (size_t)xq[q] * 16;
    }
    float4 acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      // dmap (compact train-row dA): dD_self of u lives in row dmap[u] (-1: none)
      const int64_t du = dmap ? (u0 < n_in ? (int64_t)dmap[u0] : -1) : (u0 < n_in ? u0 : -1);
      acc[q] = (dDs && du >= 0) ? __ldcs(dDs + du * ldA4 + xq[q]) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (addend) f4acc(acc[q], __ldcs(J + u0 * ld4 + xq[q]));  // heavy-tile sums (spmm_tc) of this row, in place
    }
    const int64_t beg = trp[u0], end = trp[u0 + 1];
    for (int64_t e0 = beg; e0 < end; e0 += G) {
      const int cnt = (int)((end - e0) < G ? (end - e0) : G);
      const int my = lane < cnt ? __ldg(tcol + e0 + lane) : 0;
      int j = 0;
      for (; j + U <= cnt; j += U) {
        float4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u, G);
#pragma unroll
          for (int q = 0; q < NC; ++q) v[u][q] = __ldg(nbr(bq[q], c, row_bytes));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NC; ++q) f4acc(acc[q], v[u][q]);
      }
      if (j < cnt) {  // remainder (< U edges): one predicated batch, every load in flight at once
        float4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u < cnt ? j + u : j, G);
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = j + u < cnt ? __ldg(nbr(bq[q], c, row_bytes)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j + u < cnt)
#pragma unroll
            for (int q = 0; q < NC; ++q) f4acc(acc[q], v[u][q]);
      }
    }
    const uint64_t kr = row_key(d, gid[u0]);
    const float sr = rs ? rs[u0] : 1.f;  // GCN-sym: d~_u^-1/2 of the (inner or boundary) row u (R26)
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t x = x0 + q * G;
      if (x >= ld4) continue;
      const float4 o = drop4(rs ? f4scale(acc[q], sr) : acc[q], x, kr, 1.f, d);  // mask of R5, J's own row
      __stcs(J + u0 * ld4 + x, o);
      if (ps.mode) push_f4(ps, u0, ld4, x, o);  // N2: boundary-row gradient straight into its owner's message rows
    }
  }
}

// ---------------------------------------------------------------- bf16 gather tier (pgcn_config.gather = 1)
// The gathered table is first rounded to bf16 (k_to_bf16: rows of ld8 16-byte vectors = 8 columns,
// padding columns 0); the SpMMs then gather half the bytes and accumulate in fp32 (exact bf16 ->
// fp32 widening, FADD2 sums).  2e-2 tier (north_star), selected by pgcn_config.gather = 1.
// src: n_rows rows of stride s4 float4s, of which the first w4 are converted (the rest of the ld8
// vectors are zero padding).
__global__ void k_to_bf16(const float4* __restrict__ src, int64_t s4, int64_t w4, int64_t n_rows, int64_t ld8,
                          uint4* __restrict__ dst) {
  for (RowCursor rc(ld8); rc.r < n_rows; rc.next((int)ld8)) {
    const int64_t x0 = 2 * (int64_t)rc.x;
    const float4 a = x0 < w4 ? src[rc.r * s4 + x0] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b = x0 + 1 < w4 ? src[rc.r * s4 + x0 + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
    uint4 o;
    o.x = bf16x2_rn(a.x, a.y);
    o.y = bf16x2_rn(a.z, a.w);
    o.z = bf16x2_rn(b.x, b.y);
    o.w = bf16x2_rn(b.z, b.w);
    dst[rc.r * ld8 + rc.x] = o;
  }
}

// fp32 tier of the tensor-core tile path (spmm_tc.cu): x = hi + lo + O(2^-18 |x|) with hi = rn_bf16(x),
// lo = rn_bf16(x - hi) (x - hi is exact in fp32); same row layout as k_to_bf16, two tables.
__device__ __forceinline__ void split2(float a, float b, uint32_t& h, uint32_t& l) {
  h = bf16x2_rn(a, b);
  const float ha = __uint_as_float(h << 16), hb = __uint_as_float(h & 0xffff0000u);
  l = bf16x2_rn(a - ha, b - hb);
}
__global__ void k_split_bf16(const float4* __restrict__ src, int64_t s4, int64_t w4, int64_t n_rows, int64_t ld8,
                             uint4* __restrict__ hi, uint4* __restrict__ lo) {
  for (RowCursor rc(ld8); rc.r < n_rows; rc.next((int)ld8)) {
    const int64_t x0 = 2 * (int64_t)rc.x;
    const float4 a = x0 < w4 ? src[rc.r * s4 + x0] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 b = x0 + 1 < w4 ? src[rc.r * s4 + x0 + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
    uint4 h, l;
    split2(a.x, a.y, h.x, l.x);
    split2(a.z, a.w, h.y, l.y);
    split2(b.x, b.y, h.z, l.z);
    split2(b.z, b.w, h.w, l.w);
    hi[rc.r * ld8 + rc.x] = h;
    lo[rc.r * ld8 + rc.x] = l;
  }
}

__device__ __forceinline__ void acc8(float (&a)[8], const uint4& w) {
  bf16x2_acc(a[0], a[1], w.x);
  bf16x2_acc(a[2], a[3], w.y);
  bf16x2_acc(a[4], a[5], w.z);
  bf16x2_acc(a[6], a[7], w.w);
}
__device__ __forceinline__ void set8(float (&a)[8], const uint4& w) {
  a[0] = __uint_as_float(w.x << 16); a[1] = __uint_as_float(w.x & 0xffff0000u);
  a[2] = __uint_as_float(w.y << 16); a[3] = __uint_as_float(w.y & 0xffff0000u);
  a[4] = __uint_as_float(w.z << 16); a[5] = __uint_as_float(w.z & 0xffff0000u);
  a[6] = __uint_as_float(w.w << 16); a[7] = __uint_as_float(w.w & 0xffff0000u);
}

// S3 on a bf16 table: same work items / scheduling as k_spmm_fwd, a lane owns 8 columns (one
// 16-byte bf16 vector) per chunk q; fp32 output (stride ld4 float4s).
template <int G, int NC, int U, int MINB, bool CHK>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_fwd16(const int64_t* __restrict__ rp,
                                                               const int32_t* __restrict__ col,
                                                               const float* __restrict__ inv_deg,
                                                               const uint4* __restrict__ D, int64_t ld8,
                                                               int64_t n_rows, int64_t n_valid, int nchunk,
                                                               float4* __restrict__ Z, int64_t ld4,
                                                               unsigned long long* work, int grabk, int self,
                                                               const float* __restrict__ bias, int64_t n_bias,
                                                               int relu, const int32_t* __restrict__ rows,
                                                               int addend, int compact) {
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const int64_t n_items = n_rows * nchunk;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  const uint32_t row_bytes = (uint32_t)ld8 * 16u;
  const uint32_t nv = (uint32_t)n_valid;
  int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
  int64_t cend = 0;
  if (work) first = next_item<G>(work, lane, gm, -1, 0, grabk, cend);
  for (int64_t it = first; it < n_items; it = next_item<G>(work, lane, gm, it, stride, grabk, cend)) {
    // item -> (chunk, row), chunk-major: with several column chunks every row's chunk 0 is gathered
    // before any chunk 1, so each phase's working set is 1/nchunk of the table (L2-resident when the
    // launcher picks nchunk for that); rows: optional row list
    const int64_t ch = nchunk > 1 ? it / n_rows : 0;
    const int64_t ri = it - ch * n_rows;
    const int64_t row = rows ? (int64_t)rows[ri] : ri;
    const int64_t x0 = ch * (NC * G) + lane;
    const char* bq[NC];
    float acc[NC][8];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t xq = x0 + q * G < ld8 ? x0 + q * G : ld8 - 1;
      bq[q] = reinterpret_cast<const char*>(D + xq);
      if (self) set8(acc[q], __ldg(D + row * ld8 + xq));
      else
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[q][j] = 0.f;
      if (addend) {  // heavy-tile sums (spmm_tc) of this row, in place
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t xf = 2 * xq + h;
          if (xf < ld4) {
            const float4 a = __ldcs(Z + row * ld4 + xf);
            acc[q][4 * h] += a.x; acc[q][4 * h + 1] += a.y; acc[q][4 * h + 2] += a.z; acc[q][4 * h + 3] += a.w;
          }
        }
      }
    }
    const int64_t beg = rp[row], end = rp[row + 1];
    for (int64_t e0 = beg; e0 < end; e0 += G) {
      const int cnt = (int)((end - e0) < G ? (end - e0) : G);
      const int my = lane < cnt ? __ldg(col + e0 + lane) : 0;
      int j = 0;
      for (; j + U <= cnt; j += U) {
        uint4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u, G);
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = (!CHK || c < nv) ? __ldg(reinterpret_cast<const uint4*>(nbr(bq[q], c, row_bytes)))
                                       : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NC; ++q) acc8(acc[q], v[u][q]);
      }
      if (j < cnt) {  // remainder (< U edges): one predicated batch, every load in flight at once
        uint4 v[U][NC];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u < cnt ? j + u : j, G);
          ok[u] = j + u < cnt && (!CHK || c < nv);
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = ok[u] ? __ldg(reinterpret_cast<const uint4*>(nbr(bq[q], c, row_bytes))) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ok[u])
#pragma unroll
            for (int q = 0; q < NC; ++q) acc8(acc[q], v[u][q]);
      }
    }
    const float s = inv_deg[row];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t x = x0 + q * G;
      if (x >= ld8) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t xf = 2 * x + h;
        if (xf >= ld4) continue;
        float o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v = acc[q][4 * h + j] * s;
          if (bias) {
            v += 4 * xf + j < n_bias ? bias[4 * xf + j] : 0.f;
            if (relu) v = fmaxf(v, 0.f);
          }
          o[j] = v;
        }
        __stcs(Z + (compact ? ri : row) * ld4 + xf, make_float4(o[0], o[1], o[2], o[3]));
      }
    }
  }
}

// S8 on a bf16 copy of dZs (ld8 vectors per row, n_in rows); dDs stays fp32 (stride ldA4).
template <int G, int NC, int U, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_spmm_bwd16(const int64_t* __restrict__ trp,
                                                               const int32_t* __restrict__ tcol,
                                                               const uint4* __restrict__ dZs, int64_t ld8,
                                                               const float4* __restrict__ dDs, int64_t ldA4,
                                                               int64_t n_in, int64_t n_all, int nchunk,
                                                               float4* __restrict__ J, int64_t ld4,
                                                               const int64_t* __restrict__ gid, DropSpec d,
                                                               unsigned long long* work, int grabk, const float* __restrict__ rs,
                                                               int addend, const int32_t* __restrict__ dmap,
                                                               const __grid_constant__ PushSpec ps) {
  const int lane = threadIdx.x % G;
  const unsigned gm = group_mask<G>();
  const int64_t n_items = n_all * nchunk;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  const uint32_t row_bytes = (uint32_t)ld8 * 16u;
  int64_t first = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G;
  int64_t cend = 0;
  if (work) first = next_item<G>(work, lane, gm, -1, 0, grabk, cend);
  for (int64_t it = first; it < n_items; it = next_item<G>(work, lane, gm, it, stride, grabk, cend)) {
    const int64_t ch = nchunk > 1 ? it / n_all : 0;  // chunk-major, see k_spmm_fwd
    const int64_t u0 = it - ch * n_all;
    const int64_t x0 = ch * (NC * G) + lane;
    const char* bq[NC];
    float acc[NC][8];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t xq = x0 + q * G < ld8 ? x0 + q * G : ld8 - 1;
      bq[q] = reinterpret_cast<const char*>(dZs + xq);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t xf = 2 * xq + h;
        const int64_t du = dmap ? (u0 < n_in ? (int64_t)dmap[u0] : -1) : (u0 < n_in ? u0 : -1);
        float4 a = (dDs && du >= 0 && xf < ld4) ? __ldcs(dDs + du * ldA4 + xf) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (addend && xf < ld4) f4acc(a, __ldcs(J + u0 * ld4 + xf));  // heavy-tile sums (spmm_tc) of this row, in place
        acc[q][4 * h] = a.x; acc[q][4 * h + 1] = a.y; acc[q][4 * h + 2] = a.z; acc[q][4 * h + 3] = a.w;
      }
    }
    const int64_t beg = trp[u0], end = trp[u0 + 1];
    for (int64_t e0 = beg; e0 < end; e0 += G) {
      const int cnt = (int)((end - e0) < G ? (end - e0) : G);
      const int my = lane < cnt ? __ldg(tcol + e0 + lane) : 0;
      int j = 0;
      for (; j + U <= cnt; j += U) {
        uint4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u, G);
#pragma unroll
          for (int q = 0; q < NC; ++q) v[u][q] = __ldg(reinterpret_cast<const uint4*>(nbr(bq[q], c, row_bytes)));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NC; ++q) acc8(acc[q], v[u][q]);
      }
      if (j < cnt) {  // remainder (< U edges): one predicated batch, every load in flight at once
        uint4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t c = (uint32_t)__shfl_sync(gm, my, j + u < cnt ? j + u : j, G);
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = j + u < cnt ? __ldg(reinterpret_cast<const uint4*>(nbr(bq[q], c, row_bytes))) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (j + u < cnt)
#pragma unroll
            for (int q = 0; q < NC; ++q) acc8(acc[q], v[u][q]);
      }
    }
    const uint64_t kr = row_key(d, gid[u0]);
    const float sr = rs ? rs[u0] : 1.f;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      const int64_t x = x0 + q * G;
      if (x >= ld8) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t xf = 2 * x + h;
        if (xf >= ld4) continue;
        float4 o = make_float4(acc[q][4 * h], acc[q][4 * h + 1], acc[q][4 * h + 2], acc[q][4 * h + 3]);
        if (rs) o = f4scale(o, sr);
        o = drop4(o, xf, kr, 1.f, d);
        __stcs(J + u0 * ld4 + xf, o);
        if (ps.mode) push_f4(ps, u0, ld4, xf, o);
      }
    }
  }
}

// ---------------------------------------------------------------- compact train rows (N1(ii))
// dst[map[r]] = src[r] over n rows of ld4 float4s
__global__ void k_scatter_rows(const float4* __restrict__ src, const int32_t* __restrict__ map, int64_t n, int64_t ld4,
                               float4* __restrict__ dst) {
  for (RowCursor rc(ld4); rc.r < n; rc.next((int)ld4)) dst[(int64_t)map[rc.r] * ld4 + rc.x] = src[rc.r * ld4 + rc.x];
}
// pos[v] = k where list[k] = v, else -1 (pos pre-filled with -1)
__global__ void k_positions(const int32_t* __restrict__ list, int64_t n, int32_t* __restrict__ pos) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    pos[list[k]] = (int32_t)k;
}
// a[e] = pos[a[e]] (in place)
__global__ void k_remap(int32_t* __restrict__ a, int64_t n, const int32_t* __restrict__ pos) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    a[e] = pos[a[e]];
}
// dst[k * w + j] = src[list[k] * w + j] (bytes)
__global__ void k_gather_bytes(const uint8_t* __restrict__ src, const int32_t* __restrict__ list, int64_t n, int64_t w,
                               uint8_t* __restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * w; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = i / w, j = i - k * w;
    dst[i] = src[(int64_t)list[k] * w + j];
  }
}

// ---------------------------------------------------------------- gather rows / EMA install (S1, S2)
__global__ void k_gather(const __grid_constant__ SegTable t, const int32_t* __restrict__ row_map, int64_t n_rows,
                         int64_t ld4, float4* __restrict__ dst, const float4* __restrict__ prev, float gamma, int ema,
                         int first) {
  for (RowCursor rc(ld4); rc.r < n_rows; rc.next((int)ld4)) {
    const int64_t r = rc.r, x = rc.x, i = r * ld4 + x;
    const int s = find_seg(t, r);
    const int64_t srow = row_map ? (int64_t)row_map[r] : r - t.off[s];
    float4 v = __ldg(reinterpret_cast<const float4*>(t.base[s]) + srow * ld4 + x);
    if (ema && !first) {
      const float4 p = prev[i];
      const float a = gamma, b = 1.0f - gamma;
      v = make_float4(a * p.x + b * v.x, a * p.y + b * v.y, a * p.z + b * v.z, a * p.w + b * v.w);
    }
    dst[i] = v;
  }
}

// bf16 exchange payloads (pgcn_config.halo_payload = 1): a float4 of a row travels as
// one uint2 (4 bf16, round to nearest even) and is widened exactly on receipt.
__device__ __forceinline__ uint2 f4_to_bf16x4(const float4 v) {
  return make_uint2(bf16x2_rn(v.x, v.y), bf16x2_rn(v.z, v.w));
}
__device__ __forceinline__ float4 bf16x4_to_f4(const uint2 w) {
  return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u), __uint_as_float(w.y << 16),
                     __uint_as_float(w.y & 0xffff0000u));
}
// S2 pack in bf16: dst[r] = bf16(src(r)), src row = row_map[r] (or r) of one fp32 table
__global__ void k_pack_bf16(const float4* __restrict__ src, const int32_t* __restrict__ row_map, int64_t n_rows,
                            int64_t ld4, uint2* __restrict__ dst) {
  for (RowCursor rc(ld4); rc.r < n_rows; rc.next((int)ld4)) {
    const int64_t srow = row_map ? (int64_t)row_map[rc.r] : rc.r;
    dst[rc.r * ld4 + rc.x] = f4_to_bf16x4(__ldg(src + srow * ld4 + rc.x));
  }
}
// S1 install of bf16 payloads: dst[r] = widen(src[r]) or EMA: gamma * prev[r] + (1 - gamma) * widen(src[r])
__global__ void k_install_bf16(const uint2* __restrict__ src, int64_t n_rows, int64_t ld4, float4* __restrict__ dst,
                               const float4* __restrict__ prev, float gamma, int ema) {
  for (RowCursor rc(ld4); rc.r < n_rows; rc.next((int)ld4)) {
    const int64_t i = rc.r * ld4 + rc.x;
    float4 v = bf16x4_to_f4(__ldg(src + i));
    if (ema) {
      const float4 p = prev[i];
      const float a = gamma, b = 1.0f - gamma;
      v = make_float4(a * p.x + b * v.x, a * p.y + b * v.y, a * p.z + b * v.z, a * p.w + b * v.w);
    }
    dst[i] = v;
  }
}
// Delay injection on the comm stream (tests of the stream/event contract): one thread spins on the
// global nanosecond timer.
__global__ void k_spin(int64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while ((int64_t)(t - t0) < ns);
}

// lo = x - trunc_tf32(x) (exact): the 3xTF32 GEMMs' second operand term (tc_ptx.cuh tf32_lo_trunc, the
// converter warps' split -- kind::tf32 reads the raw word's top 19 bits as hi), written by the producers
// of M so the GEMMs that read M load it instead of recomputing it per tile (gemm_tc.cu pre_a / pre_b).
__device__ __forceinline__ float lo_tf32(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ float4 lo_tf32(float4 v) {
  return make_float4(lo_tf32(v.x), lo_tf32(v.y), lo_tf32(v.z), lo_tf32(v.w));
}

// ---------------------------------------------------------------- stale gradient accumulate + M (S9)
__global__ void k_grad_reduce(const int64_t* __restrict__ inv_ptr, const int32_t* __restrict__ inv_pos,
                              const __grid_constant__ SegTable msg, const int32_t* __restrict__ row_map,
                              float4* __restrict__ ema, float gamma, int use_ema, int first, float4* __restrict__ J,
                              int write_j, const float4* __restrict__ Hprev, float4* __restrict__ M, int64_t n_in,
                              int64_t ld4, int msg16, float4* __restrict__ Mlo) {
  const int64_t total = n_in * ld4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / ld4, x = i - v * ld4;
    float4 acc = J[i];
    if (msg.n_seg > 0) {
      const int64_t kb = inv_ptr[v], ke = inv_ptr[v + 1];
      for (int64_t q = kb; q < ke; ++q) {
        const int64_t k = inv_pos[q];
        const int s = find_seg(msg, k);
        const int64_t srow = row_map ? (int64_t)row_map[k] : k - msg.off[s];
        float4 c = msg16 ? bf16x4_to_f4(__ldg(reinterpret_cast<const uint2*>(msg.base[s]) + srow * ld4 + x))
                         : __ldg(reinterpret_cast<const float4*>(msg.base[s]) + srow * ld4 + x);
        if (use_ema) {
          if (!first) {
            const float4 e = ema[k * ld4 + x];
            const float a = gamma, b = 1.0f - gamma;
            c = make_float4(a * e.x + b * c.x, a * e.y + b * c.y, a * e.z + b * c.z, a * e.w + b * c.w);
          }
          ema[k * ld4 + x] = c;
        }
        acc = f4add(acc, c);
      }
    }
    if (write_j) J[i] = acc;
    const float4 h = Hprev[v * ld4 + x];
    const float4 m = make_float4(h.x > 0.f ? acc.x : 0.f, h.y > 0.f ? acc.y : 0.f, h.z > 0.f ? acc.z : 0.f,
                                 h.w > 0.f ? acc.w : 0.f);
    M[i] = m;
    if (Mlo) Mlo[i] = lo_tf32(m);
  }
}

// ---------------------------------------------------------------- loss (S5)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Y and M may alias (compact train rows: the logits become J^(L) in place, each row read before written)
__global__ void k_loss_ce(const float* Y, int64_t n, int64_t C, int64_t ld, const int32_t* __restrict__ lab,
                          const uint8_t* __restrict__ train, float inv_nt, float* M, float* __restrict__ rl,
                          float* __restrict__ Mlo, const int32_t* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t wpg = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; k < n; k += wpg) {
    const int64_t v = rows ? (int64_t)rows[k] : k;  // rows: the train row list (row loss at position k)
    const float* y = Y + v * ld;
    float* m = M + v * ld;
    if (!rows && train && !train[v]) {  // J^(L) = 0 off the train set: 16-byte stores (ld is a multiple of 4)
      for (int64_t c = lane; c < ld / 4; c += 32) {
        reinterpret_cast<float4*>(m)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (Mlo) reinterpret_cast<float4*>(Mlo + v * ld)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) rl[v] = 0.f;
      continue;
    }
    float mx = -INFINITY;
    for (int64_t c = lane; c < C; c += 32) mx = fmaxf(mx, y[c]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int64_t c = lane; c < C; c += 32) s += expf(y[c] - mx);
    s = warp_sum(s);
    const int32_t t = lab[v];
    const float ls = logf(s);
    const float yt = y[t];
    __syncwarp();
    for (int64_t c = lane; c < ld; c += 32) {
      float g = 0.f;
      if (c < C) g = (expf(y[c] - mx) / s - (c == t ? 1.f : 0.f)) * inv_nt;
      m[c] = g;
      if (Mlo) Mlo[v * ld + c] = lo_tf32(g);
    }
    if (lane == 0) rl[k] = (ls + mx - yt) * inv_nt;
  }
}

__global__ void k_loss_bce(const float* Y, int64_t n, int64_t C, int64_t ld, const uint8_t* __restrict__ lab,
                           const uint8_t* __restrict__ train, float inv_ntc, float* M, float* __restrict__ rl,
                           float* __restrict__ Mlo, const int32_t* __restrict__ rows) {
  const int lane = threadIdx.x & 31;
  const int64_t wpg = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; k < n; k += wpg) {
    const int64_t v = rows ? (int64_t)rows[k] : k;  // rows: the train row list (row loss at position k)
    const float* y = Y + v * ld;
    float* m = M + v * ld;
    const bool tr = rows || !train || train[v] != 0;
    if (!tr) {
      for (int64_t c = lane; c < ld / 4; c += 32) {
        reinterpret_cast<float4*>(m)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (Mlo) reinterpret_cast<float4*>(Mlo + v * ld)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (lane == 0) rl[v] = 0.f;
      continue;
    }
    float l = 0.f;
    for (int64_t c = lane; c < ld; c += 32) {
      float g = 0.f;
      if (tr && c < C) {
        const float yc = y[c], lb = (float)lab[v * C + c];
        g = (1.f / (1.f + expf(-yc)) - lb) * inv_ntc;
        l += fmaxf(yc, 0.f) + log1pf(expf(-fabsf(yc))) - lb * yc;
      }
      m[c] = g;
      if (Mlo) Mlo[v * ld + c] = lo_tf32(g);
    }
    l = warp_sum(l);
    if (lane == 0) rl[k] = l * inv_ntc;
  }
}

__global__ void k_reduce_sum(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
  // one block, fixed assignment (deterministic); 16-byte loads with 4 independent accumulators per
  // thread when x is 16-byte aligned, so a single SM streams the 13.9M row losses of a
  // papers-shaped partition at its full load bandwidth
  __shared__ double sh[1024];
  double a = 0.0;
  int64_t head = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int64_t n4 = n / 4;
    double b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
    for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
      const float4 v = x4[i];
      b0 += (double)v.x; b1 += (double)v.y; b2 += (double)v.z; b3 += (double)v.w;
    }
    a = (b0 + b1) + (b2 + b3);
    head = n4 * 4;
  }
  for (int64_t i = head + threadIdx.x; i < n; i += blockDim.x) a += (double)x[i];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = (float)sh[0];
}

// ---------------------------------------------------------------- SIMT fp32 GEMMs (parity path)
constexpr int BM = 64, BN = 64, BK = 16;

// A_ext(m, k) = [Z | D | 1](m, k), K = 2F + 1
__device__ __forceinline__ float a_ext(const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, int64_t m,
                                       int64_t k) {
  if (m >= M) return 0.f;
  if (k < F) return __ldg(Z + m * ldA + k);
  if (k < 2 * F) return __ldg(D + m * ldA + (k - F));
  return k == 2 * F ? 1.f : 0.f;
}

template <int RELU>
__global__ void __launch_bounds__(256) k_gemm_fwd(const float* __restrict__ Z, const float* __restrict__ D, int64_t ldA,
                                                  int64_t M, int64_t F, const float* __restrict__ W, int64_t N,
                                                  float* __restrict__ Y, int64_t ldY) {
  __shared__ float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t K = 2 * F + 1;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty + 16 * i;
      As[tx][r] = a_ext(Z, D, ldA, M, F, m0 + r, k0 + tx);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = ty, nn = tx + 16 * i;
      const int64_t k = k0 + kk, n = n0 + nn;
      Bs[kk][nn] = (k < K && n < N) ? __ldg(W + k * N + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n < N) Y[m * ldY + n] = RELU ? fmaxf(acc[i][j], 0.f) : acc[i][j];
      else if (n < ldY) Y[m * ldY + n] = 0.f;
    }
  }
}

// partial[s][k][n] = sum_{m in chunk s} A_ext(m, k) Mg(m, n)
__global__ void __launch_bounds__(256) k_gemm_dw(const float* __restrict__ Z, const float* __restrict__ D, int64_t ldA,
                                                 int64_t M, int64_t F, const float* __restrict__ Mg, int64_t ldM, int64_t N,
                                                 int64_t rows_per_split, float* __restrict__ part) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t k0 = (int64_t)blockIdx.x * BM, n0 = (int64_t)blockIdx.y * BN;
  const int64_t K = 2 * F + 1;
  const int64_t r_beg = (int64_t)blockIdx.z * rows_per_split;
  const int64_t r_end = r_beg + rows_per_split < M ? r_beg + rows_per_split : M;
  float acc[4][4] = {};
  for (int64_t r0 = r_beg; r0 < r_end; r0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // As[r][k]: 16 rows x 64 k
      const int kk = tx + 16 * i, rr = ty;
      const int64_t r = r0 + rr;
      As[rr][kk] = (r < r_end && k0 + kk < K) ? a_ext(Z, D, ldA, M, F, r, k0 + kk) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int nn = tx + 16 * i, rr = ty;
      const int64_t r = r0 + rr, n = n0 + nn;
      Bs[rr][nn] = (r < r_end && n < N) ? __ldg(Mg + r * ldM + n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int rr = 0; rr < BK; ++rr) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[rr][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[rr][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* out = part + (int64_t)blockIdx.z * K * N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t k = k0 + ty * 4 + i;
    if (k >= K) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t n = n0 + tx * 4 + j;
      if (n < N) out[k * N + n] = acc[i][j];
    }
  }
}

// G[r * N + c] = sum_s part[s][r * NP + c]  (ascending s)
__global__ void k_split_reduce_strided(const float* __restrict__ part, int64_t splits, int64_t rows, int64_t N,
                                       int64_t NP, float* __restrict__ G) {
  const int64_t len = rows * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i - r * N;
    float a = 0.f;
    for (int64_t s = 0; s < splits; ++s) a += part[s * rows * NP + r * NP + c];
    G[i] = a;
  }
}

// dW partial reduce with per-row-range split counts: rows [0, F) sum zc[0] splits, [F, 2F) zc[1]
// (nseg == 2), the bias row zc[2]; partial z holds (nseg F + 1) rows of stride NP.
__global__ void k_split_reduce_dw(const float* __restrict__ part, int64_t z0, int64_t z1, int64_t zb, int64_t F,
                                  int64_t rows, int64_t N, int64_t NP, float* __restrict__ G) {
  const int64_t len = rows * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i - r * N;
    const int64_t splits = r == rows - 1 ? zb : (r < F ? z0 : z1);
    float a = 0.f;
    for (int64_t s = 0; s < splits; ++s) a += part[s * rows * NP + r * NP + c];
    G[i] = a;
  }
}

__global__ void k_split_reduce(const float* __restrict__ part, int64_t splits, int64_t len, float* __restrict__ G) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int64_t s = 0; s < splits; ++s) a += part[s * len + i];
    G[i] = a;
  }
}

// dA(m, oc), oc in [0, 2 ld): half h = oc / ld, c = oc % ld; value = sum_j Mg(m, j) W(hF + c, j)
__global__ void __launch_bounds__(256) k_gemm_da(const float* __restrict__ Mg, int64_t ldM, int64_t M, int64_t N,
                                                 const float* __restrict__ W, int64_t F, const float* __restrict__ inv_deg,
                                                 float* __restrict__ dA, int64_t ld) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.x * BM, o0 = (int64_t)blockIdx.y * BN;
  float acc[4][4] = {};
  for (int64_t j0 = 0; j0 < N; j0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = ty + 16 * i;
      const int64_t m = m0 + r, j = j0 + tx;
      As[tx][r] = (m < M && j < N) ? __ldg(Mg + m * ldM + j) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int oo = ty + 16 * i;   // output column within tile
      const int64_t oc = o0 + oo, j = j0 + tx;
      float w = 0.f;
      if (oc < 2 * ld && j < N) {
        const int64_t h = oc / ld, c = oc - h * ld;
        if (c < F) w = __ldg(W + (h * F + c) * N + j);
      }
      Bs[tx][oo] = w;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + ty * 4 + i;
    if (m >= M) continue;
    const float s = inv_deg[m];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t oc = o0 + tx * 4 + j;
      if (oc >= 2 * ld) continue;
      const int64_t h = oc / ld, c = oc - h * ld;
      float v = c < F ? acc[i][j] : 0.f;
      if (h == 0) v *= s;
      dA[m * 2 * ld + oc] = v;
    }
  }
}

// out[v] = s[v] * M[v] (row scaling, e.g. inv_deg o M before the transposed aggregation)
__global__ void k_scale_rows(const float4* __restrict__ M, const float* __restrict__ sc, int64_t n, int64_t ld4,
                             float4* __restrict__ out) {
  for (RowCursor rc(ld4); rc.r < n; rc.next((int)ld4)) {
    const int64_t i = rc.r * ld4 + rc.x;
    out[i] = f4scale(M[i], sc[rc.r]);
  }
}

// ---------------------------------------------------------------- staleness diagnostics (N4)
// out += sum over rows r, cols c < F of (used(r) - fresh(r))^2, where used(r) is used + r*ld (or 0 if
// used is null, or the second table `ustab` row) and fresh(r) comes from the segment table `ftab`.
__global__ void k_stale_err(const __grid_constant__ SegTable ftab, const int32_t* __restrict__ fmap,
                            const __grid_constant__ SegTable utab, const int32_t* __restrict__ umap,
                            const float* __restrict__ used, int use_tab, int64_t n_rows, int64_t ld, int64_t F,
                            double* out) {
  double a = 0.0;
  const int64_t total = n_rows * F;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, c = i - r * F;
    const int s = find_seg(ftab, r);
    const int64_t fr = fmap ? (int64_t)fmap[r] : r - ftab.off[s];
    const float f = ftab.base[s][fr * ld + c];
    float u = 0.f;
    if (use_tab) {
      const int su = find_seg(utab, r);
      const int64_t ur = umap ? (int64_t)umap[r] : r - utab.off[su];
      u = utab.base[su][ur * ld + c];
    } else if (used) {
      u = used[r * ld + c];
    }
    const double d = (double)u - (double)f;
    a += d * d;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = a;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(out, sh[0]);
}

// ---------------------------------------------------------------- optimiser (S11, S12)
__global__ void k_sum_grads(const __grid_constant__ PtrList G, int64_t P, float* __restrict__ grads) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    float a = G.p[0][i];
    for (int k = 1; k < G.n; ++k) a += G.p[k][i];
    grads[i] = a;
  }
}

__global__ void k_opt(const float* __restrict__ grads, int64_t P, float* __restrict__ w, float* __restrict__ m,
                      float* __restrict__ v, OptSpec o) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const float g = grads[i];
    if (!o.adam) {
      w[i] = w[i] - o.lr * g;
    } else {
      const float mi = o.beta1 * m[i] + (1.f - o.beta1) * g;
      const float vi = o.beta2 * v[i] + (1.f - o.beta2) * g * g;
      m[i] = mi;
      v[i] = vi;
      w[i] = w[i] - o.step_size * mi / (sqrtf(vi) * o.inv_sqrt_bc2 + o.eps);
    }
  }
}

// ---------------------------------------------------------------- SpMM dispatch
// (G, NC, U, min blocks/SM) per row width, measured in the full Reddit-shaped step on B200
// (tools/ab_r1/spmm_sweep.sh; tools/ab_r1/spmm_lab.py for the isolated kernel): rows of <= 32 float4 use one
// lane per float4 (G = next pow2, NC = 1, U = 8); wider rows use 32 lanes and NC = ceil(ld4/32)
// float4 per lane, U ~ 8/NC rows in flight (whole row per warp); register caps chosen for 3-4
// resident blocks (NC = 5: 3 blocks beat 2 by 15%; NC = 2: 4 blocks).
struct SpmmShape {
  int G, NC, U, MB, nchunk;
};
#define PGCN_SPMM_CASES(X)                                                                                     \
  X(32, 3, 2, 3) X(32, 8, 1, 2) X(32, 12, 1, 1) X(32, 16, 1, 1) X(32, 1, 8, 3) X(32, 2, 4, 3)             \
  X(32, 1, 8, 4) X(16, 1, 8, 4) X(8, 1, 8, 4) X(4, 1, 8, 4) X(32, 2, 4, 4) X(32, 5, 1, 3) X(32, 6, 1, 3) \
  X(32, 4, 2, 3) X(32, 2, 8, 2) X(16, 1, 8, 3) X(4, 3, 4, 3) X(4, 3, 8, 2) X(4, 3, 2, 4) X(8, 2, 4, 3)          \
  X(8, 2, 8, 2)

static bool dyn_enabled() { return knobs().spmm_dyn != 0; }

bool spmm_instantiated(int G, int NC, int U, int MB) {
#define X(G_, NC_, U_, MB_) \
  if (G == G_ && NC == NC_ && U == U_ && MB == MB_) return true;
  PGCN_SPMM_CASES(X)
#undef X
  return false;
}

// Dev knob (not part of the ABI): PGCN_SPMM_TABLE="ld4=G,NC,U,MB;..." overrides the table for the
// listed widths (used by the in-situ sweep in tools/); combinations that are not instantiated are
// ignored (the default shape is used), so a kernel is never skipped.
bool spmm_override(int64_t ld4, SpmmShape& s) {
  const char* e = knobs().spmm_table;
  if (!e) return false;
  const char* p = e;
  while (*p) {
    long long w;
    int g, nc, u, mb, n = 0;
    if (std::sscanf(p, "%lld=%d,%d,%d,%d%n", &w, &g, &nc, &u, &mb, &n) == 5) {
      if (w == ld4 && (ld4 >= 1000000 || spmm_instantiated(g, nc, u, mb))) {
        const int64_t w4 = ld4 >= 1000000 ? ld4 - 1000000 : ld4;
        s = SpmmShape{g, nc, u, mb, (int)((w4 + (int64_t)g * nc - 1) / ((int64_t)g * nc))};
        return true;
      }
      p += n;
    } else {
      break;
    }
    while (*p == ';' || *p == ' ') ++p;
  }
  return false;
}

SpmmShape spmm_shape(int64_t ld4) {
  SpmmShape s{32, 1, 8, 4, 1};
  if (spmm_override(ld4, s)) return s;
  if (ld4 <= 32) {
    int g = 4;
    while (g < ld4) g *= 2;
    s.G = g;
    return s;
  }
  int64_t nc = (ld4 + 31) / 32;
  static const int NCs[] = {2, 3, 4, 5, 6, 8, 12, 16};
  int pick = 16;
  for (int c : NCs)
    if (c >= nc) { pick = c; break; }
  s.NC = pick;
  // 256-wide rows (pick 2): 8 neighbours in flight x 2 float4 per lane, 2 blocks/SM (in-situ sweep
  // after the 32-bit-addressing rewrite, tools/ab_r1/spmm_sweep5.sh: Reddit step 49.0 -> 46.5 ms).
  s.U = pick == 2 ? 8 : (pick <= 4 ? 2 : 1);
  s.MB = pick == 2 ? 2 : (pick <= 6 ? 3 : (pick <= 8 ? 2 : 1));
  s.nchunk = (int)((ld4 + 32 * pick - 1) / (32 * pick));
  return s;
}

// Transposed SpMM, rows of 9-12 float4 (papers-shaped 48 wide): 8 lanes x 2 float4 per lane beat the
// 16-lane x 1 float4 forward shape (papers-q step: spmm_bwd 41.1 -> 37.3 ms; the forward is faster with
// the default shape, 27.1 vs 28.4 ms).
SpmmShape spmm_bwd_shape(int64_t ld4) {
  SpmmShape s{8, 2, 4, 3, 1};
  if (ld4 > 8 && ld4 <= 12 && !spmm_override(ld4, s)) return s;
  return spmm_shape(ld4);
}

// bf16 tier: a lane owns one 16-byte vector (8 columns) per chunk; rows of ld8 vectors.
#define PGCN_SPMM16_CASES(X) \
  X(32, 1, 16, 2) X(32, 1, 8, 4) X(16, 1, 8, 4) X(8, 1, 8, 4) X(4, 1, 8, 4) X(32, 2, 4, 3) X(32, 3, 2, 3) X(32, 6, 1, 2) \
  X(8, 1, 16, 2) X(32, 1, 12, 3) X(16, 1, 16, 2)

SpmmShape spmm16_shape(int64_t ld8) {
  SpmmShape s{32, 1, 8, 4, 1};
  if (spmm_override(1000000 + ld8, s)) return s;  // PGCN_SPMM_TABLE key 1000000 + ld8 (dev sweeps)
  if (ld8 <= 16) {
    int g = 4;
    while (g < ld8) g *= 2;
    s.G = g;
  } else if (ld8 <= 32) {
    // (32, 1, 8, 4): measured best for 256-wide rows (tools/spmm16_sweep.sh)
  } else if (ld8 <= 64) {
    s.NC = 2; s.U = 4; s.MB = 3;
  } else if (ld8 <= 96) {
    s.NC = 3; s.U = 2; s.MB = 3;
  } else {
    s.NC = 6; s.U = 1; s.MB = 2;
  }
  s.nchunk = (int)((ld8 + (int64_t)s.G * s.NC - 1) / ((int64_t)s.G * s.NC));
  return s;
}

// Column chunks for L2 residency: a gathered table larger than the
// L2 budget (dev knob PGCN_SPMM_L2MB, MB; 0 = off) is processed in nchunk column chunks, chunk-major, so
// the rows being gathered at any time span table_bytes / nchunk.  The shape is the one for the chunk
// width; the row's other chunks are separate items.
// Only two halves, and only for tables up to 3x the budget: measured on B200 (PGCN_SPMM_L2MB sweep,
// profiles/r2_spmm_chunks.md) the Reddit-shaped step gains 3 % at 96 MB (its 238 MB forward and 119 MB
// transposed tables), while splitting GB-sized tables (products) into many narrow chunks loses 70 %.
SpmmShape chunked(SpmmShape (*shape)(int64_t), int64_t w, double table_bytes) {
  const double budget = (double)knobs().spmm_l2mb * 1048576.0;
  if (budget <= 0.0 || table_bytes <= budget || table_bytes > 3.0 * budget) return shape(w);
  const int64_t nch = knobs().spmm_nch;  // (dev knob PGCN_SPMM_NCH, default 2)
  int64_t cw = (w + nch - 1) / nch;
  cw = (cw + 3) / 4 * 4;  // chunk width in vectors: a multiple of 4 (whole 64-byte fp32 / bf16 segments)
  if (cw >= w) return shape(w);
  SpmmShape sh = shape(cw);
  sh.nchunk = (int)((w + (int64_t)sh.G * sh.NC - 1) / ((int64_t)sh.G * sh.NC));
  return sh;
}


}  // namespace

// Items per atomic grab of the dynamic SpMM scheduler: ~128 edges per grab, 1..64 rows (sweep
// tools/grab_sweep.sh: 64-256 best on Reddit / products / papers-q; 512+ loses L2 locality).
static int grab_items(int64_t nnz, int64_t rows) {
  const int64_t target = knobs().spmm_grab;  // dev knob PGCN_SPMM_GRAB: edges per grab (sweeps)
  if (nnz < 0 || rows <= 0) return 1;
  const int64_t k = (target * rows) / (nnz > 0 ? nnz : 1);
  return (int)(k < 1 ? 1 : (k > 64 ? 64 : k));
}

static void count(const Launch& L, int64_t n = 1) {
  if (L.count) *L.count += n;
}

void dropout_fwd(Launch L, const float* H, float* D, int64_t ld, int64_t n_rows, int64_t n_valid,
                 const int64_t* gid, const DropSpec& d, const float* rs) {
  const int64_t ld4 = ld / 4;
  if (n_rows <= 0) return;
  k_dropout<<<grid_for(n_rows * ld4, kThreads), kThreads, 0, L.s>>>(
      reinterpret_cast<const float4*>(H), reinterpret_cast<float4*>(D), ld4, n_rows, n_valid, gid, d, rs);
  count(L);
}

// Sub-interval timing of the tile part (Launch::mark): executed MMA flops (0/1 tile x 64 table rows per
// heavy tile, every table, columns rounded to whole 64-column atoms) and TMA bytes (64 rows per tile and
// table + the 1 KB bitmask).
struct TileMark {
  const Launch& L;
  int kind;
  TileMark(const Launch& l, int k, const TileDev& T, int64_t width, bool b16) : L(l), kind(k) {
    if (!L.mark) return;
    const double nt = b16 ? 1.0 : 2.0, cols = (double)((width + 63) / 64 * 64), tiles = (double)T.n_tiles;
    L.mark(L.mctx, kind, 1, 2.0 * 128.0 * 64.0 * cols * nt * tiles, tiles * (64.0 * cols * 2.0 * nt + 1024.0));
  }
  ~TileMark() {
    if (L.mark) L.mark(L.mctx, kind, 0, 0.0, 0.0);
  }
};

// Tile path (tiles != nullptr, every neighbour row valid): the heavy tiles go to the tensor cores
// (spmm_tc, writing the tile sums into the output rows) and the gather kernel then walks the light
// edges on top of them (addend) and applies the epilogue.  (Running the light gather concurrently
// on a side stream, one block per SM next to the tile kernel's CTA, measured 15-25 % slower: both
// passes contend for the same L2 / DRAM path.)

int spmm_fwd(Launch L, const int64_t* row_ptr, const int32_t* col, const float* inv_deg, const float* D, int64_t ld,
              int64_t n_rows, int64_t n_valid, float* Z, unsigned long long* work, int self, const float* bias,
              int64_t n_bias, int relu, int64_t n_cols, void* g16, const int32_t* rows, int64_t nnz,
              const TileDev* tiles, void* t16, int compact) {
  if (n_rows <= 0) return 0;
  const int tcu = tiles && tiles->n_tiles > 0 && !rows && n_cols >= 0 && n_valid >= n_cols && tiles->n_rows == n_rows;
  if (tcu) {
    row_ptr = tiles->lrp;
    col = tiles->lcol;
    nnz = tiles->nnz_light;
  }
  const int64_t ld4 = ld / 4, ld8 = (ld + 7) / 8;
  const bool b16 = g16 != nullptr;
  if ((b16 ? ld8 * 16 : ld4 * 16) >= (int64_t(1) << 32) || n_valid >= (int64_t(1) << 31)) {
    return fail(PGCN_EUNSUPPORTED, "spmm_fwd: row stride / id range exceeds 32-bit addressing");
  }
  const int K = grab_items(nnz, n_rows);
  if (!dyn_enabled()) work = nullptr;
  const bool chk = !tcu && (n_cols < 0 || n_valid < n_cols);  // some neighbour rows are not valid yet
  auto Z4 = reinterpret_cast<float4*>(Z);
  auto D4 = reinterpret_cast<const float4*>(D);
  auto G16 = static_cast<uint4*>(g16);
  if (b16) {  // bf16 gather tier: round the table's valid rows to bf16, then gather those
    k_to_bf16<<<grid_for(n_valid * ld8, kThreads), kThreads, 0, L.s>>>(D4, ld4, ld4, n_valid, ld8, G16);
    count(L);
  }
  auto gather = [&](cudaStream_t st, unsigned long long* wk, int slf, int add) -> int {
    if (wk) cudaMemsetAsync(wk, 0, sizeof(unsigned long long), st);
    if (b16) {
      const SpmmShape sh = chunked(spmm16_shape, ld8, (double)n_valid * ld8 * 16);
      const int grid = grid_for(n_rows * sh.nchunk, kThreads / sh.G, sm_count() * 64);
#define X(G_, NC_, U_, MB_)                                                                                     \
  if (sh.G == G_ && sh.NC == NC_ && sh.U == U_ && sh.MB == MB_) {                                              \
    if (chk)                                                                                                   \
      k_spmm_fwd16<G_, NC_, U_, MB_, true><<<grid, kThreads, 0, st>>>(row_ptr, col, inv_deg, G16, ld8, n_rows,   \
                                                                      n_valid, sh.nchunk, Z4, ld4, wk, K, slf,    \
                                                                      bias, n_bias, relu, rows, add, compact);    \
    else                                                                                                       \
      k_spmm_fwd16<G_, NC_, U_, MB_, false><<<grid, kThreads, 0, st>>>(row_ptr, col, inv_deg, G16, ld8, n_rows,  \
                                                                       n_valid, sh.nchunk, Z4, ld4, wk, K, slf,   \
                                                                       bias, n_bias, relu, rows, add, compact);   \
  } else
      PGCN_SPMM16_CASES(X) { return fail(PGCN_EUNSUPPORTED, "no bf16 spmm_fwd shape for ld8=%lld", (long long)ld8); }
#undef X
    } else {
      const SpmmShape sh = chunked(spmm_shape, ld4, (double)n_valid * ld4 * 16);
      const int grid = grid_for(n_rows * sh.nchunk, kThreads / sh.G, sm_count() * 64);
#define X(G_, NC_, U_, MB_)                                                                                     \
  if (sh.G == G_ && sh.NC == NC_ && sh.U == U_ && sh.MB == MB_) {                                              \
    if (chk)                                                                                                   \
      k_spmm_fwd<G_, NC_, U_, MB_, true><<<grid, kThreads, 0, st>>>(row_ptr, col, inv_deg, D4, ld4, n_rows,      \
                                                                    n_valid, sh.nchunk, Z4, wk, K, slf, bias,     \
                                                                    n_bias, relu, rows, add, compact);            \
    else                                                                                                       \
      k_spmm_fwd<G_, NC_, U_, MB_, false><<<grid, kThreads, 0, st>>>(row_ptr, col, inv_deg, D4, ld4, n_rows,     \
                                                                     n_valid, sh.nchunk, Z4, wk, K, slf, bias,    \
                                                                     n_bias, relu, rows, add, compact);           \
  } else
      PGCN_SPMM_CASES(X) { return fail(PGCN_EUNSUPPORTED, "no spmm_fwd shape for ld4=%lld", (long long)ld4); }
#undef X
    }
    count(L);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : fail(PGCN_ECUDA, "SpMM launch failed");
  };
  L2Window l2w(L.s, b16 ? g16 : (const void*)D, (size_t)n_valid * (b16 ? ld8 * 16 : ld4 * 16));
  if (!tcu) return gather(L.s, work, self, 0);
  auto tile = [&](float* out) -> int {
    int rc;
    TileMark tm(L, PGCN_K_SPMM_TILE_FWD, *tiles, ld, b16);
    if (b16) {
      rc = spmm_tc(L, *tiles, G16, nullptr, ld8 * 8, n_valid, ld8 * 8, out, ld, ld);
    } else {  // fp32 tier: bf16 hi/lo split of the table, then the tile sums (2 MMAs per k-step)
      auto H16 = static_cast<uint4*>(t16);
      k_split_bf16<<<grid_for(n_valid * ld8, kThreads), kThreads, 0, L.s>>>(D4, ld4, ld4, n_valid, ld8, H16,
                                                                               H16 + n_valid * ld8);
      count(L);
      rc = spmm_tc(L, *tiles, H16, H16 + n_valid * ld8, ld8 * 8, n_valid, ld8 * 8, out, ld, ld);
    }
    return rc ? fail(PGCN_ECUDA, "tensor-core tile SpMM (fwd) launch failed") : 0;
  };
  if (int rc = tile(Z)) return rc;
  return gather(L.s, work, self, 1);
}

int spmm_bwd(Launch L, const int64_t* t_row_ptr, const int32_t* t_col, const float* dZs, const float* dDs,
              int64_t ld_dA, int64_t n_in, int64_t n_all, float* J, int64_t ld, const int64_t* gid,
              const DropSpec& d, unsigned long long* work, const float* rs, void* g16, int64_t nnz,
              const TileDev* tiles, void* t16, const int32_t* dmap, const PushSpec* push) {
  PushSpec ps{};
  if (push) ps = *push;
  if (n_all <= 0) return 0;
  const int tcu = tiles && tiles->n_tiles > 0 && tiles->n_rows == n_all;  // see spmm_fwd
  if (tcu) {
    t_row_ptr = tiles->lrp;
    t_col = tiles->lcol;
    nnz = tiles->nnz_light;
  }
  const int64_t ld4 = ld / 4, ld8 = (ld + 7) / 8;
  const bool b16 = g16 != nullptr;
  if ((b16 ? ld8 * 16 : ld_dA * 4) >= (int64_t(1) << 32) || n_in >= (int64_t(1) << 31)) {
    return fail(PGCN_EUNSUPPORTED, "spmm_bwd: row stride / id range exceeds 32-bit addressing");
  }
  const int K = grab_items(nnz, n_all);
  if (!dyn_enabled()) work = nullptr;
  auto J4 = reinterpret_cast<float4*>(J);
  const int64_t lda4 = ld_dA / 4;
  auto a = reinterpret_cast<const float4*>(dZs);
  auto G16 = static_cast<uint4*>(g16);
  if (b16) {  // bf16 gather tier: dZs (n_in rows of stride ld_dA) -> bf16 rows of ld8 vectors
    k_to_bf16<<<grid_for(n_in * ld8, kThreads), kThreads, 0, L.s>>>(a, lda4, ld4, n_in, ld8, G16);
    count(L);
  }
  auto gather = [&](cudaStream_t st, unsigned long long* wk, const float* dD, int add) -> int {
    if (wk) cudaMemsetAsync(wk, 0, sizeof(unsigned long long), st);
    auto b = reinterpret_cast<const float4*>(dD);
    if (b16) {
      const SpmmShape sh = chunked(spmm16_shape, ld8, (double)n_in * ld8 * 16);
      const int grid = grid_for(n_all * sh.nchunk, kThreads / sh.G, sm_count() * 64);
#define X(G_, NC_, U_, MB_)                                                                                     \
  if (sh.G == G_ && sh.NC == NC_ && sh.U == U_ && sh.MB == MB_) {                                              \
    k_spmm_bwd16<G_, NC_, U_, MB_><<<grid, kThreads, 0, st>>>(t_row_ptr, t_col, G16, ld8, b, lda4, n_in, n_all,  \
                                                              sh.nchunk, J4, ld4, gid, d, wk, K, rs, add, dmap, ps);                                     \
  } else
      PGCN_SPMM16_CASES(X) { return fail(PGCN_EUNSUPPORTED, "no bf16 spmm_bwd shape for ld8=%lld", (long long)ld8); }
#undef X
    } else {
      const SpmmShape sh = chunked(spmm_bwd_shape, ld4, (double)n_in * ld4 * 16);
      const int grid = grid_for(n_all * sh.nchunk, kThreads / sh.G, sm_count() * 64);
#define X(G_, NC_, U_, MB_)                                                                                     \
  if (sh.G == G_ && sh.NC == NC_ && sh.U == U_ && sh.MB == MB_) {                                              \
    k_spmm_bwd<G_, NC_, U_, MB_><<<grid, kThreads, 0, st>>>(t_row_ptr, t_col, a, b, lda4, n_in, n_all,          \
                                                            sh.nchunk, J4, ld4, gid, d, wk, K, rs, add, dmap, ps);                                       \
  } else
      PGCN_SPMM_CASES(X) { return fail(PGCN_EUNSUPPORTED, "no spmm_bwd shape for ld4=%lld", (long long)ld4); }
#undef X
    }
    count(L);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : fail(PGCN_ECUDA, "SpMM launch failed");
  };
  L2Window l2w(L.s, b16 ? g16 : (const void*)a, (size_t)n_in * (b16 ? ld8 * 16 : (size_t)lda4 * 16));
  if (!tcu) return gather(L.s, work, dDs, 0);
  auto tile = [&](float* out) -> int {
    int rc;
    TileMark tm(L, PGCN_K_SPMM_TILE_BWD, *tiles, ld, b16);
    if (b16) {
      rc = spmm_tc(L, *tiles, G16, nullptr, ld8 * 8, n_in, ld8 * 8, out, ld, ld);
    } else {  // fp32 tier: bf16 hi/lo split of dZs, then the tile sums
      auto H16 = static_cast<uint4*>(t16);
      k_split_bf16<<<grid_for(n_in * ld8, kThreads), kThreads, 0, L.s>>>(a, lda4, ld4, n_in, ld8, H16,
                                                                            H16 + n_in * ld8);
      count(L);
      rc = spmm_tc(L, *tiles, H16, H16 + n_in * ld8, ld8 * 8, n_in, ld8 * 8, out, ld, ld);
    }
    return rc ? fail(PGCN_ECUDA, "tensor-core tile SpMM (bwd) launch failed") : 0;
  };
  if (int rc = tile(J)) return rc;
  return gather(L.s, work, dDs, 1);
}

void gather_rows(Launch L, const SegTable& src, const int32_t* row_map, int64_t n_rows, int64_t ld, float* dst,
                 const float* prev, float gamma, int ema, int first) {
  if (n_rows <= 0) return;
  const int64_t ld4 = ld / 4;
  k_gather<<<grid_for(n_rows * ld4, kThreads), kThreads, 0, L.s>>>(src, row_map, n_rows, ld4,
                                                                   reinterpret_cast<float4*>(dst),
                                                                   reinterpret_cast<const float4*>(prev), gamma, ema,
                                                                   first);
  count(L);
}

void grad_reduce(Launch L, const int64_t* inv_ptr, const int32_t* inv_pos, const SegTable& msg, const int32_t* row_map,
                 float* ema, float gamma, int use_ema, int first, float* J, int write_j, const float* Hprev, float* M,
                 int64_t n_in, int64_t ld, int msg16, float* Mlo) {
  if (n_in <= 0) return;
  const int64_t ld4 = ld / 4;
  k_grad_reduce<<<grid_for(n_in * ld4, kThreads), kThreads, 0, L.s>>>(
      inv_ptr, inv_pos, msg, row_map, reinterpret_cast<float4*>(ema), gamma, use_ema, first,
      reinterpret_cast<float4*>(J), write_j, reinterpret_cast<const float4*>(Hprev), reinterpret_cast<float4*>(M), n_in,
      ld4, msg16, reinterpret_cast<float4*>(Mlo));
  count(L);
}

void pack_rows_bf16(Launch L, const float* src, const int32_t* row_map, int64_t n_rows, int64_t ld, void* dst) {
  if (n_rows <= 0) return;
  const int64_t ld4 = ld / 4;
  k_pack_bf16<<<grid_for(n_rows * ld4, kThreads), kThreads, 0, L.s>>>(reinterpret_cast<const float4*>(src), row_map,
                                                                      n_rows, ld4, static_cast<uint2*>(dst));
  count(L);
}

void install_bf16(Launch L, const void* src, int64_t n_rows, int64_t ld, float* dst, const float* prev, float gamma,
                  int ema) {
  if (n_rows <= 0) return;
  const int64_t ld4 = ld / 4;
  k_install_bf16<<<grid_for(n_rows * ld4, kThreads), kThreads, 0, L.s>>>(
      static_cast<const uint2*>(src), n_rows, ld4, reinterpret_cast<float4*>(dst),
      reinterpret_cast<const float4*>(prev), gamma, ema);
  count(L);
}

void spin_ns(cudaStream_t s, int64_t ns) {
  if (ns > 0) k_spin<<<1, 1, 0, s>>>(ns);
}

void scatter_rows(Launch L, const float* src, const int32_t* map, int64_t n, int64_t ld, float* dst) {
  if (n <= 0) return;
  const int64_t ld4 = ld / 4;
  k_scatter_rows<<<grid_for(n * ld4, kThreads), kThreads, 0, L.s>>>(reinterpret_cast<const float4*>(src), map, n, ld4,
                                                                    reinterpret_cast<float4*>(dst));
  count(L);
}

void compact_train_setup(Launch L, const int32_t* list, int64_t n_tr, int64_t n_in, int32_t* pos, int32_t* cols,
                         int64_t n_cols) {
  cudaMemsetAsync(pos, 0xff, sizeof(int32_t) * (size_t)n_in, L.s);
  if (n_tr > 0) {
    k_positions<<<grid_for(n_tr, kThreads), kThreads, 0, L.s>>>(list, n_tr, pos);
    count(L);
  }
  if (n_cols > 0) {
    k_remap<<<grid_for(n_cols, kThreads), kThreads, 0, L.s>>>(cols, n_cols, pos);
    count(L);
  }
}

void gather_bytes(Launch L, const void* src, const int32_t* list, int64_t n, int64_t w, void* dst) {
  if (n <= 0 || w <= 0) return;
  k_gather_bytes<<<grid_for(n * w, kThreads), kThreads, 0, L.s>>>(static_cast<const uint8_t*>(src), list, n, w,
                                                                   static_cast<uint8_t*>(dst));
  count(L);
}

void loss_rows(Launch L, int kind, const float* Y, int64_t n, int64_t C, int64_t ld, const void* labels,
               const uint8_t* train, double n_train, float* M, float* row_loss, float* Mlo, const int32_t* rows) {
  if (n <= 0) return;
  const int grid = grid_for(n, kThreads / 32, sm_count() * 32);
  if (kind == 0)
    k_loss_ce<<<grid, kThreads, 0, L.s>>>(Y, n, C, ld, static_cast<const int32_t*>(labels), train,
                                          (float)(1.0 / n_train), M, row_loss, Mlo, rows);
  else
    k_loss_bce<<<grid, kThreads, 0, L.s>>>(Y, n, C, ld, static_cast<const uint8_t*>(labels), train,
                                           (float)(1.0 / (n_train * (double)C)), M, row_loss, Mlo, rows);
  count(L);
}

void reduce_sum(Launch L, const float* x, int64_t n, float* out) {
  k_reduce_sum<<<1, 1024, 0, L.s>>>(x, n, out);
  count(L);
}

void gemm_fwd_f32(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* Wext,
                  int64_t N, float* Y, int64_t ldY, int relu) {
  if (M <= 0) return;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((ldY + BN - 1) / BN));
  if (relu) k_gemm_fwd<1><<<grid, 256, 0, L.s>>>(Z, D, ldA, M, F, Wext, N, Y, ldY);
  else k_gemm_fwd<0><<<grid, 256, 0, L.s>>>(Z, D, ldA, M, F, Wext, N, Y, ldY);
  count(L);
}

int64_t gemm_dw_ws_floats(int64_t M, int64_t F, int64_t N) {
  const int64_t K = 2 * F + 1;
  const int64_t tiles = ((K + BM - 1) / BM) * ((N + BN - 1) / BN);
  int64_t splits = (2 * sm_count() + tiles - 1) / tiles;
  const int64_t max_splits = (M + 255) / 256;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits * K * N;
}

void gemm_dw_f32(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* Mg,
                 int64_t ldM, int64_t N, float* G, float* ws, int64_t ws_floats) {
  const int64_t K = 2 * F + 1;
  int64_t splits = gemm_dw_ws_floats(M, F, N) / (K * N);
  if (splits * K * N > ws_floats) splits = ws_floats / (K * N);
  if (splits < 1) splits = 1;
  if (M <= 0) {
    cudaMemsetAsync(G, 0, sizeof(float) * K * N, L.s);
    return;
  }
  const int64_t rps = ((M + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (M + rps - 1) / rps;
  dim3 grid((unsigned)((K + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)splits);
  k_gemm_dw<<<grid, 256, 0, L.s>>>(Z, D, ldA, M, F, Mg, ldM, N, rps, ws);
  k_split_reduce<<<grid_for(K * N, kThreads), kThreads, 0, L.s>>>(ws, splits, K * N, G);
  count(L, 2);
}

void split_reduce(Launch L, const float* part, int64_t splits, int64_t len, float* G) {
  k_split_reduce<<<grid_for(len, kThreads), kThreads, 0, L.s>>>(part, splits, len, G);
  count(L);
}

void split_reduce_strided(Launch L, const float* part, int64_t splits, int64_t rows, int64_t N, int64_t NP,
                          float* G) {
  k_split_reduce_strided<<<grid_for(rows * N, kThreads), kThreads, 0, L.s>>>(part, splits, rows, N, NP, G);
  count(L);
}

void split_reduce_dw(Launch L, const float* part, const int64_t zc[3], int64_t F, int nseg, int64_t N, int64_t NP,
                     float* G) {
  const int64_t rows = nseg * F + 1;
  k_split_reduce_dw<<<grid_for(rows * N, kThreads), kThreads, 0, L.s>>>(part, zc[0], zc[1], zc[2], F, rows, N, NP, G);
  count(L);
}

void gemm_da_f32(Launch L, const float* Mg, int64_t ldM, int64_t M, int64_t N, const float* W, int64_t F,
                 const float* inv_deg, float* dA, int64_t ld) {
  if (M <= 0) return;
  dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((2 * ld + BN - 1) / BN));
  k_gemm_da<<<grid, 256, 0, L.s>>>(Mg, ldM, M, N, W, F, inv_deg, dA, ld);
  count(L);
}

void stale_err(Launch L, const SegTable& fresh, const int32_t* fmap, const SegTable* used_tab, const int32_t* umap,
               const float* used, int64_t n_rows, int64_t ld, int64_t F, double* out) {
  if (n_rows <= 0) return;
  SegTable none{};
  k_stale_err<<<grid_for(n_rows * F, 256, sm_count() * 4), 256, 0, L.s>>>(fresh, fmap, used_tab ? *used_tab : none, umap, used,
                                                                    used_tab ? 1 : 0, n_rows, ld, F, out);
  count(L);
}

void scale_rows(Launch L, const float* M, const float* s, int64_t n, int64_t ld, float* out) {
  if (n <= 0) return;
  k_scale_rows<<<grid_for(n * (ld / 4), kThreads), kThreads, 0, L.s>>>(reinterpret_cast<const float4*>(M), s, n,
                                                                      ld / 4, reinterpret_cast<float4*>(out));
  count(L);
}

void sum_grads(Launch L, const PtrList& G, int64_t P, float* grads) {
  k_sum_grads<<<grid_for(P, kThreads), kThreads, 0, L.s>>>(G, P, grads);
  count(L);
}

void opt_update(Launch L, const float* grads, int64_t P, float* params, float* m, float* v, const OptSpec& o) {
  k_opt<<<grid_for(P, kThreads), kThreads, 0, L.s>>>(grads, P, params, m, v, o);
  count(L);
}

namespace {
// Random-row gather ceiling (roofline denominator for the DRAM-served aggregation): groups of G lanes
// read whole rows idx[k] (row4 float4 each, row4 <= G) with U rows in flight per group, and fold them
// into one checksum per thread.  No arithmetic beyond the adds: the hardware's random-row read rate.
template <int G, int U>
__global__ void __launch_bounds__(256) k_gather_read(const float4* __restrict__ tab, int64_t row4,
                                                     const int32_t* __restrict__ idx, int64_t n_idx,
                                                     float* __restrict__ out) {
  const int lane = threadIdx.x & (G - 1);
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t n_grp = (int64_t)gridDim.x * blockDim.x / G;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t k0 = grp * U; k0 < n_idx; k0 += n_grp * U) {
    for (int64_t x = lane; x < row4 || x == lane; x += G) {  // rows wider than G float4: several passes
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t k = k0 + u;
        v[u] = (k < n_idx && x < row4) ? __ldg(tab + (int64_t)__ldg(idx + k) * row4 + x) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc = f4add(acc, v[u]);
    }
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int U>
__global__ void __launch_bounds__(256) k_l2_read(const float4* __restrict__ buf, int64_t n4, int reps,
                                                 float* __restrict__ out) {
  // Each warp streams contiguous 512*U-byte chunks (U independent 512-byte LDG.128 per lane in
  // flight), chunks handed out grid-stride over warps; 32-bit indexing.
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = a;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t n_chunks = (uint32_t)(n4 / (32 * U));
  const uint32_t w0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = 0; r < reps; ++r) {
    for (uint32_t c = w0; c < n_chunks; c += nw) {
      const float4* p = buf + (size_t)c * (32 * U) + lane;
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(p + 32 * u);
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        f4acc(a, v[u]);
        if (u + 1 < U) f4acc(b, v[u + 1]);
      }
    }
  }
  float s = a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ float sh[8];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += sh[w];
    out[blockIdx.x] = t;
  }
}
}  // namespace
}  // namespace pgcn

extern "C" int pgcn_dev_spmm(const int64_t* row_ptr, const int32_t* col, const float* inv_deg, const float* D,
                             int64_t ld, int64_t n_rows, int64_t n_valid, float* Z, void* stream) {
  if (!row_ptr || !col || !inv_deg || !D || !Z || ld % 4 || n_rows < 0) return -1;
  const int rc = pgcn::spmm_fwd(pgcn::Launch{static_cast<cudaStream_t>(stream), nullptr}, row_ptr, col, inv_deg, D,
                                ld, n_rows, n_valid, Z, nullptr, 0, nullptr, 0, 0, n_valid);
  return rc ? rc : (cudaGetLastError() == cudaSuccess ? 0 : -3);
}

extern "C" int pgcn_dev_gather_read(const float* tab, int64_t row_floats, const int32_t* idx, int64_t n_idx,
                                    float* out, int32_t variant, void* stream) {
  if (!tab || !idx || !out || row_floats % 4 || row_floats <= 0 || n_idx < 0) return -1;
  const int64_t row4 = row_floats / 4;
  const int blocks = pgcn::sm_count() * 8;  // out holds blocks * 256 floats
  auto s = static_cast<cudaStream_t>(stream);
  auto t4 = reinterpret_cast<const float4*>(tab);
  const int U = variant == 1 ? 16 : 8;
  if (row4 <= 4) {
    if (U == 8) pgcn::k_gather_read<4, 8><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
    else pgcn::k_gather_read<4, 16><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
  } else if (row4 <= 8) {
    if (U == 8) pgcn::k_gather_read<8, 8><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
    else pgcn::k_gather_read<8, 16><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
  } else if (row4 <= 16) {
    if (U == 8) pgcn::k_gather_read<16, 8><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
    else pgcn::k_gather_read<16, 16><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
  } else {
    if (U == 8) pgcn::k_gather_read<32, 8><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
    else pgcn::k_gather_read<32, 16><<<blocks, 256, 0, s>>>(t4, row4, idx, n_idx, out);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

extern "C" int pgcn_dev_l2_read(const void* buf, int64_t bytes, int32_t reps, float* out, void* stream) {
  if (!buf || !out || bytes < 16 || reps < 1) return -1;
  // variant (reps' high byte): 0 = 4 x 512 B in flight per warp, 8 blocks/SM; 1 = 8 x 512 B,
  // 8 blocks/SM; 2 = 8 x 512 B, 4 blocks/SM.  The caller takes the best as the L2 read peak.
  const int variant = (reps >> 24) & 0xff;
  reps &= 0xffffff;
  auto s = static_cast<cudaStream_t>(stream);
  auto b4 = static_cast<const float4*>(buf);
  const int sms = pgcn::sm_count();  // out holds up to sms x 8 floats
  if (variant == 0) pgcn::k_l2_read<4><<<sms * 8, 256, 0, s>>>(b4, bytes / 16, reps, out);
  else if (variant == 1) pgcn::k_l2_read<8><<<sms * 8, 256, 0, s>>>(b4, bytes / 16, reps, out);
  else pgcn::k_l2_read<8><<<sms * 4, 256, 0, s>>>(b4, bytes / 16, reps, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}
