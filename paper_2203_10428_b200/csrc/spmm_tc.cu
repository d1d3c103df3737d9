// Heavy-tile part of the aggregation SpMMs (S3 forward, S8 transposed) on the tensor cores.
//
// Eq. 3 sums gathered rows: out[v] = sum_{u in N(v)} B[u].  Where a 128-row block
// of the pattern and a 64-column tile hold many edges (dense communities: Reddit-shaped rows have
// ~490 neighbours, 90 % inside their community), that block of the sum is the dense product
// A_tile (128 x 64, entries 0/1 -- exactly the pattern) x B[64 rows of the tile, :].  Gathering
// those edges one row per edge moves 64 x F x 4 bytes per ~(tile edges) uses; the product reads
// each of the 64 rows once per tile, so the gather bytes drop by the tile's edge count / 64 and
// the contraction itself runs on tcgen05:
//   fp32 tier: B = B_hi + B_lo split (kind::tf32; hi = the fp32 word, truncated by the tensor
//              core; lo = x - trunc(x)); A is exact in tf32, so 2 MMAs give fp32-grade sums
//              (the dropped lo truncation is <= 2^-20 relative, fp32 accumulation).
//   bf16 tier: B = the bf16 table the gather tier already rounds to (kind::f16, 1 MMA).
// Output: out[r, 0:width) = sum over the heavy tiles of row block r / 128 (zeros where a block has
// none); the gather SpMM then adds the light edges on top (its `addend`), applies inv_deg, the
// self term, bias / ReLU or the dropout mask -- so the result is the same sum, reassociated.
//
// Roles (320 threads): warp 0 TMA producer (B boxes + the tile's 1 KB bitmask by bulk copy), warp 1
// TMEM owner + single-thread MMA issuer, warps 2-5 builders (bitmask -> A tile in the UMMA K-major
// SW128 layout; fp32 tier: B_lo), warps 6-9 epilogue (tcgen05.ld -> float4 stores).  Work list:
// (row block, n-tile) items in the host's descending-tile-count order, strided over a persistent
// grid of one CTA per SM.  Operand layouts are the proven ones of gemm_tc.cu: A as its FWD
// K-major A, B as its DW MN-major B (tf32: 32x32 boxes, SWIZZLE_128B_ATOM_32B; bf16: 64x32 boxes,
// SWIZZLE_128B).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace pgcn {
namespace tcs {

using namespace pgcn::tc;

constexpr int kBuildWarps = 4;
constexpr int kBuildThreads = 32 * kBuildWarps;
constexpr int kThreads = 64 + kBuildThreads + 128;
constexpr int BM = 128;

struct Params {
  CUtensorMap map_b;
  const int32_t* rb_ptr;
  const int32_t* order;
  const int32_t* tile_col;
  const uint64_t* mask;
  float* out;
  int64_t n_rows, ld_out;
  int n_rb, n_nt, BN, stages, tmem_cols, width;
};

// Per-stage geometry.  tf32: one stage = half a tile (32 columns of k): A 128x32 fp32 (16 KB) |
// B 32 rows x BN fp32 | B_lo | mask 1 KB.  bf16: one stage = a whole tile (64 k): A 128x64 bf16
// (16 KB) | B two k-halves of 32 rows x BN bf16 | mask.
struct Geo {
  uint32_t a, b, blo, mask;
  __host__ __device__ uint32_t stage() const { return a + b + blo + mask; }
};
__host__ __device__ inline Geo geometry(int BF, int BN) {
  Geo g;
  g.a = 16384;
  g.b = BF ? (uint32_t)BN * 64 * 2 : (uint32_t)BN * 32 * 4;
  g.blo = BF ? 0u : (uint32_t)BN * 32 * 4;
  g.mask = BM * 8;
  return g;
}

template <int BF>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_tc(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const Geo geo = geometry(BF, p.BN);
  const uint32_t stage_bytes = geo.stage();
  constexpr int HALVES = BF ? 1 : 2;  // stages per tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = bars + 3 * S + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_items = p.n_rb * p.n_nt;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kBuildThreads);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"((uint32_t)p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ===================================================== TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t tx = geo.b + geo.mask;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int rb = p.order[it / p.n_nt];
        const int n0 = (it % p.n_nt) * p.BN;
        for (int k = p.rb_ptr[rb]; k < p.rb_ptr[rb + 1]; ++k) {
          const int row0 = p.tile_col[k] * 64;
          for (int h = 0; h < HALVES; ++h) {
            mbar_wait(&empty[s], ph ^ 1, 11);
            uint8_t* st = smem + (size_t)s * stage_bytes;
            uint8_t* B = st + geo.a;
            uint8_t* Mk = st + geo.a + geo.b + geo.blo;
            mbar_expect_tx(&full[s], tx);
            if (BF) {
              // two k-halves of 32 rows, each BN/64 SW128 atoms of 64 bf16 x 32 rows (4 KB)
              for (int kh = 0; kh < 2; ++kh)
                for (int j = 0; j < p.BN / 64; ++j)
                  tma_load_2d(B + (kh * (p.BN / 64) + j) * 4096, &p.map_b, &full[s], n0 + 64 * j, row0 + 32 * kh);
            } else {
              for (int j = 0; j < p.BN / 32; ++j)
                tma_load_2d(B + j * 4096, &p.map_b, &full[s], n0 + 32 * j, row0 + 32 * h);
            }
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(Mk)),
                "l"(reinterpret_cast<uint64_t>(p.mask + (size_t)k * BM)), "r"((uint32_t)(BM * 8)),
                "r"(smem_u32(&full[s]))
                : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      const uint32_t fmt = BF ? 1u : 2u;
      // A K-major (bit 15 = 0), B MN-major (bit 16 = 1), F32 accumulators
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) | ((uint32_t)(p.BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int rb = p.order[it / p.n_nt];
        mbar_wait(&tempty[acc], acc_ph ^ 1, 12);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * p.BN);
        uint32_t accum = 0;
        const int nst = (p.rb_ptr[rb + 1] - p.rb_ptr[rb]) * HALVES;
        for (int i = 0; i < nst; ++i) {
          mbar_wait(&conv[s], ph, 13);
          tc_fence_after();
          const uint32_t A = smem_u32(smem + (size_t)s * stage_bytes);
          const uint32_t B = A + geo.a;
          if (BF) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // k-steps of 16: A 32 bytes apart; B 16-row steps in k-half kk/2
              const uint32_t Bk = B + (uint32_t)((kk >> 1) * (p.BN / 64) * 4096 + (kk & 1) * 2048);
              mma_bf16(d, make_desc(A + kk * 32, 16, 1024), make_desc(Bk, 4096, 1024), idesc, accum);
              accum = 1u;
            }
          } else {
            const uint32_t Blo = B + geo.b;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // k-steps of 8: A 32 bytes apart, B 8 rows = 1 KB apart
              const uint64_t a = make_desc(A + kk * 32, 16, 1024);
              mma_tf32(d, a, make_desc(B + kk * 1024, 4096, 512, 1), idesc, accum);
              mma_tf32(d, a, make_desc(Blo + kk * 1024, 4096, 512, 1), idesc, 1u);
              accum = 1u;
            }
          }
          tc_commit(&empty[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp < 2 + kBuildWarps) {
    // ===================================================== builders: bitmask -> A (0/1), B -> B_lo
    const int ct = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int rb = p.order[it / p.n_nt];
      const int nt = p.rb_ptr[rb + 1] - p.rb_ptr[rb];
      for (int k = 0; k < nt; ++k) {
        for (int h = 0; h < HALVES; ++h) {
          mbar_wait(&full[s], ph, 14);
          uint8_t* st = smem + (size_t)s * stage_bytes;
          const uint64_t* Mk = reinterpret_cast<const uint64_t*>(st + geo.a + geo.b + geo.blo);
          // A row r = 128 bytes (32 tf32 or 64 bf16 of k); 16-byte chunk j at r*128 + ((j ^ (r&7)) << 4)
          for (int i = ct; i < BM * 8; i += kBuildThreads) {
            const int r = i >> 3, j = i & 7;
            uint4 o;
            if (BF) {
              const uint32_t bits = (uint32_t)(Mk[r] >> (8 * j)) & 0xFFu;
              const uint32_t one = 0x3F80u;  // bf16 1.0
              o.x = ((bits & 1u) ? one : 0u) | ((bits & 2u) ? one << 16 : 0u);
              o.y = ((bits & 4u) ? one : 0u) | ((bits & 8u) ? one << 16 : 0u);
              o.z = ((bits & 16u) ? one : 0u) | ((bits & 32u) ? one << 16 : 0u);
              o.w = ((bits & 64u) ? one : 0u) | ((bits & 128u) ? one << 16 : 0u);
            } else {
              const uint32_t bits = (uint32_t)(Mk[r] >> (32 * h + 4 * j)) & 0xFu;
              const uint32_t one = 0x3F800000u;  // 1.0f
              o.x = (bits & 1u) ? one : 0u;
              o.y = (bits & 2u) ? one : 0u;
              o.z = (bits & 4u) ? one : 0u;
              o.w = (bits & 8u) ? one : 0u;
            }
            *reinterpret_cast<uint4*>(st + r * 128 + ((j ^ (r & 7)) << 4)) = o;
          }
          if (!BF) {
            const float4* B = reinterpret_cast<const float4*>(st + geo.a);
            float4* Blo = reinterpret_cast<float4*>(st + geo.a + geo.b);
            for (int i = ct; i < (int)(geo.b / 16); i += kBuildThreads) {
              const float4 x = B[i];
              Blo[i] = make_float4(tf32_lo_trunc(x.x), tf32_lo_trunc(x.y), tf32_lo_trunc(x.z), tf32_lo_trunc(x.w));
            }
          }
          fence_async_smem();
          mbar_arrive(&conv[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else {
    // ===================================================== epilogue: TMEM -> out rows
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int rb = p.order[it / p.n_nt];
      const int n0 = (it % p.n_nt) * p.BN;
      const bool none = p.rb_ptr[rb + 1] == p.rb_ptr[rb];
      mbar_wait(&tfull[acc], acc_ph, 15);
      __syncwarp();
      tc_fence_after();
      const int64_t row = (int64_t)rb * BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * p.BN);
      float* out = p.out + row * p.ld_out;
      for (int c0 = 0; c0 < p.BN; c0 += 16) {
        if (n0 + c0 >= p.width) break;  // warp-uniform
        uint32_t r[16];
        TMEM_LD16(tbase + c0, r);
        tmem_ld_wait();
        if (row < p.n_rows) {
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4) {
            const int n = n0 + c0 + 4 * g4;
            if (n >= p.width) break;
            const float4 o = none ? make_float4(0.f, 0.f, 0.f, 0.f)
                                  : make_float4(__uint_as_float(r[4 * g4]), __uint_as_float(r[4 * g4 + 1]),
                                                __uint_as_float(r[4 * g4 + 2]), __uint_as_float(r[4 * g4 + 3]));
            *reinterpret_cast<float4*>(out + n) = o;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_ph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"((uint32_t)p.tmem_cols));
  }
}

}  // namespace tcs

// out[r, 0:width) = sum of the heavy-tile edges of row r over the table B (rows b_rows, row stride
// b_ld elements, fp32 or bf16).  Returns 0, or < 0 when the table cannot be mapped for TMA.
int spmm_tc(Launch L, const TileDev& T, const void* B, int bf, int64_t b_cols, int64_t b_rows, int64_t b_ld,
            float* out, int64_t ld_out, int64_t width) {
  using namespace tcs;
  if (T.n_rb <= 0) return 0;
  Params p{};
  const int atom = bf ? 64 : 32;
  int64_t bn = (width + atom - 1) / atom * atom;
  if (bn > 256) bn = 256;
  p.BN = (int)bn;
  p.n_nt = (int)((width + bn - 1) / bn);
  p.n_rb = (int)T.n_rb;
  p.rb_ptr = T.rb_ptr;
  p.order = T.order;
  p.tile_col = T.tile_col;
  p.mask = T.mask;
  p.out = out;
  p.n_rows = T.n_rows;
  p.ld_out = ld_out;
  p.width = (int)width;
  p.tmem_cols = tc_tmem_cols(p.BN);
  const uint32_t stage = geometry(bf, p.BN).stage();
  int S = (int)((200 * 1024) / stage);
  p.stages = S > 6 ? 6 : (S < 2 ? 2 : S);
  const size_t smem = 1024 + (size_t)p.stages * stage + (3 * p.stages + 4) * 8 + 16;
  if (!tc_map_table(&p.map_b, B, bf != 0, b_cols, b_rows, b_ld, atom, 32)) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_spmm_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_spmm_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int n_items = p.n_rb * p.n_nt;
  const int grid = n_items < 148 ? n_items : 148;
  if (bf) k_spmm_tc<1><<<grid, kThreads, smem, L.s>>>(p);
  else k_spmm_tc<0><<<grid, kThreads, smem, L.s>>>(p);
  if (L.count) *L.count += 1;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace pgcn
