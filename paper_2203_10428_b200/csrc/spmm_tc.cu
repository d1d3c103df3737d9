// Heavy-tile part of the aggregation SpMMs (S3 forward, S8 transposed) on the tensor cores.
//
// Eq. 3 sums gathered rows: out[v] = sum_{u in N(v)} B[u].  Where a 128-row block
// of the pattern and a 64-column tile hold many edges (dense communities: Reddit-shaped rows have
// ~490 neighbours, 90 % inside their community), that block of the sum is the dense product
// A_tile (128 x 64, entries 0/1 -- exactly the pattern) x B[64 rows of the tile, :].  Gathering
// those edges one row per edge moves 64 x F x 4 bytes per ~(tile edges) uses; the product reads
// each of the 64 rows once per tile, so the gather bytes drop by the tile's edge count / 64 and
// the contraction itself runs on tcgen05 (kind::f16, A = 0/1 exact in bf16, fp32 accumulation):
//   fp32 tier: B = B_hi + B_lo, both bf16 (hi = rn(x), lo = rn(x - hi); |x - hi - lo| <= 2^-18 |x|),
//              two MMAs per k-step -- fp32-grade sums at twice the tf32 rate per k.
//   bf16 tier: B = the bf16 table the gather tier already rounds to (one MMA).
// The split tables are written by k_split_bf16 (kernels.cu) right before the launch.
// Output: out[r, 0:width) = sum over the heavy tiles of row block r / 128 (zeros where a block has
// none); the gather SpMM then adds the light edges on top (its `addend`), applies inv_deg, the
// self term, bias / ReLU or the dropout mask -- so the result is the same sum, reassociated.
//
// Roles (320 threads): warp 0 TMA producer (B boxes; in SS mode also the tile's 1 KB bitmask by bulk
// copy on its own barrier), warp 1 TMEM owner + single-thread MMA issuer, warps 2-5 build the A tile:
// TS mode (default) -- each thread reads its row's 64-bit mask word from global two tiles ahead and
// writes 32 columns of bf16 0/1 pairs to TMEM with tcgen05.st (A from TMEM); SS mode (bf16 tier,
// BN = 256) -- expand the bitmask into the UMMA K-major SW128 layout in shared memory.  Warps 6-9:
// epilogue (tcgen05.ld -> float4 stores).  Work list: (row block, n-tile) items in the host's
// descending-tile-count order, strided over a persistent grid of two CTAs per SM (one TMEM
// accumulator each; the kernel is latency-bound and two independent pipelines per SM beat one
// deeper one).  Operand layouts are the proven ones of gemm_tc.cu's bf16 variant: A as its FWD
// K-major A (128-byte rows of 64 bf16), B MN-major SW128 (atoms of 64 bf16 columns; 64-row boxes of
// 8 KB, LBO = atom stride -- or two k-halves of 32-row boxes, PGCN_TC_SPMM_BOX64=0).
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
  CUtensorMap map_b[2];  // bf16 tables: [0] hi (or the only table), [1] lo
  const int32_t* rb_ptr;
  const int32_t* order;
  const int32_t* tile_col;
  const uint64_t* mask;
  float* out;
  int64_t n_rows, ld_out;
  int n_rb, n_nt, BN, stages, tmem_cols, width;
  int nacc;   // TMEM accumulator buffers: 2 (epilogue overlaps the next item) or 1 (two CTAs per SM)
  int box64;  // B boxes of 64 rows (one SW128 atom column of 8 KB per 64 table columns) instead of two
              // k-halves of 32-row boxes
  int dbg;   // dev knob PGCN_TC_SPMM_DBG (bottleneck probes, wrong results): 1 skip B loads, 2 skip MMAs
};

// Per-stage geometry (one stage = one 128 x 64 tile): A 128 x 64 bf16 (16 KB) | NT tables x (64 rows
// x BN bf16) | mask 1 KB.  Every piece is a multiple of 1 KB (SW128 atoms stay 1024-aligned).
// TS = 1 (A in TMEM, written by tcgen05.st): no A in shared memory.
__host__ __device__ inline uint32_t table_bytes(int BN) { return (uint32_t)BN * 64 * 2; }
__host__ __device__ inline uint32_t a_bytes(int TS) { return TS ? 0u : 16384u; }
__host__ __device__ inline uint32_t stage_bytes(int NT, int BN, int TS) {
  return a_bytes(TS) + NT * table_bytes(BN) + BM * 8;
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, {%5, %5, %5, %5}, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}

// One 32-column tcgen05.st of this warp's TMEM lane quarter (thread i -> lane 32 q + i).
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// TS = 1: the 128 x 64 A tile of stage s lives in TMEM columns [2 BN + 32 s, + 32) (lane = row, two
// bf16 k per 32-bit column, k even in the low half -- the UMMA "A from TMEM" layout), written by the
// builders with tcgen05.st; otherwise in shared memory (SS mode).
template <int NT, int TS>
__global__ void __launch_bounds__(kThreads, 1) k_spmm_tc(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const uint32_t tb = table_bytes(p.BN), sb = stage_bytes(NT, p.BN, TS), ab = a_bytes(TS);
  const uint32_t mask_off = ab + NT * tb;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * sb);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = bars + 3 * S + 2;
  uint64_t* mfull = bars + 3 * S + 4;  // the tile's bitmask only: the builders need not wait for B
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 4 * S + 4);
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_items = p.n_rb * p.n_nt;
  const int natom = p.BN / 64;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kBuildThreads);
      mbar_init(&empty[s], 1);
      mbar_init(&mfull[s], 1);
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
      const uint32_t tx = (p.dbg & 1) ? 0u : NT * tb;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int rb = p.order ? p.order[it / p.n_nt] : it / p.n_nt;
        const int n0 = (it % p.n_nt) * p.BN;
        for (int k = p.rb_ptr[rb]; k < p.rb_ptr[rb + 1]; ++k) {
          const int row0 = p.tile_col[k] * 64;
          mbar_wait(&empty[s], ph ^ 1, 11);
          uint8_t* st = smem + (size_t)s * sb;
          if (!TS) {  // SS mode: the builders read the bitmask from shared memory
          mbar_expect_tx(&mfull[s], BM * 8);
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(st + mask_off)),
              "l"(reinterpret_cast<uint64_t>(p.mask + (size_t)k * BM)), "r"((uint32_t)(BM * 8)),
              "r"(smem_u32(&mfull[s]))
              : "memory");
          }
          mbar_expect_tx(&full[s], tx);
          if (tx && p.box64)
            for (int t = 0; t < NT; ++t)
              for (int j = 0; j < natom; ++j)  // natom SW128 atoms of 64 columns x 64 rows (8 KB)
                tma_load_2d(st + ab + t * tb + j * 8192, &p.map_b[t], &full[s], n0 + 64 * j, row0);
          else if (tx)
            for (int t = 0; t < NT; ++t)
              for (int kh = 0; kh < 2; ++kh)  // two k-halves of 32 rows, natom SW128 atoms of 64 x 32 each
                for (int j = 0; j < natom; ++j)
                  tma_load_2d(st + ab + t * tb + (kh * natom + j) * 4096, &p.map_b[t], &full[s], n0 + 64 * j,
                              row0 + 32 * kh);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      // bf16 A and B, F32 accumulators, A K-major (bit 15 = 0), B MN-major (bit 16 = 1)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(p.BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int rb = p.order ? p.order[it / p.n_nt] : it / p.n_nt;
        mbar_wait(&tempty[acc], acc_ph ^ 1, 12);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * p.BN);
        uint32_t accum = 0;
        const int nst = p.rb_ptr[rb + 1] - p.rb_ptr[rb];
        for (int i = 0; i < nst; ++i) {
          mbar_wait(&conv[s], ph, 13);
          mbar_wait(&full[s], ph, 16);
          tc_fence_after();
          const uint32_t A = sbase + (uint32_t)s * sb;
          const uint32_t ta = tmem_base + (uint32_t)(p.nacc * p.BN + 32 * s);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // k-steps of 16: A 32 bytes (SS) / 8 columns (TS) apart;
                                            // B 16-row steps in k-half kk/2
            const uint64_t a = make_desc(A + kk * 32, 16, 1024);
            const uint32_t boff =
                ab + (p.box64 ? (uint32_t)(kk * 2048) : (uint32_t)((kk >> 1) * natom * 4096 + (kk & 1) * 2048));
            const uint32_t lbo = p.box64 ? 8192u : 4096u;  // MN-direction atom stride
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const uint64_t b = make_desc(A + boff + t * tb, lbo, 1024);
              if (p.dbg & 2) continue;
              if (TS) mma_bf16_ts(d, ta + 8 * kk, b, idesc, accum);
              else mma_bf16(d, a, b, idesc, accum);
              accum = 1u;
            }
          }
          tc_commit(&empty[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc_commit(&tfull[acc]);
        if (++acc == p.nacc) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp < 2 + kBuildWarps) {
    // ===================================================== builders: bitmask -> A (0/1 bf16)
    const int ct = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    if (TS) {
      // A in TMEM: each thread owns row r = 32 (warp % 4) + lane and reads that row's 64-bit mask word
      // straight from global memory, two tiles ahead, so the build of stage s waits only for the MMAs
      // that last read A[s] (empty[s]) -- not for any copy.  64 bits -> 32 columns of bf16 pairs.
      const int q = warp & 3, r = 32 * q + lane;
      int nit = blockIdx.x, kk = 0, ke = 0;
      auto next_tile = [&]() -> int {  // this CTA's (item, tile) sequence, as the producer / MMA walk it
        while (kk >= ke) {
          if (nit >= n_items) return -1;
          const int rb = p.order ? p.order[nit / p.n_nt] : nit / p.n_nt;
          kk = p.rb_ptr[rb];
          ke = p.rb_ptr[rb + 1];
          nit += gridDim.x;
        }
        return kk++;
      };
      auto load_mask = [&](int t) -> uint64_t { return t >= 0 ? __ldg(p.mask + (size_t)t * BM + r) : 0ull; };
      int t0 = next_tile(), t1 = next_tile();
      uint64_t m0 = load_mask(t0), m1 = load_mask(t1);
      const uint32_t trow = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(p.nacc * p.BN);
      while (t0 >= 0) {
        const int t2 = next_tile();
        const uint64_t m2 = load_mask(t2);
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = (((m0 >> (2 * c)) & 1ull) ? 0x3F80u : 0u) | (((m0 >> (2 * c + 1)) & 1ull) ? 0x3F800000u : 0u);
        mbar_wait(&empty[s], ph ^ 1, 14);
        tc_fence_after();
        tmem_st32(trow + (uint32_t)(32 * s), v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&conv[s]);
        if (++s == S) { s = 0; ph ^= 1; }
        t0 = t1;
        m0 = m1;
        t1 = t2;
        m1 = m2;
      }
    } else
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int rb = p.order ? p.order[it / p.n_nt] : it / p.n_nt;
      const int nt = p.rb_ptr[rb + 1] - p.rb_ptr[rb];
      for (int k = 0; k < nt; ++k) {
        mbar_wait(&mfull[s], ph, 14);
        const uint32_t st = sbase + (uint32_t)s * sb;
        // row r = 128 bytes (64 bf16 of k); 16-byte chunk j (k = 8j..8j+7) at r*128 + ((j ^ (r&7)) << 4)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int i = ct + q * kBuildThreads, r = i >> 3, j = i & 7;
          const uint32_t bits = (uint32_t)(lds64(st + mask_off + r * 8) >> (8 * j)) & 0xFFu;
          const uint32_t one = 0x3F80u;  // bf16 1.0
          sts128(st + r * 128 + ((j ^ (r & 7)) << 4), ((bits & 1u) ? one : 0u) | ((bits & 2u) ? one << 16 : 0u),
                 ((bits & 4u) ? one : 0u) | ((bits & 8u) ? one << 16 : 0u),
                 ((bits & 16u) ? one : 0u) | ((bits & 32u) ? one << 16 : 0u),
                 ((bits & 64u) ? one : 0u) | ((bits & 128u) ? one << 16 : 0u));
        }
        fence_async_smem();
        mbar_arrive(&conv[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ===================================================== epilogue: TMEM -> out rows
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int rb = p.order ? p.order[it / p.n_nt] : it / p.n_nt;
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
            __stcs(reinterpret_cast<float4*>(out + n), o);  // streamed: keep L2 for the B tiles
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == p.nacc) { acc = 0; acc_ph ^= 1; }
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

// out[r, 0:width) = sum of the heavy-tile edges of row r over the bf16 table(s) hi (+ lo): rows
// b_rows, b_cols columns, row stride b_ld elements.  Returns 0, or < 0 when a table cannot be mapped.
int spmm_tc(Launch L, const TileDev& T, const void* hi, const void* lo, int64_t b_cols, int64_t b_rows, int64_t b_ld,
            float* out, int64_t ld_out, int64_t width) {
  using namespace tcs;
  if (T.n_rb <= 0) return 0;
  const int NT = lo ? 2 : 1;
  const DevKnobs& kn = knobs();
  const int env_cap = kn.tc_spmm_bn;
  const int bn_cap = env_cap ? env_cap : (NT == 2 ? 128 : 256);
  Params p{};
  int64_t bn = (width + 63) / 64 * 64;
  if (bn > bn_cap) bn = bn_cap;
  p.BN = (int)bn;
  p.n_nt = (int)((width + bn - 1) / bn);
  p.n_rb = (int)T.n_rb;
  p.rb_ptr = T.rb_ptr;
  const int env_order = kn.tc_spmm_order;
  p.order = env_order ? T.order : nullptr;
  const int env_dbg = kn.tc_spmm_dbg;
  p.dbg = env_dbg;
  p.tile_col = T.tile_col;
  p.mask = T.mask;
  p.out = out;
  p.n_rows = T.n_rows;
  p.ld_out = ld_out;
  p.width = (int)width;
  const int env_nacc1 = kn.tc_spmm_nacc1, env_ts = kn.tc_spmm_ts, env_ctas = kn.tc_spmm_ctas;
  // The kernel is latency-bound (one chain TMA -> build -> MMA per stage), so two CTAs per SM (two
  // independent pipelines sharing the tensor core) beat one CTA with twice the stages: 2 CTAs x
  // (<= 104 KB of stages, one TMEM accumulator, <= 256 TMEM columns).  A in TMEM (TS) when the
  // accumulator leaves room for >= 2 A buffers of 32 columns, else A in shared memory (SS).
  int ctas = env_ctas == 1 ? 1 : 2, TS = 0, S = 0, smem_budget = 0, tmem_budget = 0;
  uint32_t stage = 0;
  for (;; ctas = 1) {  // two stages must fit next to a second CTA, else one CTA per SM
    smem_budget = ctas == 2 ? 104 * 1024 : 210 * 1024;
    tmem_budget = ctas == 2 ? 256 : 512;
    p.nacc = (ctas == 2 || env_nacc1) ? 1 : 2;
    TS = env_ts && p.nacc * p.BN + 32 * 2 <= tmem_budget;
    stage = stage_bytes(NT, p.BN, TS);
    S = (int)(smem_budget / stage);
    S = S > 8 ? 8 : S;
    if (TS)
      while (S > 2 && p.nacc * p.BN + 32 * S > tmem_budget) --S;
    if (S >= 2 || ctas == 1) break;
  }
  if (S < 2) S = 2;
  p.stages = S;
  p.tmem_cols = tmem_budget == 256 ? 256 : (TS ? 512 : tc_tmem_cols(p.BN));
  const size_t smem = 1024 + (size_t)p.stages * stage + (4 * p.stages + 4) * 8 + 16;
  const int env_box = kn.tc_spmm_box64;
  p.box64 = env_box ? 1 : 0;
  const int box_rows = p.box64 ? 64 : 32;
  if (!tc_map_table(&p.map_b[0], hi, true, b_cols, b_rows, b_ld, 64, box_rows)) return -1;
  if (NT == 2 && !tc_map_table(&p.map_b[1], lo, true, b_cols, b_rows, b_ld, 64, box_rows)) return -1;
  if (smem_attr_once((const void*)k_spmm_tc<1, 0>, 227 * 1024) || smem_attr_once((const void*)k_spmm_tc<2, 0>, 227 * 1024) ||
      smem_attr_once((const void*)k_spmm_tc<1, 1>, 227 * 1024) || smem_attr_once((const void*)k_spmm_tc<2, 1>, 227 * 1024))
    return -2;
  const int n_items = p.n_rb * p.n_nt;
  const int grid_cap = ctas * sm_count();
  const int grid = n_items < grid_cap ? n_items : grid_cap;
  if (NT == 2) {
    if (TS) k_spmm_tc<2, 1><<<grid, kThreads, smem, L.s>>>(p);
    else k_spmm_tc<2, 0><<<grid, kThreads, smem, L.s>>>(p);
  } else {
    if (TS) k_spmm_tc<1, 1><<<grid, kThreads, smem, L.s>>>(p);
    else k_spmm_tc<1, 0><<<grid, kThreads, smem, L.s>>>(p);
  }
  if (L.count) *L.count += 1;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace pgcn
