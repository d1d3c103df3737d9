// Node-update GEMMs of the GraphSAGE layer (S4 fwd, S6 dW, S7 dA) on the 5th-generation tensor
// cores: TMA-fed, tcgen05.mma with fp32 accumulators in TMEM, warp-specialised, persistent.
//
// Precision: "3xTF32" -- every fp32 operand x is split as x = hi + lo with hi = x truncated to
// tf32 (the raw fp32 word: kind::tf32 reads its top 19 bits) and lo = x - hi (exact), and
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi (kind::tf32, fp32 accumulate).  The dropped A_lo B_lo
// term and the truncation of lo are O(2^-20) relative, so the result is fp32-grade (the 1e-4
// parity tier of the north_star) while running on the tensor pipe.  Weights are pre-split
// (hi = rna_tf32(W), lo = rna_tf32(W - hi)) by k_wprep.
//
// Roles (384 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA issuer (one lane),
// warps 2-7 = converters (split fp32 tiles into hi/lo in shared memory, in the UMMA layout),
// warps 8-11 = epilogue (tcgen05.ld TMEM -> registers -> global; warp % 4 = its TMEM lane quarter).
// Pipelines: full[s] (TMA -> converters), conv[s] (converters -> MMA), empty[s] (MMA commit ->
// TMA), tfull[a] / tempty[a] (MMA <-> epilogue, two accumulator buffers in TMEM).
//
// Modes:
//   FWD : Y[m, n]   = sum_k [Z | D][m, k] W[k, n] + b[n]  (ReLU)   A K-major (2 segments),
//         B = W^T pre-split into hi/lo [N x 2Fp] K-major.
//   DA  : dA[m, hF+c] = sum_j M[m, j] W[hF + c, j]  (h = 0 scaled by inv_deg[m])  A = M K-major,
//         B = W pre-split [2F x Kp] K-major.
//   DW  : part[z][segF + f, n] = sum_{r in split z} A_s[r, f] M[r, n]   both operands MN-major
//         (row-major activations read "transposed"), both split by the converters.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "pgcn_dev.h"

#include "common.h"
#include "gemm_tc.cuh"
#include "tc_ptx.cuh"
#include "kernels.cuh"

namespace pgcn {
namespace tc {

// ------------------------------------------------------------------------------------------------ kernel
constexpr int kConvWarps = 6;                       // warps 2..7 split fp32 tiles into tf32 hi/lo
constexpr int kConvThreads = 32 * kConvWarps;
constexpr int kThreads = 64 + kConvThreads + 128;   // + TMA warp, MMA warp, 4 epilogue warps
constexpr int BM = 128;   // UMMA M (rows of A, TMEM lanes)
constexpr int BK = 32;    // fp32 elements per k-block = one 128-byte swizzle row

struct Tile {
  int m0, n0, kb_begin, kb_end, z, seg, half;
};

// Per-stage shared-memory geometry.  tf32 (BF = 0): A | A_lo | B | B_lo, k-block = 32 elements
// (FWD/DA) or 32 rows (DW).  bf16 (BF = 1): A_raw (fp32 as loaded) | A_bf16 | B (bf16 weights, or
// raw fp32 for DW) | B_bf16 (DW only); k-block = 64 elements (FWD/DA) or 32 rows (DW).
struct Geo {
  uint32_t a_raw, a_cvt, b_raw, b_cvt;
  __host__ __device__ uint32_t stage() const { return a_raw + a_cvt + b_raw + b_cvt; }
};
// DW with one f-tile of F <= 96 features stores only afeat (32 / 64 / 96) of the 128 A features per
// stage: the MMA still reads 128 (its last atoms overlap the next buffer of the stage) but those TMEM
// lanes are output rows >= F, never stored.  Smaller stages -> more of them in flight (the narrow dW of
// papers-shaped layers, 48 x 48, is latency-bound on bytes in flight).
__host__ __device__ inline Geo geometry(int bf, int mode, int BN, int afeat = BM, int kbw = BK) {
  Geo g;
  if (!bf) {
    const int af = mode == TC_DW ? afeat : BM;
    const int kw = kbw <= 0 ? BK : kbw;  // (DW: rows per k-block)
    g.a_raw = (uint32_t)af * kw * 4;
    g.a_cvt = (uint32_t)af * kw * 4;
    g.b_raw = (uint32_t)BN * kw * 4;
    g.b_cvt = (uint32_t)BN * kw * 4;
  } else if (mode == TC_DW) {
    g.a_raw = (uint32_t)afeat * 32 * 4;                // afeat features x 32 rows fp32
    g.a_cvt = (uint32_t)((afeat + 63) / 64) * 64 * 32 * 2;  // bf16 MN-major, 64-feature atoms
    g.b_raw = (uint32_t)BN * 32 * 4;
    g.b_cvt = (uint32_t)BN * 32 * 2;
  } else {
    g.a_raw = BM * 64 * 4;           // 128 rows x 64 k fp32 (two boxes)
    g.a_cvt = BM * 64 * 2;           // bf16 K-major, 128-byte rows
    g.b_raw = (uint32_t)BN * 64 * 2; // bf16 weights straight from TMA
    g.b_cvt = 0;
  }
  return g;
}

// FWD/DA: tile = (m-tile, n-tile), K loop over the A segments (FWD) or F_out (DA).
// DW: tile = (segment, split z, f-tile, n-tile); K loop = the split's row blocks of that segment.
__device__ __forceinline__ void decode(const TcParams& p, int t, Tile& T) {
  if (p.mode == TC_DW) {
    const int seg0 = p.Zseg[0] * p.n_ftiles * p.n_ntiles;  // segment-major, per-segment split counts
    T.seg = t < seg0 ? 0 : 1;
    int r = t - (T.seg ? seg0 : 0);
    const int nt = r % p.n_ntiles;
    r /= p.n_ntiles;
    const int ft = r % p.n_ftiles;
    T.z = r / p.n_ftiles;
    T.m0 = ft * BM;
    T.n0 = nt * p.BN;
    T.kb_begin = T.z * p.kb_per_split[T.seg];
    T.kb_end = min(T.kb_begin + p.kb_per_split[T.seg], p.kb_seg[T.seg]);
    if (T.kb_end < T.kb_begin) T.kb_end = T.kb_begin;
    T.half = 0;
  } else {
    const int nt = t % p.n_ntiles;
    const int mt = t / p.n_ntiles;
    T.m0 = mt * BM;
    T.z = 0;
    T.seg = 0;
    if (p.mode == TC_DA) {
      T.half = nt / p.n_ntiles_half;
      T.n0 = (nt % p.n_ntiles_half) * p.BN;
    } else {
      T.half = 0;
      T.n0 = nt * p.BN;
    }
    T.kb_begin = 0;
    T.kb_end = p.kb_seg[0] + (p.nseg > 1 ? p.kb_seg[1] : 0);
  }
}

// Bits 40..63 of SplitMix64(z) (dropout mask, reading R5); the output xorshift z ^ (z >> 31) does not
// touch them and is skipped.
__device__ __forceinline__ uint32_t smix_top24(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(z >> 40);
}

// PUSH (N2): the epilogue also stores the rows peers consume (p.push) -- a separate instantiation so the
// push loop's registers do not weigh on the launches without it.
template <int BF, int PUSH>
__global__ void __launch_bounds__(kThreads, 1) k_umma_gemm(const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int S = p.stages;
  const Geo geo = geometry(BF, p.mode, p.BN, p.a_feat, p.kbw);
  const int kw = p.kbw > 0 ? p.kbw : BK;  // tf32 FWD / DA k-block width (fp32 elements)
  const uint32_t a_bytes = geo.a_raw;
  const uint32_t b_bytes = geo.b_raw;
  const uint32_t stage_bytes = geo.stage();
  uint8_t* stA = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_bytes);
  uint64_t* full = bars;
  uint64_t* conv = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = bars + 3 * S + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * S + 4);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kConvThreads);
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
  const bool split_b = p.mode == TC_DW;

  if (warp == 0) {
    // ===================================================== TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        Tile T;
        decode(p, t, T);
        for (int kb = T.kb_begin; kb < T.kb_end; ++kb) {
          mbar_wait(&empty[s], ph ^ 1, 1);
          uint8_t* A = stA + (size_t)s * stage_bytes;
          uint8_t* B = A + geo.a_raw + geo.a_cvt;
          uint8_t* Blo = B + geo.b_raw;
          if (BF) {
            mbar_expect_tx(&full[s], geo.a_raw + geo.b_raw);
            if (p.mode == TC_DW) {
              const int r0 = kb * 32;
              for (int j = 0; j < p.a_feat / 32; ++j)
                tma_load_2d(A + j * 4096, &p.map_a[p.merged ? (j >> 1) : T.seg], &full[s],
                            p.merged ? 32 * (j & 1) : T.m0 + 32 * j, r0);
              for (int j = 0; j < p.BN / 32; ++j)
                tma_load_2d(B + j * 4096, &p.map_b[T.seg], &full[s], T.n0 + 32 * j, r0);
            } else if (p.mode == TC_FWD) {
              const int seg = kb < p.kb_seg[0] ? 0 : 1;
              const int kl = kb - (seg ? p.kb_seg[0] : 0);
              tma_load_2d(A, &p.map_a[seg], &full[s], kl * 64, T.m0);
              tma_load_2d(A + BM * 128, &p.map_a[seg], &full[s], kl * 64 + 32, T.m0);
              tma_load_2d(B, &p.map_b[0], &full[s], (p.kb_off_b[seg] + kl) * 64, T.n0);
            } else {  // TC_DA
              tma_load_2d(A, &p.map_a[0], &full[s], kb * 64, T.m0);
              tma_load_2d(A + BM * 128, &p.map_a[0], &full[s], kb * 64 + 32, T.m0);
              tma_load_2d(B, &p.map_b[0], &full[s], kb * 64, T.half * p.F + T.n0);
            }
          } else {
          const bool pb = split_b && ((p.pre_b >> T.seg) & 1), pa = p.mode == TC_DA && p.pre_a;
          mbar_expect_tx(&full[s], (pa ? 2 : 1) * a_bytes + (split_b && !pb ? b_bytes : 2 * b_bytes));
          if (p.mode == TC_DW) {  // atoms of 32 features x kw rows (128 kw bytes)
            const int r0 = kb * kw;
            const int ab = 128 * kw;
            for (int j = 0; j < p.a_feat / 32; ++j)
              tma_load_2d(A + j * ab, &p.map_a[p.merged ? (j >> 1) : T.seg], &full[s],
                          p.merged ? 32 * (j & 1) : T.m0 + 32 * j, r0);
            for (int j = 0; j < p.BN / 32; ++j) {
              tma_load_2d(B + j * ab, &p.map_b[T.seg], &full[s], T.n0 + 32 * j, r0);
              if (pb) tma_load_2d(Blo + j * ab, &p.map_lo[T.seg], &full[s], T.n0 + 32 * j, r0);
            }
          } else if (p.mode == TC_FWD) {
            const int seg = kb < p.kb_seg[0] ? 0 : 1;
            const int kl = kb - (seg ? p.kb_seg[0] : 0);
            tma_load_2d(A, &p.map_a[seg], &full[s], kl * kw, T.m0);
            const int kcol = p.kb_off_b[seg] * BK + kl * kw;  // (kb_off_b in 32-element units)
            tma_load_2d(B, &p.map_b[0], &full[s], kcol, T.n0);
            tma_load_2d(Blo, &p.map_b_lo, &full[s], kcol, T.n0);
          } else {  // TC_DA
            tma_load_2d(A, &p.map_a[0], &full[s], kb * kw, T.m0);
            if (pa) tma_load_2d(A + a_bytes, &p.map_lo[0], &full[s], kb * kw, T.m0);
            const int brow = T.half * p.F + T.n0;
            tma_load_2d(B, &p.map_b[0], &full[s], kb * kw, brow);
            tma_load_2d(Blo, &p.map_b_lo, &full[s], kb * kw, brow);
          }
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer
    if (lane == 0) {
      const uint32_t fmt = BF ? 1u : 2u;  // BF16 (kind::f16) or TF32 (kind::tf32) operands, F32 accumulators
      const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (p.mode == TC_DW ? (1u << 15) | (1u << 16) : 0u) |
                             ((uint32_t)(p.BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
        Tile T;
        decode(p, t, T);
        mbar_wait(&tempty[acc], acc_ph ^ 1, 2);
        tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * p.BN);
        uint32_t accum = 0;
        for (int kb = T.kb_begin; kb < T.kb_end; ++kb) {
          mbar_wait(&conv[s], ph, 3);
          tc_fence_after();
          const uint32_t A = smem_u32(stA + (size_t)s * stage_bytes);
          if (BF) {
            const uint32_t Ab = A + geo.a_raw, Bb = A + geo.a_raw + geo.a_cvt;
            if (p.mode == TC_DW) {  // bf16 MN-major SW128: 64-wide atoms 4 KB apart, 8-row groups 1 KB apart
              const uint32_t Bc = Bb + geo.b_raw;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                mma_bf16(d, make_desc(Ab + kk * 2048, 4096, 1024), make_desc(Bc + kk * 2048, 4096, 1024), idesc,
                         accum);
                accum = 1u;
              }
            } else {  // bf16 K-major SW128: k-step of 16 elements = 32 bytes
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                mma_bf16(d, make_desc(Ab + kk * 32, 16, 1024), make_desc(Bb + kk * 32, 16, 1024), idesc, accum);
                accum = 1u;
              }
            }
            tc_commit(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
            continue;
          }
          const uint32_t Alo = A + a_bytes, B = A + 2 * a_bytes, Blo = B + b_bytes;
          if (p.mode != TC_DW && kw == 16) {  // K-major SW64: 64-byte rows, 8-row groups 512 B apart, 2 k-steps
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint64_t ah = make_desc(A + kk * 32, 16, 512, 4), al = make_desc(Alo + kk * 32, 16, 512, 4);
              const uint64_t bh = make_desc(B + kk * 32, 16, 512, 4), bl = make_desc(Blo + kk * 32, 16, 512, 4);
              mma_tf32(d, ah, bh, idesc, accum);
              mma_tf32(d, ah, bl, idesc, 1u);
              mma_tf32(d, al, bh, idesc, 1u);
              accum = 1u;
            }
            tc_commit(&empty[s]);
            if (++s == S) { s = 0; ph ^= 1; }
            continue;
          }
          const int nk = p.mode == TC_DW ? kw / 8 : BK / 8;
          const uint32_t lbo = 128u * (uint32_t)kw;  // DW: MN-atom stride (32 features x kw rows)
#pragma unroll 4
          for (int kk = 0; kk < nk; ++kk) {
            uint64_t ah, al, bh, bl;
            if (p.mode == TC_DW) {  // MN-major: MN atoms lbo apart (LBO), 4-row k-groups 512 B apart (SBO)
              ah = make_desc(A + kk * 1024, lbo, 512, 1);
              al = make_desc(Alo + kk * 1024, lbo, 512, 1);
              bh = make_desc(B + kk * 1024, lbo, 512, 1);
              bl = make_desc(Blo + kk * 1024, lbo, 512, 1);
            } else {  // K-major: 8-row groups 1 KB apart (SBO); k-step = 32 bytes inside the swizzle row
              ah = make_desc(A + kk * 32, 16, 1024);
              al = make_desc(Alo + kk * 32, 16, 1024);
              bh = make_desc(B + kk * 32, 16, 1024);
              bl = make_desc(Blo + kk * 32, 16, 1024);
            }
            mma_tf32(d, ah, bh, idesc, accum);
            mma_tf32(d, ah, bl, idesc, 1u);
            mma_tf32(d, al, bh, idesc, 1u);
            accum = 1u;
          }
          tc_commit(&empty[s]);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tc_commit(&tfull[acc]);  // also for an empty K range: the epilogue then writes zeros
        if (++acc == 2) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp < 2 + kConvWarps) {
    // ===================================================== converters: x -> (hi, lo)
    const int ct = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      Tile T;
      decode(p, t, T);
      for (int kb = T.kb_begin; kb < T.kb_end; ++kb) {
        mbar_wait(&full[s], ph, 4);
        if (BF) {
          uint8_t* base = stA + (size_t)s * stage_bytes;
          if (p.mode == TC_DW) {
            // raw fp32 box jb (32 features x 32 rows, 128-byte rows, no swizzle) -> bf16 MN-major SW128:
            // chunk (atom a, row r, h) = features 64a + 8h .. +7 at a*4096 + r*128 + ((h ^ (r & 7)) << 4)
            for (int part = 0; part < 2; ++part) {
              const uint8_t* raw = part == 0 ? base : base + geo.a_raw + geo.a_cvt;
              uint8_t* cvt = part == 0 ? base + geo.a_raw : base + geo.a_raw + geo.a_cvt + geo.b_raw;
              const int nf = part == 0 ? p.a_feat : p.BN;
              const int nch = nf / 8, items = nch * 32;
              for (int i = ct; i < items; i += kConvThreads) {
                // chunk index fastest across a warp: its LDS.128s walk along 128-byte rows of the raw box
                // (a row-fastest order put 8 threads of a phase on one bank group, 8-way conflicts)
                const int hc = i % nch, r = i / nch;  // hc: 8-feature chunk index
                const float4* src = reinterpret_cast<const float4*>(raw + (hc >> 2) * 4096 + r * 128 + (hc & 3) * 32);
                const float4 x = src[0], y = src[1];
                uint4 o;
                o.x = pack_bf16(x.x, x.y); o.y = pack_bf16(x.z, x.w); o.z = pack_bf16(y.x, y.y); o.w = pack_bf16(y.z, y.w);
                const int a = hc >> 3, h = hc & 7;
                *reinterpret_cast<uint4*>(cvt + a * 4096 + r * 128 + ((h ^ (r & 7)) << 4)) = o;
              }
            }
          } else {
            // raw fp32 (two 32-column boxes, 128-byte rows, no swizzle) -> bf16 K-major SW128 rows
            const uint8_t* raw = base;
            uint8_t* cvt = base + geo.a_raw;
            for (int i = ct; i < BM * 8; i += kConvThreads) {
              const int r = i >> 3, j = i & 7;
              const float4* src = reinterpret_cast<const float4*>(raw + (j >> 2) * (BM * 128) + r * 128 + (j & 3) * 32);
              const float4 x = src[0], y = src[1];
              uint4 o;
              o.x = pack_bf16(x.x, x.y); o.y = pack_bf16(x.z, x.w); o.z = pack_bf16(y.x, y.y); o.w = pack_bf16(y.z, y.w);
              *reinterpret_cast<uint4*>(cvt + r * 128 + ((j ^ (r & 7)) << 4)) = o;
            }
          }
          fence_async_smem();
          mbar_arrive(&conv[s]);
          if (++s == S) { s = 0; ph ^= 1; }
          continue;
        }
        float4* A = reinterpret_cast<float4*>(stA + (size_t)s * stage_bytes);
        float4* Alo = A + a_bytes / 16;
#if PGCN_TF32_TRUNC_HI
        // (operands whose lo arrived by TMA -- p.pre_a / p.pre_b -- are not converted)
        if (!(p.mode == TC_DA && p.pre_a))
          for (int i = ct; i < (int)(a_bytes / 16); i += kConvThreads) {
            const float4 x = A[i];
            Alo[i] = make_float4(tf32_lo_trunc(x.x), tf32_lo_trunc(x.y), tf32_lo_trunc(x.z), tf32_lo_trunc(x.w));
          }
        if (split_b && !((p.pre_b >> T.seg) & 1)) {
          const float4* B = A + 2 * (a_bytes / 16);
          float4* Blo = A + 2 * (a_bytes / 16) + b_bytes / 16;
          for (int i = ct; i < (int)(b_bytes / 16); i += kConvThreads) {
            const float4 x = B[i];
            Blo[i] = make_float4(tf32_lo_trunc(x.x), tf32_lo_trunc(x.y), tf32_lo_trunc(x.z), tf32_lo_trunc(x.w));
          }
        }
#else
        for (int i = ct; i < (int)(a_bytes / 16); i += kConvThreads) {
          float4 x = A[i], h, l;
          h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
          h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
          h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
          h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
          A[i] = h;
          Alo[i] = l;
        }
        if (split_b) {
          float4* B = A + 2 * (a_bytes / 16);
          float4* Blo = B + b_bytes / 16;
          for (int i = ct; i < (int)(b_bytes / 16); i += kConvThreads) {
            float4 x = B[i], h, l;
            h.x = tf32_rna(x.x); l.x = tf32_rna(x.x - h.x);
            h.y = tf32_rna(x.y); l.y = tf32_rna(x.y - h.y);
            h.z = tf32_rna(x.z); l.z = tf32_rna(x.z - h.z);
            h.w = tf32_rna(x.w); l.w = tf32_rna(x.w - h.w);
            B[i] = h;
            Blo[i] = l;
          }
        }
#endif
        fence_async_smem();
        mbar_arrive(&conv[s]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else {
    // ===================================================== epilogue: TMEM -> registers -> global
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_ph = 0;
    for (int t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
      Tile T;
      decode(p, t, T);
      mbar_wait(&tfull[acc], acc_ph, 5);
      __syncwarp();
      tc_fence_after();
      const bool empty_k = T.kb_end <= T.kb_begin;
      const int row = T.m0 + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * p.BN);
      for (int c0 = 0; c0 < p.BN; c0 += 16) {
        uint32_t r[16];
        TMEM_LD16(tbase + c0, r);
        tmem_ld_wait();
        if (empty_k) {
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = 0u;
        }
        // 16 accumulator columns of this thread's row -> four float4 groups (16-byte aligned:
        // every output stride is a multiple of 4 floats and n0 + c0 a multiple of 16).
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
        if (p.epi == EPI_ACT) {
          if (row < p.M) {
            float* out = p.out + (int64_t)row * p.ld_out;
            const float* add = p.addend ? p.addend + (int64_t)row * p.ld_add : nullptr;
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const int n = T.n0 + c0 + 4 * g4;
              if (n >= p.ld_out) break;
              float4 o = make_float4(v[4 * g4], v[4 * g4 + 1], v[4 * g4 + 2], v[4 * g4 + 3]);
              if (n + 3 < p.N) {
                if (add) {
                  const float4 a4 = *reinterpret_cast<const float4*>(add + n);
                  o.x += a4.x; o.y += a4.y; o.z += a4.z; o.w += a4.w;
                }
                if (p.bias) {
                  o.x += p.bias[n]; o.y += p.bias[n + 1]; o.z += p.bias[n + 2]; o.w += p.bias[n + 3];
                }
                if (p.relu) {
                  o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f);
                }
              } else {
                float e[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  if (n + j < p.N) {
                    if (add) e[j] += add[n + j];
                    if (p.bias) e[j] += p.bias[n + j];
                    if (p.relu) e[j] = fmaxf(e[j], 0.f);
                  } else {
                    e[j] = 0.f;
                  }
                }
                o = make_float4(e[0], e[1], e[2], e[3]);
              }
              *reinterpret_cast<float4*>(out + n) = o;
              if constexpr (PUSH) push_f4(p.push, row, p.ld_out / 4, n / 4, o);  // N2: rows peers consume
            }
          }
        } else if (p.epi == EPI_MASK) {  // dropout backward of the layer input (R5)
          if (row < p.M) {
            float* out = p.out + (int64_t)row * p.ld_out;
            const uint64_t kr = ((uint64_t)p.key_base + (uint64_t)p.gid[row]) * (uint64_t)p.width;
            const float rs = p.rscale ? p.rscale[row] : 1.f;  // GCN-sym: d~_u^-1/2 (R26)
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const int n = T.n0 + c0 + 4 * g4;
              if (n >= p.ld_out) break;
              float e[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                float x = v[4 * g4 + j] * rs;
                if (n + j >= p.N) {
                  x = 0.f;
                } else if (p.mask_on) {
                  x = smix_top24((kr + (uint64_t)(n + j)) ^ p.seed) >= p.thr ? x * p.scale : 0.f;
                }
                e[j] = x;
              }
              const float4 o = make_float4(e[0], e[1], e[2], e[3]);
              *reinterpret_cast<float4*>(out + n) = o;
              if constexpr (PUSH) push_f4(p.push, row, p.ld_out / 4, n / 4, o);  // N2: boundary rows to owners
            }
          }
        } else if (p.epi == EPI_DA) {
          if (row < p.M) {
            float* out = p.out + (int64_t)row * p.ld_out + (int64_t)T.half * p.ld_half;
            const float sc = T.half == 0 ? p.inv_deg[row] : 1.f;
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const int c = T.n0 + c0 + 4 * g4;
              if (c >= p.ld_half) break;
              float e[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) e[j] = (c + j < p.F) ? v[4 * g4 + j] * sc : 0.f;
              *reinterpret_cast<float4*>(out + c) = make_float4(e[0], e[1], e[2], e[3]);
            }
          }
        } else {  // EPI_PART: dW partial of split z, row stride ld_out = round_up(N, 4)
          const int sg = p.merged ? (row >> 6) : T.seg, r = p.merged ? (row & 63) : row;  // merged: lanes 64+ = seg 1
          if (r < p.F) {
            float* out = p.out + ((int64_t)T.z * p.K_out + (int64_t)p.out_row_off[sg] + r) * p.ld_out;
#pragma unroll
            for (int g4 = 0; g4 < 4; ++g4) {
              const int n = T.n0 + c0 + 4 * g4;
              if (n >= p.ld_out) break;
              *reinterpret_cast<float4*>(out + n) =
                  make_float4(v[4 * g4], v[4 * g4 + 1], v[4 * g4 + 2], v[4 * g4 + 3]);
            }
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

// W prep: for layer weights W [ns F x N] (ns = 2 GraphSAGE [W_neigh; W_self], ns = 1 GCN-sym), write
// the tf32 hi/lo splits in the two TMA layouts used above: WT [N x ns Fp] (FWD operand B, K-major;
// segment s = cols [s Fp, s Fp + F)) and Wp [ns F x Kp] (DA operand B, K-major).
// WJ [F x ns Kq] (Kq = round_up(N, 32)): row f = [W_neigh[f, :] | W_self[f, :]] (GCN: W[f, :]), the
// B operand of the transform-first input gradient J = [Q | M] [W_neigh | W_self]^T (null to skip).
__global__ void k_wprep(const float* __restrict__ W, int F, int N, int Fp, int Kp, int Kq, int ns, float* WT_hi,
                        float* WT_lo, float* Wp_hi, float* Wp_lo, float* WJ_hi, float* WJ_lo) {
  const int64_t total_t = (int64_t)N * ns * Fp, total_p = (int64_t)ns * F * Kp;
  const int64_t total_j = WJ_hi ? (int64_t)F * ns * Kq : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total_t + total_p + total_j;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = 0.f;
    if (i >= total_t + total_p) {
      const int64_t j = i - total_t - total_p, f = j / (ns * Kq), k = j % (ns * Kq);
      const int seg = (int)(k / Kq), c = (int)(k % Kq);
      if (c < N) x = W[((int64_t)seg * F + f) * N + c];
      const float h = tf32_rna(x);
      WJ_hi[j] = h;
      WJ_lo[j] = tf32_rna(x - h);
    } else if (i < total_t) {
      const int64_t n = i / (ns * Fp), k = i % (ns * Fp);
      const int seg = (int)(k / Fp), f = (int)(k % Fp);
      if (f < F) x = W[((int64_t)seg * F + f) * N + n];
      const float h = tf32_rna(x);
      WT_hi[i] = h;
      WT_lo[i] = tf32_rna(x - h);
    } else {
      const int64_t j = i - total_t, r = j / Kp, c = j % Kp;
      if (c < N) x = W[r * N + c];
      const float h = tf32_rna(x);
      Wp_hi[j] = h;
      Wp_lo[j] = tf32_rna(x - h);
    }
  }
}

// bf16 operand copies of W [ns F x N] (RNE): WT [N x ns Fp] (FWD B), Wp [ns F x Kp] (DA B) and
// optionally WJ [F x ns Kq] (transform-first J), Fp/Kq multiples of 64 elements, Kp of 8.
__global__ void k_wprep_bf16(const float* __restrict__ W, int F, int N, int Fp, int Kp, int Kq, int ns,
                             __nv_bfloat16* WT, __nv_bfloat16* Wp, __nv_bfloat16* WJ) {
  const int64_t total_t = (int64_t)N * ns * Fp, total_p = (int64_t)ns * F * Kp;
  const int64_t total_j = WJ ? (int64_t)F * ns * Kq : 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total_t + total_p + total_j;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = 0.f;
    if (i >= total_t + total_p) {
      const int64_t j = i - total_t - total_p, f = j / (ns * Kq), k = j % (ns * Kq);
      const int seg = (int)(k / Kq), c = (int)(k % Kq);
      if (c < N) x = W[((int64_t)seg * F + f) * N + c];
      WJ[j] = __float2bfloat16_rn(x);
    } else if (i < total_t) {
      const int64_t n = i / (ns * Fp), k = i % (ns * Fp);
      const int seg = (int)(k / Fp), f = (int)(k % Fp);
      if (f < F) x = W[((int64_t)seg * F + f) * N + n];
      WT[i] = __float2bfloat16_rn(x);
    } else {
      const int64_t j = i - total_t, r = j / Kp, c = j % Kp;
      if (c < N) x = W[r * N + c];
      Wp[j] = __float2bfloat16_rn(x);
    }
  }
}

// db partial: part[z][row_off + n] = sum_{r in split z} M[r, n]  (fixed order; the bias row of
// the dW output, reduced over splits together with the tensor-core rows)
__global__ void k_colsum(const float* __restrict__ Mg, int64_t M, int64_t ld, int N, int64_t rps,
                         float* __restrict__ part, int64_t zstride, int64_t row_off) {
  __shared__ float sh[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rps, r1 = r0 + rps < M ? r0 + rps : M;
  float a = 0.f;
  if (n < N)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) a += Mg[r * ld + n];
  sh[threadIdx.y][threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float s = 0.f;
    for (int y = 0; y < 8; ++y) s += sh[y][threadIdx.x];
    part[(int64_t)blockIdx.y * zstride + row_off + n] = s;
  }
}

// Same partial with `sub` row chunks per split (more blocks for narrow N / few splits): chunk s of
// split z sums rows [z rps + s rpsub, ...) into scratch[(z sub + s) N + n]; k_colsum_fin then adds the
// sub partials of each split in ascending s (fixed order, deterministic).
__global__ void k_colsum_sub(const float* __restrict__ Mg, int64_t M, int64_t ld, int N, int64_t rps, int sub,
                             int64_t rpsub, float* __restrict__ scratch) {
  __shared__ float sh[8][33];
  const int n = blockIdx.x * 32 + threadIdx.x;
  const int z = blockIdx.y / sub, sc = blockIdx.y % sub;
  const int64_t zend = (int64_t)(z + 1) * rps < M ? (int64_t)(z + 1) * rps : M;
  const int64_t r0 = (int64_t)z * rps + (int64_t)sc * rpsub, r1 = r0 + rpsub < zend ? r0 + rpsub : zend;
  float a = 0.f;
  if (n < N)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) a += Mg[r * ld + n];
  sh[threadIdx.y][threadIdx.x] = a;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float s = 0.f;
    for (int y = 0; y < 8; ++y) s += sh[y][threadIdx.x];
    scratch[(int64_t)blockIdx.y * N + n] = s;
  }
}
__global__ void k_colsum_fin(const float* __restrict__ scratch, int sub, int N, int Zs, float* __restrict__ part,
                             int64_t zstride, int64_t row_off) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)Zs * N) return;
  const int z = (int)(i / N), n = (int)(i - (int64_t)z * N);
  float s = 0.f;
  for (int k = 0; k < sub; ++k) s += scratch[((int64_t)z * sub + k) * N + n];
  part[(int64_t)z * zstride + row_off + n] = s;
}

}  // namespace tc

// ------------------------------------------------------------------------------------------------ host side
namespace {
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}
}  // namespace

// swz: 0 none, 1 128B (K-major UMMA operands), 2 128B_ATOM_32B (tf32 MN-major operands), 3 64B (K-major
// tf32 operands in 16-element k-blocks).
static bool tc_map(CUtensorMap* m, const void* base, bool bf16, int64_t cols, int64_t rows, int64_t ld, int box_cols,
                   int box_rows, int swz) {
  EncodeFn f = encode_fn();
  if (!f || cols <= 0 || rows <= 0) return false;
  const size_t es_b = bf16 ? 2 : 4;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es_b};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapSwizzle sw = swz == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                         : (swz == 1 ? CU_TENSOR_MAP_SWIZZLE_128B
                                                     : (swz == 3 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B));
  return f(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
           dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tc_map_2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, int box_cols, int box_rows,
               bool mn_major) {
  return tc_map(m, base, false, cols, rows, ld, box_cols, box_rows, mn_major ? 2 : 1);
}

// Gathered table of the tensor-core SpMM (spmm_tc.cu): MN-major B operand boxes, fp32 with
// SWIZZLE_128B_ATOM_32B (tf32) or bf16 with SWIZZLE_128B.
bool tc_map_table(CUtensorMap* m, const void* base, bool bf16, int64_t cols, int64_t rows, int64_t ld, int box_cols,
                  int box_rows) {
  return tc_map(m, base, bf16, cols, rows, ld, box_cols, box_rows, bf16 ? 1 : 2);
}

int tc_stages(int BN, int bf, int mode, int afeat, int kbw) {
  const int stage = (int)tc::geometry(bf, mode, BN, afeat, kbw).stage();
  int S = (200 * 1024) / stage;
  const int cap = mode == TC_DW ? 8 : 4;  // dW: stream of 32-row k-blocks, latency-bound on bytes in flight
  return S > cap ? cap : (S < 2 ? 2 : S);
}

size_t tc_smem_bytes(int BN, int S, int bf, int mode, int afeat, int kbw) {
  const size_t stage = tc::geometry(bf, mode, BN, afeat, kbw).stage();
  return 1024 + S * stage + (3 * S + 4) * 8 + 16;
}

int tc_bn(int64_t N) {
  const int cap = knobs().tc_bnmax;  // dev knob PGCN_TC_BNMAX: cap the FWD/DA n-tile (A/B experiments)
  int64_t bn = (N + 15) / 16 * 16;
  if (bn > cap) bn = cap;
  if (bn < 16) bn = 16;
  return (int)bn;
}

int tc_tmem_cols(int BN) {
  int need = 2 * BN, c = 32;
  while (c < need) c *= 2;
  return c;
}

// Narrow forward / dA GEMMs (TMEM accumulators <= 256 columns, >= 2 stages in 104 KB) run two CTAs per
// SM: their pipelines are TMA-latency bound (memory-bound shapes: papers-shaped 48-wide layers), and
// two independent pipelines per SM hide more of it (papers-q forward GEMMs 18.9 -> 15.7 ms per step;
// the dW GEMM measured slower, its split-K plan fills 148-CTA waves).  Dev knob PGCN_TC_GEMM_CTAS=1.
static int gemm_ctas() { return knobs().tc_gemm_ctas; }
// dev knob PGCN_PRESPLIT=1: the engine allocates M_lo and the GEMMs load it (default 0, see engine.cu)
static bool presplit_enabled() { return knobs().presplit != 0; }

cudaError_t tc_launch(const TcParams& p0, cudaStream_t s, int sms) {
  if (smem_attr_once((const void*)tc::k_umma_gemm<0, 0>, 227 * 1024) ||
      smem_attr_once((const void*)tc::k_umma_gemm<1, 0>, 227 * 1024) ||
      smem_attr_once((const void*)tc::k_umma_gemm<0, 1>, 227 * 1024) ||
      smem_attr_once((const void*)tc::k_umma_gemm<1, 1>, 227 * 1024))
    return cudaErrorInvalidValue;
  TcParams p = p0;
  int ctas = 1;
  // (the PUSH instantiation needs > 85 registers per thread: one CTA of 384 threads per SM)
  // dW: its split-K plan is sized for sm_count() x PGCN_TC_DW_CTAS concurrent CTAs
  const bool two = p.mode == TC_DW ? knobs().tc_dw_ctas == 2 : gemm_ctas() == 2;
  if (two && p.tmem_cols <= 256 && !p.push.mode) {
    const size_t stage = tc::geometry(p.bf, p.mode, p.BN, p.a_feat, p.kbw).stage();
    int S = (int)((104 * 1024 - 1024 - 64) / stage);
    if (S >= 2) {
      p.stages = S < p.stages ? S : p.stages;
      ctas = 2;
    }
  }
  const size_t smem = tc_smem_bytes(p.BN, p.stages, p.bf, p.mode, p.a_feat, p.kbw);
  const int cap = ctas * sms;
  int grid = p.n_tiles < cap ? p.n_tiles : cap;
  if (grid < 1) return cudaSuccess;
  const bool push = p.push.mode != 0;
  if (p.bf) {
    if (push) tc::k_umma_gemm<1, 1><<<grid, tc::kThreads, smem, s>>>(p);
    else tc::k_umma_gemm<1, 0><<<grid, tc::kThreads, smem, s>>>(p);
  } else {
    if (push) tc::k_umma_gemm<0, 1><<<grid, tc::kThreads, smem, s>>>(p);
    else tc::k_umma_gemm<0, 0><<<grid, tc::kThreads, smem, s>>>(p);
  }
  return cudaGetLastError();
}

void tc_wprep_bf16(const float* W, int F, int N, int Fp, int Kp, int Kq, int ns, void* WT, void* Wp, void* WJ,
                   cudaStream_t s) {
  const int64_t total = (int64_t)N * ns * Fp + (int64_t)ns * F * Kp + (WJ ? (int64_t)F * ns * Kq : 0);
  int grid = (int)((total + 255) / 256);
  if (grid > sm_count() * 8) grid = sm_count() * 8;
  tc::k_wprep_bf16<<<grid, 256, 0, s>>>(W, F, N, Fp, Kp, Kq, ns, static_cast<__nv_bfloat16*>(WT),
                                        static_cast<__nv_bfloat16*>(Wp), static_cast<__nv_bfloat16*>(WJ));
}

void tc_wprep(const float* W, int F, int N, int Fp, int Kp, int Kq, int ns, float* WT_hi, float* WT_lo, float* Wp_hi,
              float* Wp_lo, float* WJ_hi, float* WJ_lo, cudaStream_t s) {
  const int64_t total = (int64_t)N * ns * Fp + (int64_t)ns * F * Kp + (WJ_hi ? (int64_t)F * ns * Kq : 0);
  int grid = (int)((total + 255) / 256);
  if (grid > sm_count() * 8) grid = sm_count() * 8;
  tc::k_wprep<<<grid, 256, 0, s>>>(W, F, N, Fp, Kp, Kq, ns, WT_hi, WT_lo, Wp_hi, Wp_lo, WJ_hi, WJ_lo);
}

// ---------------------------------------------------------------------------------------- mode wrappers
// bf = 1: bf16 operands (kind::f16; k-block 64 elements; B = bf16 weight copy, SW128); bf = 0: 3xTF32.
static void tc_common(TcParams& p, int BN, int bf, int mode) {
  p.BN = BN;
  p.bf = bf;
  if (!p.a_feat) p.a_feat = tc::BM;
  // 3xTF32 K-major modes: 16-element k-blocks -- half-size stages, twice as many in flight (256-wide n-tiles:
  // four 48 KB stages instead of two 96 KB ones; narrow n-tiles: enough stages for two CTAs per SM).
  // Dev knob PGCN_TC_BK16: 0 off, 1 n-tiles > 128 only, 2 (default) every n-tile (profiles/r2r_bk16.md)
  const int bk16 = knobs().tc_bk16;
  if (!bf && mode != TC_DW && (bk16 == 2 || (bk16 == 1 && BN > 128))) p.kbw = 16;
  // dW: 16-row k-blocks with dev knob PGCN_TC_DW16=1 (half-size stages; measured slower on every config:
  // the dW's bytes in flight do not change and the k-block count doubles -- profiles/r2r_bk16.md)
  if (!bf && mode == TC_DW && knobs().tc_dw16) p.kbw = 16;
  p.stages = tc_stages(BN, bf, mode, p.a_feat, p.kbw);
  p.tmem_cols = tc_tmem_cols(BN);
}

// dW reads activations "transposed" (MN-major): N tiles are whole swizzle atoms (32 fp32 / 64 bf16).
static int dw_bn(int64_t N, int bf) {
  const int64_t atom = bf ? 64 : 32;
  int64_t bn = (N + atom - 1) / atom * atom;
  const int64_t cap = bf ? 256 : knobs().tc_dw_bnmax;  // (dev knob PGCN_TC_DW_BNMAX, 3xTF32 A/B tests)
  return (int)(bn > cap ? cap : bn);
}

// Split-K plan of the dW GEMM: each of the n_seg segments (row counts kb_s k-blocks of 32 rows) is cut
// into Z_s splits so that every tile (segment, split, f-tile, n-tile) carries about the same number of
// k-blocks and the tile count fits W whole waves of the 148-CTA persistent grid (W = 1..3, the cheapest
// by "W x largest tile + per-tile overhead").  Balancing per segment matters for transform-first layers,
// whose two segments have n_all and n_in rows.
constexpr int kDwMaxWaves = 3;
constexpr int kColsumSub = 16;  // max row chunks per split of the bias-row column sums
static int dw_base(int64_t F, int64_t N) { return (int)(((F + 127) / 128) * ((N + dw_bn(N, 0) - 1) / dw_bn(N, 0))); }
// Longest accumulation chain of one dW tile, in k-blocks of 32 rows (dev knob PGCN_DW_KMAX; 0 = none;
// default 128).  The tensor core's fp32 accumulation does not round to nearest, so its error grows with
// the chain length instead of averaging out.  Measured on B200 against fp64 (tools/r2/dw_chain.py,
// 13.9M x 48 x 48, 3xTF32): chains of 2935 / 1024 / 256 / 64 k-blocks -> 1.2e-3 / 2.0e-4 / 6.2e-5 /
// 1.5e-5 relative error, at 4.84 / 5.04 / 5.09 / 6.08 ms; Reddit's 116K-row dW is unaffected (2.2e-5).
// Splitting long reductions into more tiles (summed in fp32 round-to-nearest by the fixed-order second
// pass) keeps every chain short.
static int64_t dw_kmax() { return knobs().dw_kmax; }
static int64_t zmin_for(int64_t kb) {
  const int64_t km = dw_kmax();
  return km > 0 ? std::max<int64_t>(1, (kb + km - 1) / km) : 1;
}
static void dw_plan(int64_t kb0, int64_t kb1, int nseg, int base, int Z[2], int slots_sm) {
  const int64_t ovh = 6;  // per-tile fill / drain, in k-block units
  int64_t best = INT64_MAX;
  const int64_t zm0 = zmin_for(kb0), zm1 = nseg > 1 ? zmin_for(kb1) : 0;
  Z[0] = (int)zm0;
  Z[1] = (int)zm1;
  if ((zm0 + zm1) * base > (int64_t)kDwMaxWaves * slots_sm) return;  // chains cap the split count
  for (int W = 1; W <= kDwMaxWaves; ++W) {
    const int slots = W * slots_sm / base;
    if (slots < nseg) continue;
    const int lo = 1, hi = nseg > 1 ? slots - 1 : slots;
    for (int z0 = lo; z0 <= hi; ++z0) {
      int64_t a = z0 < kb0 ? z0 : (kb0 > 0 ? kb0 : 1);
      int64_t b = nseg > 1 ? (slots - z0 < kb1 ? slots - z0 : (kb1 > 0 ? kb1 : 1)) : 0;
      if (a < zm0 || (nseg > 1 && b < zm1)) continue;
      const int64_t kpt = std::max((kb0 + a - 1) / a, nseg > 1 ? (kb1 + b - 1) / b : (int64_t)0);
      const int64_t waves = ((a + b) * base + slots_sm - 1) / slots_sm;
      const int64_t cost = waves * (kpt + ovh);
      if (cost < best) {
        best = cost;
        Z[0] = (int)a;
        Z[1] = (int)b;
      }
    }
  }
}

int64_t tc_dw_ws_floats(int64_t M, int64_t F, int64_t N) {
  int64_t Z = kDwMaxWaves * sm_count() * knobs().tc_dw_ctas / dw_base(F, N);
  const int64_t kb = (M + 31) / 32;
  if (Z > kb) Z = kb;
  Z = std::max(Z, zmin_for(kb));
  if (Z < 1) Z = 1;
  return Z * (2 * F + 1) * ((N + 3) / 4 * 4) + Z * kColsumSub * N;  // + the bias-row sub partials
}

// FWD-mode launch with 1 or 2 K-major A segments sharing one pre-converted B operand copy
// (tf32: hi/lo fp32 [N x ldB]; bf16: [N x ldB] bf16).  kb_off in k-blocks of the variant.
static int launch_fwd(Launch L, int nseg, const float* const* A, const int64_t* rowsA, int64_t ldA, int64_t K,
                      const void* B_hi, const void* B_lo, int64_t ldB, const int* kb_off, int64_t M, int64_t N,
                      TcParams& p, int bf) {
  const int BN = tc_bn(N);
  tc_common(p, BN, bf, TC_FWD);
  bool ok;
  const int kw = p.kbw > 0 ? p.kbw : 32, sw = kw == 16 ? 3 : 1;  // tf32 k-block width and its swizzle
  if (bf) ok = tc_map(&p.map_b[0], B_hi, true, ldB, N, ldB, 64, BN, 1);
  else
    ok = tc_map(&p.map_b[0], B_hi, false, ldB, N, ldB, kw, BN, sw) && tc_map(&p.map_b_lo, B_lo, false, ldB, N, ldB, kw, BN, sw);
  for (int s = 0; s < nseg && ok; ++s)
    ok = tc_map(&p.map_a[s], A[s], false, K, rowsA[s] > 0 ? rowsA[s] : 1, ldA, bf ? 32 : kw, 128, bf ? 0 : sw);
  if (!ok) return -1;
  const int kbk = bf ? 64 : kw;
  p.mode = TC_FWD;
  p.nseg = nseg;
  for (int s = 0; s < nseg; ++s) {
    p.kb_seg[s] = (int)((K + kbk - 1) / kbk);
    p.kb_off_b[s] = kb_off[s];
  }
  p.n_ntiles = (int)((N + BN - 1) / BN);
  p.n_tiles = (int)((M + 127) / 128) * p.n_ntiles;
  p.M = (int)M;
  p.N = (int)N;
  if (L.count) *L.count += 1;
  return tc_launch(p, L.s, sm_count()) == cudaSuccess ? 0 : -2;
}

int64_t tc_kpad(int64_t K, int bf) { return bf ? (K + 63) / 64 * 64 : (K + 31) / 32 * 32; }

int gemm_fwd_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const void* WT_hi,
                const void* WT_lo, const float* bias, int64_t N, float* Y, int64_t ldY, int relu, int bf,
                const PushSpec* push) {
  if (M <= 0) return 0;
  TcParams p{};
  if (push) p.push = *push;
  const int64_t Fp = tc_kpad(F, bf);
  const float* A[2] = {Z, D};
  const int64_t rows[2] = {M, M};
  const int off[2] = {0, (int)(Fp / (bf ? 64 : 32))};
  p.epi = EPI_ACT;
  p.ld_out = ldY;
  p.out = Y;
  p.bias = bias;
  p.relu = relu;
  return launch_fwd(L, 2, A, rows, ldA, F, WT_hi, WT_lo, 2 * Fp, off, M, N, p, bf);
}

int tc_fwd_1seg(Launch L, const float* A, int64_t M, int64_t ldA, int64_t K, const void* WT_hi, const void* WT_lo,
                int64_t ldB, int kb_off, int64_t N, float* out, int64_t ld_out, const float* bias,
                const float* addend, int64_t ld_add, int relu, int bf, const PushSpec* push) {
  if (M <= 0) return 0;
  TcParams p{};
  if (push) p.push = *push;
  const float* As[1] = {A};
  const int64_t rows[1] = {M};
  const int off[1] = {kb_off};
  p.epi = EPI_ACT;
  p.ld_out = ld_out;
  p.out = out;
  p.bias = bias;
  p.addend = addend;
  p.ld_add = ld_add;
  p.relu = relu;
  return launch_fwd(L, 1, As, rows, ldA, K, WT_hi, WT_lo, ldB, off, M, N, p, bf);
}

int tc_fwd_mask(Launch L, const float* Q, int64_t M, const float* Mg, int64_t M_inner, int64_t ld, int64_t K,
                const void* WJ_hi, const void* WJ_lo, int64_t Kq, int64_t F, float* J, int64_t ldJ,
                const int64_t* gid, const DropSpec& d, int bf, const float* rscale, const PushSpec* push) {
  if (M <= 0) return 0;
  TcParams p{};
  if (push) p.push = *push;
  const float* A[2] = {Q, Mg};
  const int64_t rows[2] = {M, M_inner};
  const int off[2] = {0, (int)(Kq / (bf ? 64 : 32))};
  p.epi = EPI_MASK;
  p.ld_out = ldJ;
  p.out = J;
  p.gid = gid;
  p.seed = d.seed;
  p.key_base = d.key_base;
  p.thr = d.thr;
  p.scale = d.scale;
  p.width = d.width;
  p.mask_on = d.on;
  p.rscale = rscale;
  const int64_t ldB = Mg ? 2 * Kq : Kq;  // GCN-sym: one segment (Mg == nullptr), B = WJ [F x Kq]
  if (M_inner <= 0 || !Mg) return launch_fwd(L, 1, A, rows, ld, K, WJ_hi, WJ_lo, ldB, off, M, F, p, bf);
  return launch_fwd(L, 2, A, rows, ld, K, WJ_hi, WJ_lo, ldB, off, M, F, p, bf);
}

int gemm_da_tc(Launch L, const float* Mg, int64_t ldM, int64_t M, int64_t N, const void* Wp_hi, const void* Wp_lo,
               int64_t Kp, int64_t F, const float* inv_deg, float* dA, int64_t ld, int bf, int halves,
               const float* Mlo) {
  if (M <= 0) return 0;
  if (halves != 1 && halves != 2) return -1;
  TcParams p{};
  const int BN = tc_bn(F);
  tc_common(p, BN, bf, TC_DA);
  const int kw = p.kbw > 0 ? p.kbw : 32, sw = kw == 16 ? 3 : 1;  // tf32 k-block width and its swizzle
  bool ok = tc_map(&p.map_a[0], Mg, false, N, M, ldM, bf ? 32 : kw, 128, bf ? 0 : sw);
  p.pre_a = !bf && Mlo && PGCN_TF32_TRUNC_HI && presplit_enabled();
  if (p.pre_a) ok = ok && tc_map(&p.map_lo[0], Mlo, false, N, M, ldM, kw, 128, sw);
  if (bf) ok = ok && tc_map(&p.map_b[0], Wp_hi, true, N, halves * F, Kp, 64, BN, 1);
  else
    ok = ok && tc_map(&p.map_b[0], Wp_hi, false, N, halves * F, Kp, kw, BN, sw) &&
         tc_map(&p.map_b_lo, Wp_lo, false, N, halves * F, Kp, kw, BN, sw);
  if (!ok) return -1;
  p.mode = TC_DA;
  p.epi = EPI_DA;
  p.nseg = 1;
  p.n_ntiles_half = (int)((F + BN - 1) / BN);
  p.n_ntiles = halves * p.n_ntiles_half;
  p.n_tiles = (int)((M + 127) / 128) * p.n_ntiles;
  p.kb_seg[0] = (int)((N + (bf ? 64 : kw) - 1) / (bf ? 64 : kw));
  p.M = (int)M;
  p.N = (int)N;
  p.F = (int)F;
  p.ld_out = halves * ld;
  p.ld_half = ld;
  p.out = dA;
  p.inv_deg = inv_deg;
  if (L.count) *L.count += 1;
  return tc_launch(p, L.s, sm_count()) == cudaSuccess ? 0 : -2;
}

int tc_dw_general(Launch L, const float* A0, const float* B0, int64_t rows0, const float* A1, const float* B1,
                  int64_t rows1, int64_t ldA, int64_t ldB, int64_t F, int64_t N, const float* Mb, int64_t rowsMb,
                  float* G, float* ws, int64_t ws_floats, int bf, const float* B0lo, const float* B1lo) {
  const int nseg = A1 ? 2 : 1;  // GCN-sym: G = [A0^T B0 ; colsum(Mb)]
  if (!A1) rows1 = 0;
  const int64_t K = nseg * F + 1;
  const int64_t rmax = rows0 > rows1 ? rows0 : rows1;
  if (rmax <= 0) {
    cudaMemsetAsync(G, 0, sizeof(float) * K * N, L.s);
    return 0;
  }
  TcParams p{};
  const int BN = dw_bn(N, bf);
  // Two segments over the same rows and the same B (aggregate-first GraphSAGE: [Z | D]^T M) with F <= 64
  // share one 128-row M tile: B (M) is streamed once instead of once per segment and the k-block loop
  // runs once (papers-shaped 48-wide layers).
  p.merged = nseg == 2 && rows0 == rows1 && B0 == B1 && F <= 64 && knobs().dw_merge;
  p.a_feat = p.merged ? tc::BM : (F <= 96 ? (int)((F + 31) / 32 * 32) : tc::BM);
  tc_common(p, BN, bf, TC_DW);
  // PGCN_TC_DW_CTAS=2 (default): the split plan fills waves of 2 x sm_count() CTAs, and tc_launch runs two
  // CTAs per SM where their accumulators and two stages each fit (narrow n-tiles).  The finer split pays
  // even where one CTA runs (products-shaped 128-wide dW: 5.06 -> 4.45 ms per step; r2x / r2y)
  const int slots_sm = sm_count() * knobs().tc_dw_ctas;
  int Zseg[2];
  if (p.merged) {
    dw_plan((rows0 + 31) / 32, 0, 1, dw_base(F, N), Zseg, slots_sm);
    Zseg[1] = Zseg[0];
  } else {
    dw_plan((rows0 + 31) / 32, (rows1 + 31) / 32, nseg, dw_base(F, N), Zseg, slots_sm);
  }
  const int Zs = std::max(Zseg[0], Zseg[1]);
  const int64_t NP = (N + 3) / 4 * 4;  // partial row stride (16-byte aligned epilogue stores)
  if ((int64_t)Zs * K * NP > ws_floats) return -3;
  const float* As[2] = {A0, A1};
  const float* Bs[2] = {B0, B1};
  const int64_t rows[2] = {rows0, rows1};
  const float* Blos[2] = {B0lo, B1lo};
  const int kr = bf ? 32 : (p.kbw > 0 ? p.kbw : 32);  // rows per k-block (3xTF32: 16 with PGCN_TC_DW16)
  bool ok = true;
  for (int s = 0; s < nseg && ok; ++s) {
    ok = tc_map(&p.map_a[s], As[s], false, F, rows[s] > 0 ? rows[s] : 1, ldA, 32, kr, bf ? 0 : 2) &&
         tc_map(&p.map_b[s], Bs[s], false, N, rows[s] > 0 ? rows[s] : 1, ldB, 32, kr, bf ? 0 : 2);
    if (ok && !bf && Blos[s] && PGCN_TF32_TRUNC_HI && presplit_enabled()) {
      ok = tc_map(&p.map_lo[s], Blos[s], false, N, rows[s] > 0 ? rows[s] : 1, ldB, 32, kr, 2);
      p.pre_b |= 1 << s;
    }
  }
  if (!ok) return -1;
  p.mode = TC_DW;
  p.epi = EPI_PART;
  p.nseg = p.merged ? 1 : nseg;
  p.Z = Zs;
  for (int s = 0; s < nseg; ++s) {
    p.Zseg[s] = Zseg[s];
    // the split plan is in 32-row k-blocks; the kernel walks kr-row k-blocks (same row ranges per split)
    const int64_t kb32 = (rows[s] + 31) / 32;
    int64_t kps = (kb32 + Zseg[s] - 1) / Zseg[s];
    if (kps < 1) kps = 1;
    p.kb_seg[s] = (int)((rows[s] + kr - 1) / kr);
    p.kb_per_split[s] = (int)(kps * (32 / kr));
    p.out_row_off[s] = (int)(s * F);
  }
  p.n_ftiles = (int)((F + 127) / 128);
  p.n_ntiles = (int)((N + BN - 1) / BN);
  p.n_tiles = (Zseg[0] + (nseg > 1 && !p.merged ? Zseg[1] : 0)) * p.n_ftiles * p.n_ntiles;
  p.M = (int)rmax;
  p.N = (int)N;
  p.F = (int)F;
  p.K_out = (int)K;
  p.ld_out = NP;
  p.out = ws;
  if (tc_launch(p, L.s, sm_count()) != cudaSuccess) return -2;
  // bias row: colsum of Mb in the same Z splits (rows per split = a multiple of 32)
  const int64_t kbb = (rowsMb + 31) / 32;
  const int64_t rps = ((kbb + Zs - 1) / Zs) * 32;
  dim3 block(32, 8), grid((unsigned)((N + 31) / 32), (unsigned)Zs);
  // narrow N / few splits leave most SMs idle: split each split's rows into `sub` chunks (>= 4 blocks per
  // SM in total) with a fixed-order second pass, when the workspace has room for the sub partials
  int sub = (int)((4 * sm_count() + (int64_t)grid.x * Zs - 1) / ((int64_t)grid.x * Zs));
  sub = sub > kColsumSub ? kColsumSub : sub;
  const int64_t room = ws_floats - (int64_t)Zs * K * NP;
  while (sub > 1 && (int64_t)Zs * sub * N > room) --sub;
  const int64_t rpsub = ((rps + sub - 1) / sub + 7) / 8 * 8;  // sub chunks cover the split
  if (rowsMb > 0 && sub > 1) {
    float* scratch = ws + (int64_t)Zs * K * NP;
    tc::k_colsum_sub<<<dim3(grid.x, (unsigned)(Zs * sub)), block, 0, L.s>>>(Mb, rowsMb, ldB, (int)N,
                                                                           rps > 0 ? rps : 32, sub, rpsub, scratch);
    const int64_t tot = (int64_t)Zs * N;
    tc::k_colsum_fin<<<(unsigned)((tot + 255) / 256), 256, 0, L.s>>>(scratch, sub, (int)N, Zs, ws, K * NP,
                                                                      nseg * F * NP);
    if (L.count) *L.count += 1;
  } else if (rowsMb > 0) {
    tc::k_colsum<<<grid, block, 0, L.s>>>(Mb, rowsMb, ldB, (int)N, rps > 0 ? rps : 32, ws, K * NP, nseg * F * NP);
  } else {
    for (int z = 0; z < Zs; ++z) cudaMemsetAsync(ws + z * K * NP + nseg * F * NP, 0, sizeof(float) * N, L.s);
  }
  const int64_t zc[3] = {Zseg[0], nseg > 1 ? Zseg[1] : 0, Zs};  // splits of rows [0,F), [F,2F), bias row
  split_reduce_dw(L, ws, zc, F, nseg, N, NP, G);
  if (L.count) *L.count += 2;
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

int gemm_dw_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* Mg,
               int64_t ldM, int64_t N, float* G, float* ws, int64_t ws_floats, int bf, const float* Mlo) {
  return tc_dw_general(L, Z, Mg, M, D, Mg, M, ldA, ldM, F, N, Mg, M, G, ws, ws_floats, bf, Mlo, Mlo);
}

}  // namespace pgcn

// ------------------------------------------------------------------------------------------------ diagnostics ABI
namespace {
int64_t r256(int64_t b) { return (b + 255) / 256 * 256; }
}  // namespace

extern "C" size_t pgcn_dev_gemm_scratch_bytes(int64_t M, int64_t F, int64_t N) {
  const int64_t Fp = (F + 63) / 64 * 64, Kp = (N + 7) / 8 * 8;  // covers the tf32 and bf16 layouts
  int64_t ws = pgcn::tc_dw_ws_floats(M, F, N);
  const int64_t ws2 = pgcn::gemm_dw_ws_floats(M, F, N);
  if (ws2 > ws) ws = ws2;
  return (size_t)(2 * r256(4 * N * 2 * Fp) + 2 * r256(4 * 2 * F * Kp) + r256(4 * ws));
}

extern "C" int pgcn_dev_gemm(int32_t op, int32_t variant, const float* A0, const float* A1, int64_t ldA, int64_t M,
                             int64_t F, const float* W, int64_t N, const float* Mg, int64_t ldM, const float* inv_deg,
                             float* out, int64_t ld_out, int32_t relu, void* scratch, size_t scratch_bytes,
                             void* stream) {
  using namespace pgcn;
  if (op < 0 || op > 2 || variant < 0 || variant > 2) return fail(PGCN_EINVAL, "pgcn_dev_gemm: bad op/variant");
  if (!out || !W || M < 0 || F < 1 || N < 1) return fail(PGCN_EINVAL, "pgcn_dev_gemm: bad shape/pointer");
  if (scratch_bytes < pgcn_dev_gemm_scratch_bytes(M, F, N)) return fail(PGCN_ENOMEM, "pgcn_dev_gemm: scratch too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t Fp = (F + 31) / 32 * 32, Kp = (N + 3) / 4 * 4;
  char* base = static_cast<char*>(scratch);
  float* WT_hi = reinterpret_cast<float*>(base);
  float* WT_lo = reinterpret_cast<float*>(base + r256(4 * N * 2 * Fp));
  float* Wp_hi = reinterpret_cast<float*>(base + 2 * r256(4 * N * 2 * Fp));
  float* Wp_lo = reinterpret_cast<float*>(base + 2 * r256(4 * N * 2 * Fp) + r256(4 * 2 * F * Kp));
  float* ws = reinterpret_cast<float*>(base + 2 * r256(4 * N * 2 * Fp) + 2 * r256(4 * 2 * F * Kp));
  const int64_t ws_floats = (int64_t)(scratch_bytes - (size_t)(2 * r256(4 * N * 2 * Fp) + 2 * r256(4 * 2 * F * Kp))) / 4;
  Launch L{s, nullptr};
  int rc = 0;
  if (variant == 0) {
    if (op != 1) tc_wprep(W, (int)F, (int)N, (int)Fp, (int)Kp, 0, 2, WT_hi, WT_lo, Wp_hi, Wp_lo, nullptr, nullptr, s);
    if (op == 0) rc = gemm_fwd_tc(L, A0, A1, ldA, M, F, WT_hi, WT_lo, W + 2 * F * N, N, out, ld_out, relu, 0);
    else if (op == 1) rc = gemm_dw_tc(L, A0, A1, ldA, M, F, Mg, ldM, N, out, ws, ws_floats, 0);
    else rc = gemm_da_tc(L, Mg, ldM, M, N, Wp_hi, Wp_lo, Kp, F, inv_deg, out, ld_out / 2, 0, 2);
  } else if (variant == 1) {
    const int64_t Fb = (F + 63) / 64 * 64, Kb = (N + 7) / 8 * 8;
    if (op != 1) tc_wprep_bf16(W, (int)F, (int)N, (int)Fb, (int)Kb, 0, 2, WT_hi, Wp_hi, nullptr, s);
    if (op == 0) rc = gemm_fwd_tc(L, A0, A1, ldA, M, F, WT_hi, nullptr, W + 2 * F * N, N, out, ld_out, relu, 1);
    else if (op == 1) rc = gemm_dw_tc(L, A0, A1, ldA, M, F, Mg, ldM, N, out, ws, ws_floats, 1);
    else rc = gemm_da_tc(L, Mg, ldM, M, N, Wp_hi, nullptr, Kb, F, inv_deg, out, ld_out / 2, 1, 2);
  } else {
    if (op == 0) gemm_fwd_f32(L, A0, A1, ldA, M, F, W, N, out, ld_out, relu);
    else if (op == 1) gemm_dw_f32(L, A0, A1, ldA, M, F, Mg, ldM, N, out, ws, ws_floats);
    else gemm_da_f32(L, Mg, ldM, M, N, W, F, inv_deg, out, ld_out / 2);
  }
  if (rc) return fail(PGCN_ECUDA, "pgcn_dev_gemm: tensor-core path failed (%d)", rc);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PGCN_ECUDA, "pgcn_dev_gemm: %s", cudaGetErrorString(e));
  return PGCN_OK;
}
