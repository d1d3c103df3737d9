// SpMM tile-reuse lab (diagnostics only): Z[v] = inv[v] * sum_{u in N(v)} D[u] for 256-wide rows with
// the edges of each 128-row block split into "heavy" 64-column tiles (processed tile-synchronously by
// all 16 warps of the CTA so the tile's 64 KB of D is reused from L1 or shared memory) and "light"
// leftover edges (plain gathers).  MODE 0: heavy tiles read through L1 (ld.global); MODE 1: each heavy
// tile is staged into shared memory with cp.async.bulk (double buffered) and read from there.
// Measured on the Reddit-shaped partition (tools/spmm_tile_lab.py, B200): fwd 3.82 -> 3.43 ms,
// transposed 3.67 -> 3.04 ms (mode 1) vs the product row kernel -- ~1.1-1.2x, not integrated
// (DESIGN.md "SpMM").  Caching the column bytes in registers per warp made it slower.
#include <cuda_runtime.h>

#include <cstdint>

namespace {
constexpr int R = 128, C = 64, WARPS = 16, RPW = R / WARPS;  // 8 rows per warp

__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1)
k_tiled(const int32_t* __restrict__ blk_tile_ptr, const int32_t* __restrict__ tile_col0, const int32_t* __restrict__ tile_off,
        const uint8_t* __restrict__ tile_col, const int64_t* __restrict__ light_ptr, const int32_t* __restrict__ light_col,
        const float* __restrict__ inv, const float4* __restrict__ D, int64_t n_rows, int64_t n_cols, float4* __restrict__ Z,
        unsigned long long* work) {
  extern __shared__ __align__(128) float4 sm[];  // MODE 1: 2 x 64 rows x 64 float4
  __shared__ long long s_blk;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n_blk = (n_rows + R - 1) / R;
  if (MODE == 1 && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase[2] = {0, 0};
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_blk = (long long)atomicAdd(work, 1ull);
    __syncthreads();
    const long long blk = s_blk;
    __syncthreads();
    if (blk >= n_blk) break;
    float4 acc[RPW][2];
#pragma unroll
    for (int r = 0; r < RPW; ++r) acc[r][0] = acc[r][1] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int t0 = blk_tile_ptr[blk], t1 = blk_tile_ptr[blk + 1];
    auto issue = [&](int t, int buf) {
      const int64_t c0 = tile_col0[t];
      const int64_t rows = (c0 + C <= n_cols) ? C : (n_cols - c0);
      const uint32_t bytes = (uint32_t)(rows * 64 * 16);
      const uint32_t b = smem_u32(&bar[buf]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(sm + buf * C * 64)),
                   "l"(D + c0 * 64), "r"(bytes), "r"(b)
                   : "memory");
    };
    if (MODE == 1 && threadIdx.x == 0 && t0 < t1) issue(t0, 0);
    for (int t = t0; t < t1; ++t) {
      const int buf = (t - t0) & 1;
      const float4* src_base;
      if (MODE == 1) {
        if (threadIdx.x == 0 && t + 1 < t1) issue(t + 1, buf ^ 1);
        const uint32_t b = smem_u32(&bar[buf]);
        uint32_t done = 0;
        while (!done)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(done)
                       : "r"(b), "r"(phase[buf])
                       : "memory");
        phase[buf] ^= 1;
        src_base = sm + buf * C * 64;
      } else {
        src_base = D + (int64_t)tile_col0[t] * 64;
      }
      const int32_t* off = tile_off + (int64_t)t * (R + 1) + warp * RPW;
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int e0 = off[r], e1 = off[r + 1];
        int e = e0;
        for (; e + 4 <= e1; e += 4) {
          float4 v[4][2];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float4* s = src_base + (int)tile_col[e + u] * 64;
            v[u][0] = s[lane];
            v[u][1] = s[lane + 32];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            acc[r][0] = add4(acc[r][0], v[u][0]);
            acc[r][1] = add4(acc[r][1], v[u][1]);
          }
        }
        for (; e < e1; ++e) {
          const float4* s = src_base + (int)tile_col[e] * 64;
          acc[r][0] = add4(acc[r][0], s[lane]);
          acc[r][1] = add4(acc[r][1], s[lane + 32]);
        }
      }
      __syncthreads();  // all warps done with this tile (buffer reuse / L1 locality)
    }
    // light edges: plain gathers
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int64_t row = blk * R + warp * RPW + r;
      if (row >= n_rows) continue;
      const int64_t e0 = light_ptr[row], e1 = light_ptr[row + 1];
      int64_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        float4 v[4][2];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float4* s = D + (int64_t)light_col[e + u] * 64;
          v[u][0] = __ldg(s + lane);
          v[u][1] = __ldg(s + lane + 32);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[r][0] = add4(acc[r][0], v[u][0]);
          acc[r][1] = add4(acc[r][1], v[u][1]);
        }
      }
      for (; e < e1; ++e) {
        const float4* s = D + (int64_t)light_col[e] * 64;
        acc[r][0] = add4(acc[r][0], __ldg(s + lane));
        acc[r][1] = add4(acc[r][1], __ldg(s + lane + 32));
      }
      const float sc = inv[row];
      Z[row * 64 + lane] = make_float4(acc[r][0].x * sc, acc[r][0].y * sc, acc[r][0].z * sc, acc[r][0].w * sc);
      Z[row * 64 + lane + 32] = make_float4(acc[r][1].x * sc, acc[r][1].y * sc, acc[r][1].z * sc, acc[r][1].w * sc);
    }
  }
}
}  // namespace

extern "C" int lab_tiled(int mode, const int32_t* blk_tile_ptr, const int32_t* tile_col0, const int32_t* tile_off,
                         const uint8_t* tile_col, const int64_t* light_ptr, const int32_t* light_col, const float* inv,
                         const float* D, int64_t n_rows, int64_t n_cols, float* Z, unsigned long long* work,
                         void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(work, 0, 8, s);
  const size_t smem = mode == 1 ? 2 * C * 64 * 16 : 0;
  if (mode == 1) {
    cudaFuncSetAttribute(k_tiled<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_tiled<1><<<148, WARPS * 32, smem, s>>>(blk_tile_ptr, tile_col0, tile_off, tile_col, light_ptr, light_col, inv,
                                            reinterpret_cast<const float4*>(D), n_rows, n_cols,
                                            reinterpret_cast<float4*>(Z), work);
  } else {
    k_tiled<0><<<148 * 2, WARPS * 32, 0, s>>>(blk_tile_ptr, tile_col0, tile_off, tile_col, light_ptr, light_col, inv,
                                             reinterpret_cast<const float4*>(D), n_rows, n_cols,
                                             reinterpret_cast<float4*>(Z), work);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
