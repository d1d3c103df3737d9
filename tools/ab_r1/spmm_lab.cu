// SpMM design lab (diagnostics only, not linked into libpgcn.so): parameterised variants of the
// row-gather aggregation Z[v] = inv_deg[v] * sum_{u in N(v)} D[u], timed from tools/spmm_lab.py.
//   item = (row, chunk): a group of G lanes owns NC*G float4 columns of one row, U neighbour rows
//   in flight per step.  POLICY 0 = default caching, 1 = L2 evict_last on feature loads.
#include <cuda_runtime.h>

#include <cstdint>

namespace {
__device__ __forceinline__ float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

template <int G>
__device__ __forceinline__ unsigned gmask() {
  if (G == 32) return 0xffffffffu;
  return ((1u << G) - 1u) << ((threadIdx.x & 31u) & ~(unsigned)(G - 1));
}

template <int POLICY>
__device__ __forceinline__ float4 ldf(const float4* p, uint64_t pol) {
  if (POLICY == 1) {
    float4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
  }
  return __ldg(p);
}

template <int G, int NC, int U, int POLICY, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmm(const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                    const float* __restrict__ inv, const float4* __restrict__ D,
                                                    int64_t ld4, int64_t n_rows, int nchunk, float4* __restrict__ Z) {
  uint64_t pol = 0;
  if (POLICY == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const int lane = threadIdx.x % G;
  const unsigned gm = gmask<G>();
  const int64_t n_items = n_rows * nchunk;
  const int64_t stride = (int64_t)gridDim.x * (blockDim.x / G);
  for (int64_t it = (int64_t)blockIdx.x * (blockDim.x / G) + threadIdx.x / G; it < n_items; it += stride) {
    const int64_t row = it / nchunk;
    const int64_t x0 = (it - row * nchunk) * (NC * G) + lane;
    float4 acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t beg = rp[row], end = rp[row + 1];
    for (int64_t e0 = beg; e0 < end; e0 += G) {
      const int cnt = (int)((end - e0) < G ? (end - e0) : G);
      const int my = lane < cnt ? __ldg(col + e0 + lane) : 0;
      int j = 0;
      for (; j + U <= cnt; j += U) {
        float4 v[U][NC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = __shfl_sync(gm, my, j + u, G);
          const float4* src = D + (int64_t)c * ld4 + x0;
#pragma unroll
          for (int q = 0; q < NC; ++q)
            v[u][q] = (x0 + q * G < ld4) ? ldf<POLICY>(src + q * G, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < NC; ++q) acc[q] = add4(acc[q], v[u][q]);
      }
      for (; j < cnt; ++j) {
        const int c = __shfl_sync(gm, my, j, G);
        const float4* src = D + (int64_t)c * ld4 + x0;
#pragma unroll
        for (int q = 0; q < NC; ++q)
          if (x0 + q * G < ld4) acc[q] = add4(acc[q], ldf<POLICY>(src + q * G, pol));
      }
    }
    const float s = inv[row];
#pragma unroll
    for (int q = 0; q < NC; ++q)
      if (x0 + q * G < ld4) Z[row * ld4 + x0 + q * G] = make_float4(acc[q].x * s, acc[q].y * s, acc[q].z * s, acc[q].w * s);
  }
}

template <int G, int NC, int U, int POLICY, int MINB>
int run(const int64_t* rp, const int32_t* col, const float* inv, const float* D, int64_t ld, int64_t n_rows, float* Z,
        int grid_mult, cudaStream_t s) {
  const int64_t ld4 = ld / 4;
  const int nchunk = (int)((ld4 + NC * G - 1) / (NC * G));
  int64_t items = n_rows * nchunk;
  int64_t blocks = (items + (256 / G) - 1) / (256 / G);
  const int64_t cap = (int64_t)148 * grid_mult;
  if (blocks > cap) blocks = cap;
  k_spmm<G, NC, U, POLICY, MINB><<<(int)blocks, 256, 0, s>>>(rp, col, inv, reinterpret_cast<const float4*>(D), ld4,
                                                             n_rows, nchunk, reinterpret_cast<float4*>(Z));
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
}  // namespace

#define V(ID, G, NC, U, P, MB) \
  case ID: return run<G, NC, U, P, MB>(rp, col, inv, D, ld, n_rows, Z, grid_mult, s);

extern "C" int lab_spmm(int variant, const int64_t* rp, const int32_t* col, const float* inv, const float* D, int64_t ld,
                        int64_t n_rows, float* Z, int grid_mult, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (variant) {
    V(0, 32, 5, 1, 0, 1)   // round-1 original: whole row per warp
    V(1, 32, 5, 2, 0, 1)
    V(2, 32, 1, 8, 0, 4)   // current: 128-float chunks
    V(3, 32, 2, 4, 0, 4)
    V(4, 32, 2, 8, 0, 2)
    V(5, 32, 3, 4, 0, 2)
    V(6, 32, 1, 16, 0, 2)
    V(7, 32, 1, 8, 1, 4)   // + evict_last
    V(8, 32, 2, 4, 1, 4)
    V(9, 32, 5, 1, 1, 1)
    V(10, 32, 1, 4, 0, 8)
    V(11, 32, 2, 2, 0, 8)
    V(12, 16, 1, 8, 0, 4)
    V(13, 32, 3, 2, 0, 4)
    default: return -2;
  }
}
extern "C" int lab_n_variants() { return 14; }
