// tcgen05 (5th-gen tensor core) GEMMs of the GraphSAGE node update -- see gemm_tc.cu.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace pgcn {

enum { TC_FWD = 0, TC_DA = 1, TC_DW = 2 };

struct alignas(64) TcParams {
  CUtensorMap map_a0, map_a1, map_b, map_b_lo;
  int mode, BN, stages, tmem_cols;
  int n_tiles, n_ntiles, n_ntiles_half, n_ftiles, n_seg;
  int kb_total, kb_seg0, kb_per_split;
  int M, N, F, K_out;
  int64_t ld_out, ld_half;
  float* out;
  const float* bias;
  const float* inv_deg;
  int relu;
};

bool tc_map_2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, int box_cols, int box_rows,
               bool mn_major = false);
int tc_stages(int BN);
size_t tc_smem_bytes(int BN, int S);
int tc_bn(int64_t N);
int tc_tmem_cols(int BN);
cudaError_t tc_launch(const TcParams& p, cudaStream_t s, int sms);
void tc_wprep(const float* W, int F, int N, int Fp, int Kp, float* WT_hi, float* WT_lo, float* Wp_hi, float* Wp_lo,
              cudaStream_t s);
struct Launch;
// Mode wrappers (return 0 on success, < 0 if the shape could not be mapped / launched).
int64_t tc_dw_ws_floats(int64_t M, int64_t F, int64_t N);
int gemm_fwd_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* WT_hi,
                const float* WT_lo, const float* bias, int64_t N, float* Y, int64_t ldY, int relu);
int gemm_da_tc(Launch L, const float* Mg, int64_t ldM, int64_t M, int64_t N, const float* Wp_hi, const float* Wp_lo,
               int64_t Kp, int64_t F, const float* inv_deg, float* dA, int64_t ld);
int gemm_dw_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* Mg,
               int64_t ldM, int64_t N, float* G, float* ws, int64_t ws_floats);

}  // namespace pgcn
