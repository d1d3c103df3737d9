// tcgen05 (5th-gen tensor core) GEMMs of the GraphSAGE node update -- see gemm_tc.cu.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "push.cuh"

namespace pgcn {

enum { TC_FWD = 0, TC_DA = 1, TC_DW = 2 };
enum { EPI_ACT = 0, EPI_DA = 1, EPI_MASK = 2, EPI_PART = 3 };

struct alignas(64) TcParams {
  CUtensorMap map_a[2], map_b[2], map_b_lo;
  int mode, epi, BN, stages, tmem_cols;
  int nseg, kb_seg[2], kb_off_b[2], kb_per_split[2], Zseg[2];
  int n_tiles, n_ntiles, n_ntiles_half, n_ftiles, Z;
  int M, N, F, K_out;
  int out_row_off[2];
  int64_t ld_out, ld_half, ld_add;
  float* out;
  const float* bias;
  const float* inv_deg;
  const float* addend;
  int relu;
  const int64_t* gid;
  uint64_t seed, key_base;
  uint32_t thr;
  float scale;
  int width, mask_on;
  const float* rscale;  // EPI_MASK: optional per-row scale (GCN-sym d~^-1/2)
  PushSpec push;        // EPI_ACT / EPI_MASK: N2 fused push of the rows peers consume (mode 0: off)
  int bf;  // 1: bf16 operands (kind::f16), 0: 3xTF32 (kind::tf32)
  int a_feat;  // DW: A features stored per stage (32 / 64 / 96 / 128; see geometry()); other modes 128
  int merged;  // DW with two segments over the same rows and operand B, F <= 64: one M tile holds both
               // (A atoms 0-1 = segment 0's features, 2-3 = segment 1's; TMEM lanes 0-63 / 64-127)
  // 3xTF32 operands whose lo = x - trunc_tf32(x) was written by their producer (the loss / the stale-
  // gradient accumulate write M and M_lo): TMA loads lo from map_lo instead of the converter warps
  // computing it once per tile that reads the operand.  pre_a: DA's A (M); pre_b: bit s = DW segment s's B.
  CUtensorMap map_lo[2];
  int pre_a, pre_b;
  // 3xTF32 FWD / DA: fp32 elements per k-block, 32 (one 128-byte SW128 row; 0 = 32) or 16 (one 64-byte SW64
  // row): half-size stages, twice as many in flight, for the 256-wide n-tiles whose 96 KB stages fit twice
  int kbw;
};

bool tc_map_2d(CUtensorMap* m, const float* base, int64_t cols, int64_t rows, int64_t ld, int box_cols, int box_rows,
               bool mn_major = false);
bool tc_map_table(CUtensorMap* m, const void* base, bool bf16, int64_t cols, int64_t rows, int64_t ld, int box_cols,
                  int box_rows);
int tc_stages(int BN, int bf, int mode, int afeat, int kbw = 32);
size_t tc_smem_bytes(int BN, int S, int bf, int mode, int afeat, int kbw = 32);
void tc_wprep_bf16(const float* W, int F, int N, int Fp, int Kp, int Kq, int ns, void* WT, void* Wp, void* WJ,
                   cudaStream_t s);
int tc_bn(int64_t N);
int tc_tmem_cols(int BN);
cudaError_t tc_launch(const TcParams& p, cudaStream_t s, int sms);
// W [ns F x N] (ns = 2 GraphSAGE, 1 GCN-sym) -> tf32 hi/lo operand copies: WT [N x ns Fp] (FWD B),
// Wp [ns F x Kp] (DA B), optionally WJ [F x ns Kq] (transform-first input-gradient B; null to skip).
void tc_wprep(const float* W, int F, int N, int Fp, int Kp, int Kq, int ns, float* WT_hi, float* WT_lo, float* Wp_hi,
              float* Wp_lo, float* WJ_hi, float* WJ_lo, cudaStream_t s);
struct Launch;
struct DropSpec;
// Mode wrappers (return 0 on success, < 0 if the shape could not be mapped / launched).
int64_t tc_dw_ws_floats(int64_t M, int64_t F, int64_t N);
// K padded to whole k-blocks of the variant (32 for 3xTF32, 64 for bf16)
int64_t tc_kpad(int64_t K, int bf);
// Node-update GEMMs; bf = 0: 3xTF32 (B operand copies are tf32 hi/lo fp32 arrays), bf = 1: bf16
// (B operand copy is bf16, *_lo unused).  Return 0 on success, < 0 on mapping / launch failure.
int gemm_fwd_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const void* WT_hi,
                const void* WT_lo, const float* bias, int64_t N, float* Y, int64_t ldY, int relu, int bf,
                const PushSpec* push = nullptr);
// dA = Mg W^T; halves = 2: [dZ' | dD] (GraphSAGE, first half scaled by inv_deg, row stride 2 ld),
// halves = 1: inv_deg o (Mg W^T) (GCN-sym, row stride ld).
// Mlo (optional, 3xTF32 only): the producer-written lo = x - trunc_tf32(x) of Mg, same layout.
int gemm_da_tc(Launch L, const float* Mg, int64_t ldM, int64_t M, int64_t N, const void* Wp_hi, const void* Wp_lo,
               int64_t Kp, int64_t F, const float* inv_deg, float* dA, int64_t ld, int bf, int halves,
               const float* Mlo = nullptr);
int gemm_dw_tc(Launch L, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F, const float* Mg,
               int64_t ldM, int64_t N, float* G, float* ws, int64_t ws_floats, int bf, const float* Mlo = nullptr);
// Transform-before-aggregate pieces (N1: P(DW) = (PD)W for F_out < F_in):
//   out[M x N] = act(A[M x K] W_seg^T + addend + bias), W_seg = W_neigh (kb_off 0) or W_self
//   (kb_off = Fp / k-block) read from the WT operand copy (ldB = 2Fp columns).
int tc_fwd_1seg(Launch L, const float* A, int64_t M, int64_t ldA, int64_t K, const void* WT_hi, const void* WT_lo,
                int64_t ldB, int kb_off, int64_t N, float* out, int64_t ld_out, const float* bias,
                const float* addend, int64_t ld_add, int relu, int bf, const PushSpec* push = nullptr);
//   J[M x F] = mask o s o rscale o ([Q | Mg] [W_neigh | W_self]^T), Q rows M, Mg rows M_inner (rows
//   beyond are zero), B = WJ [F x 2Kq]; mask / gid / key per DropSpec (R5).  GCN-sym: Mg = nullptr,
//   J = mask o s o rscale o (Q W^T) with B = WJ [F x Kq]; rscale (per row) may be null.
int tc_fwd_mask(Launch L, const float* Q, int64_t M, const float* Mg, int64_t M_inner, int64_t ld, int64_t K,
                const void* WJ_hi, const void* WJ_lo, int64_t Kq, int64_t F, float* J, int64_t ldJ,
                const int64_t* gid, const DropSpec& d, int bf, const float* rscale, const PushSpec* push = nullptr);
//   G[(2F+1) x N] = [A0^T B0 ; A1^T B1 ; colsum(Mb)], A_s/B_s over their own row counts;
//   A1 == nullptr: G[(F+1) x N] = [A0^T B0 ; colsum(Mb)] (GCN-sym).
//   B0lo / B1lo (optional, 3xTF32): producer-written lo of B0 / B1.
int tc_dw_general(Launch L, const float* A0, const float* B0, int64_t rows0, const float* A1, const float* B1,
                  int64_t rows1, int64_t ldA, int64_t ldB, int64_t F, int64_t N, const float* Mb, int64_t rowsMb,
                  float* G, float* ws, int64_t ws_floats, int bf, const float* B0lo = nullptr,
                  const float* B1lo = nullptr);

}  // namespace pgcn
