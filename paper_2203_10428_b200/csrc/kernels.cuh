// Launchers of the sm_100a kernels of the PipeGCN hot path (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pgcn.h"
#include "push.cuh"

namespace pgcn {

// Rows [off[s], off[s+1]) of a gathered block come from base[s] + row_map[r] * ld.
struct SegTable {
  const float* base[PGCN_MAX_PARTS];
  int64_t off[PGCN_MAX_PARTS + 1];
  int32_t n_seg;
};

// Dropout of one layer input (reading R5): keep iff (SplitMix64(key ^ seed) >> 40) >= thr,
// key = (key_base + gid) * width + col, key_base = (t (L+1) + l) N.
struct DropSpec {
  uint64_t seed;
  uint64_t key_base;
  uint32_t thr;
  float scale;
  int32_t width;
  int32_t on;
};

// Launch counter (per context) incremented by every launcher.
struct Launch {
  cudaStream_t s;
  int64_t* count;
  // optional sub-interval timing (engine, pgcn_timing_*): mark(mctx, kind, begin, flops, bytes) brackets the
  // tensor-core tile part of an aggregation launch (kind PGCN_K_SPMM_TILE_FWD / _BWD)
  void (*mark)(void* mctx, int kind, int begin, double flops, double bytes) = nullptr;
  void* mctx = nullptr;
};

// Device copy of a dense-tile decomposition (tiles.h) of an SpMM pattern.
struct TileDev {
  const int32_t* rb_ptr = nullptr;
  const int32_t* order = nullptr;
  const int32_t* tile_col = nullptr;
  const uint64_t* mask = nullptr;
  const int64_t* lrp = nullptr;   // light CSR (columns ascending within a row)
  const int32_t* lcol = nullptr;
  int64_t n_rows = 0, n_cols = 0, n_rb = 0, n_tiles = 0, nnz_light = 0;
};
// Heavy-tile sums on the tensor cores (spmm_tc.cu): out[r, 0:width) = sum over the heavy-tile edges
// (r, c) of B[c, 0:width), B = hi (+ lo when non-null): bf16 tables of b_rows rows, row stride b_ld
// elements (fp32 tier: the hi/lo split of the fp32 table; bf16 tier: the rounded table).  0 on success.
int spmm_tc(Launch L, const TileDev& T, const void* hi, const void* lo, int64_t b_cols, int64_t b_rows, int64_t b_ld,
            float* out, int64_t ld_out, int64_t width);

// S3 prologue: D = dropout(H) over rows [0, n_rows); rows >= n_valid are written as 0.
// rs (optional, per row): D[r] *= rs[r] (GCN-sym prescale by d~^-1/2, R26); with d.on == 0 a plain
// (row-scaled) copy.
void dropout_fwd(Launch, const float* H, float* D, int64_t ld, int64_t n_rows, int64_t n_valid,
                 const int64_t* gid, const DropSpec& d, const float* rs = nullptr);

// S3: Z[v] = inv_deg[v] * sum_{e in row v} D[col[e]]   (neighbours >= n_valid contribute 0)
// work: per-launch atomic item counter (8 bytes of device scratch) for dynamic row scheduling,
// or nullptr for static grid-stride.
// GCN-sym (R26): self = 1 adds the row's own D[v] (A + I); inv_deg then holds d~_v^-1/2.
// bias (optional, n_bias entries): Z = act(Z + b) epilogue (relu = ReLU), fusing the node update of
// a transform-first GCN layer.  n_cols: rows of D (neighbour ids < n_cols); -1 = unknown (ids are
// then checked against n_valid on every edge).
int spmm_fwd(Launch, const int64_t* row_ptr, const int32_t* col, const float* inv_deg,
              const float* D, int64_t ld, int64_t n_rows, int64_t n_valid, float* Z, unsigned long long* work,
              int self = 0, const float* bias = nullptr, int64_t n_bias = 0, int relu = 0, int64_t n_cols = -1,
              void* g16 = nullptr, const int32_t* rows = nullptr, int64_t nnz = -1, const TileDev* tiles = nullptr,
              void* t16 = nullptr, int compact = 0);
// rows (optional): aggregate only the n_rows rows listed (local ids; N1(ii) train-row-sparse last
// layer); the other output rows are left untouched.  compact: output row k of the list goes to Z[k].
// dmap (spmm_bwd, optional): dDs of inner row u is row dmap[u] of dDs (-1: none) -- compact train rows.

// S8: J[u] = mask_u * s * ( [u < n_in] dDs[u] + sum_{v in T(u)} dZs[v] ),  u in [0, n_all)
//     dZs = inv_deg-scaled dZ (first half of dA), dDs = second half; both stride ld_dA.
//     rs (optional, GCN-sym R26): the sum is scaled by rs[u] = d~_u^-1/2 before the mask (dDs = dZs
//     then realises the self loop).
int spmm_bwd(Launch, const int64_t* t_row_ptr, const int32_t* t_col, const float* dZs,
              const float* dDs, int64_t ld_dA, int64_t n_in, int64_t n_all, float* J, int64_t ld,
              const int64_t* gid, const DropSpec& d, unsigned long long* work, const float* rs = nullptr,
              void* g16 = nullptr, int64_t nnz = -1, const TileDev* tiles = nullptr, void* t16 = nullptr,
              const int32_t* dmap = nullptr, const PushSpec* push = nullptr);
// Both SpMMs return 0, or a PGCN_E* code (message set) when a launch cannot be made.
// tiles (both SpMMs, optional): dense-tile decomposition of the pattern (tiles.h); its heavy tiles are
// summed by spmm_tc into the output rows first and the gather kernel walks only the light CSR, adding
// the tile sums (fwd: used only when n_valid >= n_cols and rows == nullptr).  t16 (fp32 tier with tiles):
// scratch for the bf16 hi/lo split of the table, 2 x (table rows) x round_up(ld, 8) bf16.
// nnz (both SpMMs): edges the launch visits (sizes the dynamic scheduler's grabs); -1 = one row per grab.
// g16 (both SpMMs): bf16 gather tier (pgcn_config.gather = 1) -- scratch of at least
// (rows of the gathered table) x round_up(ld, 8) bf16; the table is rounded to bf16 there first and
// the kernel gathers the bf16 rows (fp32 accumulation, fp32 output).  nullptr = fp32 gathers.

// N1(ii) train-row-sparse last layer.  From the train mask of the n_in inner rows: tr_list = inner ids
// with train != 0 (ascending) and *tr_count; and the transposed CSR restricted to train sources:
// t_row_ptr_tr[u] / t_col_tr keep, in order, the entries v of P_i^T row u with train[v] != 0.  tmp:
// device scratch of train_rows_tmp_bytes(n_in, n_all) bytes; counts[n_all + 1] int64 scratch.
size_t train_rows_tmp_bytes(int64_t n_in, int64_t n_all);
void build_train_rows(Launch, const uint8_t* train, int64_t n_in, const int64_t* t_row_ptr, const int32_t* t_col,
                      int64_t n_all, int32_t* tr_list, int64_t* tr_count, int64_t* counts, int64_t* t_row_ptr_tr,
                      int32_t* t_col_tr, void* tmp, size_t tmp_bytes);

// Compact train rows of the last layer (N1(ii)): dst[map[r]] = src[r]; pos[v] = index of v in list (or
// -1) and cols[e] = pos[cols[e]] in place; dst[k] = src[list[k]] for rows of w bytes.
void scatter_rows(Launch, const float* src, const int32_t* map, int64_t n, int64_t ld, float* dst);
void compact_train_setup(Launch, const int32_t* list, int64_t n_tr, int64_t n_in, int32_t* pos, int32_t* cols,
                         int64_t n_cols);
void gather_bytes(Launch, const void* src, const int32_t* list, int64_t n, int64_t w, void* dst);

// N4 diagnostics: out[0] += sum_{r < n_rows, c < F} (used(r, c) - fresh(r, c))^2 with fresh rows from a
// segment table (row_map fmap) and used rows from a segment table (umap), a plain array, or 0.
void stale_err(Launch, const SegTable& fresh, const int32_t* fmap, const SegTable* used_tab, const int32_t* umap,
               const float* used, int64_t n_rows, int64_t ld, int64_t F, double* out);

// out[v] = s[v] * M[v] over n rows of stride ld
void scale_rows(Launch, const float* M, const float* s, int64_t n, int64_t ld, float* out);

// S1 / S2: dst[r] = src(r) (copy) or EMA: dst[r] = first ? src : gamma*prev[r] + (1-gamma)*src.
void gather_rows(Launch, const SegTable& src, const int32_t* row_map, int64_t n_rows, int64_t ld,
                 float* dst, const float* prev, float gamma, int ema, int first);

// S9 + M: J[v] += sum_{k in inv(v)} C_hat[k] (ascending k; C_hat = message or its EMA, state in
// ema[k]); M[v] = J[v] o 1[Hprev[v] > 0].  msg may have n_seg == 0 (nothing received).
// msg16: the message rows are bf16 (halo_payload = 1; 4 bf16 per float4 of the row, row stride ld).
void grad_reduce(Launch, const int64_t* inv_ptr, const int32_t* inv_pos, const SegTable& msg,
                 const int32_t* row_map, float* ema, float gamma, int use_ema, int first, float* J,
                 int write_j, const float* Hprev, float* M, int64_t n_in, int64_t ld, int msg16 = 0,
                 float* Mlo = nullptr);

// bf16 exchange payloads (pgcn_config.halo_payload = 1).  Rows of ld bf16 (ld % 4 == 0).
// pack:    dst[r] = bf16_rn(src[row_map ? row_map[r] : r])                     (S2 / S10 pack)
// install: dst[r] = widen(src[r]), or EMA gamma * prev[r] + (1 - gamma) * widen(src[r])   (S1)
void pack_rows_bf16(Launch, const float* src, const int32_t* row_map, int64_t n_rows, int64_t ld, void* dst);
void install_bf16(Launch, const void* src, int64_t n_rows, int64_t ld, float* dst, const float* prev, float gamma,
                  int ema);
// Delay injection: one thread spinning `ns` nanoseconds on stream s (not counted as a launch).
void spin_ns(cudaStream_t s, int64_t ns);

// S5: CE (labels int32) or BCE (labels uint8 [n x C]) on rows with train[v] != 0 (train == nullptr:
// every row is a train row).
// M = J^(L) (zero outside the train set), row_loss[v] = loss term of v (already / n_train).
// Mlo (optional; also grad_reduce): M's 3xTF32 lo term, x - trunc_tf32(x), for the GEMMs that read M.
// rows (optional): only the listed rows (the train row list; n = its length), row_loss[k] for the k-th --
// the caller zero-fills M elsewhere.
void loss_rows(Launch, int kind, const float* Y, int64_t n, int64_t C, int64_t ld, const void* labels,
               const uint8_t* train, double n_train, float* M, float* row_loss, float* Mlo = nullptr,
               const int32_t* rows = nullptr);
// out[0] = sum of x[0..n) (single block, fixed order -> deterministic)
void reduce_sum(Launch, const float* x, int64_t n, float* out);

// GEMMs (fp32 SIMT, parity path).  A_ext = [Z | D | 1] (K = 2F + 1), W_ext = [W; b].
// fwd: Y = A_ext W_ext, ReLU if relu, written to Y (ldY) rows [0, M), padding cols zeroed.
void gemm_fwd_f32(Launch, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F,
                  const float* Wext, int64_t N, float* Y, int64_t ldY, int relu);
// dW: G[(2F+1) x N] = A_ext^T Mg  (split over rows into ws[splits][(2F+1) N], fixed-order reduce)
void gemm_dw_f32(Launch, const float* Z, const float* D, int64_t ldA, int64_t M, int64_t F,
                 const float* Mg, int64_t ldM, int64_t N, float* G, float* ws, int64_t ws_floats);
int64_t gemm_dw_ws_floats(int64_t M, int64_t F, int64_t N);
// G[i] = sum_{s < splits} part[s * len + i]  (ascending s)
void split_reduce(Launch, const float* part, int64_t splits, int64_t len, float* G);
// G[r * N + c] = sum_s part[s][r * NP + c] over rows x N (partials with row stride NP)
void split_reduce_strided(Launch, const float* part, int64_t splits, int64_t rows, int64_t N, int64_t NP, float* G);
// dW partials (tc_dw_general): rows [0, F) reduce zc[0] splits, [F, 2F) zc[1] (nseg 2), bias row zc[2]
void split_reduce_dw(Launch, const float* part, const int64_t zc[3], int64_t F, int nseg, int64_t N, int64_t NP,
                     float* G);
// dA = Mg W^T ([M x 2F]); first half scaled by inv_deg[row] (dZ' of S7), into dA (ld_dA = 2 ld)
void gemm_da_f32(Launch, const float* Mg, int64_t ldM, int64_t M, int64_t N, const float* W, int64_t F,
                 const float* inv_deg, float* dA, int64_t ld);

// S11 + S12: g = sum_i G_i (ascending i); grads = g; SGD or Adam update of params.
struct OptSpec {
  int32_t adam;
  float lr, beta1, beta2, eps;
  float step_size;       // lr / (1 - beta1^t)
  float inv_sqrt_bc2;    // 1 / sqrt(1 - beta2^t)
  int32_t apply;         // 0: only write grads (cross-rank all-reduce follows)
};
struct PtrList {
  const float* p[PGCN_MAX_PARTS];
  int32_t n;
};
void sum_grads(Launch, const PtrList& G, int64_t P, float* grads);
void opt_update(Launch, const float* grads, int64_t P, float* params, float* m, float* v, const OptSpec& o);

}  // namespace pgcn
