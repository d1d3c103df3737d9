/*
 * pgcn_dev.h -- diagnostics entry points of libpgcn.so (not needed to train; used by the GPU unit
 * tests to check one kernel in isolation).  Same conventions as pgcn.h: 0 / negative PGCN_E*
 * codes, message in pgcn_last_error(), device pointers, asynchronous on `stream`.
 */
#ifndef PGCN_DEV_H
#define PGCN_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The three node-update GEMMs of a GraphSAGE layer (Alg. 1 l.14, l.18, l.20), with
 * A_ext = [A0 | A1 | 1] ([M x (2F+1)], A0 / A1 row-major with row stride ldA) and
 * W_ext = [W; b] ([(2F+1) x N] row-major, the layer's slice of theta):
 *   op 0 (forward)  out[M x ld_out]      = act(A_ext W_ext), act = ReLU if relu; cols [N, ld_out) = 0
 *   op 1 (dW)       out[(2F+1) x N]      = A_ext^T Mg            (Mg: [M x N], row stride ldM)
 *   op 2 (dA)       out[M x 2 ld_out/2]  = [inv_deg o (Mg W_neigh^T) | Mg W_self^T], halves padded
 * variant: 0 = tcgen05 3xTF32 tensor cores, 2 = fp32 SIMT.  scratch: device buffer of at least
 * pgcn_dev_gemm_scratch_bytes(M, F, N) bytes (256-byte aligned).                                  */
size_t pgcn_dev_gemm_scratch_bytes(int64_t M, int64_t F, int64_t N);
int pgcn_dev_gemm(int32_t op, int32_t variant, const float* A0, const float* A1, int64_t ldA, int64_t M, int64_t F,
                  const float* W_ext, int64_t N, const float* Mg, int64_t ldM, const float* inv_deg, float* out,
                  int64_t ld_out, int32_t relu, void* scratch, size_t scratch_bytes, void* stream);

/* The aggregation kernel of S3 (Eq. 3): Z[v] = inv_deg[v] * sum_{e in row v} D[col[e]] for rows
 * [0, n_rows); D holds n_valid rows and every column id must be < n_valid (the unchecked product
 * variant, as in a step where every boundary row is installed); D, Z row stride ld (multiple of 4). */
int pgcn_dev_spmm(const int64_t* row_ptr, const int32_t* col, const float* inv_deg, const float* D, int64_t ld,
                  int64_t n_rows, int64_t n_valid, float* Z, void* stream);

/* Random-row gather microbenchmark (roofline denominator for DRAM-served aggregation): reads rows
 * idx[0 .. n_idx) (row_floats floats each, multiple of 4) of tab in full, U rows in flight per
 * lane group (variant 0: U = 8, 1: U = 16), and writes checksums to out[] (sm_count x 8 x 256 floats).
 * Bytes moved = n_idx x 4 x row_floats; the caller times it.                                       */
int pgcn_dev_gather_read(const float* tab, int64_t row_floats, const int32_t* idx, int64_t n_idx, float* out,
                         int32_t variant, void* stream);

/* L2 streaming-read microbenchmark (roofline denominator for L2-served kernels): warps stream
 * contiguous chunks of buf[0 .. bytes) with __ldcg, `reps` passes (low 24 bits of reps), and write
 * one checksum per block to out[] (up to 148 x 8 blocks of 256 threads).  reps bits 24..31 pick the
 * variant (0: 4 loads in flight per lane, 8 blocks/SM; 1: 8 loads, 8 blocks/SM; 2: 8 loads, 4
 * blocks/SM).  Keep `bytes` well below the 126 MB L2.                                          */
int pgcn_dev_l2_read(const void* buf, int64_t bytes, int32_t reps, float* out, void* stream);

/* Dense-tile decomposition used by the tensor-core aggregation (pgcn_config.spmm_tiles; host only,
 * no GPU): which = 0 -> P_i (n_inner rows x (n_inner + n_halo) columns), 1 -> P_i^T.  Row blocks of
 * 128 rows x column tiles of 64 columns; a tile with >= tile_min edges is "heavy" and stored as a
 * bitmask (mask[128 k + r] bit c = edge (128 b + r, 64 tile_col[k] + c), tiles of block b at
 * [rb_ptr[b], rb_ptr[b+1]), column tiles ascending); the other edges (and a repeated (row, col)
 * pair) form the light CSR lrp / lcol, columns ascending within a row.  order = row blocks by
 * descending tile count (stable).  sizes[6] receives n_rows, n_rb, n_tiles, nnz_heavy, nnz_light,
 * n_cols; any array pointer may be NULL (sizes only).  Arrays are caller-owned host buffers of
 * those sizes (rb_ptr n_rb + 1, order n_rb, tile_col n_tiles, mask 128 n_tiles, lrp n_rows + 1,
 * lcol nnz_light).                                                                           */
typedef struct pgcn_partitioning pgcn_partitioning;
int pgcn_dev_tiles(const pgcn_partitioning* p, int32_t part, int32_t which, int32_t tile_min, int64_t* sizes,
                   int32_t* rb_ptr, int32_t* order, int32_t* tile_col, uint64_t* mask, int64_t* lrp, int32_t* lcol);

/* Exchange hook of the posted transports (pgcn_config.transport = LOOPBACK, or NCCL), used by the
 * stream/event-contract tests (SURVEY 4.6 delay injection) and the exposed-communication ablation:
 *   spin_ns   > 0: before every transfer (forward and backward, every layer) a one-thread kernel
 *             spins this many nanoseconds on the comm stream, delaying the messages.  With the
 *             contract intact results are bit-identical to spin_ns = 0.
 *   flags     PGCN_XH_SKIP_F_WAIT / PGCN_XH_SKIP_B_WAIT: fault injection -- drop the compute stream's
 *             wait for the forward / backward exchange events (results must then change under delay);
 *             PGCN_XH_NOCOMM: skip the transfers themselves (everything else runs; boundary rows keep
 *             whatever they held -- a timing ablation, T_PIPE - T_nocomm = exposed communication).
 * Applies to every later call on ctx.  PGCN_EUNSUPPORTED on a LOCAL-transport context.             */
typedef struct pgcn_ctx pgcn_ctx;
enum { PGCN_XH_SKIP_F_WAIT = 1, PGCN_XH_SKIP_B_WAIT = 2, PGCN_XH_NOCOMM = 4 };
int pgcn_dev_exchange_hook(pgcn_ctx* ctx, int64_t spin_ns, int32_t flags);
/* Payload bytes this context has posted to peers so far (forward features, backward gradients; counted
 * at enqueue; 0 on a LOCAL-transport context, whose install reads the owners' rows in place).        */
int pgcn_dev_exchange_bytes(const pgcn_ctx* ctx, int64_t* fwd_bytes, int64_t* bwd_bytes);

#ifdef __cplusplus
}
#endif
#endif /* PGCN_DEV_H */
