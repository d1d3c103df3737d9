/*
 * pgcn.h -- C ABI of the B200-native PipeGCN training step (arXiv 2203.10428).
 *
 * The calls follow the paper's problem statement, Alg. 1 (PAPER.md:104 header + lines 1-7,
 * PAPER.md:450 lines 8-35):  Input: partition id i, partition count n, G_i, P_i, X_i, Y_i,
 * B_i, L, eta, W_0.  Output: W_T.
 *
 *   pgcn_partition      Alg. 1 l.1-5   inner / boundary sets, send / receive sets, P_i
 *   pgcn_layer_fwd      Alg. 1 l.9-14  install stale boundary rows, exchange, H^(l) = s(P_i H W)
 *   pgcn_loss           Alg. 1 l.16    J^(L) = dLoss/dH^(L)
 *   pgcn_layer_bwd      Alg. 1 l.18-27 G_i^(l), J^(l-1), stale gradient accumulation, exchange
 *   pgcn_update         Alg. 1 l.31-32 G = AllReduce(G_i); W_t = W_{t-1} - eta G (or Adam, Table 3)
 *   pgcn_step           one iteration t of Alg. 1 l.8-32 (all of the above, in order)
 *
 * Readings of ambiguous passages (R1..R24) are listed in DESIGN.md; the ones that fix a
 * computed value are cited where they apply below.
 *
 * Conventions
 * - Every call returns 0 (PGCN_OK) or a negative PGCN_E* code; pgcn_last_error() returns a
 *   thread-local message describing the last failure on the calling thread.
 * - Host pointers are borrowed for the duration of the call.  Device memory is owned by the
 *   caller: the context carves everything it needs out of one caller-allocated workspace
 *   (size from pgcn_workspace_bytes); the library never calls cudaMalloc.  NCCL may allocate
 *   internally.
 * - Arguments are validated before any work is enqueued.  A CUDA or NCCL failure is sticky:
 *   every later call on that context returns PGCN_ESTATE.
 * - Order: within iteration t the calls must be layer_fwd(1..L), loss, layer_bwd(L..1),
 *   update (pgcn_step does exactly that), and t must increase by exactly 1 starting at 1.
 *   Violations return PGCN_ESTATE.  This is what keeps "one iteration stale" well defined.
 * - Device work is asynchronous on the stream given to pgcn_ctx_create; no call synchronises
 *   the host except pgcn_ctx_create (index upload) and pgcn_ctx_destroy.
 * - A context hosts one or more partitions on one GPU.  Peers hosted by the same context
 *   exchange through device gathers ("local transport"); peers in other processes through
 *   NCCL point-to-point on a dedicated comm stream (one partition per process).
 * - Row-major everywhere.  Feature rows are padded to ld = round_up(F, 4) floats (16 B) in
 *   the context's internal buffers; the public X / params layouts below are unpadded.
 */
#ifndef PGCN_H
#define PGCN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PGCN_OK = 0,
  PGCN_EINVAL = -1,      /* bad argument (null pointer, size, range, layout) */
  PGCN_ESTATE = -2,      /* call out of Alg. 1 order, or context poisoned by an earlier failure */
  PGCN_ECUDA = -3,       /* CUDA runtime error */
  PGCN_ENCCL = -4,       /* NCCL error */
  PGCN_ENOMEM = -5,      /* workspace too small / host allocation failed */
  PGCN_EUNSUPPORTED = -6 /* configuration not implemented */
};

#define PGCN_MAX_LAYERS 16
#define PGCN_MAX_PARTS 64
#define PGCN_MAX_DEPTH 3

const char* pgcn_last_error(void);
int pgcn_version(void); /* 100 * major + minor */

/* ------------------------------------------------------------------------------------------
 * (1) Alg. 1 l.1-5.  Host only, deterministic, multithreaded.
 *
 * n_nodes   : N (< 2^31).
 * row_ptr   : [N+1] int64, CSR of the in-neighbour lists N(v) (the aggregation of Eq. 1 reads
 *             h_u for u in N(v)); col_idx: [nnz] int32 in [0, N).  Self loops and duplicate
 *             entries are kept as given (the generator emits neither).
 * n_parts   : 1..PGCN_MAX_PARTS.
 * part_of   : [N] int32 map node -> partition, or NULL for contiguous node-balanced ranges
 *             lo_p = floor(p*N/n_parts) (reading R19; METIS, is out of scope).
 * n_threads : host threads (<= 0: hardware concurrency).
 * out       : receives an opaque handle owning every array returned by pgcn_partition_view.
 * Errors    : PGCN_EINVAL (null / out-of-range ids, non-monotone row_ptr), PGCN_ENOMEM.
 * ---------------------------------------------------------------------------------------- */
typedef struct pgcn_partitioning pgcn_partitioning;

int pgcn_partition(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col_idx, int32_t n_parts,
                   const int32_t* part_of, int32_t n_threads, pgcn_partitioning** out);

/* Per-partition arrays (borrowed; valid until pgcn_partition_free).  Canonical orders
 * (reading R20) make "bit-exact" well defined:
 *   inner_gid [n_inner]      V_i, ascending gid                                  (l.1)
 *   halo_gid  [n_halo]       B_i, sorted by (owner, gid)                         (l.1)
 *   halo_off  [n_parts+1]    segment of B_i owned by j = S_{j,i} = B_i ∩ V_j      (l.4-5)
 *   send_off  [n_parts+1], send_idx [n_send]
 *                            S_{i,j} = B_j ∩ V_i as local inner ids, ascending gid;
 *                            element-wise equal to j's halo segment for owner i  (l.2-3)
 *   row_ptr [n_inner+1], col_idx [nnz]
 *                            pattern of P_i: row v's neighbours in global order, local ids
 *                            (inner: [0,n_inner), boundary: n_inner + position in B_i)
 *   inv_deg [n_inner]        fp32(1)/fp32(d_v), d_v the FULL-graph degree (Eq. 3-4,
 *                            PAPER.md:456-462; reading R1); 0 for isolated v
 *   t_row_ptr [n_inner+n_halo+1], t_col_idx [nnz]
 *                            pattern of P_i^T (Alg. 1 l.20): for local row u, the inner v
 *                            with u in N(v), ascending v
 *   inv_ptr [n_inner+1], inv_pos [n_send]
 *                            inverse send map: positions k with send_idx[k] == v, ascending k
 *                            (Alg. 1 l.23-25 accumulation)
 *   deg [n_inner+n_halo]     full-graph degree d_u of every local row (inner then boundary);
 *                            the GCN-sym weights 1/sqrt((d_v+1)(d_u+1)) of App. A.1
 *                            need it for boundary columns too (reading R26)                  */
typedef struct {
  int32_t part, n_parts;
  int64_t n_inner, n_halo, nnz, n_send;
  const int64_t* inner_gid;
  const int64_t* halo_gid;
  const int64_t* halo_off;
  const int64_t* send_off;
  const int32_t* send_idx;
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const float* inv_deg;
  const int64_t* t_row_ptr;
  const int32_t* t_col_idx;
  const int64_t* inv_ptr;
  const int32_t* inv_pos;
  const int64_t* deg;
} pgcn_part_view;

int pgcn_partition_view(const pgcn_partitioning* p, int32_t part, pgcn_part_view* out);
int64_t pgcn_partition_n_nodes(const pgcn_partitioning* p);
void pgcn_partition_free(pgcn_partitioning* p);

/* ------------------------------------------------------------------------------------------
 * (2) Training configuration.
 *   width[0..n_layers]  F_0 (input features) .. F_L (classes).  GraphSAGE-mean layers
 *                       (Table 3): Y = [Z | D] W + b,  W = [W_neigh; W_self].
 *   mode                0 VANILLA (Fig. 1(a): exchange consumed in the same iteration),
 *                       1 PIPE (Alg. 1: exchange consumed one iteration later).
 *   smooth_f, smooth_g  PipeGCN-F / -G: EMA of stale boundary features (layers >= 2, R14) /
 *                       of each received gradient message (R13); Sec. 3.4 PAPER.md:478-486.
 *   gamma               EMA decay (default 0.95).
 *   ema_init            0 = first receipt initialises the state (R12), 1 = zero state.
 *   dropout, seed       p and the mask seed: keep iff (SplitMix64(key ^ seed) >> 40) >=
 *                       floor(p*2^24 + 0.5), key = ((t(L+1)+l)N + gid)F_{l-1} + col, applied
 *                       to every layer's input after the exchange (App. F; R5).
 *   gemm                0 fp32-grade on the tensor cores: tcgen05 kind::tf32 with the 3xTF32 split
 *                       (hi/lo operands, 1e-4 tier; default); 1 BF16 tensor cores (kind::f16, 2e-2
 *                       tier); 2 fp32 SIMT CUDA-core GEMMs (reference kernels).
 *   loss                0 softmax cross-entropy (labels int32 [n_inner]), 1 sigmoid BCE
 *                       (labels uint8 [n_inner x F_L]); mean over the GLOBAL train set (R6).
 *   n_global            N (dropout keys); n_train_global: |train set| over the whole graph.
 *   opt                 0 SGD (Alg. 1 l.32), 1 Adam (Table 3; PyTorch defaults, R7).
 *   dump_j              1: also store the accumulated J^(l) inner rows (parity checks only).
 *   transform_first     0: aggregate then transform everywhere (Eq. 3 then the update, as written);
 *                       1 (auto): per layer, compute P(D W_neigh) instead of (P D) W_neigh where that
 *                       gathers fewer bytes -- layer 1 if 2 F_1 < F_0, layers >= 2 if F_l < F_{l-1}
 *                       (same mathematics, fp32 reassociation only).  Tensor-core GEMMs only.
 *   staleness_stats     1: measure the staleness errors of Fig. 5/7 (see pgcn_staleness); local
 *                       transport only (adds one reduction kernel per layer and direction).
 *   depth               pipeline depth s of PIPE (0 or 1: Alg. 1; 2..PGCN_MAX_DEPTH: App. C's "two
 *                       iterations of compute to hide one iteration of communication", PAPER.md:923,
 *                       reading R27): the exchange posted at t is consumed at t + s; boundary rows
 *                       are 0 and no gradient is accumulated for t <= s.  Activation / gradient
 *                       buffers rotate over s + 1 slots.
 *   model               0 GraphSAGE-mean (above); 1 GCN-sym (SURVEY N3, App. A.1 PAPER.md:637-647,
 *                       reading R26): Y = P D W + b with P = D~^-1/2 (A + I) D~^-1/2, D~ = d + 1
 *                       (full-graph degrees), W [F_{l-1} x F_l]; tensor-core GEMMs only (gemm 0/1).
 *   gather              0 fp32 aggregation tables (default); 1 bf16 gather tier (2e-2
 *                       tier): every table an SpMM gathers (dropout output / T / dZ') is rounded to
 *                       bf16 first, the SpMMs gather bf16 rows and accumulate in fp32 -- half the
 *                       gathered bytes.  Everything else (H, J, exchange payloads, GEMM outputs)
 *                       stays fp32.
 *   train_sparse        1: N1(ii) train-row-sparse last layer (same loss, gradients and weights): the
 *                       last layer's aggregation runs only on train rows (Y^(L) of other rows is not
 *                       computed: logits there are stale) and its transposed aggregation only over
 *                       train sources.  pgcn_set_inputs then builds the train row list and the
 *                       restricted P_i^T and synchronises the stream (their sizes size the launches).
 *   spmm_tiles          1: dense-tile aggregation (exact reassociation of Eq. 3's sum, DESIGN.md
 *                       "Tensor-core tiles"): 128-row x 64-column blocks of P_i / P_i^T holding
 *                       >= tile_min edges are summed on the tensor cores as a 0/1 block times the 64
 *                       gathered rows (fp32 tier: 2-term tf32 split of the rows, fp32-grade; bf16
 *                       tier: bf16 rows), the other edges by the gather SpMM.  Used only where the
 *                       heavy tiles hold >= 25 % of a pattern's edges and every neighbour row is
 *                       valid (t > s).  0: gather SpMM only.
 *   tile_min            heavy-tile threshold in edges per 128 x 64 tile (0: default 96).
 *   transport           single-process contexts (multi-process runs use NCCL, plus PUSH over peer memory when
 *                       transport = 2 -- see pgcn_ipc_export):
 *                       0 LOCAL    -- the install reads the owners' rows straight out of their buffers
 *                                     and the accumulate reads the peers' boundary-row gradients (one
 *                                     gather kernel each, no message buffers);
 *                       1 LOOPBACK -- the posted exchange of the NCCL transport (Alg. 1 l.12-13, l.27;
 *                                     App. F: a second stream carries all communication):
 *                                     pack S_{i,j} rows on the compute stream, event, then on the comm
 *                                     stream one cudaMemcpyAsync per (sender, receiver) segment into the
 *                                     receiver's boundary rows / gradient message buffer, event; the
 *                                     consumer waits for the event of the iteration it consumes.  Same
 *                                     buffers, rotation, events and waits as NCCL; the transfer is a
 *                                     device copy instead of ncclSend/ncclRecv.
 *                       2 PUSH     -- SURVEY N2, fusion with the exchange: the kernel that produces rows a
 *                                     peer consumes stores them straight into the peer's receive rows
 *                                     from its epilogue (forward: the node-update GEMM's epilogue stores
 *                                     each S_{i,j} row into j's boundary rows of the slot read at t + s;
 *                                     backward: the transposed SpMM / input-gradient GEMM epilogue stores
 *                                     each boundary row of J^(l-1) into its owner's message rows).  No
 *                                     pack kernel, no copy; same slots and rotation as LOOPBACK, ordered
 *                                     by the compute stream.  Layers whose output comes from the SpMM
 *                                     (GCN-sym transform-first) or a SIMT GEMM keep LOOPBACK's pack +
 *                                     copy; layer 1's X exchange (once, R10) too.  fp32 payloads only.
 *   halo_payload        posted transports (LOOPBACK, NCCL): 0 fp32 exchange payloads; 1 bf16 payloads
 *                       (SURVEY N1(iv), 2e-2 tier): the packed boundary features and the boundary-row
 *                       gradients are rounded to bf16 (round to nearest even) for the transfer and
 *                       widened on receipt (EMA and sums in fp32) -- half the exchanged bytes.
 *   lean                1: lean-memory mode (same results bit for bit, fewer bytes of
 *                       workspace): (a) the aggregation Z of every layer lives in one shared scratch and
 *                       is recomputed by the backward before the weight gradient (one more forward SpMM
 *                       per aggregate-first layer); (b) T = D W_neigh of transform-first layers shares one
 *                       scratch (it is dead between a layer's forward and its backward); (c) J^(l) and
 *                       the packed feature messages keep one slot instead of s + 1 -- the backward of
 *                       layer l+1 at t waits for the transfer of t-1 to have read J^(l)'s boundary rows,
 *                       the pack at t for the transfer of t-1 (s = 1: already implied by Alg. 1's wait);
 *                       (d) with the compact last layer (train_sparse, aggregate-first GraphSAGE) the
 *                       last layer's logits / M / D_tr rows are sized by min(n_inner, n_train_global)
 *                       and Y^(L) of non-train rows is not stored at all (pgcn_tensor of the last
 *                       layer's H is then unavailable; pgcn_set_inputs fails with PGCN_EINVAL if a
 *                       partition holds more train rows than n_train_global).  Needs a posted transport
 *                       (LOOPBACK, PUSH, NCCL) when n_parts > 1: LOCAL reads the peers' gradient rows of
 *                       an earlier slot in place.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_layers;
  int32_t width[PGCN_MAX_LAYERS + 1];
  int32_t mode;
  int32_t smooth_f, smooth_g;
  int32_t ema_init;
  double gamma;
  double dropout;
  uint64_t seed;
  int32_t gemm;
  int32_t loss;
  int64_t n_global;
  int64_t n_train_global;
  int32_t opt;
  int32_t dump_j;
  double lr, beta1, beta2, eps;
  int32_t transform_first;
  int32_t staleness_stats;
  int32_t model;
  int32_t depth;
  int32_t gather;
  int32_t train_sparse;
  int32_t spmm_tiles;
  int32_t tile_min;
  int32_t transport;
  int32_t halo_payload;
  int32_t lean;
} pgcn_config;

/* Cross-process transport.  NULL (or nranks == 1) = every partition is hosted by this
 * context.  Otherwise one partition per rank (rank r hosts partition r) and nccl_id_halo /
 * nccl_id_reduce point to two 128-byte ncclUniqueId blobs shared by all ranks (the caller
 * broadcasts them, e.g. with torch.distributed).                                           */
typedef struct {
  int32_t rank, nranks;
  const void* nccl_id_halo;
  const void* nccl_id_reduce;
} pgcn_comm;

/* NCCL bootstrap: size of an ncclUniqueId (0 if the library was built without NCCL) and a fresh
 * id written to out (rank 0 calls it; the caller broadcasts the bytes to every rank).          */
int pgcn_nccl_id_bytes(void);
int pgcn_nccl_unique_id(void* out);


typedef struct pgcn_ctx pgcn_ctx;

/* N2 over NVLink (App. F PAPER.md:981 puts the exchange on a second stream, here it rides in the
 * producing epilogues): a multi-process context created with cfg.transport = 2 (PUSH) in PIPE mode with fp32
 * payloads stores the rows its peers consume straight into their workspaces -- the node-update GEMM epilogue
 * writes S_{i,j} rows of H^(l) into peer j's boundary rows of the slot read at t + s, the transposed SpMM /
 * input-gradient GEMM epilogue writes J^(l-1)'s boundary rows into their owners' message rows -- instead of
 * pack + ncclSend/ncclRecv (layer 1's one X exchange and GCN-sym transform-first layers keep NCCL).  Ordering:
 * the per-iteration gradient all-reduce completes on a rank only after every rank's iteration-t kernels,
 * pushes included, have run, so pushes of t are visible at t + 1 and a slot is rewritten only after its last
 * reader (the rotation of the posted exchange).  Setup, after pgcn_ctx_create on every rank: each rank exports
 * its workspace (a CUDA IPC handle of the allocation holding it, pgcn_ipc_handle_bytes() bytes, and the
 * workspace's offset in it), the caller all-gathers the (handle, offset) pairs (e.g. torch.distributed), and
 * each rank imports every peer's; pgcn_layer_fwd returns PGCN_ESTATE until all nranks - 1 peers are imported.
 * Errors: PGCN_ESTATE (context not created for PUSH across ranks; rank imported twice), PGCN_EINVAL (bad rank /
 * pointer), PGCN_ECUDA (the allocation cannot be exported / opened, e.g. no peer access).  VANILLA or bf16
 * payloads with PUSH across ranks fall back to NCCL send / recv (no export needed).                       */
int pgcn_ipc_handle_bytes(void);
int pgcn_ipc_export(pgcn_ctx* ctx, void* handle /* [pgcn_ipc_handle_bytes()] out */, int64_t* offset);
int pgcn_ipc_import(pgcn_ctx* ctx, int32_t rank, const void* handle, int64_t offset);

/* Workspace bytes for hosting partitions local_parts[0..n_local) of p under cfg. */
int pgcn_workspace_bytes(const pgcn_partitioning* p, const int32_t* local_parts, int32_t n_local,
                         const pgcn_config* cfg, size_t* bytes);

/* Create a context.  ws: device buffer of ws_bytes (256-byte aligned); stream: cudaStream_t
 * (NULL = legacy default) on which all compute is enqueued.  Uploads the index arrays and
 * zero-fills the activations (boundary rows start at 0, Alg. 1 l.6), synchronously.       */
int pgcn_ctx_create(const pgcn_partitioning* p, const int32_t* local_parts, int32_t n_local,
                    const pgcn_config* cfg, const pgcn_comm* comm, void* ws, size_t ws_bytes,
                    void* stream, pgcn_ctx** out);
int pgcn_ctx_destroy(pgcn_ctx* ctx);

/* Inputs of hosted partition `local` (0..n_local-1): X_i [n_inner x F_0] fp32 row-major
 * (unpadded), labels (see cfg.loss), train_mask uint8 [n_inner].  Host (pageable or pinned)
 * or device pointers; copied asynchronously on the context stream into the workspace.     */
int pgcn_set_inputs(pgcn_ctx* ctx, int32_t local, const float* X, const void* labels,
                    const uint8_t* train_mask);

/* Streaming re-upload of a hosted partition's inputs between iterations (the end-to-end path: inputs
 * live in host memory and are copied every iteration).  Same layouts as pgcn_set_inputs, except that X
 * has row stride ld_x = F_0 or round_up(F_0, 4) (the context's own padded layout: one contiguous copy
 * instead of n_inner row copies); X, labels and train_mask are HOST pointers (pinned memory makes the
 * copy asynchronous).  The copies run on the
 * library's copy stream and overlap the iteration in flight: X is overwritten only after that
 * iteration's last read of X (layer 1's dropout, or layer 1's weight gradient when dropout = 0),
 * labels / mask only after its loss; the next pgcn_layer_fwd(layer 1) waits for the copies.  The train
 * set must be the one given to pgcn_set_inputs (the train row lists are not rebuilt), and X must hold
 * the same values (X's boundary rows are exchanged once, reading R10).  Caller keeps the host buffers
 * alive until the next iteration's layer 1 has been enqueued and the stream has passed it.
 * Errors: PGCN_EINVAL (null / range), PGCN_ESTATE (poisoned, or pgcn_set_inputs never called).     */
int pgcn_stage_inputs(pgcn_ctx* ctx, int32_t local, const float* X, int64_t ld_x, const void* labels,
                      const uint8_t* train_mask);

/* Flat parameter vector theta = vec[W^(1), b^(1), ..., W^(L), b^(L)], fp32,
 * unpadded: W^(l) is [2F_{l-1} x F_l] row-major (rows 0..F_{l-1}-1 multiply z, the rest h;
 * CONCAT(z_v, h_v) PAPER.md:44, reading R3), b^(l) is [F_l].  GCN-sym (cfg.model 1): W^(l) is
 * [F_{l-1} x F_l].                                                                          */
int64_t pgcn_param_count(const pgcn_config* cfg);

/* (3) Alg. 1 l.9-14 for layer `layer` (1..L) of every hosted partition, iteration t.
 * params: device pointer to theta (W_{t-1}).                                               */
int pgcn_layer_fwd(pgcn_ctx* ctx, int64_t t, int32_t layer, const float* params);

/* (4) Alg. 1 l.16.  loss_dev: device fp32 scalar receiving the sum of the hosted partitions'
 * loss terms (each already divided by the global train count), or NULL.                    */
int pgcn_loss(pgcn_ctx* ctx, int64_t t, float* loss_dev);

/* (5) Alg. 1 l.18-27 for layer `layer` (L..1): G_i^(l) (kept in the context), J^(l-1) with
 * stale (PIPE) or fresh (VANILLA) boundary gradients accumulated, and the exchange.        */
int pgcn_layer_bwd(pgcn_ctx* ctx, int64_t t, int32_t layer, const float* params);

/* (6) Alg. 1 l.31-32: grads = sum_i G_i (ascending i, then NCCL all-reduce SUM across ranks);
 * params updated in place.  opt_state: [2 * param_count] fp32 device (Adam m, v; zero at t=1),
 * may be NULL for SGD.                                                                     */
int pgcn_update(pgcn_ctx* ctx, int64_t t, float* params, float* grads, float* opt_state);

/* (3') / (5') Caller-buffer forms of the per-layer calls (SURVEY 8(b) signatures): the same Alg. 1 steps
 * as pgcn_layer_fwd / pgcn_layer_bwd (and the same call-order rules -- they count as those calls), with
 * the layer's weights and the activations in caller-owned device buffers.  Pointer arrays are indexed
 * by hosted partition k = 0..n_local-1 (n_inner_k rows each); a NULL array or entry means "not given".
 *   W [ns F_{l-1} x F_l] row-major (ns = 2 GraphSAGE [W_neigh; W_self], 1 GCN-sym), b [F_l]: the layer's
 *       weights W_{t-1}; the context stages them in theta layout (the backward call must pass the same
 *       weights as the forward call of iteration t).
 *   fwd h_in[k]  [n_inner_k x F_{l-1}], row stride ld_in: replaces the inner rows of the layer input
 *       H^(l-1) (layer 1: X, constant by reading R10) before the layer runs -- this is what is sent to
 *       the peers (Alg. 1 l.12-13); NULL keeps the output of the previous layer call.
 *   fwd h_out[k] [n_inner_k x F_l], row stride ld_out: receives H^(l) (ReLU for l < L; logits for l = L,
 *       valid on train rows only under train_sparse).
 *   bwd j_out[k] [n_inner_k x F_l], row stride ld_jo: replaces the accumulated J^(l) of the layer's output
 *       (l = L: dLoss/dH^(L); EUNSUPPORTED for l = L with train_sparse on a GraphSAGE aggregate-first last
 *       layer, whose rows are compact); NULL keeps the context's own (from pgcn_loss / the layer above).
 *   bwd dW_local [ns F_{l-1} x F_l], db_local [F_l]: sum over the hosted partitions (ascending i) of G_i^(l)
 *       (Alg. 1 l.18) -- this context's contribution before the all-reduce of pgcn_update.
 *   bwd j_in[k] [n_inner_k x F_{l-1}] (l >= 2), row stride ld_ji: receives J^(l-1) after the stale-
 *       gradient accumulation (l.22-25).
 * Asynchronous on the context stream; buffers must stay valid until the stream has passed the call.   */
int pgcn_layer_fwd_io(pgcn_ctx* ctx, int64_t t, int32_t layer, const float* W, const float* b,
                      const float* const* h_in, int64_t ld_in, float* const* h_out, int64_t ld_out);
int pgcn_layer_bwd_io(pgcn_ctx* ctx, int64_t t, int32_t layer, const float* W, const float* b,
                      const float* const* j_out, int64_t ld_jo, float* dW_local, float* db_local,
                      float* const* j_in, int64_t ld_ji);

/* (7) One iteration t of Alg. 1 (l.8-32).                                                   */
int pgcn_step(pgcn_ctx* ctx, int64_t t, float* params, float* grads, float* opt_state,
              float* loss_dev);

/* Device views of internal buffers for parity checks and diagnostics (not needed to train).
 * kind: PGCN_T_H   layer-l output H^(l) (l = 1..L; l = L: logits), inner rows, parity of t
 *       PGCN_T_HIN layer-l input buffer [inner; boundary] rows (l = 1..L)
 *       PGCN_T_Z   aggregated Z of layer l (inner rows); with transform-first S = P_i (D W_neigh)
 *                  (GraphSAGE) -- not kept for GCN-sym transform-first layers (PGCN_EINVAL)
 *       PGCN_T_J   accumulated J^(l) inner rows (needs cfg.dump_j; l = 1..L-1), t's parity
 *       PGCN_T_G   this partition's G_i, flat like theta
 * The returned pointer is valid until the next call that writes that buffer.               */
enum { PGCN_T_H = 0, PGCN_T_HIN = 1, PGCN_T_Z = 2, PGCN_T_J = 3, PGCN_T_G = 4 };
typedef struct {
  void* ptr;
  int64_t rows, cols, ld; /* elements; ld = row stride */
} pgcn_tensor_desc;
int pgcn_tensor(pgcn_ctx* ctx, int32_t local, int32_t kind, int32_t layer, int64_t t,
                pgcn_tensor_desc* out);

/* Fig. 5/7 staleness errors of the last completed iteration for `layer` (1..L):
 *   feat_err = ||boundary rows of the layer-l input used - the owners' fresh rows||_F (before dropout)
 *   grad_err = ||feature-gradient messages accumulated into J^(l-1) - the fresh ones||_F
 * summed over the hosted partitions ("used" = 0 when nothing was received, t = 1; the smoothed
 * value under EMA).  Needs cfg.staleness_stats and the local transport.  Synchronises.          */
int pgcn_staleness(pgcn_ctx* ctx, int32_t layer, double* feat_err, double* grad_err);

/* Number of kernels this library launched on the context so far (counted at launch). */
int64_t pgcn_launch_count(const pgcn_ctx* ctx);

/* Per-kernel device timing (diagnostics / roofline).  When enabled, every launch of the listed
 * kernel kinds is bracketed by CUDA events on the context stream; pgcn_timing_read synchronises
 * the stream and returns the summed elapsed milliseconds, launch count and the algorithmic bytes
 * (or flops for GEMMs) those launches were charged with.      */
enum {
  PGCN_K_SPMM_FWD = 0, PGCN_K_SPMM_BWD = 1, PGCN_K_GEMM_FWD = 2, PGCN_K_GEMM_DW = 3, PGCN_K_GEMM_DA = 4,
  PGCN_K_DROPOUT = 5, PGCN_K_GATHER = 6, PGCN_K_GRAD_REDUCE = 7, PGCN_K_LOSS = 8, PGCN_K_UPDATE = 9,
  PGCN_K_SPMM_TILE_FWD = 10, PGCN_K_SPMM_TILE_BWD = 11,
  PGCN_K_COUNT = 12
};
/* PGCN_K_SPMM_TILE_FWD / _BWD are sub-intervals of PGCN_K_SPMM_FWD / _BWD: the tensor-core tile part of an
 * aggregation launch on the tile path (bf16 split of the table + k_spmm_tc), charged with the MMA flops it
 * executes (2 x 128 x 64 x round_up(width, 64) per heavy tile and table: the 0/1 tile times the table's
 * 64 rows, zeros included) and the bytes its TMA loads (64 table rows per tile and table + the 1 KB mask).
 * The rest of the SPMM interval is the gather kernel (light edges and the epilogue).                */
int pgcn_timing_enable(pgcn_ctx* ctx, int32_t on); /* also resets the accumulators */
int pgcn_timing_read(pgcn_ctx* ctx, int32_t kind, double* ms, int64_t* launches, double* alg_bytes,
                     double* alg_flops);
/* For the aggregation kinds (PGCN_K_SPMM_*), alg_bytes above is SURVEY 8(d)'s compulsory B_min (the
 * gathered table read once); this returns the per-edge B_gather of the same launches (the table row
 * read once per edge).  Other kinds: equal to alg_bytes.                                            */
int pgcn_timing_read_gather(pgcn_ctx* ctx, int32_t kind, double* gather_bytes);

#ifdef __cplusplus
}
#endif
#endif /* PGCN_H */
