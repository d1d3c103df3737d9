// Step engine: per-partition device context and the Alg. 1 state machine.
//
// Data layout in the caller's workspace, per hosted partition i:
//   X        [n_all x ld0]         layer-1 input; rows [0,n_in) = X_i, [n_in,n_all) = boundary
//   H[l][b]  [n_all x ld_l]        layer-l output / layer-(l+1) input, b = t mod (s + 1) for
//                                  pipeline depth s (R27; s = 1: parity double buffer -- the
//                                  PIPE install at t reads owners' buffer of t - s)
//   logits   [n_in  x ld_L]
//   D[l]     [n_all x ld_{l-1}]    dropout(layer-l input) (absent when p = 0: D = input)
//   Z[l]     [n_in  x ld_{l-1}]    aggregated neighbours (S3)
//   M        [n_in  x max ld]      J o sigma' of the layer being back-propagated
//   dA       [n_in  x 2 max ld]    [inv_deg * dZ | dD_self] (S7)
//   J[l][b]  [n_all x ld_l]        J^(l) for inner + boundary rows (S8), s + 1 rotating buffers
//   emaG[l]  [n_send x ld_l]       EMA-G state per received gradient row (Sec. 3.4)
//   G        [P]                   this partition's G_i, laid out like theta
// ld_l = round_up(F_l, 4).  Boundary rows start at 0 (workspace zero-filled; Alg. 1 l.6).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "common.h"
#include "gemm_tc.cuh"
#include "kernels.cuh"
#include "tiles.h"
#include "pgcn.h"
#include "pgcn_dev.h"
#ifdef PGCN_WITH_NCCL
#include <nccl.h>
#endif

namespace pgcn {

constexpr int kMaxBuf = PGCN_MAX_DEPTH + 1;  // rotating activation / gradient buffers (depth s + 1)

struct PartCtx {
  int32_t part = 0;
  pgcn_part_view v{};
  int64_t n_in = 0, n_bd = 0, n_all = 0, nnz = 0, n_send = 0;
  int64_t *rp = nullptr, *trp = nullptr, *inv_ptr = nullptr, *gid = nullptr;
  int32_t *col = nullptr, *tcol = nullptr, *halo_map = nullptr, *msg_map = nullptr, *send_idx = nullptr,
          *inv_pos = nullptr;
  float* inv_deg = nullptr;
  float* sym = nullptr;  // GCN-sym: d~_u^-1/2 = 1/sqrt(d_u + 1) of inner then boundary rows (R26)
  float* X = nullptr;
  float* H[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};
  float* logits = nullptr;
  float* D[PGCN_MAX_LAYERS + 1] = {};
  float* Z[PGCN_MAX_LAYERS + 1] = {};
  float* T[PGCN_MAX_LAYERS + 1] = {};
  int64_t n_valid[PGCN_MAX_LAYERS + 1] = {};  // rows of the layer input valid this iteration
  float* M = nullptr;
  float* Mlo = nullptr;  // 3xTF32 tier: lo = M - trunc_tf32(M), written with M (the GEMMs reading M load it)
  float* dA = nullptr;
  float* J[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};
  float* emaG[PGCN_MAX_LAYERS + 1] = {};
  void* labels = nullptr;
  uint8_t* train = nullptr;
  float* row_loss = nullptr;
  float* G = nullptr;
  uint16_t* T16 = nullptr;  // fp32 tier with tiles: bf16 hi/lo split of the table the tile kernel reads
  uint16_t* G16 = nullptr;  // bf16 gather tier (cfg.gather): rounded copy of the table an SpMM gathers
  // N1(ii) train-row-sparse last layer (cfg.train_sparse): train row list, P_i^T restricted to train
  // sources, and their sizes (read back by pgcn_set_inputs)
  int32_t* tr_list = nullptr;
  int64_t* tr_count = nullptr;
  int64_t* tr_counts = nullptr;
  int64_t* trp_tr = nullptr;
  int32_t* tcol_tr = nullptr;
  int64_t n_tr = 0, nnz_tr = 0;
  // the last layer runs on train rows only (N1(ii)) -- unless its patterns have dense tiles and more than
  // a quarter of the rows are train rows: the tile path over every row is then cheaper than the gather
  // over the train rows (Reddit-shaped, 66 % train rows: step 24.4 -> 23.3 ms).  Exact either way.
  bool last_sparse = false;
  // compact train rows of an aggregate-first GraphSAGE last layer (pgcn_ctx::cl): row k = tr_list[k]
  int32_t* tr_pos = nullptr;   // [n_in] position of inner row v in tr_list, or -1
  float* Dtr = nullptr;        // [n_tr x ld_{L-1}] layer-L input rows of the train rows (aliases dA)
  float* Ytr = nullptr;        // [n_tr x ld_L] logits of the train rows (aliases M)
  void* lab_tr = nullptr;      // labels of the train rows
  float* invdeg_tr = nullptr;  // [n_tr]
  // dense-tile decompositions (cfg.spmm_tiles): [0] P_i (forward), [1] P_i^T (transposed)
  const TileSet* ts[2] = {nullptr, nullptr};
  TileDev td[2];
  const TileDev* tiles(int w) const { return ts[w] ? &td[w] : nullptr; }
  // posted-exchange message buffers (LOOPBACK / NCCL transports; fp32, or bf16 with halo_payload = 1),
  // rotating over the pipeline depth (slot = t mod (s + 1); layer 1 has one slot: X is exchanged once)
  void* send_f[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};  // packed S_{i,j} rows of the layer-l input   [n_send x ld]
  void* recv_f[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};  // staged boundary rows (EMA-F or bf16)     [n_bd x ld]
  void* send_b[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};  // bf16 boundary-row gradients (bf16 only)  [n_bd x ld]
  void* recv_b[PGCN_MAX_LAYERS + 1][kMaxBuf] = {};  // received gradient rows, send order       [n_send x ld]
  // N2 fused push (PUSH transport): destination (peer, receive row) of every send position k and of
  // every boundary row r
  int32_t *fpush_part = nullptr, *fpush_row = nullptr, *bpush_part = nullptr, *bpush_row = nullptr;
};

enum { XP_LOCAL = 0, XP_LOOPBACK = 1, XP_NCCL = 2, XP_PUSH = 3 };

struct Arena {
  char* base = nullptr;
  size_t off = 0;
  template <class T>
  T* take(int64_t n) {
    off = (size_t)round_up((int64_t)off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += sizeof(T) * (size_t)(n > 0 ? n : 0);
    return p;
  }
};

enum { K_FWD = 0, K_LOSS = 1, K_BWD = 2, K_UPD = 3 };

struct KTimer {
  std::vector<cudaEvent_t> ev;  // (start, stop) pairs
  size_t used = 0;
  int64_t n = 0;
  double bytes = 0.0, flops = 0.0, gbytes = 0.0;
};

// Algorithmic bytes of an aggregation launch: B_min reads the gathered table once
// (compulsory), B_gather once per edge (the per-edge model); both add the index stream, the output
// and the epilogue operands (`rest`).
struct SpmmBytes {
  double min, gather;
};

}  // namespace pgcn

struct pgcn_ctx {
  pgcn_config cfg{};
  int L = 0;
  int64_t F[PGCN_MAX_LAYERS + 1] = {}, ld[PGCN_MAX_LAYERS + 1] = {}, woff[PGCN_MAX_LAYERS + 2] = {};
  int64_t P = 0, ldmax = 0;
  int32_t n_parts = 0;
  std::vector<pgcn::PartCtx> parts;
  cudaStream_t s = nullptr;
  float* dw_ws = nullptr;
  int64_t dw_ws_floats = 0;
  // tensor-core operand prep per layer: W_ext^T and W (tf32 hi/lo splits, TMA-legal strides)
  float* WT_hi[PGCN_MAX_LAYERS + 1] = {};
  float* WT_lo[PGCN_MAX_LAYERS + 1] = {};
  float* Wp_hi[PGCN_MAX_LAYERS + 1] = {};
  float* Wp_lo[PGCN_MAX_LAYERS + 1] = {};
  float* WJ_hi[PGCN_MAX_LAYERS + 1] = {};
  float* WJ_lo[PGCN_MAX_LAYERS + 1] = {};
  int64_t Fp[PGCN_MAX_LAYERS + 1] = {}, Kp[PGCN_MAX_LAYERS + 1] = {}, Kq[PGCN_MAX_LAYERS + 1] = {};
  // N1 transform-before-aggregate per layer: Y = P(D W_neigh) + D W_self + b instead of (PD) W_neigh
  int tf[PGCN_MAX_LAYERS + 1] = {};
  int gcn = 0, ns = 2;  // cfg.model == 1 (GCN-sym, R26); weight row segments
  // N1(ii) with an aggregate-first GraphSAGE last layer on the tensor cores: the whole last layer (SpMM
  // output, [Z | D] W, loss, dW, dA) runs on compact train rows; only the transposed aggregation
  // scatters back to every local row.  (papers-shaped: 1.1 % train rows.)
  int cl = 0;
  int64_t depth = 1;    // pipeline depth s (R27): an exchange posted at t is consumed at t + s
  float* part_loss = nullptr;
  float* theta_io = nullptr;  // [P] weights staged by the caller-buffer layer calls (theta layout)
  unsigned long long* work = nullptr;  // SpMM dynamic-scheduling counter
  char* sp_tmp = nullptr;               // CUB scratch of the train-row builders (cfg.train_sparse)
  int64_t sp_tmp_bytes = 0;
  double* diag = nullptr;              // N4: [2][L+1] squared staleness errors of the current iteration
  int64_t exp_t = 1;
  int exp_kind = pgcn::K_FWD, exp_layer = 1;
  int poisoned = 0;
  int64_t launches = 0;
  int timing = 0;
  pgcn::KTimer kt[PGCN_K_COUNT];
  // ---- exchange transport: LOCAL gathers, or the posted exchange on the comm
  // stream -- LOOPBACK (device copies between the hosted partitions) or NCCL (one partition per rank)
  int nccl = 0, rank = 0, nranks = 1;
  int xp = pgcn::XP_LOCAL;
  // N2 over NVLink (multi-process PUSH, PIPE): producers store exchanged rows straight into the peers'
  // workspaces, mapped with CUDA IPC (pgcn_ipc_export / pgcn_ipc_import); peer[j] = partition j's buffers
  // laid out in peer j's workspace, addressed in this process
  int ipc_push = 0;
  std::vector<pgcn::PartCtx> peer;
  std::vector<void*> ipc_open;  // mapped peer allocations (closed on destroy)
  int n_imported = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  const pgcn_partitioning* part = nullptr;
  int posted = 0;           // xp != XP_LOCAL
  int p16 = 0;              // bf16 payloads (cfg.halo_payload)
  int64_t hook_spin_ns = 0; // pgcn_dev_exchange_hook: delay injected on the comm stream before each transfer
  int32_t hook_flags = 0;   // PGCN_XH_* (pgcn_dev.h)
  int64_t xbytes[2] = {0, 0};  // payload bytes posted by this context's transfers (fwd, bwd)
  // PUSH: iteration in which layer l's input boundary rows / J^(l-1) messages were pushed by their producer
  int64_t fpushed[PGCN_MAX_LAYERS + 2] = {}, bpushed[PGCN_MAX_LAYERS + 2] = {};
  // ---- streaming inputs (pgcn_stage_inputs): copy stream and its events
  cudaStream_t cps = nullptr;
  cudaEvent_t ev_x_free = nullptr, ev_lab_free = nullptr, ev_in_ready = nullptr;
  int in_pending = 0, inputs_set = 0;
  int force_write_j = 0;  // pgcn_layer_bwd_io with j_in: the stale-gradient accumulate writes J^(l-1) inner rows
  int mlo_stale = 0;      // pgcn_layer_bwd_io(layer L, j_out): M came from the caller, Mlo was not written
#ifdef PGCN_WITH_NCCL
  ncclComm_t ch = nullptr, cr = nullptr;  // halo exchange / weight-gradient all-reduce
#endif
  cudaStream_t cs = nullptr;              // comm stream (high priority)
  pgcn::Launch launch();
  cudaEvent_t ev_f_pack[PGCN_MAX_LAYERS + 1] = {}, ev_b_ready[PGCN_MAX_LAYERS + 1] = {};
  cudaEvent_t ev_f_done[PGCN_MAX_LAYERS + 1][pgcn::kMaxBuf] = {}, ev_b_done[PGCN_MAX_LAYERS + 1][pgcn::kMaxBuf] = {};
  int nb = 2;                                              // buffers in rotation = depth + 1
  int bi(int64_t t) const { return (int)(((t % nb) + nb) % nb); }
  ~pgcn_ctx() {
    for (auto& k : kt)
      for (auto e : k.ev) cudaEventDestroy(e);
    for (int l = 0; l <= PGCN_MAX_LAYERS; ++l) {
      if (ev_f_pack[l]) cudaEventDestroy(ev_f_pack[l]);
      if (ev_b_ready[l]) cudaEventDestroy(ev_b_ready[l]);
      for (int b = 0; b < pgcn::kMaxBuf; ++b) {
        if (ev_f_done[l][b]) cudaEventDestroy(ev_f_done[l][b]);
        if (ev_b_done[l][b]) cudaEventDestroy(ev_b_done[l][b]);
      }
    }
#ifdef PGCN_WITH_NCCL
    if (ch) ncclCommDestroy(ch);
    if (cr) ncclCommDestroy(cr);
#endif
    if (cs) cudaStreamDestroy(cs);
    if (ev_x_free) cudaEventDestroy(ev_x_free);
    if (ev_lab_free) cudaEventDestroy(ev_lab_free);
    if (ev_in_ready) cudaEventDestroy(ev_in_ready);
    if (cps) cudaStreamDestroy(cps);
    for (void* q : ipc_open) cudaIpcCloseMemHandle(q);
  }
};

namespace pgcn {
namespace {

// Launch::mark of a timed context: the tile part of an aggregation launch as its own timing kind
void tile_mark(void* mctx, int kind, int begin, double flops, double bytes) {
  pgcn_ctx* C = static_cast<pgcn_ctx*>(mctx);
  KTimer& t = C->kt[kind];
  if (begin) {
    if (t.used + 2 > t.ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      t.ev.push_back(a);
      t.ev.push_back(b);
    }
    cudaEventRecord(t.ev[t.used], C->s);
    t.n += 1;
    t.flops += flops;
    t.bytes += bytes;
    t.gbytes += bytes;
  } else {
    cudaEventRecord(t.ev[t.used + 1], C->s);
    t.used += 2;
  }
}

int validate_cfg(const pgcn_config* c) {
  if (!c) return fail(PGCN_EINVAL, "config is NULL");
  if (c->n_layers < 1 || c->n_layers > PGCN_MAX_LAYERS) return fail(PGCN_EINVAL, "n_layers out of range");
  for (int l = 0; l <= c->n_layers; ++l)
    if (c->width[l] < 1) return fail(PGCN_EINVAL, "width[%d] < 1", l);
  if (c->mode != 0 && c->mode != 1) return fail(PGCN_EINVAL, "mode must be 0 (VANILLA) or 1 (PIPE)");
  if (!(c->dropout >= 0.0 && c->dropout < 1.0)) return fail(PGCN_EINVAL, "dropout must be in [0,1)");
  if (c->gemm < 0 || c->gemm > 2) return fail(PGCN_EINVAL, "gemm must be 0 (3xTF32), 1 (bf16) or 2 (SIMT)");
  if (c->loss != 0 && c->loss != 1) return fail(PGCN_EINVAL, "loss must be 0 (CE) or 1 (BCE)");
  if (c->opt != 0 && c->opt != 1) return fail(PGCN_EINVAL, "opt must be 0 (SGD) or 1 (Adam)");
  if (c->n_train_global < 1) return fail(PGCN_EINVAL, "n_train_global < 1");
  if (!(c->gamma >= 0.0 && c->gamma <= 1.0)) return fail(PGCN_EINVAL, "gamma out of [0,1]");
  if (c->model != 0 && c->model != 1) return fail(PGCN_EINVAL, "model must be 0 (GraphSAGE) or 1 (GCN-sym)");
  if (c->model == 1 && c->gemm == 2) return fail(PGCN_EUNSUPPORTED, "GCN-sym needs the tensor-core GEMMs (gemm 0/1)");
  if (c->depth < 0 || c->depth > PGCN_MAX_DEPTH) return fail(PGCN_EINVAL, "depth must be in 0..%d", PGCN_MAX_DEPTH);
  if (c->gather != 0 && c->gather != 1) return fail(PGCN_EINVAL, "gather must be 0 (fp32) or 1 (bf16)");
  if (c->train_sparse != 0 && c->train_sparse != 1) return fail(PGCN_EINVAL, "train_sparse must be 0 or 1");
  if (c->spmm_tiles != 0 && c->spmm_tiles != 1) return fail(PGCN_EINVAL, "spmm_tiles must be 0 or 1");
  if (c->tile_min < 0 || c->tile_min > 128 * 64) return fail(PGCN_EINVAL, "tile_min out of range");
  if (c->transport < 0 || c->transport > 2)
    return fail(PGCN_EINVAL, "transport must be 0 (LOCAL), 1 (LOOPBACK) or 2 (PUSH)");
  if (c->halo_payload != 0 && c->halo_payload != 1) return fail(PGCN_EINVAL, "halo_payload must be 0 (fp32) or 1 (bf16)");
  if (c->lean != 0 && c->lean != 1) return fail(PGCN_EINVAL, "lean must be 0 or 1");
  return PGCN_OK;
}

int64_t param_count(const pgcn_config* c) {
  int64_t P = 0;
  const int64_t k = c->model == 1 ? 1 : 2;
  for (int l = 1; l <= c->n_layers; ++l) P += (k * (int64_t)c->width[l - 1] + 1) * c->width[l];
  return P;
}

// Posted exchange: boundary features are received into a staging buffer (and installed from it at
// consume time) under EMA-F (the smoothing needs the previous value) or bf16 payloads;
// otherwise they land straight in the boundary rows of the layer input that consumes them.
bool staged_recv(const pgcn_ctx* C, int l) {
  return C->p16 || (C->cfg.smooth_f && C->cfg.mode == 1 && l >= 2);
}

// PUSH: whether layer l's output (layer l + 1's input) is stored into the receivers by its producer --
// the node-update GEMM's epilogue; not GCN-sym transform-first layers (the SpMM produces H) or SIMT GEMMs.
bool pushing(const pgcn_ctx* C) { return C->xp == XP_PUSH || C->ipc_push; }
bool fwd_push_capable(const pgcn_ctx* C, int l) {
  return pushing(C) && l < C->L && !(C->gcn && C->tf[l]) && C->cfg.gemm != 2;
}

// Lays out every buffer (dry run when A.base == nullptr).
int layout(pgcn_ctx* C, const pgcn_partitioning* part, const int32_t* local, int32_t n_local, Arena& A) {
  const int L = C->L;
  C->parts.assign(n_local, PartCtx{});
  int64_t dw_need = 0;
  for (int i = 0; i < n_local; ++i) {
    PartCtx& p = C->parts[i];
    p.part = local[i];
    int rc = pgcn_partition_view(part, local[i], &p.v);
    if (rc) return rc;
    p.n_in = p.v.n_inner;
    p.n_bd = p.v.n_halo;
    p.n_all = p.n_in + p.n_bd;
    p.nnz = p.v.nnz;
    p.n_send = p.v.n_send;
    p.rp = A.take<int64_t>(p.n_in + 1);
    p.col = A.take<int32_t>(p.nnz);
    p.inv_deg = A.take<float>(p.n_in);
    if (C->cfg.model == 1) p.sym = A.take<float>(p.n_all);
    p.trp = A.take<int64_t>(p.n_all + 1);
    p.tcol = A.take<int32_t>(p.nnz);
    p.gid = A.take<int64_t>(p.n_all);
    p.send_idx = A.take<int32_t>(p.n_send);
    p.inv_ptr = A.take<int64_t>(p.n_in + 1);
    p.inv_pos = A.take<int32_t>(p.n_send);
    p.halo_map = A.take<int32_t>(p.n_bd);
    p.msg_map = A.take<int32_t>(p.n_send);
    if (pushing(C)) {
      p.fpush_part = A.take<int32_t>(p.n_send);
      p.fpush_row = A.take<int32_t>(p.n_send);
      p.bpush_part = A.take<int32_t>(p.n_bd);
      p.bpush_row = A.take<int32_t>(p.n_bd);
    }
    p.X = A.take<float>(p.n_all * C->ld[0]);
    for (int l = 1; l < L; ++l)
      for (int b = 0; b < C->nb; ++b) p.H[l][b] = A.take<float>(p.n_all * C->ld[l]);
    // lean (N1(iii)): with the compact last layer only the train rows' logits exist (Y_tr in M)
    const bool lean = C->cfg.lean != 0;
    const int64_t n_trb = std::min(p.n_in, (int64_t)C->cfg.n_train_global);  // bound on a partition's train rows
    if (!(lean && C->cl)) p.logits = A.take<float>(p.n_in * C->ld[L]);
    int64_t zw = 0, tw = 0;  // lean: widths of the shared Z and T scratches
    for (int l = 1; l <= L; ++l) {
      if (C->cfg.dropout > 0.0 || C->cfg.model == 1) p.D[l] = A.take<float>(p.n_all * C->ld[l - 1]);
      zw = std::max(zw, C->tf[l] ? C->ld[l] : C->ld[l - 1]);
      if (C->tf[l]) tw = std::max(tw, C->ld[l]);
      if (lean) continue;
      p.Z[l] = A.take<float>(p.n_in * (C->tf[l] ? C->ld[l] : C->ld[l - 1]));   // Z, or S = inv_deg P T
      if (C->tf[l]) p.T[l] = A.take<float>(p.n_all * C->ld[l]);                 // T = D W_neigh, then Q
    }
    if (lean) {  // one Z scratch (recomputed by the backward) and one T scratch (dead between fwd and bwd)
      float* zs = A.take<float>(p.n_in * zw);
      float* tsc = tw ? A.take<float>(p.n_all * tw) : nullptr;
      for (int l = 1; l <= L; ++l) {
        p.Z[l] = zs;
        if (C->tf[l]) p.T[l] = tsc;
      }
    }
    // M: J^(l) o ReLU' at width F_l (l >= 1); dA: scale_rows output of transform-first layers (width
    // F_l) or dA = M W^T of aggregate-first layers l >= 2 (width 2 F_{l-1}, F_{l-1} for GCN-sym)
    int64_t ld_m = 0, ld_da = 0;
    for (int l = 1; l <= L; ++l) {
      if (!(lean && C->cl && l == L)) ld_m = std::max(ld_m, C->ld[l]);
      if (C->tf[l]) ld_da = std::max(ld_da, C->ld[l]);
      else if (l >= 2) ld_da = std::max(ld_da, (C->cfg.model == 1 ? 1 : 2) * C->ld[l - 1]);
    }
    // lean + compact last layer: M^(L) / Y_tr has at most n_trb rows
    const int64_t m_floats = lean && C->cl ? std::max(p.n_in * ld_m, n_trb * C->ld[L]) : p.n_in * ld_m;
    p.M = A.take<float>(m_floats);
    // M's lo term: where GEMMs read M in several tiles (widths >= 128; narrow layers read it about once) and
    // not for the compact last layer (n_tr rows); lean: the converters split M
    int64_t ld_mlo = 0;
    for (int l = 1; l <= L; ++l)
      if (!(C->cl && l == L)) ld_mlo = std::max(ld_mlo, C->ld[l]);
    // Dev knob PGCN_PRESPLIT=1 (default off): measured on B200 (profiles/r2p_presplit.md) the GEMMs gain
    // 1.6 ms per Yelp-shaped step (dW 16.2 -> 15.0, dA 10.1 -> 9.6) and the M_lo stores cost 0.8 ms in the
    // stale-gradient accumulate -- the converter warps are not what bounds these GEMMs
    if (C->cfg.gemm == 0 && !lean && ld_mlo >= 128 && knobs().presplit) p.Mlo = A.take<float>(p.n_in * ld_mlo);
    if (ld_da > 0) p.dA = A.take<float>(p.n_in * ld_da);
    for (int l = 1; l < L; ++l) {
      for (int b = 0; b < C->nb; ++b)  // lean: one slot (the next writer waits for the transfer, see layer_bwd)
        p.J[l][b] = (lean && b > 0) ? p.J[l][0] : A.take<float>(p.n_all * C->ld[l]);
      if (C->cfg.smooth_g) p.emaG[l] = A.take<float>(p.n_send * C->ld[l]);
    }
    p.labels = C->cfg.loss == 0 ? (void*)A.take<int32_t>(p.n_in) : (void*)A.take<uint8_t>(p.n_in * C->F[L]);
    p.train = A.take<uint8_t>(p.n_in);
    p.row_loss = A.take<float>(p.n_in);
    p.G = A.take<float>(C->P);
    if (C->cfg.gather == 1) p.G16 = A.take<uint16_t>(p.n_all * round_up(C->ldmax, 8));
    if (C->cfg.spmm_tiles) {  // heavy tiles must carry >= 25 % of the edges to pay for the extra pass
      const int32_t tmin = C->cfg.tile_min > 0 ? C->cfg.tile_min : 96;
      for (int w = 0; w < 2; ++w) {
        const TileSet* ts = part_tiles(part, local[i], w, tmin);
        p.ts[w] = nullptr;
        if (!ts || ts->n_tiles == 0 || 4 * ts->nnz_heavy < p.nnz) continue;
        p.ts[w] = ts;
        TileDev& d = p.td[w];
        d.rb_ptr = A.take<int32_t>(ts->n_rb + 1);
        d.order = A.take<int32_t>(ts->n_rb);
        d.tile_col = A.take<int32_t>(ts->n_tiles);
        d.mask = A.take<uint64_t>(ts->n_tiles * kTileRows);
        d.lrp = A.take<int64_t>(ts->n_rows + 1);
        d.lcol = A.take<int32_t>(ts->nnz_light);
        d.n_rows = ts->n_rows;
        d.n_cols = ts->n_cols;
        d.n_rb = ts->n_rb;
        d.n_tiles = ts->n_tiles;
        d.nnz_light = ts->nnz_light;
      }
      if ((p.ts[0] || p.ts[1]) && C->cfg.gather == 0) p.T16 = A.take<uint16_t>(2 * p.n_all * round_up(C->ldmax, 8));
    }
    if (C->cfg.train_sparse) {
      p.tr_list = A.take<int32_t>(p.n_in);
      p.tr_count = A.take<int64_t>(1);
      p.tr_counts = A.take<int64_t>(p.n_all + 1);
      p.trp_tr = A.take<int64_t>(p.n_all + 1);
      p.tcol_tr = A.take<int32_t>(p.nnz);
      if (C->cl) {  // Y_tr lives in M (free until the loss, which turns it into M_tr in place); D_tr in dA
        p.tr_pos = A.take<int32_t>(p.n_in);
        p.Ytr = p.M;
        const int64_t ntr = lean ? n_trb : p.n_in;
        p.Dtr = (p.dA && ld_da >= C->ld[L - 1]) ? p.dA : A.take<float>(ntr * C->ld[L - 1]);
        p.lab_tr = C->cfg.loss == 0 ? (void*)A.take<int32_t>(ntr) : (void*)A.take<uint8_t>(ntr * C->F[L]);
        p.invdeg_tr = A.take<float>(ntr);
      }
      const size_t tb = train_rows_tmp_bytes(p.n_in, p.n_all);
      if ((int64_t)tb > C->sp_tmp_bytes) C->sp_tmp_bytes = (int64_t)tb;
    }
    for (int l = 1; l <= L; ++l) {
      int64_t w = gemm_dw_ws_floats(p.n_in, C->F[l - 1], C->F[l]);
      if (w > dw_need) dw_need = w;
      w = tc_dw_ws_floats(C->tf[l] ? p.n_all : p.n_in, C->F[l - 1], C->F[l]);
      if (w > dw_need) dw_need = w;
    }
  }
  C->dw_ws_floats = dw_need;
  C->dw_ws = A.take<float>(dw_need);
  if (C->sp_tmp_bytes > 0) C->sp_tmp = A.take<char>(C->sp_tmp_bytes);
  if (C->posted) {  // message buffers of the posted exchange (per hosted partition, per rotation slot)
    const int64_t eb = C->p16 ? 2 : 4;  // payload bytes per element
    for (auto& p : C->parts)
      for (int l = 1; l <= L; ++l)
        for (int b = 0; b < (l == 1 ? 1 : C->nb); ++b) {
          const int64_t ld = C->ld[l - 1];
          if (l == 1 || !fwd_push_capable(C, l - 1))  // lean: one slot (the pack waits for the previous send)
            p.send_f[l][b] = (C->cfg.lean && b > 0) ? p.send_f[l][0] : A.take<char>(eb * p.n_send * ld);
          if (staged_recv(C, l)) p.recv_f[l][b] = A.take<char>(eb * p.n_bd * ld);
          if (l >= 2) {
            if (C->p16) p.send_b[l][b] = A.take<char>(eb * p.n_bd * ld);
            p.recv_b[l][b] = A.take<char>(eb * p.n_send * ld);
          }
        }
  }
  const int64_t ns = C->ns;  // weight row segments: 2 GraphSAGE [W_neigh; W_self], 1 GCN-sym
  if (C->cfg.gemm == 0) {     // 3xTF32 operand copies: fp32 hi/lo, k-blocks of 32
    for (int l = 1; l <= L; ++l) {
      C->Fp[l] = round_up(C->F[l - 1], 32);
      C->Kp[l] = round_up(C->F[l], 4);
      C->WT_hi[l] = A.take<float>(C->F[l] * ns * C->Fp[l]);
      C->WT_lo[l] = A.take<float>(C->F[l] * ns * C->Fp[l]);
      C->Wp_hi[l] = A.take<float>(ns * C->F[l - 1] * C->Kp[l]);
      C->Wp_lo[l] = A.take<float>(ns * C->F[l - 1] * C->Kp[l]);
      if (C->tf[l]) {
        C->Kq[l] = round_up(C->F[l], 32);
        C->WJ_hi[l] = A.take<float>(C->F[l - 1] * ns * C->Kq[l]);
        C->WJ_lo[l] = A.take<float>(C->F[l - 1] * ns * C->Kq[l]);
      }
    }
  } else if (C->cfg.gemm == 1) {  // bf16 operand copies, k-blocks of 64 (stored in the *_hi slots)
    for (int l = 1; l <= L; ++l) {
      C->Fp[l] = round_up(C->F[l - 1], 64);
      C->Kp[l] = round_up(C->F[l], 8);
      C->WT_hi[l] = reinterpret_cast<float*>(A.take<uint16_t>(C->F[l] * ns * C->Fp[l]));
      C->Wp_hi[l] = reinterpret_cast<float*>(A.take<uint16_t>(ns * C->F[l - 1] * C->Kp[l]));
      if (C->tf[l]) {
        C->Kq[l] = round_up(C->F[l], 64);
        C->WJ_hi[l] = reinterpret_cast<float*>(A.take<uint16_t>(C->F[l - 1] * ns * C->Kq[l]));
      }
    }
  }
  C->part_loss = A.take<float>(n_local);
  C->theta_io = A.take<float>(C->P);
  C->work = A.take<unsigned long long>(4);
  C->diag = A.take<double>(2 * (PGCN_MAX_LAYERS + 1));
  return PGCN_OK;
}

int init_ctx_shapes(pgcn_ctx* C, const pgcn_partitioning* part, const int32_t* local, int32_t n_local,
                    const pgcn_config* cfg, const pgcn_comm* comm) {
  int rc = validate_cfg(cfg);
  if (rc) return rc;
  if (!part) return fail(PGCN_EINVAL, "partition is NULL");
  if (!local || n_local < 1) return fail(PGCN_EINVAL, "no local partitions");
  pgcn_part_view v0;
  rc = pgcn_partition_view(part, local[0], &v0);
  if (rc) return rc;
  if (comm && comm->nranks > 1) {
#ifndef PGCN_WITH_NCCL
    return fail(PGCN_EUNSUPPORTED, "library built without NCCL");
#else
    if (comm->nranks != v0.n_parts || n_local != 1 || local[0] != comm->rank || comm->rank < 0 ||
        comm->rank >= comm->nranks)
      return fail(PGCN_EUNSUPPORTED, "multi-process runs host exactly partition `rank` of n_parts == nranks");
    if (!comm->nccl_id_halo || !comm->nccl_id_reduce) return fail(PGCN_EINVAL, "NCCL unique ids missing");
    C->nccl = 1;
    C->rank = comm->rank;
    C->nranks = comm->nranks;
    C->xp = XP_NCCL;
    // transport PUSH across ranks (N2 over NVLink): PIPE only -- the per-iteration gradient all-reduce orders
    // iteration t's pushes before every rank's iteration t + 1 (VANILLA would need a signal per layer)
    C->ipc_push = cfg->transport == 2 && cfg->mode == 1 && cfg->halo_payload == 0;
#endif
  } else {
    if (n_local != v0.n_parts)
      return fail(PGCN_EUNSUPPORTED, "a single-process context hosts all %d partitions (got %d)", v0.n_parts, n_local);
    for (int i = 0; i < n_local; ++i)
      if (local[i] != i) return fail(PGCN_EINVAL, "local_parts must be 0..n_parts-1 in order");
    C->xp = cfg->transport == 1 ? XP_LOOPBACK : (cfg->transport == 2 ? XP_PUSH : XP_LOCAL);
  }
  C->posted = C->xp != XP_LOCAL;
  C->p16 = cfg->halo_payload == 1;
  if (C->p16 && !C->posted)
    return fail(PGCN_EUNSUPPORTED, "bf16 exchange payloads need a posted transport (LOOPBACK or NCCL)");
  if (C->p16 && C->xp == XP_PUSH) return fail(PGCN_EUNSUPPORTED, "the PUSH transport moves fp32 payloads");
  if (cfg->lean && !C->posted && v0.n_parts > 1)
    return fail(PGCN_EUNSUPPORTED, "lean mode needs a posted transport (LOOPBACK, PUSH or NCCL): LOCAL reads the "
                                   "peers' gradient rows of an earlier slot in place");
  if (cfg->n_global != pgcn_partition_n_nodes(part)) return fail(PGCN_EINVAL, "cfg.n_global != partition N");
  C->cfg = *cfg;
  C->L = cfg->n_layers;
  C->n_parts = v0.n_parts;
  C->ldmax = 0;
  for (int l = 0; l <= C->L; ++l) {
    C->F[l] = cfg->width[l];
    C->ld[l] = ld_of(cfg->width[l]);
    if (C->ld[l] > C->ldmax) C->ldmax = C->ld[l];
  }
  C->gcn = cfg->model == 1;
  C->ns = C->gcn ? 1 : 2;
  C->depth = cfg->depth > 1 ? cfg->depth : 1;
  C->nb = (int)C->depth + 1;
  C->woff[1] = 0;
  for (int l = 1; l <= C->L; ++l) C->woff[l + 1] = C->woff[l] + (C->ns * C->F[l - 1] + 1) * C->F[l];
  // N1 traffic rule (gathered row widths per iteration): layer 1 aggregates F_0 forward only
  // (no J^(0), R11) vs F_1 forward + F_1 backward; layers >= 2 aggregate F_in both ways vs F_out.
  for (int l = 1; l <= C->L; ++l) {
    const int64_t fi = C->ld[l - 1], fo = C->ld[l];
    C->tf[l] = (cfg->transform_first == 1 && cfg->gemm != 2) ? (l == 1 ? 2 * fo < fi : fo < fi) : 0;
    if ((knobs().tf_off >> l) & 1) C->tf[l] = 0;  // dev knob PGCN_TF_OFF: layers forced aggregate-first
  }
  C->cl = cfg->train_sparse && !C->tf[C->L] && cfg->model == 0 && cfg->gemm != 2;
  C->P = C->woff[C->L + 1];
  return PGCN_OK;
}

DropSpec drop_spec(const pgcn_ctx* C, int64_t t, int l) {
  DropSpec d{};
  const double p = C->cfg.dropout;
  d.on = p > 0.0;
  d.seed = C->cfg.seed;
  d.key_base = ((uint64_t)t * (uint64_t)(C->L + 1) + (uint64_t)l) * (uint64_t)C->cfg.n_global;
  d.thr = (uint32_t)std::floor(p * 16777216.0 + 0.5);
  d.scale = d.on ? (float)(1.0 / (1.0 - p)) : 1.0f;
  d.width = (int32_t)C->F[l - 1];
  return d;
}

// A failed launch leaves the context's buffers in an unknown state: every later call returns PGCN_ESTATE.
int poison(pgcn_ctx* C, int rc) {
  C->poisoned = 1;
  return rc;
}

int check_cuda(pgcn_ctx* C, const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    C->poisoned = 1;
    return fail(PGCN_ECUDA, "%s: %s", where, cudaGetErrorString(e));
  }
  return PGCN_OK;
}

int expect(pgcn_ctx* C, int64_t t, int kind, int layer, const char* name) {
  if (C->poisoned) return fail(PGCN_ESTATE, "%s: context poisoned by an earlier failure", name);
  if (t != C->exp_t || kind != C->exp_kind || (kind == K_FWD || kind == K_BWD ? layer != C->exp_layer : false)) {
    static const char* kn[] = {"layer_fwd", "loss", "layer_bwd", "update"};
    return fail(PGCN_ESTATE, "%s(t=%lld, layer=%d) out of Alg. 1 order: expected %s(t=%lld, layer=%d)", name,
                (long long)t, layer, kn[C->exp_kind], (long long)C->exp_t, C->exp_layer);
  }
  return PGCN_OK;
}

void advance(pgcn_ctx* C) {
  switch (C->exp_kind) {
    case K_FWD:
      if (C->exp_layer < C->L) ++C->exp_layer;
      else C->exp_kind = K_LOSS;
      break;
    case K_LOSS:
      C->exp_kind = K_BWD;
      C->exp_layer = C->L;
      break;
    case K_BWD:
      if (C->exp_layer > 1) --C->exp_layer;
      else C->exp_kind = K_UPD;
      break;
    default:
      C->exp_kind = K_FWD;
      C->exp_layer = 1;
      ++C->exp_t;
  }
}

inline float* layer_in(PartCtx& p, int l, int b) { return l == 1 ? p.X : p.H[l - 1][b]; }

// Brackets one launch with CUDA events (only when timing is enabled) and charges it with its
// algorithmic bytes / flops.
struct Scope {
  pgcn_ctx* C;
  int k;
  Scope(pgcn_ctx* c, int kind, SpmmBytes sb) : Scope(c, kind, sb.min, 0.0, sb.gather) {}
  Scope(pgcn_ctx* c, int kind, double bytes, double flops = 0.0, double gbytes = -1.0) : C(c), k(kind) {
    if (!C->timing) return;
    KTimer& t = C->kt[k];
    if (t.used + 2 > t.ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      t.ev.push_back(a);
      t.ev.push_back(b);
    }
    cudaEventRecord(t.ev[t.used], C->s);
    t.n += 1;
    t.bytes += bytes;
    t.flops += flops;
    t.gbytes += gbytes >= 0.0 ? gbytes : bytes;
  }
  ~Scope() {
    if (!C->timing) return;
    KTimer& t = C->kt[k];
    cudaEventRecord(t.ev[t.used + 1], C->s);
    t.used += 2;
  }
};

#ifdef PGCN_WITH_NCCL
int nccl_fail(pgcn_ctx* C, ncclResult_t r, const char* where) {
  C->poisoned = 1;
  return fail(PGCN_ENCCL, "%s: %s", where, ncclGetErrorString(r));
}
#endif

// ---------------------------------------------------------------------------------------------------
// Posted exchange (LOOPBACK / NCCL transports).  One code path for both; only the transfer of a
// segment differs (ncclSend/ncclRecv across ranks vs one cudaMemcpyAsync from the sender's buffer into
// the receiver's, both on the comm stream).  Stream/event contract, per layer l:
//   forward  (Alg. 1 l.9-13)  consume: the compute stream waits ev_f_done[l][t-s] (PIPE) before the
//                             install / the layer reads its boundary rows;
//                             post:    pack S_{i,j} rows (compute stream) -> ev_f_pack -> comm stream
//                             transfers into the receivers' rows read at t+s (PIPE) or t (VANILLA, which
//                             then waits at once) -> ev_f_done[l][t].
//   backward (Alg. 1 l.22-27) post:    ev_b_ready (J^(l-1) complete) -> comm stream transfers of the
//                             boundary-row gradients into the owners' recv_b[l][t] -> ev_b_done[l][t];
//                             consume: wait ev_b_done[l][t-s] (PIPE) or [t] (VANILLA), then accumulate.
// Rotation over s + 1 slots makes every buffer's next writer wait (through these events) for its
// last reader: send_f[t] is repacked at t+s+1 after the wait at t+s for ev_f_done[t]; recv_b[t] is
// rewritten at t+s+1 after ev_b_ready, recorded behind the accumulate of t+s that consumed it; the J
// boundary rows sent at t are rewritten at t+s+1, after the wait for ev_b_done[t] at t+s.
namespace {

// destination of the boundary-row features received at (t, l) by hosted partition q, and whether the
// receive goes to the staging buffer (installed at consume time) instead of the consuming rows
void* fwd_dst(pgcn_ctx* C, PartCtx& q, int64_t t, int l) {
  const int64_t ldi = C->ld[l - 1];
  const bool pipe = C->cfg.mode == 1;
  if (staged_recv(C, l)) return q.recv_f[l][l == 1 ? 0 : C->bi(t)];
  if (l == 1) return q.X + q.n_in * ldi;
  if (!pipe) return q.H[l - 1][C->bi(t)] + q.n_in * ldi;
  return q.H[l - 1][C->bi(t + C->depth)] + q.n_in * ldi;  // lands in the buffer read at t + s
}

// Alg. 1 l.12-13 / l.27 transfers of hosted partition i (sender) for one direction.  fwd: i's packed
// S_{i,j} rows -> j's boundary segment for owner i; bwd: i's boundary rows owned by j -> j's message
// rows for i (send order).  NCCL: one grouped send/recv per peer; LOOPBACK: one copy per segment.
int transfer(pgcn_ctx* C, int64_t t, int l, bool fwd) {
  const int64_t ldi = C->ld[l - 1];
  const int64_t eb = C->p16 ? 2 : 4;
  const int b = C->bi(t);
  if (C->hook_spin_ns > 0) spin_ns(C->cs, C->hook_spin_ns);
  if (C->hook_flags & PGCN_XH_NOCOMM) return PGCN_OK;
  if (C->xp == XP_LOOPBACK || C->xp == XP_PUSH) {  // (PUSH: layers whose producer could not push)
    for (auto& pi : C->parts) {
      const int i = pi.part;
      for (auto& pj : C->parts) {
        const int j = pj.part;
        if (j == i) continue;
        if (fwd) {
          const int64_t n = pi.v.send_off[j + 1] - pi.v.send_off[j];
          if (!n) continue;
          const char* src = static_cast<const char*>(pi.send_f[l][l == 1 ? 0 : b]) + eb * pi.v.send_off[j] * ldi;
          char* dst = static_cast<char*>(fwd_dst(C, pj, t, l));
          const int64_t row_b = staged_recv(C, l) ? eb * ldi : 4 * ldi;  // unstaged receives are fp32 rows
          cudaMemcpyAsync(dst + row_b * pj.v.halo_off[i], src, (size_t)(eb * n * ldi), cudaMemcpyDeviceToDevice, C->cs);
          C->xbytes[0] += eb * n * ldi;
        } else {
          const int64_t n = pi.v.halo_off[j + 1] - pi.v.halo_off[j];
          if (!n) continue;
          const char* src = C->p16 ? static_cast<const char*>(pi.send_b[l][b]) + eb * pi.v.halo_off[j] * ldi
                                   : reinterpret_cast<const char*>(pi.J[l - 1][b] + (pi.n_in + pi.v.halo_off[j]) * ldi);
          char* dst = static_cast<char*>(pj.recv_b[l][b]) + eb * pj.v.send_off[i] * ldi;
          cudaMemcpyAsync(dst, src, (size_t)(eb * n * ldi), cudaMemcpyDeviceToDevice, C->cs);
          C->xbytes[1] += eb * n * ldi;
        }
      }
    }
    return PGCN_OK;
  }
#ifdef PGCN_WITH_NCCL
  PartCtx& p = C->parts[0];
  const ncclDataType_t ty = C->p16 ? ncclBfloat16 : ncclFloat;
  ncclResult_t r = ncclGroupStart();
  for (int j = 0; j < C->nranks && r == ncclSuccess; ++j) {
    if (j == C->rank) continue;
    const int64_t ns = p.v.send_off[j + 1] - p.v.send_off[j], nh = p.v.halo_off[j + 1] - p.v.halo_off[j];
    if (fwd) {
      const char* sendb = static_cast<const char*>(p.send_f[l][l == 1 ? 0 : b]);
      char* dst = static_cast<char*>(fwd_dst(C, p, t, l));
      const int64_t row_b = staged_recv(C, l) ? eb * ldi : 4 * ldi;
      if (ns) r = ncclSend(sendb + eb * p.v.send_off[j] * ldi, (size_t)(ns * ldi), ty, j, C->ch, C->cs);
      C->xbytes[0] += eb * ns * ldi;
      if (nh && r == ncclSuccess) r = ncclRecv(dst + row_b * p.v.halo_off[j], (size_t)(nh * ldi), ty, j, C->ch, C->cs);
    } else {
      const char* src = C->p16 ? static_cast<const char*>(p.send_b[l][b]) + eb * p.v.halo_off[j] * ldi
                               : reinterpret_cast<const char*>(p.J[l - 1][b] + (p.n_in + p.v.halo_off[j]) * ldi);
      if (nh) r = ncclSend(src, (size_t)(nh * ldi), ty, j, C->ch, C->cs);
      C->xbytes[1] += eb * nh * ldi;
      if (ns && r == ncclSuccess)
        r = ncclRecv(static_cast<char*>(p.recv_b[l][b]) + eb * p.v.send_off[j] * ldi, (size_t)(ns * ldi), ty, j, C->ch,
                     C->cs);
    }
  }
  ncclResult_t r2 = ncclGroupEnd();
  if (r != ncclSuccess || r2 != ncclSuccess)
    return nccl_fail(C, r != ncclSuccess ? r : r2, fwd ? "halo exchange (fwd)" : "halo exchange (bwd)");
  return PGCN_OK;
#else
  return fail(PGCN_EUNSUPPORTED, "library built without NCCL");
#endif
}

}  // namespace

// N2 fused push (PUSH transport).  Forward: hosted partition p's layer-l output rows in S_{p,j} go
// straight from the producing GEMM's epilogue into every receiver j's rows that layer l + 1 reads at
// t + s (PIPE) / t (VANILLA) -- the same slots the transfer would fill (fwd_dst).  Backward: the
// boundary rows of J^(l-1) go from the producing kernel into their owners' message rows of slot t.
// All partitions are hosted by this context and the compute stream orders every producer before its
// consumer and after the previous reader of the slot (the rotation argument of the posted exchange).
bool fwd_push(pgcn_ctx* C, PartCtx& p, int64_t t, int l, PushSpec& ps) {
  if (!pushing(C) || l >= C->L || p.n_send == 0) return false;
  ps = PushSpec{};
  for (auto& q : C->parts) ps.base[q.part] = static_cast<float*>(fwd_dst(C, q, t, l + 1));
  for (auto& q : C->peer)  // multi-process: the peers' receive rows, mapped over NVLink
    if (q.part != p.part && q.X) ps.base[q.part] = static_cast<float*>(fwd_dst(C, q, t, l + 1));
  ps.ptr = p.inv_ptr;
  ps.pos = p.inv_pos;
  ps.part = p.fpush_part;
  ps.row = p.fpush_row;
  ps.mode = 1;
  C->xbytes[0] += 4 * p.n_send * C->ld[l];
  return true;
}
bool bwd_push(pgcn_ctx* C, PartCtx& p, int64_t t, int l, PushSpec& ps) {
  if (!pushing(C) || l < 2 || p.n_bd == 0) return false;
  ps = PushSpec{};
  for (auto& q : C->parts) ps.base[q.part] = static_cast<float*>(q.recv_b[l][C->bi(t)]);
  for (auto& q : C->peer)
    if (q.part != p.part && q.X) ps.base[q.part] = static_cast<float*>(q.recv_b[l][C->bi(t)]);
  ps.part = p.bpush_part;
  ps.row = p.bpush_row;
  ps.row0 = p.n_in;
  ps.mode = 2;
  C->xbytes[1] += 4 * p.n_bd * C->ld[l - 1];
  return true;
}

// Alg. 1 l.9-13 for every hosted partition: consume the exchange of t - s (PIPE) and post this
// iteration's, consumed at t + s (PIPE) or right away (VANILLA).  X is exchanged once (R10).
// n_valid[i]: rows of partition i's layer input that hold data this iteration.
int post_fwd(pgcn_ctx* C, int64_t t, int l, const Launch& Lk, int64_t* n_valid) {
  const bool pipe = C->cfg.mode == 1;
  const int64_t s = C->depth;
  const int b = C->bi(t), bp = C->bi(t - 1), bs = C->bi(t - s);
  const int64_t ldi = C->ld[l - 1];
  const bool staged = staged_recv(C, l);
  const bool skip_wait = (C->hook_flags & PGCN_XH_SKIP_F_WAIT) != 0;
  // consume (PIPE): the exchange posted at t - s (layer 1: the one X exchange of t = 1)
  if (pipe && t > s) {
    if (!skip_wait) cudaStreamWaitEvent(C->s, C->ev_f_done[l][l == 1 ? C->bi(1) : bs], 0);
    if (staged && (l >= 2 || t == s + 1)) {
      const bool ema = C->cfg.smooth_f && l >= 2;
      const bool first = ema && C->cfg.ema_init == 0 && t == s + 1;
      for (auto& p : C->parts) {
        if (p.n_bd == 0) continue;
        float* dst = layer_in(p, l, b) + p.n_in * ldi;
        const void* src = p.recv_f[l][l == 1 ? 0 : bs];
        const float* prev = p.H[l - 1][bp] + p.n_in * ldi;  // (l >= 2) previous smoothed value
        Scope sc(C, PGCN_K_GATHER, ((C->p16 ? 6.0 : 8.0) + (ema && !first ? 4.0 : 0.0)) * C->F[l - 1] * p.n_bd);
        if (C->p16) {
          install_bf16(Lk, src, p.n_bd, ldi, dst, prev, (float)C->cfg.gamma, ema && !first);
        } else {
          SegTable tab{};
          tab.n_seg = 1;
          tab.off[1] = p.n_bd;
          tab.base[0] = static_cast<const float*>(src);
          gather_rows(Lk, tab, nullptr, p.n_bd, ldi, dst, prev, (float)C->cfg.gamma, ema, first);
        }
      }
    }
  }
  // post
  if (l >= 2 && C->fpushed[l] == t) {  // PUSH: the producer of H^(l-1) already stored the rows (N2)
    cudaEventRecord(C->ev_f_done[l][b], C->s);
  } else if (l >= 2 || t == 1) {
    // lean: one send slot -- the transfer of t - 1 must have read it (PIPE s = 1 already waited above)
    if (C->cfg.lean && l >= 2 && t > 1) cudaStreamWaitEvent(C->s, C->ev_f_done[l][C->bi(t - 1)], 0);
    for (auto& p : C->parts) {
      if (p.n_send == 0) continue;
      const float* Hin = layer_in(p, l, b);
      void* dst = p.send_f[l][l == 1 ? 0 : b];
      Scope sc(C, PGCN_K_GATHER, ((C->p16 ? 6.0 : 8.0) * C->F[l - 1] + 4.0) * p.n_send);
      if (C->p16) {
        pack_rows_bf16(Lk, Hin, p.send_idx, p.n_send, ldi, dst);
      } else {
        SegTable src{};
        src.n_seg = 1;
        src.off[1] = p.n_send;
        src.base[0] = Hin;
        gather_rows(Lk, src, p.send_idx, p.n_send, ldi, static_cast<float*>(dst), nullptr, 0.f, 0, 0);
      }
    }
    cudaEventRecord(C->ev_f_pack[l], C->s);
    cudaStreamWaitEvent(C->cs, C->ev_f_pack[l], 0);
    int rc = transfer(C, t, l, true);
    if (rc) return rc;
    cudaEventRecord(C->ev_f_done[l][b], C->cs);
    if (!pipe) {
      if (!skip_wait) cudaStreamWaitEvent(C->s, C->ev_f_done[l][b], 0);
      if (staged && (l >= 2 || t == 1))
        for (auto& p : C->parts) {  // VANILLA bf16: widen the fresh rows into the layer input
          if (p.n_bd == 0) continue;
          Scope sc(C, PGCN_K_GATHER, 6.0 * C->F[l - 1] * p.n_bd);
          install_bf16(Lk, p.recv_f[l][l == 1 ? 0 : b], p.n_bd, ldi, layer_in(p, l, b) + p.n_in * ldi, nullptr, 0.f, 0);
        }
    }
  }
  for (size_t i = 0; i < C->parts.size(); ++i)
    n_valid[i] = (pipe && l == 1 && t <= s) ? C->parts[i].n_in : C->parts[i].n_all;  // X rows not in yet (l.6)
  return PGCN_OK;
}

// Alg. 1 l.22-27 for every hosted partition (l >= 2): post the boundary-row gradients of J^(l-1)
// (slot t) to their owners and make the compute stream wait for the messages to accumulate now
// (PIPE: those posted at t - s).  have: whether there is anything to accumulate this iteration.
int post_bwd(pgcn_ctx* C, int64_t t, int l, const Launch& Lk, bool* have) {
  const bool pipe = C->cfg.mode == 1;
  const int64_t s = C->depth;
  const int b = C->bi(t);
  const int64_t ldi = C->ld[l - 1];
  if (C->p16)
    for (auto& p : C->parts) {
      if (p.n_bd == 0) continue;
      Scope sc(C, PGCN_K_GATHER, 6.0 * C->F[l - 1] * p.n_bd);
      pack_rows_bf16(Lk, p.J[l - 1][b] + p.n_in * ldi, nullptr, p.n_bd, ldi, p.send_b[l][b]);
    }
  if (C->bpushed[l] == t) {  // PUSH: the producer of J^(l-1) already stored the boundary rows (N2)
    cudaEventRecord(C->ev_b_done[l][b], C->s);
  } else {
    cudaEventRecord(C->ev_b_ready[l], C->s);
    cudaStreamWaitEvent(C->cs, C->ev_b_ready[l], 0);
    int rc = transfer(C, t, l, false);
    if (rc) return rc;
    cudaEventRecord(C->ev_b_done[l][b], C->cs);
  }
  *have = !pipe || t > s;
  if (*have && !(C->hook_flags & PGCN_XH_SKIP_B_WAIT)) cudaStreamWaitEvent(C->s, C->ev_b_done[l][pipe ? C->bi(t - s) : b], 0);
  return PGCN_OK;
}

}  // namespace
}  // namespace pgcn

using namespace pgcn;

pgcn::Launch pgcn_ctx::launch() {
  pgcn::Launch L{s, &launches};
  if (timing) {
    L.mark = tile_mark;
    L.mctx = this;
  }
  return L;
}

extern "C" int64_t pgcn_param_count(const pgcn_config* cfg) { return cfg ? param_count(cfg) : -1; }

extern "C" int pgcn_workspace_bytes(const pgcn_partitioning* part, const int32_t* local, int32_t n_local,
                                    const pgcn_config* cfg, size_t* bytes) {
  if (!bytes) return fail(PGCN_EINVAL, "bytes is NULL");
  pgcn_ctx C;
  int rc = init_ctx_shapes(&C, part, local, n_local, cfg, nullptr);
  if (rc == PGCN_EUNSUPPORTED && n_local == 1) {  // one partition of a multi-process run
    pgcn_part_view v0;
    if (pgcn_partition_view(part, local[0], &v0) == PGCN_OK && v0.n_parts > 1) {
      pgcn_comm cm{local[0], v0.n_parts, "x", "x"};
      rc = init_ctx_shapes(&C, part, local, n_local, cfg, &cm);
    }
  }
  if (rc) return rc;
  Arena A;
  rc = layout(&C, part, local, n_local, A);
  if (rc) return rc;
  *bytes = A.off + 256;
  return PGCN_OK;
}

extern "C" int pgcn_ctx_create(const pgcn_partitioning* part, const int32_t* local, int32_t n_local,
                               const pgcn_config* cfg, const pgcn_comm* comm, void* ws, size_t ws_bytes,
                               void* stream, pgcn_ctx** out) {
  if (!out) return fail(PGCN_EINVAL, "out is NULL");
  *out = nullptr;
  pgcn_ctx* C = new (std::nothrow) pgcn_ctx();
  if (!C) return fail(PGCN_ENOMEM, "host allocation failed");
  int rc = init_ctx_shapes(C, part, local, n_local, cfg, comm);
  if (rc) { delete C; return rc; }
  Arena dry;
  rc = layout(C, part, local, n_local, dry);
  if (rc) { delete C; return rc; }
  if (!ws || ((uintptr_t)ws & 255)) { delete C; return fail(PGCN_EINVAL, "workspace NULL or not 256-byte aligned"); }
  if (ws_bytes < dry.off) {
    delete C;
    return fail(PGCN_ENOMEM, "workspace too small: %zu < %zu bytes", ws_bytes, dry.off);
  }
  Arena A;
  A.base = static_cast<char*>(ws);
  layout(C, part, local, n_local, A);
  C->ws = ws;
  C->ws_bytes = ws_bytes;
  C->part = part;
  C->s = static_cast<cudaStream_t>(stream);
  cudaStream_t s = C->s;
  cudaMemsetAsync(ws, 0, A.off, s);
  // uploads (host arrays are borrowed; synchronise before returning)
  for (int i = 0; i < n_local; ++i) {
    PartCtx& p = C->parts[i];
    const pgcn_part_view& v = p.v;
    std::vector<int64_t> gid(p.n_all);
    std::memcpy(gid.data(), v.inner_gid, sizeof(int64_t) * p.n_in);
    std::memcpy(gid.data() + p.n_in, v.halo_gid, sizeof(int64_t) * p.n_bd);
    // halo_map: boundary row r (owner j) -> owner's local inner id (position in V_j, ascending gid)
    std::vector<int32_t> hmap(p.n_bd), mmap(p.n_send);
    for (int j = 0; j < C->n_parts; ++j) {
      pgcn_part_view vj;
      pgcn_partition_view(part, j, &vj);
      for (int64_t r = v.halo_off[j]; r < v.halo_off[j + 1]; ++r) {
        const int64_t g = v.halo_gid[r];
        const int64_t* it = std::lower_bound(vj.inner_gid, vj.inner_gid + vj.n_inner, g);
        hmap[r] = (int32_t)(it - vj.inner_gid);
      }
      // msg_map: my send position k for peer j -> row of peer j's J buffer (its boundary row)
      for (int64_t k = v.send_off[j]; k < v.send_off[j + 1]; ++k)
        mmap[k] = (int32_t)(vj.n_inner + vj.halo_off[p.part] + (k - v.send_off[j]));
    }
    cudaMemcpyAsync(p.rp, v.row_ptr, sizeof(int64_t) * (p.n_in + 1), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.col, v.col_idx, sizeof(int32_t) * p.nnz, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.inv_deg, v.inv_deg, sizeof(float) * p.n_in, cudaMemcpyHostToDevice, s);
    std::vector<float> sym;
    if (p.sym) {  // d~^-1/2 = 1/sqrt(d + 1), correctly rounded from double (App. A.1, R26)
      sym.resize(p.n_all);
      for (int64_t r = 0; r < p.n_all; ++r) sym[r] = (float)(1.0 / std::sqrt((double)v.deg[r] + 1.0));
      cudaMemcpyAsync(p.sym, sym.data(), sizeof(float) * p.n_all, cudaMemcpyHostToDevice, s);
    }
    cudaMemcpyAsync(p.trp, v.t_row_ptr, sizeof(int64_t) * (p.n_all + 1), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.tcol, v.t_col_idx, sizeof(int32_t) * p.nnz, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.gid, gid.data(), sizeof(int64_t) * p.n_all, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.send_idx, v.send_idx, sizeof(int32_t) * p.n_send, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.inv_ptr, v.inv_ptr, sizeof(int64_t) * (p.n_in + 1), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.inv_pos, v.inv_pos, sizeof(int32_t) * p.n_send, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.halo_map, hmap.data(), sizeof(int32_t) * p.n_bd, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(p.msg_map, mmap.data(), sizeof(int32_t) * p.n_send, cudaMemcpyHostToDevice, s);
    std::vector<int32_t> fpp, fpr, bpp, bpr;
    if (pushing(C)) {  // N2 destinations: send position k of peer j -> j's boundary row; boundary row
      fpp.resize(p.n_send);  // r of owner j -> j's message row (send order)
      fpr.resize(p.n_send);
      bpp.resize(p.n_bd);
      bpr.resize(p.n_bd);
      for (int j = 0; j < C->n_parts; ++j) {
        pgcn_part_view vj;
        pgcn_partition_view(part, j, &vj);
        for (int64_t k = v.send_off[j]; k < v.send_off[j + 1]; ++k) {
          fpp[k] = j;
          fpr[k] = (int32_t)(vj.halo_off[p.part] + (k - v.send_off[j]));
        }
        for (int64_t r = v.halo_off[j]; r < v.halo_off[j + 1]; ++r) {
          bpp[r] = j;
          bpr[r] = (int32_t)(vj.send_off[p.part] + (r - v.halo_off[j]));
        }
      }
      cudaMemcpyAsync(p.fpush_part, fpp.data(), sizeof(int32_t) * p.n_send, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(p.fpush_row, fpr.data(), sizeof(int32_t) * p.n_send, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(p.bpush_part, bpp.data(), sizeof(int32_t) * p.n_bd, cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(p.bpush_row, bpr.data(), sizeof(int32_t) * p.n_bd, cudaMemcpyHostToDevice, s);
    }
    for (int w = 0; w < 2; ++w) {
      const TileSet* ts = p.ts[w];
      if (!ts) continue;
      const TileDev& d = p.td[w];
      cudaMemcpyAsync(const_cast<int32_t*>(d.rb_ptr), ts->rb_ptr.data(), sizeof(int32_t) * (ts->n_rb + 1),
                      cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(const_cast<int32_t*>(d.order), ts->order.data(), sizeof(int32_t) * ts->n_rb,
                      cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(const_cast<int32_t*>(d.tile_col), ts->tile_col.data(), sizeof(int32_t) * ts->n_tiles,
                      cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(const_cast<uint64_t*>(d.mask), ts->mask.data(), sizeof(uint64_t) * ts->mask.size(),
                      cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(const_cast<int64_t*>(d.lrp), ts->lrp.data(), sizeof(int64_t) * (ts->n_rows + 1),
                      cudaMemcpyHostToDevice, s);
      cudaMemcpyAsync(const_cast<int32_t*>(d.lcol), ts->lcol.data(), sizeof(int32_t) * ts->nnz_light,
                      cudaMemcpyHostToDevice, s);
    }
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      delete C;
      return fail(PGCN_ECUDA, "pgcn_ctx_create upload: %s", cudaGetErrorString(e));
    }
  }
  if (cudaStreamCreateWithFlags(&C->cps, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_x_free, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_lab_free, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&C->ev_in_ready, cudaEventDisableTiming) != cudaSuccess) {
    delete C;
    return fail(PGCN_ECUDA, "copy stream / event creation failed");
  }
  if (C->posted) {  // comm stream (high priority, App. F) and the exchange events
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&C->cs, cudaStreamNonBlocking, hi) != cudaSuccess) {
      delete C;
      return fail(PGCN_ECUDA, "comm stream creation failed");
    }
    for (int l = 1; l <= C->L; ++l) {
      cudaEventCreateWithFlags(&C->ev_f_pack[l], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&C->ev_b_ready[l], cudaEventDisableTiming);
      for (int b = 0; b < C->nb; ++b) {
        cudaEventCreateWithFlags(&C->ev_f_done[l][b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&C->ev_b_done[l][b], cudaEventDisableTiming);
      }
    }
  }
  if (C->nccl) {
#ifdef PGCN_WITH_NCCL
    ncclUniqueId ih, ir;
    std::memcpy(&ih, comm->nccl_id_halo, sizeof(ih));
    std::memcpy(&ir, comm->nccl_id_reduce, sizeof(ir));
    ncclResult_t nr = ncclGroupStart();
    if (nr == ncclSuccess) nr = ncclCommInitRank(&C->ch, C->nranks, ih, C->rank);
    if (nr == ncclSuccess) nr = ncclCommInitRank(&C->cr, C->nranks, ir, C->rank);
    ncclResult_t ne = ncclGroupEnd();
    if (nr != ncclSuccess || ne != ncclSuccess) {
      const char* msg = ncclGetErrorString(nr != ncclSuccess ? nr : ne);
      delete C;
      return fail(PGCN_ENCCL, "ncclCommInitRank: %s", msg);
    }
#endif
  }
  rc = check_cuda(C, "pgcn_ctx_create");
  if (rc) { delete C; return rc; }
  *out = C;
  return PGCN_OK;
}

extern "C" int pgcn_ctx_destroy(pgcn_ctx* C) {
  if (!C) return PGCN_OK;
  if (C->s) cudaStreamSynchronize(C->s);
  if (C->cs) cudaStreamSynchronize(C->cs);
  if (C->cps) cudaStreamSynchronize(C->cps);
  delete C;
  return PGCN_OK;
}

extern "C" int pgcn_set_inputs(pgcn_ctx* C, int32_t local, const float* X, const void* labels,
                               const uint8_t* train_mask) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  if (C->poisoned) return fail(PGCN_ESTATE, "context poisoned");
  if (local < 0 || local >= (int)C->parts.size()) return fail(PGCN_EINVAL, "local index out of range");
  PartCtx& p = C->parts[local];
  if (p.n_in > 0 && (!X || !labels || !train_mask)) return fail(PGCN_EINVAL, "null input");
  if (p.n_in > 0) {
    cudaMemcpy2DAsync(p.X, sizeof(float) * C->ld[0], X, sizeof(float) * C->F[0], sizeof(float) * C->F[0], p.n_in,
                      cudaMemcpyDefault, C->s);
    const size_t lb = C->cfg.loss == 0 ? sizeof(int32_t) * p.n_in : (size_t)p.n_in * C->F[C->L];
    cudaMemcpyAsync(p.labels, labels, lb, cudaMemcpyDefault, C->s);
    cudaMemcpyAsync(p.train, train_mask, (size_t)p.n_in, cudaMemcpyDefault, C->s);
  }
  if (C->cfg.train_sparse) {  // N1(ii): train row list and P_i^T restricted to train sources
    const Launch Lk = C->launch();
    build_train_rows(Lk, p.train, p.n_in, p.trp, p.tcol, p.n_all, p.tr_list, p.tr_count, p.tr_counts, p.trp_tr,
                     p.tcol_tr, C->sp_tmp, (size_t)C->sp_tmp_bytes);
    int64_t h[2] = {0, 0};
    cudaMemcpyAsync(&h[0], p.tr_count, sizeof(int64_t), cudaMemcpyDeviceToHost, C->s);
    cudaMemcpyAsync(&h[1], p.trp_tr + p.n_all, sizeof(int64_t), cudaMemcpyDeviceToHost, C->s);
    cudaStreamSynchronize(C->s);  // sizes of the last layer's launches (documented: synchronous here)
    p.n_tr = h[0];
    p.nnz_tr = h[1];
    if (C->cfg.lean && C->cl && p.n_tr > std::min(p.n_in, (int64_t)C->cfg.n_train_global))
      return fail(PGCN_EINVAL, "lean mode: partition %d has %lld train rows > n_train_global %lld", p.part,
                  (long long)p.n_tr, (long long)C->cfg.n_train_global);
    p.last_sparse = C->cl || !(p.ts[0] && p.ts[1] && 4 * p.n_tr > p.n_in);
    if (C->cl) {  // compact train rows: positions, P_i^T restricted columns -> positions, labels, inv_deg
      compact_train_setup(Lk, p.tr_list, p.n_tr, p.n_in, p.tr_pos, p.tcol_tr, p.nnz_tr);
      const int64_t lw = C->cfg.loss == 0 ? (int64_t)sizeof(int32_t) : C->F[C->L];
      gather_bytes(Lk, p.labels, p.tr_list, p.n_tr, lw, p.lab_tr);
      gather_bytes(Lk, p.inv_deg, p.tr_list, p.n_tr, (int64_t)sizeof(float), p.invdeg_tr);
    }
  }
  C->inputs_set = 1;
  return check_cuda(C, "pgcn_set_inputs");
}

extern "C" int pgcn_stage_inputs(pgcn_ctx* C, int32_t local, const float* X, int64_t ld_x, const void* labels,
                                 const uint8_t* train_mask) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  if (C->poisoned) return fail(PGCN_ESTATE, "context poisoned");
  if (!C->inputs_set) return fail(PGCN_ESTATE, "pgcn_stage_inputs before pgcn_set_inputs");
  if (local < 0 || local >= (int)C->parts.size()) return fail(PGCN_EINVAL, "local index out of range");
  PartCtx& p = C->parts[local];
  if (p.n_in == 0) return PGCN_OK;
  if (!X || !labels || !train_mask) return fail(PGCN_EINVAL, "null input");
  if (ld_x != C->F[0] && ld_x != C->ld[0]) return fail(PGCN_EINVAL, "ld_x must be F_0 or round_up(F_0, 4)");
  // X after the in-flight iteration's last read of X; labels / mask after its loss
  cudaStreamWaitEvent(C->cps, C->ev_x_free, 0);
  if (ld_x == C->ld[0])  // the context's padded layout: one contiguous copy (full PCIe rate)
    cudaMemcpyAsync(p.X, X, sizeof(float) * C->ld[0] * p.n_in, cudaMemcpyHostToDevice, C->cps);
  else
    cudaMemcpy2DAsync(p.X, sizeof(float) * C->ld[0], X, sizeof(float) * C->F[0], sizeof(float) * C->F[0], p.n_in,
                      cudaMemcpyHostToDevice, C->cps);
  cudaStreamWaitEvent(C->cps, C->ev_lab_free, 0);
  const size_t lb = C->cfg.loss == 0 ? sizeof(int32_t) * p.n_in : (size_t)p.n_in * C->F[C->L];
  cudaMemcpyAsync(p.labels, labels, lb, cudaMemcpyHostToDevice, C->cps);
  cudaMemcpyAsync(p.train, train_mask, (size_t)p.n_in, cudaMemcpyHostToDevice, C->cps);
  cudaEventRecord(C->ev_in_ready, C->cps);
  C->in_pending = 1;
  return check_cuda(C, "pgcn_stage_inputs");
}

extern "C" int pgcn_layer_fwd(pgcn_ctx* C, int64_t t, int32_t l, const float* params) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_FWD, l, "pgcn_layer_fwd");
  if (rc) return rc;
  if (C->ipc_push && C->n_imported < C->nranks - 1)
    return fail(PGCN_ESTATE, "PUSH across ranks: pgcn_ipc_import every peer's workspace first (%d of %d)",
                C->n_imported, C->nranks - 1);
  if (!params) return fail(PGCN_EINVAL, "params is NULL");
  const Launch Lk = C->launch();
  const int b = C->bi(t), bp = C->bi(t - 1), bs = C->bi(t - C->depth);
  const bool pipe = C->cfg.mode == 1;
  const int64_t ldi = C->ld[l - 1], ldo = C->ld[l];
  const float* Wext = params + C->woff[l];
  if (l == 1 && C->cfg.staleness_stats)
    cudaMemsetAsync(C->diag, 0, sizeof(double) * 2 * (PGCN_MAX_LAYERS + 1), C->s);
  const bool tcg = C->cfg.gemm != 2;
  const int bf = C->cfg.gemm == 1;
  // algorithmic SpMM bytes: gathered rows (fp32, or bf16 in the gather tier) and, in the bf16 tier,
  // the rounding pass over the table (read fp32, write bf16)
  auto gat = [&](double F, double e) { return (C->cfg.gather ? 2.0 : 4.0) * F * e; };
  auto cvt = [&](double F, double rows) { return C->cfg.gather ? 6.0 * F * rows : 0.0; };
  const int kbk = bf ? 64 : 32;
  if (tcg) {
    Scope sc(C, PGCN_K_GEMM_FWD, 0.0);
    if (bf)
      tc_wprep_bf16(Wext, (int)C->F[l - 1], (int)C->F[l], (int)C->Fp[l], (int)C->Kp[l], (int)C->Kq[l], C->ns,
                    C->WT_hi[l], C->Wp_hi[l], C->WJ_hi[l], C->s);
    else
      tc_wprep(Wext, (int)C->F[l - 1], (int)C->F[l], (int)C->Fp[l], (int)C->Kp[l], (int)C->Kq[l], C->ns, C->WT_hi[l],
               C->WT_lo[l], C->Wp_hi[l], C->Wp_lo[l], C->WJ_hi[l], C->WJ_lo[l], C->s);
    ++C->launches;
  }
  if (l == 1 && C->in_pending) {  // streamed inputs of this iteration (pgcn_stage_inputs)
    cudaStreamWaitEvent(C->s, C->ev_in_ready, 0);
    C->in_pending = 0;
  }
  int64_t nv_posted[PGCN_MAX_PARTS];
  if (C->posted && (rc = post_fwd(C, t, l, Lk, nv_posted))) return rc;
  for (auto& p : C->parts) {
    float* Hin = layer_in(p, l, b);
    // N1(ii): the last layer's aggregation only on train rows (the loss reads Y^(L) only there)
    const bool sp = C->cfg.train_sparse && l == C->L && p.last_sparse;
    const int32_t* rl = sp ? p.tr_list : nullptr;
    const int64_t nr = sp ? p.n_tr : p.n_in;
    const double nz = sp ? (double)p.nnz_tr : (double)p.nnz;
    // gathered bytes of e edges at width F: per-edge model, or the tile path's traffic when it runs
    // table of nv rows at width F, e edges, `rest` = index / output / epilogue bytes
    auto sb = [&](double F, double nv, double e, double rest) { return SpmmBytes{gat(F, nv) + rest, gat(F, e) + rest}; };
    // S1 / S2: boundary rows of the layer input (Alg. 1 l.9-13)
    int64_t n_valid = p.n_all;
    if (C->posted) {
      n_valid = nv_posted[&p - C->parts.data()];
    } else if (C->n_parts > 1 && p.n_bd > 0) {  // local transport: device gather from the owners
      bool do_install = false, ema = false, first = false;
      const float* prev = nullptr;
      SegTable src{};
      src.n_seg = C->n_parts;
      for (int j = 0; j <= C->n_parts; ++j) src.off[j] = p.v.halo_off[j];
      if (l == 1) {
        // X is constant: one exchange at t = 1, consumed at t = 1 (VANILLA) or t = 1 + s (PIPE) (R10);
        // until then X's boundary rows are not valid (0, l.6) -- the same n_valid as the posted transports
        do_install = pipe ? t == 1 + C->depth : t == 1;
        if (pipe && t <= C->depth) n_valid = p.n_in;
        for (int j = 0; j < C->n_parts; ++j) src.base[j] = C->parts[j].X;
      } else {
        const int sb = pipe ? bs : b;  // owners' layer output of t - s (PIPE) or t (VANILLA)
        do_install = pipe ? t > C->depth : true;
        for (int j = 0; j < C->n_parts; ++j) src.base[j] = C->parts[j].H[l - 1][sb];
        if (pipe && C->cfg.smooth_f) {
          ema = true;
          first = C->cfg.ema_init == 0 && t == C->depth + 1;
          prev = p.H[l - 1][bp] + p.n_in * ldi;
        }
      }
      if (do_install) {
        const double F = (double)C->F[l - 1];
        Scope sc(C, PGCN_K_GATHER, (8.0 + (ema ? 4.0 : 0.0)) * F * p.n_bd + 4.0 * p.n_bd);
        gather_rows(Lk, src, p.halo_map, p.n_bd, ldi, Hin + p.n_in * ldi, prev, (float)C->cfg.gamma, ema, first);
      }
    }
    // N4: ||boundary rows used - owners' fresh rows||^2 (local transport only)
    if (C->cfg.staleness_stats && C->xp != XP_NCCL && C->n_parts > 1 && p.n_bd > 0) {
      SegTable fresh{};
      fresh.n_seg = C->n_parts;
      for (int j = 0; j <= C->n_parts; ++j) fresh.off[j] = p.v.halo_off[j];
      for (int j = 0; j < C->n_parts; ++j) fresh.base[j] = l == 1 ? C->parts[j].X : C->parts[j].H[l - 1][b];
      stale_err(Lk, fresh, p.halo_map, nullptr, nullptr, Hin + p.n_in * ldi, p.n_bd, ldi, C->F[l - 1], C->diag + l);
    }
    // S3: dropout after the exchange (App. F), aggregation
    const double Fi = (double)C->F[l - 1], Fo = (double)C->F[l];
    const float* D = Hin;
    if (C->cfg.dropout > 0.0 || C->gcn) {  // GCN-sym: D' = d~^-1/2 o dropout(H) (the right factor of P)
      Scope sc(C, PGCN_K_DROPOUT, 8.0 * Fi * p.n_all + 8.0 * p.n_all + (C->gcn ? 4.0 * p.n_all : 0.0));
      dropout_fwd(Lk, Hin, p.D[l], ldi, p.n_all, n_valid, p.gid, drop_spec(C, t, l), p.sym);
      D = p.D[l];
    }
    p.n_valid[l] = n_valid;
    float* out = l < C->L ? p.H[l][b] : p.logits;
    const float* bias = Wext + C->ns * C->F[l - 1] * C->F[l];
    if (C->gcn) {
      // GCN-sym (App. A.1, R26): Y = d~^-1/2 o (A + I) D' W + b
      if (C->tf[l]) {  // N1: T = D' W over the valid local rows, then H = act(d~^-1/2 o (A + I) T + b)
        {
          Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * n_valid * (Fi + Fo), 2.0 * n_valid * Fi * Fo);
          if (tc_fwd_1seg(Lk, D, n_valid, ldi, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], C->Fp[l], 0, C->F[l], p.T[l],
                          ldo, nullptr, nullptr, 0, 0, bf))
            return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM (T) failed (layer %d)", l);
        }
        Scope sc(C, PGCN_K_SPMM_FWD, sb(Fo, n_valid, nz + nr, cvt(Fo, n_valid) + 4.0 * nz + 8.0 * (nr + 1) + 4.0 * nr +
                                         4.0 * Fo * nr));
        if ((rc = spmm_fwd(Lk, p.rp, p.col, p.sym, p.T[l], ldo, nr, n_valid, out, C->work, 1, bias, C->F[l], l < C->L,
                 p.n_all, p.G16, rl,
                 (int64_t)nz, p.tiles(0), p.T16))) return poison(C, rc);
        continue;
      }
      {
        Scope sc(C, PGCN_K_SPMM_FWD, sb(Fi, n_valid, nz + nr, cvt(Fi, n_valid) + 4.0 * nz + 8.0 * (nr + 1) + 4.0 * nr +
                                         4.0 * Fi * nr));
        if ((rc = spmm_fwd(Lk, p.rp, p.col, p.sym, D, ldi, nr, n_valid, p.Z[l], C->work, 1, nullptr, 0, 0, p.n_all, p.G16, rl,
                 (int64_t)nz, p.tiles(0), p.T16))) return poison(C, rc);
      }
      Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * p.n_in * (Fi + Fo) + 4.0 * (Fi + 1) * Fo, 2.0 * p.n_in * (Fi + 1) * Fo);
      PushSpec ps;
      const bool psh = fwd_push(C, p, t, l, ps);
      if (tc_fwd_1seg(Lk, p.Z[l], p.n_in, ldi, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], C->Fp[l], 0, C->F[l], out, ldo,
                      bias, nullptr, 0, l < C->L, bf, psh ? &ps : nullptr))
        return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM launch failed (layer %d)", l);
      continue;
    }
    if (C->tf[l]) {
      // N1: T = D W_neigh (all valid local rows), S = inv_deg o P_i T, Y = D_in W_self + S + b
      {
        Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * n_valid * (Fi + Fo), 2.0 * n_valid * Fi * Fo);
        if (tc_fwd_1seg(Lk, D, n_valid, ldi, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], 2 * C->Fp[l], 0, C->F[l],
                        p.T[l], ldo, nullptr, nullptr, 0, 0, bf))
          return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM (T) failed (layer %d)", l);
      }
      {
        Scope sc(C, PGCN_K_SPMM_FWD, sb(Fo, n_valid, nz, cvt(Fo, n_valid) + 4.0 * nz + 8.0 * (nr + 1) + 4.0 * nr + 4.0 * Fo * nr));
        if ((rc = spmm_fwd(Lk, p.rp, p.col, p.inv_deg, p.T[l], ldo, nr, n_valid, p.Z[l], C->work, 0, nullptr, 0, 0, p.n_all,
                 p.G16, rl,
                 (int64_t)nz, p.tiles(0), p.T16))) return poison(C, rc);
      }
      {
        Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * p.n_in * (Fi + 2 * Fo), 2.0 * p.n_in * Fi * Fo);
        PushSpec ps;
        const bool psh = fwd_push(C, p, t, l, ps);
        if (tc_fwd_1seg(Lk, D, p.n_in, ldi, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], 2 * C->Fp[l],
                        (int)(C->Fp[l] / kbk), C->F[l], out, ldo, bias, p.Z[l], ldo, l < C->L, bf,
                        psh ? &ps : nullptr))
          return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM (self) failed (layer %d)", l);
      }
      continue;
    }
    const bool cl = C->cl && l == C->L;  // compact train rows (pgcn_ctx::cl)
    {
      Scope sc(C, PGCN_K_SPMM_FWD, sb(Fi, n_valid, nz, cvt(Fi, n_valid) + 4.0 * nz + 8.0 * (nr + 1) + 4.0 * nr + 4.0 * Fi * nr));
      if ((rc = spmm_fwd(Lk, p.rp, p.col, p.inv_deg, D, ldi, nr, n_valid, p.Z[l], C->work, 0, nullptr, 0, 0, p.n_all, p.G16, rl,
                 (int64_t)nz, p.tiles(0), p.T16, cl))) return poison(C, rc);
    }
    if (cl) {  // Z rows are compact; gather the train rows of D, Y_tr = [Z | D_tr] W + b, logits scattered
      SegTable tab{};
      tab.base[0] = D;
      tab.off[0] = 0;
      tab.off[1] = p.n_tr;
      tab.n_seg = 1;
      Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * p.n_tr * (3 * Fi + 2 * Fo) + 4.0 * (2 * Fi + 1) * Fo,
               2.0 * p.n_tr * (2 * Fi + 1) * Fo);
      gather_rows(Lk, tab, p.tr_list, p.n_tr, ldi, p.Dtr, nullptr, 0.f, 0, 0);
      if (p.n_tr > 0 && gemm_fwd_tc(Lk, p.Z[l], p.Dtr, ldi, p.n_tr, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], bias,
                                    C->F[l], p.Ytr, ldo, 0, bf))
        return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM launch failed (layer %d)", l);
      if (p.logits) scatter_rows(Lk, p.Ytr, p.tr_list, p.n_tr, ldo, p.logits);  // (lean: train rows only, in Y_tr)
      continue;
    }
    // S4: Y = [Z | D] W + b, ReLU on hidden layers
    {
      Scope sc(C, PGCN_K_GEMM_FWD, 4.0 * p.n_in * (2 * Fi + Fo) + 4.0 * (2 * Fi + 1) * Fo,
               2.0 * p.n_in * (2 * Fi + 1) * Fo);
      if (tcg) {
        PushSpec ps;
        const bool psh = fwd_push(C, p, t, l, ps);
        if (gemm_fwd_tc(Lk, p.Z[l], D, ldi, p.n_in, C->F[l - 1], C->WT_hi[l], C->WT_lo[l], bias, C->F[l], out, ldo,
                        l < C->L, bf, psh ? &ps : nullptr))
          return fail(PGCN_ECUDA, "pgcn_layer_fwd: tensor-core GEMM launch failed (layer %d)", l);
      } else {
        gemm_fwd_f32(Lk, p.Z[l], D, ldi, p.n_in, C->F[l - 1], Wext, C->F[l], out, ldo, l < C->L);
      }
    }
  }
  // X's last reader this iteration: layer 1's dropout (with p = 0 GraphSAGE reads X itself later, in
  // layer 1's weight gradient -- recorded in pgcn_layer_bwd)
  if (l == 1 && (C->cfg.dropout > 0.0 || C->gcn)) cudaEventRecord(C->ev_x_free, C->s);
  // PUSH: layer l's output rows were stored into the receivers by its GEMM epilogue (GCN-sym transform-
  // first layers produce H in the SpMM and SIMT GEMMs have no push: those layers keep pack + transfer)
  if (fwd_push_capable(C, l)) C->fpushed[l + 1] = t;
  rc = check_cuda(C, "pgcn_layer_fwd");
  if (rc) return rc;
  advance(C);
  return PGCN_OK;
}

extern "C" int pgcn_loss(pgcn_ctx* C, int64_t t, float* loss_dev) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_LOSS, 0, "pgcn_loss");
  if (rc) return rc;
  const Launch Lk = C->launch();
  const int L = C->L;
  for (size_t i = 0; i < C->parts.size(); ++i) {
    PartCtx& p = C->parts[i];
    if (C->cl) {  // compact train rows: every row of Y_tr is a train row; M rows compact too
      Scope sc(C, PGCN_K_LOSS, 8.0 * p.n_tr * C->F[L] + 8.0 * p.n_tr);
      loss_rows(Lk, C->cfg.loss, p.Ytr, p.n_tr, C->F[L], C->ld[L], p.lab_tr, nullptr, (double)C->cfg.n_train_global,
                p.M, p.row_loss);  // in place: Y_tr (in M) -> M_tr, row by row
      reduce_sum(Lk, p.row_loss, p.n_tr, C->part_loss + i);
      continue;
    }
    if (C->cfg.train_sparse && p.tr_list && 2 * p.n_tr < p.n_in) {
      // few train rows (products-shaped: 8 %): zero-fill M^(L) with one memset and run the loss warps on the
      // train row list only -- not one warp per row that mostly stores a zero row (same M, same loss terms)
      Scope sc(C, PGCN_K_LOSS, 4.0 * (p.Mlo ? 2 : 1) * p.n_in * C->ld[L] + 8.0 * p.n_tr * C->F[L] + 8.0 * p.n_tr);
      cudaMemsetAsync(p.M, 0, sizeof(float) * (size_t)(p.n_in * C->ld[L]), C->s);
      if (p.Mlo) cudaMemsetAsync(p.Mlo, 0, sizeof(float) * (size_t)(p.n_in * C->ld[L]), C->s);
      loss_rows(Lk, C->cfg.loss, p.logits, p.n_tr, C->F[L], C->ld[L], p.labels, nullptr,
                (double)C->cfg.n_train_global, p.M, p.row_loss, p.Mlo, p.tr_list);
      reduce_sum(Lk, p.row_loss, p.n_tr, C->part_loss + i);
      continue;
    }
    Scope sc(C, PGCN_K_LOSS, (p.Mlo ? 12.0 : 8.0) * p.n_in * C->F[L] + 5.0 * p.n_in);
    loss_rows(Lk, C->cfg.loss, p.logits, p.n_in, C->F[L], C->ld[L], p.labels, p.train,
              (double)C->cfg.n_train_global, p.M, p.row_loss, p.Mlo);
    reduce_sum(Lk, p.row_loss, p.n_in, C->part_loss + i);
  }
  if (loss_dev) reduce_sum(Lk, C->part_loss, (int64_t)C->parts.size(), loss_dev);
  cudaEventRecord(C->ev_lab_free, C->s);
  rc = check_cuda(C, "pgcn_loss");
  if (rc) return rc;
  advance(C);
  return PGCN_OK;
}

extern "C" int pgcn_layer_bwd(pgcn_ctx* C, int64_t t, int32_t l, const float* params) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_BWD, l, "pgcn_layer_bwd");
  if (rc) return rc;
  if (!params) return fail(PGCN_EINVAL, "params is NULL");
  const Launch Lk = C->launch();
  const int b = C->bi(t), bs = C->bi(t - C->depth);
  const bool pipe = C->cfg.mode == 1;
  const int64_t ldi = C->ld[l - 1], ldo = C->ld[l];
  const float* Wext = params + C->woff[l];
  const int bf = C->cfg.gemm == 1;
  // algorithmic SpMM bytes: gathered rows (fp32, or bf16 in the gather tier) and, in the bf16 tier,
  // the rounding pass over the table (read fp32, write bf16)
  auto gat = [&](double F, double e) { return (C->cfg.gather ? 2.0 : 4.0) * F * e; };
  auto cvt = [&](double F, double rows) { return C->cfg.gather ? 6.0 * F * rows : 0.0; };
  // lean (N1(iii)): J^(l-1) has one slot; its boundary rows posted at t - 1 must have been read by the
  // transfer before this iteration rewrites them (bf16 payloads travel from send_b, PUSH from epilogues)
  if (C->cfg.lean && C->posted && !C->p16 && l >= 2 && t > 1)
    cudaStreamWaitEvent(C->s, C->ev_b_done[l][C->bi(t - 1)], 0);
  // phase A: S6 (G_i^(l), Alg. 1 l.18), S7 + S8 (J^(l-1) for inner and boundary rows, l.20)
  for (auto& p : C->parts) {
    const double Fi = (double)C->F[l - 1], Fo = (double)C->F[l];
    // N1(ii): M^(L) is 0 outside the train rows, so the last layer's transposed aggregation only
    // needs P_i^T restricted to train sources
    const bool sp = C->cfg.train_sparse && l == C->L && p.last_sparse;
    const int64_t* trp = sp ? p.trp_tr : p.trp;
    const int32_t* tcol = sp ? p.tcol_tr : p.tcol;
    const double nz = sp ? (double)p.nnz_tr : (double)p.nnz;
    auto sb = [&](double F, double nv, double e, double rest) { return SpmmBytes{gat(F, nv) + rest, gat(F, e) + rest}; };
    const float* D = (C->cfg.dropout > 0.0 || C->gcn) ? p.D[l] : layer_in(p, l, b);
    // M's producer-written lo term (3xTF32 tier; not for the compact last layer's M_tr)
    const float* mlo = (C->mlo_stale || (C->cl && l == C->L)) ? nullptr : p.Mlo;
    if (C->cfg.lean && !C->tf[l]) {
      // N1(iii): Z^(l) was not kept (one scratch for every layer) -- recompute it with the forward's own
      // launch (same inputs: D^(l) and the boundary rows of slot t are untouched until t + 1), bit for bit
      const bool spf = C->cfg.train_sparse && l == C->L && p.last_sparse;
      const int64_t nrf = spf ? p.n_tr : p.n_in, nvf = p.n_valid[l];
      const double nzf = spf ? (double)p.nnz_tr : (double)p.nnz;
      Scope sc(C, PGCN_K_SPMM_FWD, sb(Fi, nvf, nzf + (C->gcn ? nrf : 0), cvt(Fi, nvf) + 4.0 * nzf + 8.0 * (nrf + 1) +
                                       4.0 * nrf + 4.0 * Fi * nrf));
      if ((rc = spmm_fwd(Lk, p.rp, p.col, C->gcn ? p.sym : p.inv_deg, D, ldi, nrf, nvf, p.Z[l], C->work, C->gcn ? 1 : 0,
                         nullptr, 0, 0, p.n_all, p.G16, spf ? p.tr_list : nullptr, (int64_t)nzf, p.tiles(0), p.T16,
                         C->cl && l == C->L)))
        return poison(C, rc);
    }
    if (C->gcn) {
      // GCN-sym backward (App. A.1 PAPER.md:651-657 with P = S (A + I) S, S = diag(d~^-1/2), R26)
      if (C->tf[l]) {
        // Q = (A + I)^T (S M) over inner + boundary rows; G = [D'^T Q ; colsum M]; J = mask o s o S (Q W^T)
        const int64_t nv = p.n_valid[l] ? p.n_valid[l] : p.n_all;
        {
          Scope sc(C, PGCN_K_SPMM_BWD, sb(Fo, p.n_in, nz + p.n_in, cvt(Fo, p.n_in) + 4.0 * nz + 8.0 * (p.n_all + 1) +
                                           8.0 * Fo * p.n_in + 4.0 * Fo * p.n_all));
          scale_rows(Lk, p.M, p.sym, p.n_in, ldo, p.dA);
          DropSpec none{};
          none.width = (int32_t)C->F[l];
          if ((rc = spmm_bwd(Lk, trp, tcol, p.dA, p.dA, ldo, p.n_in, p.n_all, p.T[l], ldo, p.gid, none, C->work, nullptr,
                   p.G16, (int64_t)nz, sp ? nullptr : p.tiles(1), p.T16))) return poison(C, rc);
        }
        {
          Scope sc(C, PGCN_K_GEMM_DW, 4.0 * nv * (Fi + Fo) + 4.0 * p.n_in * Fo, 2.0 * nv * Fi * Fo);
          if (tc_dw_general(Lk, D, p.T[l], nv, nullptr, nullptr, 0, ldi, ldo, C->F[l - 1], C->F[l], p.M, p.n_in,
                            p.G + C->woff[l], C->dw_ws, C->dw_ws_floats, bf))
            return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dW GEMM failed (layer %d)", l);
        }
        if (l >= 2) {
          Scope sc(C, PGCN_K_GEMM_DA, 4.0 * p.n_all * (Fo + Fi), 2.0 * p.n_all * Fo * Fi);
          PushSpec ps;
          const bool psh = bwd_push(C, p, t, l, ps);
          if (tc_fwd_mask(Lk, p.T[l], p.n_all, nullptr, 0, ldo, C->F[l], C->WJ_hi[l], C->WJ_lo[l], C->Kq[l],
                          C->F[l - 1], p.J[l - 1][b], ldi, p.gid, drop_spec(C, t, l), bf, p.sym, psh ? &ps : nullptr))
            return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core input-gradient GEMM failed (layer %d)", l);
        }
        continue;
      }
      {
        Scope sc(C, PGCN_K_GEMM_DW, 4.0 * p.n_in * (Fi + Fo), 2.0 * p.n_in * (Fi + 1) * Fo);
        if (tc_dw_general(Lk, p.Z[l], p.M, p.n_in, nullptr, nullptr, 0, ldi, ldo, C->F[l - 1], C->F[l], p.M, p.n_in,
                          p.G + C->woff[l], C->dw_ws, C->dw_ws_floats, bf, mlo))
          return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dW GEMM failed (layer %d)", l);
      }
      if (l >= 2) {
        {  // dZs = S (M W^T)
          Scope sc(C, PGCN_K_GEMM_DA, 4.0 * p.n_in * (Fi + Fo) + 4.0 * p.n_in, 2.0 * p.n_in * Fo * Fi);
          if (gemm_da_tc(Lk, p.M, ldo, p.n_in, C->F[l], C->Wp_hi[l], C->Wp_lo[l], C->Kp[l], C->F[l - 1], p.sym, p.dA,
                         ldi, bf, 1, mlo))
            return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dA GEMM failed (layer %d)", l);
        }
        // J^(l-1)_u = mask o s o d~_u^-1/2 ((A + I)^T dZs)_u over inner + boundary rows
        Scope sc(C, PGCN_K_SPMM_BWD, sb(Fi, p.n_in, nz + p.n_in, cvt(Fi, p.n_in) + 4.0 * nz + 8.0 * (p.n_all + 1) +
                                         4.0 * Fi * p.n_all + 12.0 * p.n_all));
        PushSpec ps;
        const bool psh = bwd_push(C, p, t, l, ps);
        if ((rc = spmm_bwd(Lk, trp, tcol, p.dA, p.dA, ldi, p.n_in, p.n_all, p.J[l - 1][b], ldi, p.gid, drop_spec(C, t, l),
                 C->work, p.sym, p.G16, (int64_t)nz, sp ? nullptr : p.tiles(1), p.T16, nullptr,
                 psh ? &ps : nullptr))) return poison(C, rc);
      }
      continue;
    }
    if (C->tf[l]) {
      // N1 backward: Q = P_i^T (inv_deg o M) over inner + boundary rows (width F_out);
      // G = [D^T Q ; D_in^T M ; colsum M];  J^(l-1) = mask o s o ([Q | M] [W_neigh | W_self]^T)
      const int64_t nv = p.n_valid[l] ? p.n_valid[l] : p.n_all;
      {
        Scope sc(C, PGCN_K_SPMM_BWD, sb(Fo, p.n_in, nz, cvt(Fo, p.n_in) + 4.0 * nz + 8.0 * (p.n_all + 1) + 8.0 * Fo * p.n_in +
                                         4.0 * Fo * p.n_all));
        scale_rows(Lk, p.M, p.inv_deg, p.n_in, ldo, p.dA);
        DropSpec none{};
        none.width = (int32_t)C->F[l];
        if ((rc = spmm_bwd(Lk, trp, tcol, p.dA, nullptr, ldo, p.n_in, p.n_all, p.T[l], ldo, p.gid, none, C->work, nullptr,
                 p.G16, (int64_t)nz, sp ? nullptr : p.tiles(1), p.T16))) return poison(C, rc);
      }
      {
        Scope sc(C, PGCN_K_GEMM_DW, 4.0 * (nv + p.n_in) * (Fi + Fo), 2.0 * (nv + p.n_in) * Fi * Fo);
        if (tc_dw_general(Lk, D, p.T[l], nv, D, p.M, p.n_in, ldi, ldo, C->F[l - 1], C->F[l], p.M, p.n_in,
                          p.G + C->woff[l], C->dw_ws, C->dw_ws_floats, bf, nullptr, mlo))
          return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dW GEMM failed (layer %d)", l);
      }
      if (l >= 2) {
        Scope sc(C, PGCN_K_GEMM_DA, 4.0 * (p.n_all + p.n_in) * Fo + 4.0 * p.n_all * Fi,
                 2.0 * (p.n_all + p.n_in) * Fo * Fi);
        PushSpec ps;
        const bool psh = bwd_push(C, p, t, l, ps);
        if (tc_fwd_mask(Lk, p.T[l], p.n_all, p.M, p.n_in, ldo, C->F[l], C->WJ_hi[l], C->WJ_lo[l], C->Kq[l],
                        C->F[l - 1], p.J[l - 1][b], ldi, p.gid, drop_spec(C, t, l), bf, nullptr, psh ? &ps : nullptr))
          return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core input-gradient GEMM failed (layer %d)", l);
      }
      continue;
    }
    const bool cl = C->cl && l == C->L;  // compact train rows: Z, D_tr, M and dA rows are positions
    const int64_t mr = cl ? p.n_tr : p.n_in;
    if (cl) D = p.Dtr;
    {
      Scope sc(C, PGCN_K_GEMM_DW, 4.0 * mr * (2 * Fi + Fo), 2.0 * mr * (2 * Fi + 1) * Fo);
      if (C->cfg.gemm != 2) {
        if (gemm_dw_tc(Lk, p.Z[l], D, ldi, mr, C->F[l - 1], p.M, ldo, C->F[l], p.G + C->woff[l], C->dw_ws,
                       C->dw_ws_floats, bf, mlo))
          return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dW GEMM failed (layer %d)", l);
      } else {
        gemm_dw_f32(Lk, p.Z[l], D, ldi, p.n_in, C->F[l - 1], p.M, ldo, C->F[l], p.G + C->woff[l], C->dw_ws,
                    C->dw_ws_floats);
      }
    }
    if (l >= 2) {
      {
        Scope sc(C, PGCN_K_GEMM_DA, 4.0 * mr * (2 * Fi + Fo) + 4.0 * mr, 2.0 * mr * Fo * 2 * Fi);
        if (C->cfg.gemm != 2) {
          if (mr > 0 && gemm_da_tc(Lk, p.M, ldo, mr, C->F[l], C->Wp_hi[l], C->Wp_lo[l], C->Kp[l], C->F[l - 1],
                                   cl ? p.invdeg_tr : p.inv_deg, p.dA, ldi, bf, 2, mlo))
            return fail(PGCN_ECUDA, "pgcn_layer_bwd: tensor-core dA GEMM failed (layer %d)", l);
        } else {
          gemm_da_f32(Lk, p.M, ldo, p.n_in, C->F[l], Wext, C->F[l - 1], p.inv_deg, p.dA, ldi);
        }
      }
      Scope sc(C, PGCN_K_SPMM_BWD, sb(Fi, p.n_in, nz, cvt(Fi, p.n_in) + 4.0 * nz + 8.0 * (p.n_all + 1) + 4.0 * Fi * p.n_in +
                                       4.0 * Fi * p.n_all + 8.0 * p.n_all));
      PushSpec ps;
      const bool psh = bwd_push(C, p, t, l, ps);
      if ((rc = spmm_bwd(Lk, trp, tcol, p.dA, p.dA + ldi, 2 * ldi, p.n_in, p.n_all, p.J[l - 1][b], ldi, p.gid,
               drop_spec(C, t, l), C->work, nullptr, p.G16, (int64_t)nz, sp ? nullptr : p.tiles(1), p.T16,
               cl ? p.tr_pos : nullptr, psh ? &ps : nullptr))) return poison(C, rc);
    }
  }
  // phase B: S9 stale (PIPE) / fresh (VANILLA) boundary gradients (l.22-25) and M^(l-1)
  if (l >= 2 && pushing(C)) C->bpushed[l] = t;  // every producer of J^(l-1) pushed its boundary rows
  if (l >= 2) {
    bool posted_have = false;
    if (C->posted && (rc = post_bwd(C, t, l, Lk, &posted_have))) return rc;
    for (auto& p : C->parts) {
      SegTable msg{};
      msg.n_seg = 0;
      bool use_ema = false, first = false;
      const bool have = C->n_parts > 1 && p.n_send > 0 && (!pipe || t > C->depth);
      const int sb = pipe ? bs : b;  // messages of t - s (PIPE) or t (VANILLA)
      const int32_t* row_map = C->posted ? nullptr : p.msg_map;
      if (have) {
        if (C->posted) {  // one segment: the received rows in send order
          msg.n_seg = 1;
          msg.off[1] = p.n_send;
          msg.base[0] = static_cast<const float*>(p.recv_b[l][sb]);
        } else {          // local: the peers' boundary rows of J^(l-1), read in place
          msg.n_seg = C->n_parts;
          for (int j = 0; j <= C->n_parts; ++j) msg.off[j] = p.v.send_off[j];
          for (int j = 0; j < C->n_parts; ++j) msg.base[j] = C->parts[j].J[l - 1][sb];
        }
        if (pipe && C->cfg.smooth_g) {
          use_ema = true;
          first = C->cfg.ema_init == 0 && t == C->depth + 1;
        }
      }
      const int m16 = C->posted && C->p16;
      const double Fi = (double)C->F[l - 1];
      Scope sc(C, PGCN_K_GRAD_REDUCE, 4.0 * Fi * p.n_in * (3 + C->cfg.dump_j + (p.Mlo ? 1 : 0)) + 8.0 * p.n_in +
                                          (msg.n_seg ? ((m16 ? 2.0 : 4.0) * Fi + 4.0 + (use_ema ? 8.0 * Fi : 0.0)) * p.n_send : 0.0));
      grad_reduce(Lk, p.inv_ptr, p.inv_pos, msg, row_map, p.emaG[l - 1], (float)C->cfg.gamma, use_ema, first,
                  p.J[l - 1][b], C->cfg.dump_j || C->force_write_j, p.H[l - 1][b], p.M, p.n_in, ldi, m16, p.Mlo);
      if (C->cfg.staleness_stats && C->xp != XP_NCCL && C->n_parts > 1 && p.n_send > 0) {
        // N4: ||gradient messages used - fresh ones||^2 (fresh = peers' boundary rows of this iteration;
        // used = the smoothed state, the stale messages, or 0 when nothing was received)
        SegTable fresh{};
        fresh.n_seg = C->n_parts;
        for (int j = 0; j <= C->n_parts; ++j) fresh.off[j] = p.v.send_off[j];
        for (int j = 0; j < C->n_parts; ++j) fresh.base[j] = C->parts[j].J[l - 1][b];
        if (use_ema)
          stale_err(Lk, fresh, p.msg_map, nullptr, nullptr, p.emaG[l - 1], p.n_send, ldi, C->F[l - 1],
                    C->diag + PGCN_MAX_LAYERS + 1 + l);
        else
          stale_err(Lk, fresh, p.msg_map, msg.n_seg ? &msg : nullptr, row_map, nullptr, p.n_send, ldi, C->F[l - 1],
                    C->diag + PGCN_MAX_LAYERS + 1 + l);
      }
    }
    (void)posted_have;
  }
  if (l == 1 && !(C->cfg.dropout > 0.0 || C->gcn)) cudaEventRecord(C->ev_x_free, C->s);
  rc = check_cuda(C, "pgcn_layer_bwd");
  if (rc) return rc;
  advance(C);
  return PGCN_OK;
}

extern "C" int pgcn_update(pgcn_ctx* C, int64_t t, float* params, float* grads, float* opt_state) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_UPD, 0, "pgcn_update");
  if (rc) return rc;
  if (!params || !grads) return fail(PGCN_EINVAL, "params / grads is NULL");
  if (C->cfg.opt == 1 && !opt_state) return fail(PGCN_EINVAL, "Adam needs opt_state");
  const Launch Lk = C->launch();
  PtrList G{};
  G.n = (int32_t)C->parts.size();
  for (int i = 0; i < G.n; ++i) G.p[i] = C->parts[i].G;
  Scope sc(C, PGCN_K_UPDATE, 4.0 * C->P * (G.n + 2 + (C->cfg.opt == 1 ? 4 : 1)));
  sum_grads(Lk, G, C->P, grads);
#ifdef PGCN_WITH_NCCL
  if (C->nccl) {  // l.31: G = AllReduce(G_i), SUM (R6), on the compute stream (consumed right away)
    ncclResult_t r = ncclAllReduce(grads, grads, (size_t)C->P, ncclFloat, ncclSum, C->cr, C->s);
    if (r != ncclSuccess) return nccl_fail(C, r, "pgcn_update all-reduce");
  }
#endif
  OptSpec o{};
  o.adam = C->cfg.opt == 1;
  o.lr = (float)C->cfg.lr;
  o.beta1 = (float)C->cfg.beta1;
  o.beta2 = (float)C->cfg.beta2;
  o.eps = (float)C->cfg.eps;
  o.step_size = (float)(C->cfg.lr / (1.0 - std::pow(C->cfg.beta1, (double)t)));
  o.inv_sqrt_bc2 = (float)(1.0 / std::sqrt(1.0 - std::pow(C->cfg.beta2, (double)t)));
  o.apply = 1;
  opt_update(Lk, grads, C->P, params, opt_state, opt_state ? opt_state + C->P : nullptr, o);
  rc = check_cuda(C, "pgcn_update");
  if (rc) return rc;
  advance(C);
  return PGCN_OK;
}

// ---------------------------------------------------------------------------------------------------
// Caller-buffer forms of the per-layer calls: stage W, b into theta layout, optionally
// replace the layer's input / output-gradient rows, run the layer, copy results out.
namespace {
int stage_weights(pgcn_ctx* C, int l, const float* W, const float* b) {
  if (!W || !b) return fail(PGCN_EINVAL, "W / b is NULL");
  const int64_t nW = C->ns * C->F[l - 1] * C->F[l];
  cudaMemcpyAsync(C->theta_io + C->woff[l], W, sizeof(float) * nW, cudaMemcpyDeviceToDevice, C->s);
  cudaMemcpyAsync(C->theta_io + C->woff[l] + nW, b, sizeof(float) * C->F[l], cudaMemcpyDeviceToDevice, C->s);
  return PGCN_OK;
}
void copy_rows(pgcn_ctx* C, float* dst, int64_t ldd, const float* src, int64_t lds, int64_t F, int64_t rows) {
  if (rows > 0)
    cudaMemcpy2DAsync(dst, sizeof(float) * ldd, src, sizeof(float) * lds, sizeof(float) * F, rows,
                      cudaMemcpyDeviceToDevice, C->s);
}
}  // namespace

extern "C" int pgcn_layer_fwd_io(pgcn_ctx* C, int64_t t, int32_t l, const float* W, const float* b,
                                 const float* const* h_in, int64_t ld_in, float* const* h_out, int64_t ld_out) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_FWD, l, "pgcn_layer_fwd_io");
  if (rc) return rc;
  if ((h_in && ld_in < C->F[l - 1]) || (h_out && ld_out < C->F[l])) return fail(PGCN_EINVAL, "row stride too small");
  if ((rc = stage_weights(C, l, W, b))) return rc;
  const int bb = C->bi(t);
  if (h_in)
    for (size_t k = 0; k < C->parts.size(); ++k) {
      PartCtx& p = C->parts[k];
      if (h_in[k]) copy_rows(C, layer_in(p, l, bb), C->ld[l - 1], h_in[k], ld_in, C->F[l - 1], p.n_in);
    }
  if ((rc = pgcn_layer_fwd(C, t, l, C->theta_io))) return rc;
  if (h_out)
    for (size_t k = 0; k < C->parts.size(); ++k) {
      PartCtx& p = C->parts[k];
      if (!h_out[k]) continue;
      if (l == C->L && !p.logits) return fail(PGCN_EUNSUPPORTED, "lean mode: the last layer's output rows are not kept");
      copy_rows(C, h_out[k], ld_out, l < C->L ? p.H[l][bb] : p.logits, C->ld[l], C->F[l], p.n_in);
    }
  return check_cuda(C, "pgcn_layer_fwd_io");
}

extern "C" int pgcn_layer_bwd_io(pgcn_ctx* C, int64_t t, int32_t l, const float* W, const float* b,
                                 const float* const* j_out, int64_t ld_jo, float* dW_local, float* db_local,
                                 float* const* j_in, int64_t ld_ji) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc = expect(C, t, K_BWD, l, "pgcn_layer_bwd_io");
  if (rc) return rc;
  if ((j_out && ld_jo < C->F[l]) || (j_in && l >= 2 && ld_ji < C->F[l - 1])) return fail(PGCN_EINVAL, "row stride too small");
  if (j_out && l == C->L && C->cl) return fail(PGCN_EUNSUPPORTED, "j_out of the last layer with compact train rows");
  if ((rc = stage_weights(C, l, W, b))) return rc;
  const int bb = C->bi(t);
  const Launch Lk = C->launch();
  if (j_out)
    for (size_t k = 0; k < C->parts.size(); ++k) {
      PartCtx& p = C->parts[k];
      if (!j_out[k]) continue;
      if (l == C->L) {  // M^(L) = J^(L)
        copy_rows(C, p.M, C->ld[l], j_out[k], ld_jo, C->F[l], p.n_in);
      } else {          // M^(l) = J^(l) o 1[H^(l) > 0]: the accumulate kernel with no messages
        copy_rows(C, p.J[l][bb], C->ld[l], j_out[k], ld_jo, C->F[l], p.n_in);
        SegTable none{};
        grad_reduce(Lk, p.inv_ptr, p.inv_pos, none, nullptr, nullptr, 0.f, 0, 0, p.J[l][bb], 0, p.H[l][bb], p.M,
                    p.n_in, C->ld[l], 0, p.Mlo);
      }
    }
  C->force_write_j = j_in != nullptr && l >= 2;
  C->mlo_stale = j_out != nullptr && l == C->L;  // M^(L) copied from the caller: the GEMMs split it themselves
  rc = pgcn_layer_bwd(C, t, l, C->theta_io);
  C->force_write_j = 0;
  C->mlo_stale = 0;
  if (rc) return rc;
  if (j_in && l >= 2)
    for (size_t k = 0; k < C->parts.size(); ++k) {
      PartCtx& p = C->parts[k];
      if (j_in[k]) copy_rows(C, j_in[k], ld_ji, p.J[l - 1][bb], C->ld[l - 1], C->F[l - 1], p.n_in);
    }
  const int64_t nW = C->ns * C->F[l - 1] * C->F[l];
  PtrList G{};
  G.n = (int32_t)C->parts.size();
  if (dW_local) {
    for (int i = 0; i < G.n; ++i) G.p[i] = C->parts[i].G + C->woff[l];
    sum_grads(Lk, G, nW, dW_local);
  }
  if (db_local) {
    for (int i = 0; i < G.n; ++i) G.p[i] = C->parts[i].G + C->woff[l] + nW;
    sum_grads(Lk, G, C->F[l], db_local);
  }
  return check_cuda(C, "pgcn_layer_bwd_io");
}

extern "C" int pgcn_step(pgcn_ctx* C, int64_t t, float* params, float* grads, float* opt_state, float* loss_dev) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  int rc;
  for (int l = 1; l <= C->L; ++l)
    if ((rc = pgcn_layer_fwd(C, t, l, params))) return rc;
  if ((rc = pgcn_loss(C, t, loss_dev))) return rc;
  for (int l = C->L; l >= 1; --l)
    if ((rc = pgcn_layer_bwd(C, t, l, params))) return rc;
  return pgcn_update(C, t, params, grads, opt_state);
}

extern "C" int pgcn_tensor(pgcn_ctx* C, int32_t local, int32_t kind, int32_t l, int64_t t, pgcn_tensor_desc* o) {
  if (!C || !o) return fail(PGCN_EINVAL, "null argument");
  if (local < 0 || local >= (int)C->parts.size()) return fail(PGCN_EINVAL, "local index out of range");
  PartCtx& p = C->parts[local];
  const int b = C->bi(t);
  const bool lok = l >= 1 && l <= C->L;
  switch (kind) {
    case PGCN_T_H:
      if (!lok || (l == C->L && !p.logits)) break;  // (lean + compact last layer: logits not kept)
      *o = {l < C->L ? (void*)p.H[l][b] : (void*)p.logits, p.n_in, C->F[l], C->ld[l]};
      return PGCN_OK;
    case PGCN_T_HIN:
      if (!lok) break;
      *o = {(void*)layer_in(p, l, b), p.n_all, C->F[l - 1], C->ld[l - 1]};
      return PGCN_OK;
    case PGCN_T_Z:  // Z = inv_deg P D (width F_{l-1}); transform-first layers: S = inv_deg P (D W_neigh)
      if (!lok || (C->gcn && C->tf[l])) break;
      *o = {(void*)p.Z[l], p.n_in, C->tf[l] ? C->F[l] : C->F[l - 1], C->tf[l] ? C->ld[l] : C->ld[l - 1]};
      return PGCN_OK;
    case PGCN_T_J:
      if (l < 1 || l >= C->L) break;
      *o = {(void*)p.J[l][b], p.n_in, C->F[l], C->ld[l]};
      return PGCN_OK;
    case PGCN_T_G:
      *o = {(void*)p.G, 1, C->P, C->P};
      return PGCN_OK;
    default:
      break;
  }
  return fail(PGCN_EINVAL, "pgcn_tensor: bad kind / layer");
}

extern "C" int64_t pgcn_launch_count(const pgcn_ctx* C) { return C ? C->launches : -1; }

extern "C" int pgcn_dev_exchange_bytes(const pgcn_ctx* C, int64_t* fwd_bytes, int64_t* bwd_bytes) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  if (fwd_bytes) *fwd_bytes = C->xbytes[0];
  if (bwd_bytes) *bwd_bytes = C->xbytes[1];
  return PGCN_OK;
}

extern "C" int pgcn_dev_exchange_hook(pgcn_ctx* C, int64_t spin_ns, int32_t flags) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  if (!C->posted) return fail(PGCN_EUNSUPPORTED, "exchange hook: posted transports (LOOPBACK / NCCL) only");
  if (spin_ns < 0 || (flags & ~(PGCN_XH_SKIP_F_WAIT | PGCN_XH_SKIP_B_WAIT | PGCN_XH_NOCOMM)))
    return fail(PGCN_EINVAL, "exchange hook: bad argument");
  C->hook_spin_ns = spin_ns;
  C->hook_flags = flags;
  return PGCN_OK;
}

extern "C" int pgcn_staleness(pgcn_ctx* C, int32_t layer, double* feat_err, double* grad_err) {
  if (!C || layer < 1 || layer > C->L) return fail(PGCN_EINVAL, "pgcn_staleness: bad argument");
  if (!C->cfg.staleness_stats) return fail(PGCN_ESTATE, "pgcn_staleness: context created without staleness_stats");
  if (C->nccl) return fail(PGCN_EUNSUPPORTED, "pgcn_staleness: single-process contexts only");
  double h[2];
  cudaStreamSynchronize(C->s);
  cudaMemcpy(&h[0], C->diag + layer, sizeof(double), cudaMemcpyDeviceToHost);
  cudaMemcpy(&h[1], C->diag + PGCN_MAX_LAYERS + 1 + layer, sizeof(double), cudaMemcpyDeviceToHost);
  if (feat_err) *feat_err = std::sqrt(h[0]);
  if (grad_err) *grad_err = std::sqrt(h[1]);
  return check_cuda(C, "pgcn_staleness");
}

extern "C" int pgcn_timing_enable(pgcn_ctx* C, int32_t on) {
  if (!C) return fail(PGCN_EINVAL, "ctx is NULL");
  if (C->s) cudaStreamSynchronize(C->s);
  C->timing = on ? 1 : 0;
  for (auto& k : C->kt) {
    k.used = 0;
    k.n = 0;
    k.bytes = k.flops = k.gbytes = 0.0;
  }
  return PGCN_OK;
}

extern "C" int pgcn_timing_read(pgcn_ctx* C, int32_t kind, double* ms, int64_t* launches, double* bytes,
                                double* flops) {
  if (!C || kind < 0 || kind >= PGCN_K_COUNT) return fail(PGCN_EINVAL, "bad argument");
  KTimer& k = C->kt[kind];
  double tot = 0.0;
  for (size_t i = 0; i + 1 < k.used; i += 2) {
    cudaError_t e = cudaEventSynchronize(k.ev[i + 1]);
    if (e != cudaSuccess) return fail(PGCN_ECUDA, "pgcn_timing_read: %s", cudaGetErrorString(e));
    float x = 0.f;
    cudaEventElapsedTime(&x, k.ev[i], k.ev[i + 1]);
    tot += x;
  }
  if (ms) *ms = tot;
  if (launches) *launches = k.n;
  if (bytes) *bytes = k.bytes;
  if (flops) *flops = k.flops;
  return PGCN_OK;
}

extern "C" int pgcn_timing_read_gather(pgcn_ctx* C, int32_t kind, double* gather_bytes) {
  if (!C || kind < 0 || kind >= PGCN_K_COUNT || !gather_bytes) return fail(PGCN_EINVAL, "bad argument");
  *gather_bytes = C->kt[kind].gbytes;
  return PGCN_OK;
}

// ---------------------------------------------------------------------------------------------------
// N2 over NVLink: the workspaces of the ranks mapped into each other with CUDA IPC.
namespace {
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(ptr);
  });
  return fn;
}
}  // namespace

extern "C" int pgcn_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int pgcn_ipc_export(pgcn_ctx* C, void* handle, int64_t* offset) {
  if (!C || !handle || !offset) return fail(PGCN_EINVAL, "pgcn_ipc_export: null argument");
  if (!C->ipc_push) return fail(PGCN_ESTATE, "pgcn_ipc_export: context not created for PUSH across ranks");
  AddrRangeFn f = addr_range_fn();
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!f || f(&base, &size, reinterpret_cast<CUdeviceptr>(C->ws)) != CUDA_SUCCESS)
    return fail(PGCN_ECUDA, "pgcn_ipc_export: allocation range of the workspace unavailable");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(PGCN_ECUDA, "pgcn_ipc_export: %s", cudaGetErrorString(e));
  std::memcpy(handle, &h, sizeof(h));
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(C->ws) - base);
  return PGCN_OK;
}

extern "C" int pgcn_ipc_import(pgcn_ctx* C, int32_t rank, const void* handle, int64_t offset) {
  if (!C || !handle || offset < 0) return fail(PGCN_EINVAL, "pgcn_ipc_import: bad argument");
  if (!C->ipc_push) return fail(PGCN_ESTATE, "pgcn_ipc_import: context not created for PUSH across ranks");
  if (rank < 0 || rank >= C->nranks || rank == C->rank) return fail(PGCN_EINVAL, "pgcn_ipc_import: bad rank %d", rank);
  if ((int)C->peer.size() < C->nranks) C->peer.resize(C->nranks);
  if (C->peer[rank].X) return fail(PGCN_ESTATE, "pgcn_ipc_import: rank %d already imported", rank);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* basep = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&basep, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(PGCN_ECUDA, "pgcn_ipc_import(rank %d): %s", rank, cudaGetErrorString(e));
  // partition `rank`'s buffers at the offsets its own context laid them out at (same partitioning, config)
  pgcn_ctx T;
  const int32_t loc = rank;
  pgcn_comm cm{rank, C->nranks, "x", "x"};  // shapes only (no communicator is created)
  int rc = init_ctx_shapes(&T, C->part, &loc, 1, &C->cfg, &cm);
  if (rc) { cudaIpcCloseMemHandle(basep); return rc; }
  Arena A;
  A.base = static_cast<char*>(basep) + offset;
  if ((rc = layout(&T, C->part, &loc, 1, A))) { cudaIpcCloseMemHandle(basep); return rc; }
  C->peer[rank] = T.parts[0];
  C->ipc_open.push_back(basep);
  ++C->n_imported;
  return PGCN_OK;
}

extern "C" int pgcn_nccl_id_bytes(void) {
#ifdef PGCN_WITH_NCCL
  return (int)sizeof(ncclUniqueId);
#else
  return 0;
#endif
}

extern "C" int pgcn_nccl_unique_id(void* out) {
#ifdef PGCN_WITH_NCCL
  if (!out) return fail(PGCN_EINVAL, "out is NULL");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(PGCN_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof(id));
  return PGCN_OK;
#else
  (void)out;
  return fail(PGCN_EUNSUPPORTED, "library built without NCCL");
#endif
}
