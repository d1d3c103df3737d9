// Internal helpers shared by the library's translation units (not part of the ABI).
#pragma once
#include <atomic>
#include <cstdarg>
#include <cstdint>

#include "pgcn.h"

namespace pgcn {

// Records a thread-local message (returned by pgcn_last_error) and returns `code`.
int fail(int code, const char* fmt, ...);

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Streaming multiprocessors of the current device (queried once per device; B200: 148).  Persistent
// grids and grid caps are sized from it.
int sm_count();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `func`, once per (device, kernel).  0 / -1.
int smem_attr_once(const void* func, int bytes);
// RAII L2 access-policy window on stream s over [base, base + bytes): persisting hits for the gathered table
// of a gather SpMM (dev knob PGCN_L2_PERSIST_MB = the persisting carve-out; 0 = off).
struct L2Window {
  struct CUstream_st* s = nullptr;  // cudaStream_t
  bool on = false;
  L2Window(struct CUstream_st* st, const void* base, size_t bytes);
  ~L2Window();
};

// Developer A/B knobs (PGCN_* environment variables used by the tools/ sweeps), read once per process
// (thread-safe); the defaults are the measured choices.
struct DevKnobs {
  int tc_spmm_bn = 0, tc_spmm_order = 1, tc_spmm_dbg = 0, tc_spmm_nacc1 = 0, tc_spmm_ts = 1, tc_spmm_ctas = 2,
      tc_spmm_box64 = 1, tc_bnmax = 256, tc_gemm_ctas = 2, spmm_dyn = 1, tf_off = 0;
  long long dw_kmax = 128;
  int spmm_l2mb = 96;
  int dw_merge = 1;
  int presplit = 0;
  int spmm_nch = 2;  // column chunks of an L2-chunked gather (PGCN_SPMM_NCH)
  int tc_dw_bnmax = 256;
  int tc_bk16 = 2;
  int tc_dw16 = 0;
  int l2_persist_mb = 0;
  int tc_dw_ctas = 2;  // dW CTAs per SM (PGCN_TC_DW_CTAS: 2 = two pipelines per SM where they fit, 1 = one)  // L2 persisting window over the table a gather SpMM reads (PGCN_L2_PERSIST_MB)  // 3xTF32 dW: 16-row k-blocks (PGCN_TC_DW16; measured slower, profiles/r2r_bk16.md)  // 3xTF32 K-major GEMMs: 16-element k-blocks (PGCN_TC_BK16: 0 off, 1 n-tiles > 128, 2 all)  // dW n-tile cap (PGCN_TC_DW_BNMAX: 32..256, multiple of 32)
  long long spmm_grab = 128;
  const char* spmm_table = nullptr;
};
const DevKnobs& knobs();
inline int64_t ld_of(int64_t f) { return round_up(f, 4); }

}  // namespace pgcn
