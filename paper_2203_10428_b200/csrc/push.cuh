// N2 fused push (pgcn_config.transport = PUSH): a producer kernel that writes rows peers consume also
// stores them straight into the peers' receive rows, so no pack kernel and no transfer run for them
// (PAPER.md:981 puts all communication on a second stream; here the transfer rides in the producing
// epilogue, tile by tile).  Rows of width ld floats; destinations are 16-byte aligned float4 slots.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "pgcn.h"

namespace pgcn {

struct PushSpec {
  float* base[PGCN_MAX_PARTS];  // per destination partition: its first receive row (row stride = the producer's ld)
  const int64_t* ptr;           // mode 1: [n_in + 1] inverse send map row -> positions (inv_ptr)
  const int32_t* pos;           // mode 1: positions k (inv_pos)
  const int32_t* part;          // mode 1: [n_send] destination of position k; mode 2: [n_bd] owner of boundary row r
  const int32_t* row;           // mode 1: [n_send] receive row of k;          mode 2: [n_bd] receive row of r
  int64_t row0;                 // mode 2: rows >= row0 (the boundary rows, row0 = n_in) are pushed
  int32_t mode;                 // 0 off; 1 forward: inner rows in S_{i,j}; 2 backward: boundary rows to owners
};

#ifdef __CUDACC__
// Extra stores of the float4 at column group x (ld4 float4s per row) of producer row `r`.
__device__ __forceinline__ void push_f4(const PushSpec& ps, int64_t r, int64_t ld4, int64_t x, const float4 o) {
  if (ps.mode == 1) {
    const int64_t qe = ps.ptr[r + 1];
    for (int64_t q = ps.ptr[r]; q < qe; ++q) {
      const int32_t k = ps.pos[q];
      reinterpret_cast<float4*>(ps.base[ps.part[k]])[(int64_t)ps.row[k] * ld4 + x] = o;
    }
  } else if (ps.mode == 2 && r >= ps.row0) {
    const int64_t b = r - ps.row0;
    reinterpret_cast<float4*>(ps.base[ps.part[b]])[(int64_t)ps.row[b] * ld4 + x] = o;
  }
}
#endif

}  // namespace pgcn
