// N1(ii) train-row-sparse last layer: the loss reads Y^(L) only at train rows
// (Alg. 1 l.16), so the last layer's aggregation is needed only there, and its backward
// messages P_i^T (.) only carry the train rows' gradients (M^(L) is 0 elsewhere).  Exact: the skipped
// terms are zero (backward) or unused (forward).  Built once per pgcn_set_inputs from the train mask:
//   tr_list     inner ids v with train[v] != 0, ascending (the row list of the last forward SpMM)
//   P_i^T|train  the transposed CSR with only the entries v in the train set, order kept (R20)
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <cstdint>

#include "kernels.cuh"

namespace pgcn {
namespace {

// counts[u] = #{e in row u of P_i^T : train[t_col[e]] != 0}, u < n_all; counts[n_all] = 0
__global__ void k_count_train(const int64_t* __restrict__ trp, const int32_t* __restrict__ tcol, int64_t n_all,
                              const uint8_t* __restrict__ train, int64_t* __restrict__ counts) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n_all; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = 0;
    if (u < n_all)
      for (int64_t e = trp[u]; e < trp[u + 1]; ++e) c += train[tcol[e]] != 0;
    counts[u] = c;
  }
}

__global__ void k_fill_train(const int64_t* __restrict__ trp, const int32_t* __restrict__ tcol, int64_t n_all,
                             const uint8_t* __restrict__ train, const int64_t* __restrict__ trp_tr,
                             int32_t* __restrict__ tcol_tr) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n_all; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = trp_tr[u];
    for (int64_t e = trp[u]; e < trp[u + 1]; ++e) {
      const int32_t v = tcol[e];
      if (train[v]) tcol_tr[k++] = v;
    }
  }
}

}  // namespace

size_t train_rows_tmp_bytes(int64_t n_in, int64_t n_all) {
  size_t a = 0, b = 0;
  cub::DeviceSelect::Flagged(nullptr, a, cub::CountingInputIterator<int32_t>(0), (const uint8_t*)nullptr,
                             (int32_t*)nullptr, (int64_t*)nullptr, (int)(n_in > 0 ? n_in : 1));
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int64_t*)nullptr, (int64_t*)nullptr, (int)(n_all + 1));
  return (a > b ? a : b) + 256;
}

void build_train_rows(Launch L, const uint8_t* train, int64_t n_in, const int64_t* t_row_ptr, const int32_t* t_col,
                      int64_t n_all, int32_t* tr_list, int64_t* tr_count, int64_t* counts, int64_t* t_row_ptr_tr,
                      int32_t* t_col_tr, void* tmp, size_t tmp_bytes) {
  if (n_in > 0) {
    cub::DeviceSelect::Flagged(tmp, tmp_bytes, cub::CountingInputIterator<int32_t>(0), train, tr_list, tr_count,
                               (int)n_in, L.s);
  } else {
    cudaMemsetAsync(tr_count, 0, sizeof(int64_t), L.s);
  }
  const int grid = (int)std::min<int64_t>((n_all + 256) / 256 + 1, 148 * 16);
  k_count_train<<<grid, 256, 0, L.s>>>(t_row_ptr, t_col, n_all, train, counts);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, t_row_ptr_tr, (int)(n_all + 1), L.s);
  k_fill_train<<<grid, 256, 0, L.s>>>(t_row_ptr, t_col, n_all, train, t_row_ptr_tr, t_col_tr);
  if (L.count) *L.count += 4;
}

}  // namespace pgcn
