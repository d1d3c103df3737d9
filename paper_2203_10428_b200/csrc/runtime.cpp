// Process-wide runtime helpers (internal): device properties, per-device kernel attributes and the
// developer A/B knobs, each initialised once and safe to call from several threads / contexts.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "common.h"

namespace pgcn {

int sm_count() {
  static std::atomic<int> cache[64];  // per device ordinal (0: not queried yet)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) return 148;
  if (dev >= 64) {
    int n = 0;
    return cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0 ? n : 148;
  }
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n > 0) return n;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  cache[dev].store(n, std::memory_order_relaxed);
  return n;
}

int smem_attr_once(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, func})) return 0;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return -1;
  done.insert({dev, func});
  return 0;
}

L2Window::L2Window(cudaStream_t st, const void* base, size_t bytes) : s(st) {
  const int mb = knobs().l2_persist_mb;
  if (mb <= 0 || !base || bytes == 0) return;
  static std::mutex mu;
  static std::set<int> carved;
  int dev = 0, maxw = 0, maxp = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev);
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
  size_t carve = std::min((size_t)mb << 20, (size_t)maxp);
  {
    std::lock_guard<std::mutex> g(mu);
    if (!carved.count(dev)) {
      if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) != cudaSuccess) { cudaGetLastError(); return; }
      carved.insert(dev);
    }
  }
  const size_t win = std::min(bytes, (size_t)maxw);
  if (win == 0 || carve == 0) return;
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)carve / (double)win));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  on = cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) == cudaSuccess;
  if (!on) cudaGetLastError();
}

L2Window::~L2Window() {
  if (!on) return;
  cudaStreamAttrValue v{};
  v.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v);
}

namespace {
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
}  // namespace

const DevKnobs& knobs() {
  static DevKnobs k;
  static std::once_flag once;
  std::call_once(once, [] {
    k.tc_spmm_bn = env_int("PGCN_TC_SPMM_BN", 0);
    if (k.tc_spmm_bn != 64 && k.tc_spmm_bn != 128 && k.tc_spmm_bn != 192 && k.tc_spmm_bn != 256) k.tc_spmm_bn = 0;
    k.tc_spmm_order = env_int("PGCN_TC_SPMM_ORDER", 1);
    k.tc_spmm_dbg = env_int("PGCN_TC_SPMM_DBG", 0);
    k.tc_spmm_nacc1 = env_int("PGCN_TC_SPMM_NACC1", 0);
    k.tc_spmm_ts = env_int("PGCN_TC_SPMM_TS", 1);
    k.tc_spmm_ctas = env_int("PGCN_TC_SPMM_CTAS", 2);
    k.tc_spmm_box64 = env_int("PGCN_TC_SPMM_BOX64", 1);
    k.tc_bnmax = env_int("PGCN_TC_BNMAX", 256);
    if (k.tc_bnmax < 16 || k.tc_bnmax > 256) k.tc_bnmax = 256;
    k.tc_gemm_ctas = env_int("PGCN_TC_GEMM_CTAS", 2);
    k.spmm_dyn = env_int("PGCN_SPMM_DYN", 1);
    const char* g = std::getenv("PGCN_SPMM_GRAB");
    k.spmm_grab = g ? std::atoll(g) : 128;
    if (k.spmm_grab < 1) k.spmm_grab = 128;
    k.spmm_table = std::getenv("PGCN_SPMM_TABLE");
    k.tf_off = env_int("PGCN_TF_OFF", 0);
    k.spmm_l2mb = env_int("PGCN_SPMM_L2MB", 96);
    k.dw_merge = env_int("PGCN_DW_MERGE", 1);
    k.presplit = env_int("PGCN_PRESPLIT", 0);
    k.spmm_nch = env_int("PGCN_SPMM_NCH", 2);
    k.tc_dw_bnmax = env_int("PGCN_TC_DW_BNMAX", 256);
    k.tc_bk16 = env_int("PGCN_TC_BK16", 2);
    k.tc_dw16 = env_int("PGCN_TC_DW16", 0);
    k.l2_persist_mb = env_int("PGCN_L2_PERSIST_MB", 0);
    k.tc_dw_ctas = env_int("PGCN_TC_DW_CTAS", 2) == 2 ? 2 : 1;
    if (k.tc_dw_bnmax < 32 || k.tc_dw_bnmax > 256 || k.tc_dw_bnmax % 32) k.tc_dw_bnmax = 256;
    if (k.spmm_nch < 2 || k.spmm_nch > 8) k.spmm_nch = 2;
    k.dw_kmax = env_int("PGCN_DW_KMAX", 128);
    if (k.dw_kmax < 0) k.dw_kmax = 128;
  });
  return k;
}

}  // namespace pgcn
