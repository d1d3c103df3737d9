// Seeded synthetic graph generator (input generation only; none of the
// PipeGCN method's arithmetic lives here).  Recipe: synth/graphs.py docstring
// and DESIGN.md "Input recipe".  Deterministic for a given seed regardless of
// the thread count: every random draw is a counter-based hash of
// (seed, stream, node, index), and rows are sorted + deduplicated at the end.
//
// C ABI (ctypes):
//   int64_t synth_edges(int64_t n, int32_t n_comm, double stubs_mean, double scale,
//                       double cross, uint64_t seed, int32_t n_threads,
//                       int64_t* row_ptr /*[n+1] out*/, int32_t** col_out /*malloc'd*/);
//   void synth_free(void*);
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

namespace {

inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
inline uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix64(seed ^ mix64(a ^ mix64(b)));
}
inline double u01(uint64_t h) { return (double)(h >> 11) * (1.0 / 9007199254740992.0); }

template <class F>
void parallel_for(int64_t n, int nt, F f) {
  if (nt <= 1 || n < 4096) { f(0, n, 0); return; }
  std::vector<std::thread> th;
  int64_t chunk = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    int64_t lo = t * chunk, hi = std::min<int64_t>(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=] { f(lo, hi, t); });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int64_t synth_edges(int64_t n, int32_t n_comm, double stubs_mean, double scale, double cross,
                    uint64_t seed, int32_t n_threads, int64_t* row_ptr, int32_t** col_out) {
  if (n <= 0 || n_comm <= 0 || !row_ptr || !col_out) return -1;
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t csize = std::max<int64_t>(n / n_comm, 1);
  // 1. stubs per node: k_v = floor(mean * scale * lambda_v + u), lambda ~ LogNormal(-1/2, 1) clipped at 50
  std::vector<int64_t> k(n + 1, 0);
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v) {
      double u1 = u01(h3(seed, 1, (uint64_t)v)), u2 = u01(h3(seed, 2, (uint64_t)v));
      double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
      double lam = std::min(std::exp(-0.5 + z), 50.0);
      double u3 = u01(h3(seed, 3, (uint64_t)v));
      k[v + 1] = (int64_t)std::floor(stubs_mean * scale * lam + u3);
    }
  });
  for (int64_t v = 0; v < n; ++v) k[v + 1] += k[v];
  const int64_t m = k[n];
  // 2. far end of each stub
  std::vector<int32_t> dst(m);
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v) {
      int64_t c = std::min<int64_t>(v / csize, n_comm - 1);
      int64_t start = c * csize, size = (c == n_comm - 1) ? n - start : csize;
      for (int64_t j = k[v]; j < k[v + 1]; ++j) {
        uint64_t a = h3(seed, 4, (uint64_t)j), b = h3(seed, 5, (uint64_t)j);
        int64_t d;
        if (u01(a) >= cross) d = start + std::min<int64_t>((int64_t)(u01(b) * size), size - 1);
        else d = (int64_t)(u01(b) * n) % n;
        dst[j] = (int32_t)d;
      }
    }
  });
  // 3. symmetrise into per-row buckets (counts, then fill with atomic cursors)
  std::vector<std::atomic<int64_t>> cnt(n);
  for (int64_t v = 0; v < n; ++v) cnt[v].store(0, std::memory_order_relaxed);
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v)
      for (int64_t j = k[v]; j < k[v + 1]; ++j) {
        int64_t d = dst[j];
        if (d == v) continue;
        cnt[v].fetch_add(1, std::memory_order_relaxed);
        cnt[d].fetch_add(1, std::memory_order_relaxed);
      }
  });
  std::vector<int64_t> off(n + 1, 0);
  for (int64_t v = 0; v < n; ++v) off[v + 1] = off[v] + cnt[v].load(std::memory_order_relaxed);
  std::vector<int32_t> buf(off[n]);
  for (int64_t v = 0; v < n; ++v) cnt[v].store(off[v], std::memory_order_relaxed);
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v)
      for (int64_t j = k[v]; j < k[v + 1]; ++j) {
        int64_t d = dst[j];
        if (d == v) continue;
        buf[cnt[v].fetch_add(1, std::memory_order_relaxed)] = (int32_t)d;
        buf[cnt[d].fetch_add(1, std::memory_order_relaxed)] = (int32_t)v;
      }
  });
  std::vector<int32_t>().swap(dst);
  // 4. sort + dedupe each row
  std::vector<int64_t> len(n + 1, 0);
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v) {
      int32_t* b = buf.data() + off[v];
      int64_t L = off[v + 1] - off[v];
      std::sort(b, b + L);
      len[v + 1] = std::unique(b, b + L) - b;
    }
  });
  row_ptr[0] = 0;
  for (int64_t v = 0; v < n; ++v) row_ptr[v + 1] = row_ptr[v] + len[v + 1];
  int64_t nnz = row_ptr[n];
  int32_t* col = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz, 1));
  if (!col) return -2;
  parallel_for(n, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t v = lo; v < hi; ++v)
      std::memcpy(col + row_ptr[v], buf.data() + off[v], sizeof(int32_t) * (size_t)len[v + 1]);
  });
  *col_out = col;
  return nnz;
}

// Per-row inputs for huge graphs (papers100M-shaped), generated only for the rows a rank owns: every value
// is a counter-based hash of (seed, stream, gid, column), so any subset of rows is reproducible on its own
// (synth/graphs.py rows_inputs).  Same distributions as gen_graph's numpy draws: X = N(0,1) + 1 at column
// (community mod f0); label = community mod classes w.p. 0.8 else uniform; train = U(0,1) < train_frac.
void synth_rows(uint64_t seed, int64_t n, int32_t n_comm, int32_t f0, int32_t classes, double train_frac,
                const int64_t* gids, int64_t m, int32_t n_threads, float* X, int32_t* labels, uint8_t* train) {
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  const int64_t csize = std::max<int64_t>(n / n_comm, 1);
  parallel_for(m, nt, [&](int64_t lo, int64_t hi, int) {
    for (int64_t r = lo; r < hi; ++r) {
      const uint64_t g = (uint64_t)gids[r];
      const int64_t c = std::min<int64_t>((int64_t)g / csize, n_comm - 1);
      float* x = X + r * f0;
      for (int32_t j = 0; j < f0; j += 2) {  // Box-Muller pairs
        const uint64_t k = g * (uint64_t)(f0 + 1) + (uint64_t)j;
        const double u1 = u01(h3(seed, 11, k)), u2 = u01(h3(seed, 12, k));
        const double rad = std::sqrt(-2.0 * std::log(1.0 - u1)), th = 6.283185307179586 * u2;
        x[j] = (float)(rad * std::cos(th));
        if (j + 1 < f0) x[j + 1] = (float)(rad * std::sin(th));
      }
      x[c % f0] += 1.0f;
      const bool keep = u01(h3(seed, 13, g)) < 0.8;
      labels[r] = keep ? (int32_t)(c % classes) : (int32_t)(h3(seed, 14, g) % (uint64_t)classes);
      train[r] = u01(h3(seed, 15, g)) < train_frac ? 1 : 0;
    }
  });
}

void synth_free(void* p) { std::free(p); }

}  // extern "C"
