// Host builder of the dense-tile decomposition (tiles.h).  One pass per 128-row block: count the
// edges per 64-column tile, keep the tiles with >= min_edges as bitmasks, route the rest (and any
// repeated (row, col) pair) to the light CSR, sorted by column within each row.
#include "tiles.h"

#include "common.h"
#include "pgcn_dev.h"

#include <algorithm>
#include <atomic>
#include <thread>

namespace pgcn {

namespace {

struct BlockOut {
  std::vector<int32_t> tcol;
  std::vector<uint64_t> mask;
  std::vector<int32_t> lcnt;  // light edges per row of the block
  std::vector<int32_t> lcol;
};

void one_block(const int64_t* rp, const int32_t* col, int64_t r0, int64_t r1, int32_t min_edges,
               std::vector<int32_t>& cnt, std::vector<int32_t>& slot, std::vector<int32_t>& touched, BlockOut& o) {
  touched.clear();
  for (int64_t r = r0; r < r1; ++r)
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int32_t j = col[e] / kTileCols;
      if (cnt[j]++ == 0) touched.push_back(j);
    }
  std::sort(touched.begin(), touched.end());
  for (int32_t j : touched)
    if (cnt[j] >= min_edges) {
      slot[j] = (int32_t)o.tcol.size();
      o.tcol.push_back(j);
    }
  o.mask.assign(o.tcol.size() * kTileRows, 0ull);
  o.lcnt.assign((size_t)(r1 - r0), 0);
  for (int64_t r = r0; r < r1; ++r) {
    const size_t row_begin = o.lcol.size();
    for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
      const int32_t c = col[e], j = c / kTileCols;
      if (slot[j] >= 0) {
        uint64_t& w = o.mask[(size_t)slot[j] * kTileRows + (size_t)(r - r0)];
        const uint64_t bit = 1ull << (c % kTileCols);
        if (!(w & bit)) {
          w |= bit;
          continue;
        }
      }
      o.lcol.push_back(c);
      ++o.lcnt[(size_t)(r - r0)];
    }
    std::sort(o.lcol.begin() + row_begin, o.lcol.end());
  }
  for (int32_t j : touched) {
    cnt[j] = 0;
    slot[j] = -1;
  }
}

}  // namespace

void build_tiles(const int64_t* rp, const int32_t* col, int64_t n_rows, int64_t n_cols, int32_t min_edges,
                 int32_t n_threads, TileSet& out) {
  out = TileSet{};
  out.n_rows = n_rows;
  out.n_cols = n_cols;
  out.min_edges = min_edges < 1 ? 1 : min_edges;
  out.n_rb = (n_rows + kTileRows - 1) / kTileRows;
  const int64_t n_ct = (n_cols + kTileCols - 1) / kTileCols;
  std::vector<BlockOut> blocks((size_t)out.n_rb);
  const int nt = std::max(1, std::min<int>(n_threads, (int)std::min<int64_t>(out.n_rb, 64)));
  std::atomic<int64_t> next{0};
  auto work = [&] {
    std::vector<int32_t> cnt((size_t)n_ct + 1, 0), slot((size_t)n_ct + 1, -1), touched;
    for (int64_t b = next++; b < out.n_rb; b = next++)
      one_block(rp, col, b * kTileRows, std::min(n_rows, (b + 1) * kTileRows), out.min_edges, cnt, slot, touched,
                blocks[(size_t)b]);
  };
  if (nt == 1) {
    work();
  } else {
    std::vector<std::thread> th;
    for (int k = 0; k < nt; ++k) th.emplace_back(work);
    for (auto& t : th) t.join();
  }
  out.rb_ptr.assign((size_t)out.n_rb + 1, 0);
  for (int64_t b = 0; b < out.n_rb; ++b) out.rb_ptr[b + 1] = out.rb_ptr[b] + (int32_t)blocks[b].tcol.size();
  out.n_tiles = out.rb_ptr[out.n_rb];
  out.tile_col.resize((size_t)out.n_tiles);
  out.mask.resize((size_t)out.n_tiles * kTileRows);
  out.lrp.assign((size_t)n_rows + 1, 0);
  for (int64_t b = 0; b < out.n_rb; ++b) {
    const BlockOut& o = blocks[b];
    std::copy(o.tcol.begin(), o.tcol.end(), out.tile_col.begin() + out.rb_ptr[b]);
    std::copy(o.mask.begin(), o.mask.end(), out.mask.begin() + (size_t)out.rb_ptr[b] * kTileRows);
    for (size_t i = 0; i < o.lcnt.size(); ++i) {
      const int64_t r = b * kTileRows + (int64_t)i;
      out.lrp[r + 1] = out.lrp[r] + o.lcnt[i];
    }
  }
  out.nnz_light = out.lrp[n_rows];
  out.nnz_heavy = (n_rows > 0 ? rp[n_rows] - rp[0] : 0) - out.nnz_light;
  out.lcol.resize((size_t)out.nnz_light);
  for (int64_t b = 0; b < out.n_rb; ++b) {
    const BlockOut& o = blocks[b];
    std::copy(o.lcol.begin(), o.lcol.end(), out.lcol.begin() + out.lrp[b * kTileRows]);
  }
  out.order.resize((size_t)out.n_rb);
  for (int64_t b = 0; b < out.n_rb; ++b) out.order[b] = (int32_t)b;
  std::stable_sort(out.order.begin(), out.order.end(), [&](int32_t a, int32_t b) {
    return out.rb_ptr[a + 1] - out.rb_ptr[a] > out.rb_ptr[b + 1] - out.rb_ptr[b];
  });
}

}  // namespace pgcn

extern "C" int pgcn_dev_tiles(const pgcn_partitioning* p, int32_t part, int32_t which, int32_t tile_min,
                              int64_t* sizes, int32_t* rb_ptr, int32_t* order, int32_t* tile_col, uint64_t* mask,
                              int64_t* lrp, int32_t* lcol) {
  if (!p || !sizes) return pgcn::fail(PGCN_EINVAL, "pgcn_dev_tiles: null argument");
  if (which != 0 && which != 1) return pgcn::fail(PGCN_EINVAL, "pgcn_dev_tiles: which must be 0 or 1");
  if (tile_min < 1) return pgcn::fail(PGCN_EINVAL, "pgcn_dev_tiles: tile_min < 1");
  const pgcn::TileSet* t = pgcn::part_tiles(p, part, which, tile_min);
  if (!t) return pgcn::fail(PGCN_EINVAL, "pgcn_dev_tiles: part out of range");
  sizes[0] = t->n_rows;
  sizes[1] = t->n_rb;
  sizes[2] = t->n_tiles;
  sizes[3] = t->nnz_heavy;
  sizes[4] = t->nnz_light;
  sizes[5] = t->n_cols;
  if (rb_ptr) std::copy(t->rb_ptr.begin(), t->rb_ptr.end(), rb_ptr);
  if (order) std::copy(t->order.begin(), t->order.end(), order);
  if (tile_col) std::copy(t->tile_col.begin(), t->tile_col.end(), tile_col);
  if (mask) std::copy(t->mask.begin(), t->mask.end(), mask);
  if (lrp) std::copy(t->lrp.begin(), t->lrp.end(), lrp);
  if (lcol) std::copy(t->lcol.begin(), t->lcol.end(), lcol);
  return PGCN_OK;
}
