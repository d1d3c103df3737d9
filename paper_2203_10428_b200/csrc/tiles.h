// Dense-tile decomposition of a local CSR pattern for the tensor-core SpMM (spmm_tc.cu).  Internal.
//
// A pattern of n_rows x n_cols (P_i: inner rows x local columns, or P_i^T) is cut into row blocks
// of 128 rows and column tiles of 64 columns.  A tile holding at least `min_edges` edges is
// "heavy": its edges are stored as a 128 x 64 bitmask (one uint64 per row) and aggregated as a
// dense 0/1 block times the 64 gathered rows on the tensor cores; every other edge (and a repeated
// (row, col) pair, which a bitmask cannot count twice) stays in the "light" CSR, columns ascending
// within a row, for the gather SpMM.
// sum over heavy bits + light edges = the pattern, exactly.
#pragma once
#include <cstdint>
#include <vector>

#include "pgcn.h"

namespace pgcn {

constexpr int kTileRows = 128;  // UMMA M
constexpr int kTileCols = 64;   // bits of one mask word

struct TileSet {
  int64_t n_rows = 0, n_cols = 0, n_rb = 0, n_tiles = 0, nnz_heavy = 0, nnz_light = 0;
  int32_t min_edges = 0;
  std::vector<int32_t> rb_ptr;    // [n_rb + 1] heavy tiles of row block b: [rb_ptr[b], rb_ptr[b+1])
  std::vector<int32_t> order;     // [n_rb] row blocks by descending heavy-tile count (static LPT work list)
  std::vector<int32_t> tile_col;  // [n_tiles] column tile j (columns 64 j .. 64 j + 63), ascending per block
  std::vector<uint64_t> mask;     // [n_tiles x 128] bit c of word r: edge (128 b + r, 64 j + c)
  std::vector<int64_t> lrp;       // [n_rows + 1] light CSR, columns ascending within a row
  std::vector<int32_t> lcol;      // [nnz_light]
};

// Builds the decomposition (deterministic, independent of n_threads).
void build_tiles(const int64_t* row_ptr, const int32_t* col, int64_t n_rows, int64_t n_cols, int32_t min_edges,
                 int32_t n_threads, TileSet& out);

// Cached on the partitioning handle (built on first use, freed with it): which = 0 -> P_i
// (n_inner x (n_inner + n_halo)), 1 -> P_i^T ((n_inner + n_halo) x n_inner).
const TileSet* part_tiles(const pgcn_partitioning* p, int32_t part, int which, int32_t min_edges);

}  // namespace pgcn
