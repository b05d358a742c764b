// Host-side block layout and launch plans.
//
// Layout reproduces the reference's SymTensor storage bit for bit
// (/root/reference/proj/src/symten.cpp:105-140): blocks with non-decreasing
// block index j in lexicographic order, each a dense C-order block with
// extents min(b, n - j_k b), one flat array.  The block ranker is the
// reference's lexicographic multiset rank (symten.hpp:19-59).
//
// MomentPlan is the GEMM view of one pair of orders (S, S-1) (SURVEY
// Appendix B): rows = canonical (S-1)-prefixes (i_1 <= ... <= i_{S-1}),
// grouped by the block J = i_{S-1} / b of their last index; columns =
// i_S in [J b, n).  M_S[prefix, i_S] = sum_rows A[row, prefix] x[row, i_S]
// with A the left-to-right product of the prefix columns, and
// M_{S-1}[prefix] = sum_rows A[row, prefix].
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "common.hpp"

namespace csb {

constexpr int kMaxOrder = CSB_MAX_ORDER;

struct Layout {
  int order = 0, dim = 0, block = 0, grid = 0;
  uint64_t nblocks = 0, stored = 0;
  std::vector<uint16_t> index;    // nblocks x order block coordinates
  std::vector<uint64_t> offset;   // nblocks + 1 (last = stored)
  std::vector<uint64_t> prefix;   // ranker table: order x (grid + 1)

  Layout() = default;
  Layout(int order, int dim, int block);

  int ext(int j) const { return block < dim - j * block ? block : dim - j * block; }
  uint64_t rank(const int* j) const;          // block rank of a sorted block index
  uint64_t element_offset(const int* i) const;  // at_sorted_unchecked addressing
  uint64_t volume(uint64_t r) const { return offset[r + 1] - offset[r]; }
};

uint64_t block_multiplicity(const int* j, int d);

// One prefix row of the GEMM view (48 bytes, 16-byte aligned).
struct alignas(16) PrefixRow {
  uint16_t idx[8];    // i_1..i_L (L = S-1 <= 7)
  uint64_t top_base;  // offset in M_S of block (j_1..j_L, J)
  uint64_t low_off;   // offset in M_{S-1} of this prefix's canonical element
  uint32_t vprime;    // prefix block volume prod_{k<=L} e(j_k)
  uint32_t poff;      // in-block prefix offset (Horner over o_1..o_L)
};
static_assert(sizeof(PrefixRow) == 48, "PrefixRow layout");

// One group of 8 prefix rows (pi, 8h + g), g = 0..7, for the DMMA kernel:
// pi = (i_1..i_{L-1}); rows with g < lo (i_L < i_{L-1}) or 8h + g >= n are
// not canonical and are masked.
//
// A group may also represent lower-order elements: its prefix products at
// depth s (x[pi_1] ... x[pi_s]) are the order-s moment products of the
// tuple (pi_1..pi_s); the group (pi_1..pi_s, pi_s, ..., pi_s) in its first
// window h = pi_s / 8 is that tuple's unique representative (rep_mask bit
// s-1), so the producer warps compute every order <= d-2 as well.
struct DmmaGroup {
  uint16_t pidx[6];
  uint16_t lo;
  uint16_t h;
  uint32_t rep;       // first entry in MomentPlan::rep_off (valid when rep_mask != 0)
  uint32_t rep_mask;  // bit s-1: this group represents order-s tuple (pi_1..pi_s)
  uint32_t pad[2];
};
static_assert(sizeof(DmmaGroup) == 32, "DmmaGroup layout");

struct MomTile {
  uint32_t row0, nrows;  // range in the row table
  uint32_t J;            // block of the last prefix index
  uint32_t col0, ncols;  // absolute column range [col0, col0 + ncols)
  uint32_t low;          // 1: this tile also owns the M_{S-1} sums of its rows
  uint32_t pad0, pad1;
};

// Block-prefix sharding of the top pair of orders: order-d
// blocks are owned by their first plen block coordinates (2 for d = 4, 3 for
// d >= 5, never more than d-2), in contiguous prefix ranges from a min-max
// partition of the canonical-element weight.  Ownership then depends only on the (d-2)-prefix pi of a DMMA
// group, so a shard computes whole groups, owns a contiguous range of
// order-d blocks AND a contiguous range of order-(d-1) blocks.
struct ShardPlan {
  int d = 0, n = 0, b = 0, count = 1;
  int plen = 0;                          // prefix length (block coordinates)
  std::shared_ptr<Layout> prefix_rank;   // lexicographic ranker of prefixes
  std::vector<int> shard_of_prefix;      // by lexicographic prefix rank
  std::vector<uint64_t> top_blk, low_blk;  // count + 1 block boundaries (orders d, d-1)
  void build(int d, int n, int b, int count, const Layout& top, const Layout& low);
  int owner(const int* block_prefix) const;  // shard of a block prefix (plen coords)
};

struct MomentPlan {
  int S = 0, L = 0, n = 0, b = 0;
  std::vector<PrefixRow> rows;
  std::vector<MomTile> tiles;
  DevBuf<PrefixRow> d_rows;
  DevBuf<MomTile> d_tiles;
  uint64_t scratch_per_tile = 0;  // doubles
  bool dmma = false;  // tiles are for moment_top_dmma_kernel (pad0 = column groups)
  std::vector<DmmaGroup> groups;
  DevBuf<DmmaGroup> d_groups;
  std::vector<uint64_t> rep_off;  // canonical offset in M_s (bit 63: block has copies)
  DevBuf<uint64_t> d_rep_off;
  void build(int S, int n, int b, const Layout& top, const Layout* low, int threads);
  // Tiles for the DMMA kernel: groups (pi, h) of 8 prefix rows, 8 groups per
  // warp; columns [8h, n) in ranges of at most 4 groups of 8; rows[8 g + r]
  // is the PrefixRow of row r of group g (zero for masked rows).
  // lowers[s-1] = layout of order s (s <= S-2) when the groups should also
  // compute the lower orders (unsharded plans), nullptr otherwise
  void build_dmma(int S, int n, int b, const Layout& top, const Layout* low, int warps,
                  uint64_t scratch_per_tile, const ShardPlan* shard = nullptr, int shard_index = 0,
                  const Layout* const* lowers = nullptr);
  void upload();

 private:
  std::vector<std::vector<PrefixRow>> enumerate(int S, int n, int b, const Layout& top, const Layout* low);
  PrefixRow make_row(const int* t, const Layout& top, const Layout* low) const;
};

}  // namespace csb
