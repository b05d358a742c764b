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

// kMaxOrder: the specialised kernels (DMMA / DFMA top pair, mirror lists,
// staged moms2cums up to 6); above it the any-order kernels of generic.cu
// take over, up to the reference's limits (symten.hpp:87, cumulants.hpp:24).
constexpr int kMaxOrder = 8;
constexpr int kMaxOrderAny = CSB_MAX_ORDER;  // 20
constexpr int kMaxCumOrder = 6;              // generated partition code
constexpr int kMaxCumOrderAny = 16;
static_assert(kMaxOrderAny == 20, "CSB_MAX_ORDER follows the reference's SymTensor::kMaxOrder");

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

// One pair of prefix rows (pi, a0), (pi, a1) of the DMMA kernel, pi =
// (i_1..i_{L-1}).  The kernel packs the canonical prefix rows of one
// column window h (8h <= i_L < 8h + 8) densely, two per producer lane: a
// lane forms P = x[pi_1] ... x[pi_{L-1}] once per data row and the two
// Khatri-Rao values P x[a0], P x[a1].  a1 == a0 when the pair's second
// row does not exist (its slot is masked: PrefixRow::vprime == 0).
struct DmmaPair {
  uint16_t pidx[6];
  uint16_t a0, a1;
};
static_assert(sizeof(DmmaPair) == 16, "DmmaPair layout");

// One task of the CUDA-core kernel for the narrowest column windows
// (moment_tail_kernel): prefix pi = (i_1..i_{L-1}) and a run of last
// indices i_L in [s, e).  TAIL_TRI: the run spans the rest of its window and
// the task covers the columns [i_L, e) of each row plus the rows' order-L
// sums; TAIL_RECT: e - s <= 4 and the 8 columns [c0, c0 + 8) right of the
// window.  tail_rows[row0 + i] is the PrefixRow of (pi, s + i); padding
// tasks (whole warps share kind and run length) have row0 == kNoRow.
constexpr uint32_t kNoRow = 0xffffffffu;
constexpr uint16_t TAIL_TRI = 0, TAIL_RECT = 1;
struct TailTask {
  uint16_t pidx[6];
  uint16_t s, e, c0, kind;
  uint32_t row0;
};
static_assert(sizeof(TailTask) == 24, "TailTask layout");

// DFMA kernel: rows [row0, row0 + nrows) of the row table, columns
// [col0, col0 + ncols).  DMMA kernel: row sets [row0, row0 + nrows) (64
// prefix-row slots / 32 pairs each), column tiles of 8 starting at col0,
// ncols of them, R = pad0 row-set slots per CTA (1, 2 or 4; the 4 DMMA warps
// of the CTA cover R row sets x 4/R column ranges).
struct MomTile {
  uint32_t row0, nrows;  // range in the row table (DMMA: row sets)
  uint32_t J;            // block of the last prefix index (DMMA: column window h)
  uint32_t col0, ncols;  // DFMA: absolute column range; DMMA: first column, column tiles
  uint32_t low;          // 1: this tile also owns the M_{S-1} sums of its rows
  uint32_t pad0, pad1;   // DMMA: R, tile index
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
  bool dmma = false;  // tiles are for moment_top_dmma_kernel
  std::vector<DmmaPair> pairs;  // DMMA: 32 per row set
  DevBuf<DmmaPair> d_pairs;
  // DMMA plans: the narrowest column windows run on the CUDA cores instead
  std::vector<TailTask> tail;
  std::vector<PrefixRow> tail_rows;
  DevBuf<TailTask> d_tail;
  DevBuf<PrefixRow> d_tail_rows;
  void build(int S, int n, int b, const Layout& top, const Layout* low, int threads);
  // Tiles for the DMMA kernel.  Per column window h, the canonical prefix
  // rows with 8h <= i_L < 8h + 8 are packed in pairs (lexicographic pi, then
  // i_L), 32 pairs = 64 row slots per row set; rows[64 s + 2 j + e] is the
  // PrefixRow of element e of pair j of row set s (vprime == 0: masked).
  // Columns [8h, n) are covered in tiles of 8.
  // tail_windows: the last so many column windows become TailTasks
  // (moment_tail_kernel) instead of DMMA tiles
  void build_dmma(int S, int n, int b, const Layout& top, const Layout* low, uint64_t scratch_per_tile,
                  int tail_windows, const ShardPlan* shard = nullptr, int shard_index = 0, int sm_count = 148);
  void upload();

 private:
  std::vector<std::vector<PrefixRow>> enumerate(int S, int n, int b, const Layout& top, const Layout* low);
  PrefixRow make_row(const int* t, const Layout& top, const Layout* low) const;
};

}  // namespace csb
