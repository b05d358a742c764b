// Device-side parameter blocks shared by kernels.cu and runtime.cpp.
#pragma once

#include <cstdint>

#include "layout.hpp"

namespace csb {

// Rows [0, len0) come from seg0, rows [len0, len0 + len1) from seg1
// (the ring buffer's two segments in arrival order, stream.cpp:39-66).
struct RowSource {
  const double* seg0 = nullptr;
  const double* seg1 = nullptr;
  uint32_t len0 = 0, len1 = 0;
};

struct MomParams {
  RowSource src[2];     // pass 0 (incoming / window), pass 1 (outgoing)
  int npass = 1;        // 1: assign (moment_series), 2: update (moments_update)
  uint32_t K = 0;       // rows per pass
  int n = 0, b = 0, L = 0;
  const PrefixRow* rows = nullptr;
  const MomTile* tiles = nullptr;
  const DmmaPair* pairs = nullptr;  // DMMA kernel only
  double* top = nullptr;      // M_S
  double* low = nullptr;      // M_{S-1} (nullptr: not written)
  double* scratch = nullptr;  // pass-0 stash (DMMA: per tile)
  const double* zeros = nullptr;  // DMMA: >= 16 x n zero doubles (tail rows of a pass)
  int stages = 0;                 // DMMA: row-chunk stages in shared memory
  const TailTask* tail = nullptr;  // moment_tail_kernel: tasks (32 per warp), rows = their PrefixRows
  uint32_t tail_warps = 0;
  uint32_t stash_slots = 0, stash_stride = 0;  // moment_tail_kernel: per-SM stash in scratch
  double c = 0.0;             // p / T        (moments.cpp:287)
  double inv = 1.0;           // 1.0 / rows   (moments.cpp:148)
};

struct LayoutDev {
  const uint64_t* offset = nullptr;  // nblocks + 1
  const uint16_t* index = nullptr;   // nblocks x order
  const uint64_t* prefix = nullptr;  // order x (grid + 1)
  int order = 0, grid = 0;
  uint64_t nblocks = 0;
};

struct M2CParams {
  const double* m = nullptr;        // M_S
  double* c = nullptr;              // C_S
  const double* lower[kMaxOrder];   // C_1 .. C_{S-1}
  LayoutDev lay[kMaxOrder];         // layouts of orders 1..S (index s-1)
  int n = 0, b = 0;
  uint64_t blk0 = 0;                // first block of the shard
  // (dst, src) symmetric-copy pairs of a full block per run pattern (or
  // nullptr); with them a full block is assembled in shared memory at
  // cblk (doubles past the staged sub-blocks) and written out coalesced
  const uint2* mlist = nullptr;
  const uint32_t* mlist_off = nullptr;
  uint32_t cblk = 0;
  bool inblk = false;  // launcher: the block fits beside the sub-blocks (cblk valid)
  double* mfix = nullptr;  // M_S itself: also write its symmetric copies from the staged block
  const uint64_t* subs = nullptr;   // per block, masks 1..2^S-2: offset of the sub-block in C_|mask|
  // canonical positions of a full block (all extents b) per run pattern
  // (bit k-1: j_k == j_{k-1}): canon[canon_off[pat] .. canon_off[pat + 1])
  const uint32_t* canon = nullptr;
  const uint32_t* canon_off = nullptr;
  // per canonical position (indexed like canon): its symmetric copies in the
  // block, cdst[cstart[i] .. cstart[i + 1]) -- the out-of-block pass writes
  // them and weights the norm term by 1 + copies right after computing it
  const uint32_t* cstart = nullptr;
  const uint32_t* cdst = nullptr;
  // persistent kernel: the blocks in descending order of canonical entries
  // (nullptr: block order); CTAs take them round-robin, so every CTA's -- and
  // each of its halves' -- share of the arithmetic is the same within a block
  const uint32_t* order = nullptr;
  double* partial = nullptr;        // per block: sum over stored entries of v*v
  int fold_width = 0;               // > 0: exact knorm partials (in-block path; see launch_moms2cums_v2)
};

// One canonical element of a low order (S <= d-2): indices and the offset
// of its block in M_S.
struct LowerElem {
  uint16_t idx[8];
  uint64_t blk_off;
};

struct LowerParams {
  RowSource src[2];
  int npass = 1;
  int n = 0, b = 0;
  const LowerElem* elems = nullptr;
  uint64_t count = 0;
  double* m = nullptr;
  double c = 0.0, inv = 1.0;
};

// One thread of the staged low-order kernel (orders 1..ST, ST = d-2 <= 4):
// the order-ST elements (pi, t0 + w), w < cnt (consecutive in lexicographic
// order, element ids e0 + w), and the lower-order tuples (pi_1..pi_s) it
// represents (rep[s-1], 0xffffffff: none).
struct LowerThread {
  uint32_t e0;
  uint32_t rep[3];
  uint16_t pidx[4];
  uint16_t t0, cnt;
  uint32_t pad;
};
static_assert(sizeof(LowerThread) == 32, "LowerThread layout");

struct Lower2Params {
  RowSource src[2];
  int npass = 1;
  uint32_t K = 0;
  int n = 0, b = 0;
  const LowerThread* threads = nullptr;
  uint32_t nthreads = 0;
  const LowerElem* elems[4] = {nullptr, nullptr, nullptr, nullptr};  // orders 1..ST
  double* m[4] = {nullptr, nullptr, nullptr, nullptr};                // M_1..M_ST
  double c = 0.0, inv = 1.0;
};

struct NormParams {
  const double* partial[kMaxOrderAny];  // per order, nblocks each
  const double* mult[kMaxOrderAny];     // per order block multiplicities (as double)
  uint64_t nblocks[kMaxOrderAny];
  int norders = 0;                   // orders 1..norders
  bool fold = true;                  // false: only the diagonals are gathered (the host folds the blocks)
  const double* diag_src[3];         // C_2, C_3, C_4 (nullptr if absent)
  const uint64_t* diag_off[3];       // n offsets each
  int n = 0;
  double* out = nullptr;             // [norders sums][3 x n diagonals]
};

// any-order kernels (generic.cu): one thread per stored element
struct GenMomParams {
  RowSource src[2];
  int npass = 1;
  uint32_t K = 0;
  int n = 0, b = 0;
  bool top = false;  // this is the series' top order: acc = fma(q, x, acc) (moments.cpp:47)
  double* m = nullptr;
  LayoutDev lay;
  uint64_t stored = 0;
  double c = 0.0, inv = 1.0;
};
struct GenM2CParams {
  const double* m = nullptr;  // M_s
  double* c = nullptr;        // C_s
  const double* lower[kMaxCumOrderAny];  // C_1 .. C_{s-1}
  LayoutDev lay[kMaxCumOrderAny];        // layouts of orders 1..s
  int n = 0, b = 0, s = 0;
  uint64_t stored = 0;
};
void launch_moment_generic(const GenMomParams& p, cudaStream_t st);
void launch_moms2cums_generic(const GenM2CParams& p, cudaStream_t st);

void launch_moment_pair(const MomParams& p, int ntiles, bool top_fma, cudaStream_t st);
// whether moms2cums of order S assembles every block in shared memory
// (then it can also fill M_S's symmetric copies: MomentPlan's deferred mirror)
bool m2c_fuse_ok(int S, int n, int b);
// returns whether the blocks' exact norm partials were written (p.fold_width)
bool launch_moms2cums_v2(int S, const M2CParams& p, uint64_t nblocks, cudaStream_t st);
void launch_moment_lower(int S, const LowerParams& p, cudaStream_t st);
void launch_moment_lower2(int ST, int W, const Lower2Params& p, cudaStream_t st);
// orders <= ST of few elements: one thread per element, TMA-staged rows
bool lower_tma_supported(const Lower2Params& p);
void launch_moment_lower_tma(int ST, int W, const Lower2Params& p, cudaStream_t st);
void launch_moment_lower_side(int ST, const Lower2Params& p, cudaStream_t st);
void launch_gather(const double* t, const uint64_t* off, uint64_t count, double* out, cudaStream_t st);
void launch_copy_c1(const double* m1, double* c1, double* partial, const LayoutDev& lay,
                    uint64_t nblocks, uint64_t stored, cudaStream_t st);
void launch_norm_finalize(const NormParams& p, cudaStream_t st);
// per-block sums of |e|^k of blocks [blk0, blk0 + nblk) in the reference's
// exact order (partial indexed by absolute block); width: the reference
// build's vector width of the k = 2 fold (4 or 8)
void launch_knorm_exact(const double* t, const LayoutDev& lay, uint64_t blk0, uint64_t nblk, double k, int width,
                        double* partial, cudaStream_t st);
void launch_diag_pick(const double* c, const uint64_t* off, uint64_t lo, uint64_t hi, int n, double* out,
                      cudaStream_t st);
void launch_combine(const double* a, const double* b, double w1, double w2, double* out,
                    uint64_t count, cudaStream_t st);

constexpr int kMomThreads = 256;

// Kernels this library has launched in this process (bench.py's
// gpu_launches claim).
uint64_t launch_count();
void count_launch();
void add_launches(uint64_t k);

// FP64 tensor-core (DMMA) kernel for the top pair of orders (moment_dmma.cu)
bool dmma_supported(const MomParams& p);
uint32_t dmma_chunk_rows(int n, int b);
bool tail_supported(int n, int b);  // moment_tail_kernel fits for this row length
int tail_windows(int S, int n, int b);  // column windows of order S the tail kernel takes
size_t tail_scratch_doubles();          // scratch the tail kernel needs (per-SM stash)
void launch_moment_tail(const MomParams& p, cudaStream_t st);
const char* dmma_kernel_name(int n, int b);
// every non-empty segment of the pass sources starts on a 16-byte boundary
// (the bulk copies' requirement; rows themselves are 16-byte multiples
// when n is even)
inline bool rows_aligned16(const RowSource* src, int npass) {
  for (int q = 0; q < npass; ++q) {
    if (src[q].len0 && (reinterpret_cast<uintptr_t>(src[q].seg0) & 15u)) return false;
    if (src[q].len1 && (reinterpret_cast<uintptr_t>(src[q].seg1) & 15u)) return false;
  }
  return true;
}
size_t dmma_scratch_per_tile();
void launch_moment_top_dmma(const MomParams& p, int ntiles, cudaStream_t st);
// copies of canonical entries in blocks with runs (after the DMMA kernel)
// symmetric copies of the canonical entries of the listed stored blocks
// (lists: per run pattern (dst, src) pairs of a full block, or nullptr)
void launch_mirror(int S, double* m, const LayoutDev& lay, const uint32_t* blocks, uint32_t nblocks, int n, int b,
                   const uint2* lists, const uint32_t* list_off, cudaStream_t st);

}  // namespace csb
