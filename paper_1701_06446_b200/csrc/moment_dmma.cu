// Top-order moment kernel on the FP64 tensor cores (DMMA, sm_100a).
//
// GEMM view: for the pair of orders (d, d-1),
//   M_d[prefix, col] = sum_k A[prefix, k] * x[k, col],   col >= i_L,
//   M_{d-1}[prefix]  = sum_k A[prefix, k],
// with A[prefix, k] = x[k,i_1] * x[k,i_2] * ... * x[k,i_L] (left to right,
// moments.cpp:55,71).  The contraction runs on mma.sync.m8n8k4.f64, which
// on B200 evaluates each output as the sequential FMA chain over its four
// k values in order (measured: tools/fp64_peak.cu, 0 mismatches in 12,800);
// chaining the MMAs over k in row order therefore reproduces the
// reference's row-ordered fma(A, x, acc) (moments.cpp:47) bit for bit.
//
// Work decomposition (MomentPlan::build_dmma).  The canonical prefix rows
// (i_1 <= ... <= i_L) whose last index lies in the column window
// [8h, 8h + 8) all need the output columns [8h, n); they are packed densely
// in pairs (pi, a0), (pi, a0 + 1) -- no masked rows apart from odd tails --
// into row sets of 64 rows.  A CTA takes R row sets (R = 4, 2, 1 for windows
// with <= 4, <= 8, > 8 column tiles) and a range of <= 16/R column tiles;
// its 4 DMMA warps cover R row sets x 4/R column ranges, so each Khatri-Rao
// value is formed once per CTA and reused over up to 128 columns.
//
// Per CTA: 4 DMMA (consumer) warps + up to 4 producer warps (one per row
// set).  Data rows stream through a shared-memory ring of 16-row chunks
// filled by TMA bulk copies (cp.async.bulk, mbarrier complete_tx); the last
// warp to release a stage refills it at once.  A producer
// lane owns one pair: per data row it forms P = x[pi_1] ... x[pi_{L-1}] and
// the two products P x[a0], P x[a1], adds them to its order-(d-1) row sums
// in row order and stores them in MMA fragment order into its row set's
// A ring (2 slots of one chunk each, full/empty mbarriers).  The DMMA warps
// read A fragments from the ring and B fragments (the data rows) straight
// from the staged chunk.  The incoming pass's means are stashed at the pass
// boundary; the epilogue applies M = fma(p/T, a - b, M) (moments.cpp:297) to
// the canonical entries (mirror_kernel then fixes the symmetric copies).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace csb {

namespace {

constexpr int CWARPS = 4;                 // DMMA consumer warps
constexpr int PWARPS = 4;                 // producer warps (one per row set)
constexpr int THREADS = (CWARPS + PWARPS) * 32;
constexpr int HSTEPS = 4;                 // k4 steps per chunk
constexpr int KC = 4 * HSTEPS;            // data rows per chunk / stage
constexpr int ASTRIDE = 10;               // doubles per (r, q) entry: 8 used, bank-conflict free
constexpr int ASLOT = HSTEPS * 32 * ASTRIDE;
constexpr int ASLOTS = 2;                 // A-ring slots per row set
constexpr int MAX_STAGES = 12;
constexpr int SLOTS_PER_SET = 64;         // prefix rows per row set

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ const double* row_ptr(const RowSource& s, uint32_t k, int n) {
  return k < s.len0 ? s.seg0 + static_cast<size_t>(k) * n
                    : s.seg1 + static_cast<size_t>(k - s.len0) * n;
}

__device__ __forceinline__ int ext_of(int j, int n, int b) { return b < n - j * b ? b : n - j * b; }

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// ---------------------------------------------------------------------------
// Shared state of one CTA.
struct Ring {
  double* xs;          // stages x KC x n data rows
  double* arings;      // PWARPS x ASLOTS x ASLOT
  uint64_t* xfull;     // per stage: TMA bytes landed
  uint32_t* rel;       // per stage: release counter (active warps per round)
  uint64_t* afull;     // per row set and slot: producer lanes stored
  uint64_t* aempty;    // per row set and slot: DMMA lanes consumed
  uint32_t stages;
  uint32_t active;       // warps that consume the staged chunks
  uint32_t chunks, cpp;  // chunks in total, per pass
};

// TMA bulk copies of data-row chunk i into its stage (one thread).
__device__ __forceinline__ void issue_chunk(const MomParams& P, const Ring& g, uint32_t i, uint32_t st) {
  const int n = P.n;
  const uint32_t K = P.K;
  const uint32_t rb = static_cast<uint32_t>(n) * 8u;
  const uint32_t pass = i >= g.cpp ? 1u : 0u;
  const RowSource& src = P.src[pass];
  const uint32_t a0 = (i - pass * g.cpp) * KC;
  const uint32_t kc = min(static_cast<uint32_t>(KC), K - a0);
  double* dst = g.xs + st * static_cast<size_t>(KC) * n;
  mbar_expect_tx(g.xfull + st, static_cast<uint32_t>(KC) * rb);
  // rows past the end of the pass are zero rows: they add exact zeros
  if (kc < static_cast<uint32_t>(KC))
    bulk_g2s(dst + static_cast<size_t>(kc) * n, P.zeros, (KC - kc) * rb, g.xfull + st);
  if (a0 + kc <= src.len0 || a0 >= src.len0) {
    bulk_g2s(dst, row_ptr(src, a0, n), kc * rb, g.xfull + st);
  } else {  // across the ring's wrap
    const uint32_t k1 = src.len0 - a0;
    bulk_g2s(dst, row_ptr(src, a0, n), k1 * rb, g.xfull + st);
    bulk_g2s(dst + static_cast<size_t>(k1) * n, src.seg1, (kc - k1) * rb, g.xfull + st);
  }
}

// Position in the stage ring (stage index and mbarrier phase parity).
struct Cursor {
  uint32_t st = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t stages) {
    if (++st == stages) {
      st = 0;
      ph ^= 1u;
    }
  }
};

// A warp is done with chunk c (in stage st): the last of the CTA's active
// warps to release the stage refills it with chunk c + stages right away
// (atomicInc wraps the per-stage counter at `active`).
__device__ __forceinline__ void release_chunk(const MomParams& P, const Ring& g, uint32_t c, uint32_t st) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    __threadfence_block();  // this warp's reads of the stage happen before the release
    const uint32_t old = atomicInc(g.rel + st, g.active - 1);
    if (old == g.active - 1 && c + g.stages < g.chunks) {
      __threadfence_block();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async-proxy writes
      issue_chunk(P, g, c + g.stages, st);
    }
  }
}

// Producer warp of row set rs.  Lane j owns pair j of the row set: slots
// (r, 2gp) and (r, 2gp + 1) of the MMA A operand, r = j >> 2, gp = j & 3.
// Ring layout: aring[slot][t][(r * 4 + q) * ASTRIDE + g] holds the value of
// row slot (r, g) at data row k = 4t + q of the chunk, so a DMMA lane
// (r, q) loads its 8 fragments with 4 x LDS.128.
template <int LM1, int N>
__device__ __forceinline__ void produce(const MomParams& P, const MomTile& tile, const Ring& g, int rs) {
  const int n = N ? N : P.n;
  const int lane = threadIdx.x & 31;
  const uint32_t set = tile.row0 + rs;
  const DmmaPair pr = P.pairs[static_cast<size_t>(set) * 32 + lane];
  int pidx[LM1];
#pragma unroll
  for (int t = 0; t < LM1; ++t) pidx[t] = pr.pidx[t];
  const int a0 = pr.a0, a1 = pr.a1;
  const bool update = P.npass == 2;
  const bool do_low = P.low != nullptr && tile.low;
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  double* aring = g.arings + static_cast<size_t>(rs) * ASLOTS * ASLOT;
  uint64_t* afull = g.afull + rs * ASLOTS;
  uint64_t* aempty = g.aempty + rs * ASLOTS;
  const int wofs = ((lane >> 2) * 4) * ASTRIDE + 2 * (lane & 3);
  double s0 = 0.0, s1 = 0.0, in0 = 0.0, in1 = 0.0;
  Cursor cur;
  for (uint32_t c = 0; c < g.chunks; ++c, cur.next(g.stages)) {
    const uint32_t st = cur.st;
    mbar_wait(g.xfull + st, cur.ph);
    const uint32_t slot = c % ASLOTS;
    if (c >= ASLOTS) mbar_wait(aempty + slot, ((c / ASLOTS) - 1) & 1u);
    const double* xst = g.xs + st * stage_elems;
    double* as = aring + slot * ASLOT + wofs;
#pragma unroll
    for (int t = 0; t < HSTEPS; ++t)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double* xr = xst + (4 * t + q) * n;
        double pv = xr[pidx[0]];
#pragma unroll
        for (int u = 1; u < LM1; ++u) pv = __dmul_rn(pv, xr[pidx[u]]);
        const double v0 = __dmul_rn(pv, xr[a0]);
        const double v1 = __dmul_rn(pv, xr[a1]);
        s0 = __dadd_rn(s0, v0);  // row order, plain adds (moments.cpp:44)
        s1 = __dadd_rn(s1, v1);
        *reinterpret_cast<double2*>(as + t * 32 * ASTRIDE + q * ASTRIDE) = make_double2(v0, v1);
      }
    mbar_arrive(afull + slot);  // every lane: its stores are released
    release_chunk(P, g, c, st);
    if (update && c + 1 == g.cpp) {  // end of the incoming pass
      in0 = __dmul_rn(s0, P.inv);
      in1 = __dmul_rn(s1, P.inv);
      s0 = s1 = 0.0;
    }
  }
  // ---- order L = d-1: the row sums of this lane's two slots ----
  if (!do_low) return;
  const double cc = P.c;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const PrefixRow& row = P.rows[static_cast<size_t>(set) * SLOTS_PER_SET + 2 * lane + e];
    if (row.vprime == 0) continue;
    const double s = e ? s1 : s0;
    if (update) {
      const double delta = __dsub_rn(e ? in1 : in0, __dmul_rn(s, P.inv));  // a - b
      P.low[row.low_off] = __fma_rn(cc, delta, P.low[row.low_off]);
      if (row.idx[7] & 1u) P.dlow[row.low_off] = delta;
    } else {
      P.low[row.low_off] = __dmul_rn(s, P.inv);
    }
  }
}

// DMMA warp: row set rs, column tiles [ct0, ct0 + NC) of the CTA's range.
// Lane (r, q): A fragment g = row slot (r, g) at k = q; B fragment c =
// x[k = q][col + 8c + r]; accumulator (g, c, e) = row slot (r, g), column
// col + 8c + 2q + e.
template <int NC, int N>
__device__ __forceinline__ void consume(const MomParams& P, const MomTile& tile, const Ring& g, int rs, int ct0,
                                        int warp) {
  const int n = N ? N : P.n;
  const int b = P.b;
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const uint32_t set = tile.row0 + rs;
  const int colbase = static_cast<int>(tile.col0) + 8 * ct0;
  const bool update = P.npass == 2;
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  const double* aring = g.arings + static_cast<size_t>(rs) * ASLOTS * ASLOT + (r * 4 + q) * ASTRIDE;
  uint64_t* afull = g.afull + rs * ASLOTS;
  uint64_t* aempty = g.aempty + rs * ASLOTS;
  // pass-0 means of this thread (64 doubles), in the CTA's scratch
  double* stash = P.scratch + static_cast<size_t>(blockIdx.x) * (CWARPS * 32 * 64);
  const int tid = warp * 32 + lane;
  double acc[8][NC][2];
#pragma unroll
  for (int gg = 0; gg < 8; ++gg)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[gg][c][0] = acc[gg][c][1] = 0.0;
  Cursor cur;
  for (uint32_t c = 0; c < g.chunks; ++c, cur.next(g.stages)) {
    const uint32_t st = cur.st;
    const uint32_t slot = c % ASLOTS;
    mbar_wait(g.xfull + st, cur.ph);
    mbar_wait(afull + slot, (c / ASLOTS) & 1u);
    const double* as = aring + slot * ASLOT;
    const double* xb = g.xs + st * stage_elems + static_cast<size_t>(q) * n + colbase + r;
    double a[2][8], bb[2][NC];
    auto load = [&](int t, int buf) {
      const double2* ap = reinterpret_cast<const double2*>(as + t * 32 * ASTRIDE);
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        const double2 v = ap[s2];
        a[buf][2 * s2] = v.x;
        a[buf][2 * s2 + 1] = v.y;
      }
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) bb[buf][cc] = xb[static_cast<size_t>(4 * t) * n + 8 * cc];
    };
    load(0, 0);
#pragma unroll
    for (int t = 0; t < HSTEPS; ++t) {
      if (t + 1 < HSTEPS) load(t + 1, (t + 1) & 1);
#pragma unroll
      for (int cc = 0; cc < NC; ++cc)
#pragma unroll
        for (int gg = 0; gg < 8; ++gg) dmma(acc[gg][cc][0], acc[gg][cc][1], a[t & 1][gg], bb[t & 1][cc]);
    }
    mbar_arrive(aempty + slot);  // every lane has consumed the slot
    release_chunk(P, g, c, st);
    if (update && c + 1 == g.cpp) {
      // end of the incoming pass: stash its means, restart the accumulators
#pragma unroll
      for (int gg = 0; gg < 8; ++gg)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            stash[static_cast<size_t>((gg * NC + cc) * 2 + e) * (CWARPS * 32) + tid] =
                __dmul_rn(acc[gg][cc][e], P.inv);
            acc[gg][cc][e] = 0.0;
          }
    }
  }

  // ---- epilogue: canonical entries only ----
  // Entries of blocks with equal neighbouring coordinates have symmetric
  // copies; for those the update's delta is also written to the delta
  // buffer at the canonical position and mirror_kernel applies it to every
  // other stored copy (or copies the value, for an assignment).
  const double cc = P.c;
#pragma unroll
  for (int gg = 0; gg < 8; ++gg) {
    const PrefixRow& pr = P.rows[static_cast<size_t>(set) * SLOTS_PER_SET + r * 8 + gg];
    if (pr.vprime == 0) continue;  // masked slot
    const int iL = pr.idx[P.L - 1];
    const bool row_runs = (pr.idx[7] & 1u) != 0;  // runs among (j_1..j_L)
    const int J = iL / b;
    size_t off[NC][2];
    double val[NC][2];
    bool ok[NC][2], diag[NC][2];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = colbase + 8 * c + 2 * q + e;
        const int jd = col / b;
        ok[c][e] = col < n && col >= iL;
        diag[c][e] = row_runs || jd == J;
        off[c][e] = pr.top_base + static_cast<uint64_t>(pr.vprime) * b * (jd - J) +
                    static_cast<uint64_t>(pr.poff) * ext_of(jd, n, b) + (col - jd * b);
        if (update) {
          const size_t ix = static_cast<size_t>((gg * NC + c) * 2 + e) * (CWARPS * 32) + tid;
          val[c][e] = __dsub_rn(stash[ix], __dmul_rn(acc[gg][c][e], P.inv));  // a - b
        } else {
          val[c][e] = __dmul_rn(acc[gg][c][e], P.inv);
        }
      }
    if (update) {
      double old[NC][2];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) old[c][e] = ok[c][e] ? P.top[off[c][e]] : 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (ok[c][e]) {
            P.top[off[c][e]] = __fma_rn(cc, val[c][e], old[c][e]);
            if (diag[c][e]) P.dtop[off[c][e]] = val[c][e];
          }
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (ok[c][e]) P.top[off[c][e]] = val[c][e];
    }
  }
}

// N: compile-time row length (0: runtime P.n) -- with it every shared-memory
// address of the inner loops is a register plus an immediate
template <int N>
__global__ void __launch_bounds__(THREADS, 1) moment_top_dmma_kernel(const MomParams P) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[MAX_STAGES + 2 * PWARPS * ASLOTS];
  __shared__ uint32_t rel[MAX_STAGES];
  const MomTile tile = P.tiles[blockIdx.x];
  const int R = static_cast<int>(tile.pad0);    // row-set slots of this CTA: 1, 2, 4
  const int nrs = static_cast<int>(tile.nrows); // live row sets (<= R)
  const int C = CWARPS / R;                     // column ranges
  Ring g;
  g.stages = static_cast<uint32_t>(P.stages);
  g.xs = smem;
  // reads past row n of the last stage (B fragments of the last column
  // tile) land in this padding and only feed outputs that are never stored
  g.arings = smem + static_cast<size_t>(g.stages) * KC * P.n + 64;
  g.xfull = bars;
  g.rel = rel;
  g.afull = bars + MAX_STAGES;
  g.aempty = g.afull + PWARPS * ASLOTS;
  g.cpp = (P.K + KC - 1) / KC;
  g.chunks = g.cpp * P.npass;  // incoming pass, then outgoing pass
  const int warp = threadIdx.x >> 5;
  // active warps: DMMA warps whose row set is live, one producer per live row set
  int active = nrs;
  for (int w = 0; w < CWARPS; ++w) active += (w % R) < nrs;
  g.active = static_cast<uint32_t>(active);
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < g.stages; ++s) {
      mbar_init(g.xfull + s, 1);
      rel[s] = 0;
    }
    for (int s = 0; s < PWARPS * ASLOTS; ++s) {
      mbar_init(g.afull + s, 32);
      mbar_init(g.aempty + s, 32 * C);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t i = 0; i < g.chunks && i < g.stages; ++i) issue_chunk(P, g, i, i);
  }
  __syncthreads();
  if (warp >= CWARPS) {
    const int rs = warp - CWARPS;
    if (rs >= nrs) return;
    switch (P.L) {
      case 2: produce<1, N>(P, tile, g, rs); break;
      case 3: produce<2, N>(P, tile, g, rs); break;
      case 4: produce<3, N>(P, tile, g, rs); break;
      case 5: produce<4, N>(P, tile, g, rs); break;
      default: break;
    }
    return;
  }
  const int rs = warp % R;
  if (rs >= nrs) return;
  const int part = warp / R;
  const int nct = static_cast<int>(tile.ncols);
  const int ct0 = nct * part / C, ct1 = nct * (part + 1) / C;
  switch (ct1 - ct0) {
    case 1: consume<1, N>(P, tile, g, rs, ct0, warp); break;
    case 2: consume<2, N>(P, tile, g, rs, ct0, warp); break;
    case 3: consume<3, N>(P, tile, g, rs, ct0, warp); break;
    case 4: consume<4, N>(P, tile, g, rs, ct0, warp); break;
    default: break;
  }
}

// Symmetric copies of the canonical entries written above, one CTA per
// stored block with equal neighbouring coordinates (symten.cpp:195-220):
// entry o of block j is a copy of the entry with o sorted within each run
// of equal j; an update applies the canonical delta to the copy's own old
// value (moments.cpp:294-299 RMWs every stored entry), an assignment copies.
template <int S>
__global__ void __launch_bounds__(256) mirror_kernel(double* __restrict__ m, const double* __restrict__ delta,
                                                     LayoutDev lay, const uint32_t* __restrict__ blocks, int n,
                                                     int b, bool update, double c) {
  const uint32_t blk = blocks[blockIdx.x];
  int j[S], e[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    j[k] = lay.index[static_cast<size_t>(blk) * S + k];
    e[k] = ext_of(j[k], n, b);
  }
  const uint64_t base = lay.offset[blk];
  const uint64_t vol = lay.offset[blk + 1] - base;
  for (uint64_t pos = threadIdx.x; pos < vol; pos += blockDim.x) {
    int o[S];
    uint64_t rem = pos;
#pragma unroll
    for (int k = S - 1; k >= 0; --k) {
      o[k] = static_cast<int>(rem % e[k]);
      rem /= e[k];
    }
    // sort within runs (bubble passes over a tiny array, fully unrolled)
    bool canonical = true;
#pragma unroll
    for (int k = 1; k < S; ++k)
      if (j[k] == j[k - 1] && o[k] < o[k - 1]) canonical = false;
    if (canonical) continue;
#pragma unroll
    for (int pass = 0; pass < S - 1; ++pass)
#pragma unroll
      for (int k = 1; k < S; ++k)
        if (j[k] == j[k - 1] && o[k] < o[k - 1]) {
          const int t = o[k];
          o[k] = o[k - 1];
          o[k - 1] = t;
        }
    uint64_t src = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) src = src * e[k] + o[k];
    double* p = m + base + pos;
    *p = update ? __fma_rn(c, delta[base + src], *p) : m[base + src];
  }
}

size_t smem_bytes(int n, int stages) {
  return sizeof(double) * (static_cast<size_t>(stages) * KC * n + 64 + PWARPS * ASLOTS * ASLOT);
}

// leaves room for a co-resident low-order CTA (1 KB reserved shared memory per CTA)
constexpr size_t kSmemLimit = 224 * 1024;

int stages_for(int n) {
  int s = MAX_STAGES;
  while (s > 0 && smem_bytes(n, s) > kSmemLimit) --s;
  return s;
}

}  // namespace

// per tile: the incoming pass's means (64 values per consumer thread)
size_t dmma_scratch_per_tile() { return static_cast<size_t>(CWARPS) * 32 * 64; }

bool dmma_supported(const MomParams& p) {
  // instantiated for orders 3..6 (L = 2..5); rows must be 16-byte aligned
  // for the bulk copies, and at least two stages must fit
  if (p.n % 2 != 0 || p.L < 2 || p.L > 5) return false;
  return stages_for(p.n) >= 2;
}

void launch_mirror(int S, double* m, const double* delta, const LayoutDev& lay, const uint32_t* blocks,
                   uint32_t nblocks, int n, int b, bool update, double c, cudaStream_t st) {
  if (!nblocks) return;
  switch (S) {
#define CSB_MIRROR(SS) \
  case SS: mirror_kernel<SS><<<nblocks, 256, 0, st>>>(m, delta, lay, blocks, n, b, update, c); break;
    CSB_MIRROR(2) CSB_MIRROR(3) CSB_MIRROR(4) CSB_MIRROR(5) CSB_MIRROR(6) CSB_MIRROR(7) CSB_MIRROR(8)
#undef CSB_MIRROR
    default: fail(CSB_EINVAL, "mirror: order out of range");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

void launch_moment_top_dmma(const MomParams& p_in, int ntiles, cudaStream_t st) {
  if (ntiles <= 0) return;
  MomParams p = p_in;
  p.stages = stages_for(p.n);
  if (p.stages < 2) fail(CSB_EINVAL, "moment_top_dmma: rows too wide for the staging ring");
  const size_t smem = smem_bytes(p.n, p.stages);
  auto kern = p.n == 96 ? moment_top_dmma_kernel<96>
            : p.n == 48 ? moment_top_dmma_kernel<48>
            : p.n == 24 ? moment_top_dmma_kernel<24>
            : p.n == 256 ? moment_top_dmma_kernel<256>
                         : moment_top_dmma_kernel<0>;
  CSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<ntiles, THREADS, smem, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
