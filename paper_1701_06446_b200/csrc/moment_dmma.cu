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
// Work unit: a tile = 32 groups (pi, h) of 8 prefix rows (pi, 8h + g) x up
// to 4 column groups of 8.  A CTA streams the incoming rows, stashes their
// means, streams the outgoing rows and applies the fused update
// M = fma(p/T, a - b, M) (moments.cpp:297) to the canonical entries.
//
// Per CTA (4 warps): rows of the batch stream through a 4-stage shared
// memory ring filled by cp.async.bulk (one TMA bulk copy per 32-row chunk,
// mbarrier completion; lane 0 of warp 0 is the producer and refills a stage
// once all warps released it -- no CTA-wide barrier in the loop).  Each warp
// builds its Khatri-Rao fragments in registers straight from the staged
// rows, software-pipelined so the next step's loads and products overlap
// the current step's DMMAs.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace csb {

namespace {

constexpr int CWARPS = 4;           // DMMA consumer warps
constexpr int WARPS = 2 * CWARPS;   // + one producer warp per consumer
constexpr int THREADS = WARPS * 32;
constexpr int HSTEPS = 8;           // k4 steps per A-ring slot (one 32-row chunk)
constexpr int ASTRIDE = 10;         // doubles per (r, q) entry: 8 used, bank-conflict free
constexpr int ASLOT = HSTEPS * 32 * ASTRIDE;
constexpr int STAGES = 2;
constexpr int KC = 32;        // data rows per stage


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

// Per-warp layout: lane = 4 r + q.  The warp owns 8 groups; group r is
// (pi_r, h): the 8 prefix rows (pi_r, 8h + g), g = 0..7.  For MMA fragment
// g, row m = r of A is the Khatri-Rao value of row (pi_r, 8h + g) at data
// row k = q, so each thread forms P = x[pi_r] once per k and the 8 row values
// as P * x[8h + g] (prefix sharing of moments.cpp:55,71).  B fragment c is
// x[k = q][col0 + 8c + r].  Accumulator (g, c, e) is the element
// (pi_r, 8h + g, col0 + 8c + 2q + e).
//
// The k loop runs over "steps" of 4 data rows, flat across both passes and
// all staged chunks, software-pipelined in registers: step s+1's operands
// are loaded from shared memory and multiplied out while step s's DMMAs
// occupy the FP64 tensor pipe.

// Warp-specialized tile: warps 0..CWARPS-1 are DMMA consumers, warps
// CWARPS..2*CWARPS-1 their producers.  A DMMA stalls its warp for 15 cycles
// (SASS control bits), so a warp cannot overlap its own FP64 products and
// row sums with its DMMAs; split across warps, the products, the order-L
// row sums and the DMMAs share the FP64 pipe of the SM sub-partition.
//
// Producer lane (r, gp) of producer warp w: rows (pi_r, 8h + 2gp + e),
// e = 0, 1, of the consumer warp's group r.  Per data row k it forms
// P = x[pi_1] ... x[pi_{L-1}] and the two products P * x[8h + 2gp + e]
// (moments.cpp:55,71), adds them to its row sums in row order, and stores
// them to the A ring in fragment order:
//   aring[w][slot][t][(r * 4 + q) * ASTRIDE + g],  k = 16 half + 4 t + q.
// Consumer lane (r, q): fragment g of step t is aring[...][t][(r*4+q)*10+g]
// (4 x LDS.128), B fragment c is x[k = 4 t + q][col0 + 8c + r].
template <int LM1, int NC>
__device__ __forceinline__ void run_tile(const MomParams& P, const MomTile& tile, double* xs, double* arings,
                                         uint64_t* xfull, uint64_t* xempty, uint64_t* afull, uint64_t* aempty) {
  constexpr int L = LM1 + 1;
  const int n = P.n, b = P.b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool producer = warp >= CWARPS;
  const int pw = producer ? warp - CWARPS : warp;  // pair index
  const int r = lane >> 2, q4 = lane & 3;          // (r, q) consumer / (r, gp) producer
  const int h8 = static_cast<int>(tile.J) * 8;
  const int col0 = static_cast<int>(tile.col0);
  const bool do_low = (P.low != nullptr) && tile.low;
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  const uint32_t K = P.K;
  const uint32_t cpp = (K + KC - 1) / KC;  // chunks per pass
  const uint32_t chunks = cpp * P.npass;   // incoming pass, then outgoing pass
  double* aring = arings + static_cast<size_t>(pw) * 2 * ASLOT;

  // ---- TMA producer: lane 0 of the first producer warp ----
  uint32_t next_issue = 0;
  auto pump = [&](uint32_t needed) {
    if (threadIdx.x != CWARPS * 32) return;
    while (next_issue < chunks) {
      const uint32_t i = next_issue;
      const uint32_t st = i % STAGES;
      if (i >= STAGES) {
        const uint32_t par = ((i / STAGES) - 1) & 1u;
        if (!mbar_test(xempty + st, par)) {
          if (i > needed) break;
          mbar_wait(xempty + st, par);
        }
      }
      const RowSource& src = P.src[i / cpp];
      const uint32_t a0 = (i % cpp) * KC;
      const uint32_t kc = min(static_cast<uint32_t>(KC), K - a0);
      double* dst = xs + st * stage_elems;
      const uint32_t rb = static_cast<uint32_t>(n) * 8u;
      mbar_expect_tx(xfull + st, static_cast<uint32_t>(KC) * rb);
      // rows past the end of the pass are zero rows: they add exact zeros
      if (kc < static_cast<uint32_t>(KC))
        bulk_g2s(dst + static_cast<size_t>(kc) * n, P.zeros, (KC - kc) * rb, xfull + st);
      if (a0 + kc <= src.len0 || a0 >= src.len0) {
        bulk_g2s(dst, row_ptr(src, a0, n), kc * rb, xfull + st);
      } else {  // across the ring's wrap
        const uint32_t k1 = src.len0 - a0;
        bulk_g2s(dst, row_ptr(src, a0, n), k1 * rb, xfull + st);
        bulk_g2s(dst + static_cast<size_t>(k1) * n, src.seg1, (kc - k1) * rb, xfull + st);
      }
      ++next_issue;
    }
  };

  const int gl = pw * 8 + r;  // group slot in the tile
  const bool gvalid = gl < static_cast<int>(tile.nrows);
  const uint32_t gi = tile.row0 + (gvalid ? gl : 0);
  const DmmaGroup grp = P.groups[gi];
  const int lo = grp.lo;
  const bool update = P.npass == 2;
  // pass-0 means of the consumer threads (the producers keep theirs in registers)
  double* stash = P.scratch + static_cast<size_t>(blockIdx.x) * (CWARPS * 32 * 64);

  if (producer) {
    int pidx[LM1 > 0 ? LM1 : 1];
#pragma unroll
    for (int t = 0; t < LM1; ++t) pidx[t] = grp.pidx[t];
    const int gp = q4;
    double lowacc[2] = {0.0, 0.0}, lowin[2] = {0.0, 0.0};
    // lower orders: lane gp accumulates depth gp + 1 of the prefix chain
    // (the order-(gp+1) product of (pi_1..pi_{gp+1})) when the group
    // represents that tuple; other lanes' sums are discarded
    const bool rep = do_low && P.rep_off != nullptr && gp < LM1 && ((grp.rep_mask >> gp) & 1u);
    double repacc = 0.0, repin = 0.0;
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint32_t st = c % STAGES;
      if (warp == CWARPS) pump(c);
      __syncwarp();
      mbar_wait(xfull + st, (c / STAGES) & 1u);
      const double* xst = xs + st * stage_elems;
#pragma unroll 1
      for (int hc = 0; hc < KC / (4 * HSTEPS); ++hc) {
        const uint32_t u = c * (KC / (4 * HSTEPS)) + hc;
        const int slot = u & 1;
        if (u >= 2) mbar_wait(aempty + pw * 2 + slot, ((u >> 1) - 1) & 1u);
        double* as = aring + slot * ASLOT;
#pragma unroll
        for (int t = 0; t < HSTEPS; ++t)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double* xr = xst + static_cast<size_t>(hc * 4 * HSTEPS + 4 * t + q) * n;
            double Pv = xr[pidx[0]];
            double Ps = Pv;
#pragma unroll
            for (int t2 = 1; t2 < LM1; ++t2) {
              Pv = __dmul_rn(Pv, xr[pidx[t2]]);
              if (gp >= t2) Ps = Pv;
            }
            if (LM1 > 0) repacc = __dadd_rn(repacc, Ps);  // row order, plain adds (moments.cpp:44)
            const double2 xv = *reinterpret_cast<const double2*>(xr + h8 + 2 * gp);
            double a0, a1;
            if (P.debug & 2) {
              a0 = xv.x;
              a1 = xv.y;
            } else {
              a0 = __dmul_rn(Pv, xv.x);
              a1 = __dmul_rn(Pv, xv.y);
            }
            if (do_low && !(P.debug & 1)) {
              lowacc[0] = __dadd_rn(lowacc[0], a0);  // row order, plain adds (moments.cpp:44)
              lowacc[1] = __dadd_rn(lowacc[1], a1);
            }
            *reinterpret_cast<double2*>(as + t * 32 * ASTRIDE + (r * 4 + q) * ASTRIDE + 2 * gp) =
                make_double2(a0, a1);
          }
        mbar_arrive(afull + pw * 2 + slot);  // every lane: its stores are released
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(xempty + st);
      if (warp == CWARPS) pump(0);
      if (update && c + 1 == cpp) {  // end of the incoming pass
        lowin[0] = __dmul_rn(lowacc[0], P.inv);
        lowin[1] = __dmul_rn(lowacc[1], P.inv);
        lowacc[0] = lowacc[1] = 0.0;
        repin = __dmul_rn(repacc, P.inv);
        repacc = 0.0;
      }
    }
    if (rep && gvalid) {  // order gp + 1, canonical element (pi_1..pi_{gp+1})
      const uint64_t e = P.rep_off[grp.rep + __popc(grp.rep_mask & ((1u << gp) - 1u))];
      const uint64_t off = e & ~(1ull << 63);
      double* Ms = P.lower[gp];
      if (update) {
        const double delta = __dsub_rn(repin, __dmul_rn(repacc, P.inv));
        Ms[off] = __fma_rn(P.c, delta, Ms[off]);
        if (e >> 63) P.dlower[gp][off] = delta;
      } else {
        Ms[off] = __dmul_rn(repacc, P.inv);
      }
    }
    // ---- producer epilogue: order L (= d-1) ----
    if (!gvalid || !do_low) return;
    const double cc = P.c;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 2 * gp + e;
      const int iL = h8 + g;
      if (g < lo || iL >= n) continue;
      const PrefixRow& pr = P.rows[static_cast<size_t>(gi) * 8 + g];
      if (update) {
        const double delta = __dsub_rn(lowin[e], __dmul_rn(lowacc[e], P.inv));  // a - b
        P.low[pr.low_off] = __fma_rn(cc, delta, P.low[pr.low_off]);
        if (pr.idx[7] & 1u) P.dlow[pr.low_off] = delta;
      } else {
        P.low[pr.low_off] = __dmul_rn(lowacc[e], P.inv);
      }
    }
    return;
  }

  // ================= DMMA consumer =================
  const int q = q4;
  double acc[8][NC][2];
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[g][c][0] = acc[g][c][1] = 0.0;
  for (uint32_t c = 0; c < chunks; ++c) {
    const uint32_t st = c % STAGES;
    mbar_wait(xfull + st, (c / STAGES) & 1u);
    const double* xst = xs + st * stage_elems + static_cast<size_t>(q) * n + col0 + r;
#pragma unroll 1
    for (int hc = 0; hc < KC / (4 * HSTEPS); ++hc) {
      const uint32_t u = c * (KC / (4 * HSTEPS)) + hc;
      const int slot = u & 1;
      mbar_wait(afull + pw * 2 + slot, (u >> 1) & 1u);
      const double* as = aring + slot * ASLOT + (r * 4 + q) * ASTRIDE;
      const double* xb = xst + static_cast<size_t>(hc * 4 * HSTEPS) * n;
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
          for (int g = 0; g < 8; ++g) dmma(acc[g][cc][0], acc[g][cc][1], a[t & 1][g], bb[t & 1][cc]);
      }
      mbar_arrive(aempty + pw * 2 + slot);  // every lane has consumed the slot
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty + st);
    if (update && c + 1 == cpp) {
      // end of the incoming pass: stash its means, restart the accumulators
      const int tid = pw * 32 + lane;
#pragma unroll
      for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            stash[static_cast<size_t>((g * NC + cc) * 2 + e) * (CWARPS * 32) + tid] = __dmul_rn(acc[g][cc][e], P.inv);
            acc[g][cc][e] = 0.0;
          }
    }
  }

  const int tid = pw * 32 + lane;  // consumer thread index

  // ---- epilogue: canonical entries only ----
  // Entries of blocks with equal neighbouring coordinates have symmetric
  // copies; for those the update's delta is also written to the delta
  // buffer at the canonical position and mirror_kernel applies it to every
  // other stored copy (or copies the value, for an assignment).
  if (!gvalid) return;
  const double cc = P.c;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const int iL = h8 + g;
    if (g < lo || iL >= n) continue;
    const PrefixRow& pr = P.rows[static_cast<size_t>(gi) * 8 + g];
    const bool row_runs = (pr.idx[7] & 1u) != 0;  // runs among (j_1..j_L)
    const int J = iL / b;
    size_t off[NC][2];
    double val[NC][2];
    bool ok[NC][2], diag[NC][2];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = col0 + 8 * c + 2 * q + e;
        const int jd = col / b;
        ok[c][e] = col < n && col >= iL;
        diag[c][e] = row_runs || jd == J;
        off[c][e] = pr.top_base + static_cast<uint64_t>(pr.vprime) * b * (jd - J) +
                    static_cast<uint64_t>(pr.poff) * ext_of(jd, n, b) + (col - jd * b);
        if (update) {
          const size_t ix = static_cast<size_t>((g * NC + c) * 2 + e) * (CWARPS * 32) + tid;
          val[c][e] = __dsub_rn(stash[ix], __dmul_rn(acc[g][c][e], P.inv));  // a - b
        } else {
          val[c][e] = __dmul_rn(acc[g][c][e], P.inv);
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

__global__ void __launch_bounds__(THREADS, 1) moment_top_dmma_kernel(const MomParams P) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t xfull[STAGES];
  __shared__ __align__(8) uint64_t xempty[STAGES];
  __shared__ __align__(8) uint64_t afull[CWARPS * 2];
  __shared__ __align__(8) uint64_t aempty[CWARPS * 2];
  double* xs = smem;
  // dense staging ring; reads past row n of a stage (the last 8-column
  // window / column group) only feed rows and columns that are never stored
  double* arings = xs + static_cast<size_t>(STAGES) * KC * P.n + 64;  // CWARPS x 2 x ASLOT
  const MomTile tile = P.tiles[blockIdx.x];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, WARPS);
    }
    for (int s = 0; s < CWARPS * 2; ++s) {
      mbar_init(afull + s, 32);
      mbar_init(aempty + s, 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nc = static_cast<int>(tile.pad0);
  switch (P.L * 8 + nc) {
#define CSB_CASE(LL, NCC) \
  case (LL) * 8 + (NCC): \
    run_tile<(LL) - 1, NCC>(P, tile, xs, arings, xfull, xempty, afull, aempty); break;
#define CSB_CASES(LL) CSB_CASE(LL, 1) CSB_CASE(LL, 2) CSB_CASE(LL, 3) CSB_CASE(LL, 4)
    CSB_CASES(2) CSB_CASES(3) CSB_CASES(4) CSB_CASES(5)
#undef CSB_CASES
#undef CSB_CASE
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

size_t smem_bytes(int n) {
  return sizeof(double) * (static_cast<size_t>(STAGES) * KC * n + 64 + CWARPS * 2 * ASLOT);
}

}  // namespace

int dmma_warps() { return CWARPS; }

// per tile: the incoming pass's means (64 values per consumer thread)
size_t dmma_scratch_per_tile() { return static_cast<size_t>(CWARPS) * 32 * 64; }

bool dmma_supported(const MomParams& p) {
  // instantiated for orders 3..6 (L = 2..5); the staging ring must fit
  if (p.n % 2 != 0 || p.L < 2 || p.L > 5) return false;
  if (smem_bytes(p.n) > 220 * 1024) return false;
  return true;
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

void launch_moment_top_dmma(const MomParams& p, int ntiles, cudaStream_t st) {
  if (ntiles <= 0) return;
  const size_t smem = smem_bytes(p.n);
  CSB_CUDA(cudaFuncSetAttribute(moment_top_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  moment_top_dmma_kernel<<<ntiles, THREADS, smem, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
