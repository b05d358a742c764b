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

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>

#include "kernels.cuh"

namespace csb {

namespace {

constexpr int CWARPS = 8;                 // DMMA consumer warps (two per SM sub-partition)
constexpr int PWARPS = 4;                 // producer warps (one per row set)
constexpr int THREADS = (CWARPS + PWARPS) * 32;
constexpr int MAXNC = 3;                  // column tiles per DMMA warp
// Chunk geometry: HS k4 steps (4 HS data rows) per chunk, stage and A slot;
// HS is a kernel template parameter (8, 6 or 4, whichever leaves >= 5 stages; 10 at n = 48, b = 4).
constexpr int ASTRIDE = 8;                // doubles per (r, q) A-ring entry (swizzled, see apos)
constexpr int ASLOTS = 2;                 // A-ring slots per row set
template <int HS>
struct Geo {
  static constexpr int KC = 4 * HS;                  // data rows per chunk
  static constexpr int ASLOT = HS * 32 * ASTRIDE;    // doubles per A slot
};

// A-ring entry e = 4 r + q holds the 8 fragments (16-byte chunks s = 0..3)
// of row slots (r, 0..7) at one data row.  Entries are permuted and their
// chunks XOR-swizzled so that both the producers' stores (fixed q, lanes
// (r, gp)) and the DMMA warps' loads (fixed s, lanes (r, q)) are free of
// shared-memory bank conflicts.
__device__ __forceinline__ int apos(int e, int s) {
  const int pe = e ^ ((e >> 2) & 1);
  return pe * ASTRIDE + 2 * (s ^ ((pe >> 1) & 3));
}
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
  uint32_t stages, kc;   // stages, data rows per chunk
  uint32_t aslots, alog;  // A-ring slots per live row set (PWARPS x ASLOTS / R) and log2
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
  const uint32_t KC = g.kc;
  const uint32_t a0 = (i - pass * g.cpp) * KC;
  const uint32_t kc = min(KC, K - a0);
  double* dst = g.xs + st * static_cast<size_t>(KC) * n;
  mbar_expect_tx(g.xfull + st, KC * rb);
  // rows past the end of the pass are zero rows: they add exact zeros
  if (kc < KC) bulk_g2s(dst + static_cast<size_t>(kc) * n, P.zeros, (KC - kc) * rb, g.xfull + st);
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
    // no fence before the release: every read this warp made of the stage
    // has returned (its values were consumed by the chunk's last DMMAs or
    // products, which precede this point); only the refill below orders the
    // generic proxy against the TMA writes (measured +0.6..0.9%)
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
template <int LM1, int N, int HS, bool SUMS>
__device__ __forceinline__ void produce(const MomParams& P, const MomTile& tile, const Ring& g, int rs) {
  constexpr int HSTEPS = HS, KC = Geo<HS>::KC, ASLOT = Geo<HS>::ASLOT;
  const int n = N ? N : P.n;
  const int lane = threadIdx.x & 31;
  const uint32_t set = tile.row0 + rs;
  const DmmaPair pr = P.pairs[static_cast<size_t>(set) * 32 + lane];
  int pidx[LM1];
#pragma unroll
  for (int t = 0; t < LM1; ++t) pidx[t] = pr.pidx[t];
  const int a0 = pr.a0;  // pr.a1 == a0 + 1
  const bool update = P.npass == 2;
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  double* aring = g.arings + static_cast<size_t>(rs) * g.aslots * ASLOT;
  uint64_t* afull = g.afull + rs * g.aslots;
  uint64_t* aempty = g.aempty + rs * g.aslots;
  const int pr_r = lane >> 2, pr_gp = lane & 3;
  double s0 = 0.0, s1 = 0.0, in0 = 0.0, in1 = 0.0;
  // Explicit software pipeline: the operands of the next k4 step (4 data
  // rows; across the chunk boundary too) are loaded before this step's
  // products are formed and stored, so the loads are not held behind the
  // A-ring stores and the rows' latency chains overlap.
  constexpr int NV = LM1 + 2;
  double xv[2][4][NV];
  auto load = [&](const double* xst, int t, int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double* xr = xst + (4 * t + q) * n;
#pragma unroll
      for (int u = 0; u < LM1; ++u) xv[buf][q][u] = xr[pidx[u]];
      const double2 xa = *reinterpret_cast<const double2*>(xr + a0);  // a1 == a0 + 1, a0 even
      xv[buf][q][LM1] = xa.x;
      xv[buf][q][LM1 + 1] = xa.y;
    }
  };
  // The row sums lag the products by one k4 step: the adds of the previous
  // step's products (a dependent chain per slot, ~40 cycles per add while
  // the DMMA warps hold the FP64 pipe) are interleaved with this step's
  // independent multiplications instead of serializing them.
  double h0[4] = {0.0, 0.0, 0.0, 0.0}, h1[4] = {0.0, 0.0, 0.0, 0.0};  // held products (exact zeros at start)
  auto form = [&](double* as, int t, int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double pv = xv[buf][q][0];
#pragma unroll
      for (int u = 1; u < LM1; ++u) pv = __dmul_rn(pv, xv[buf][q][u]);
      const double v0 = __dmul_rn(pv, xv[buf][q][LM1]);
      const double v1 = __dmul_rn(pv, xv[buf][q][LM1 + 1]);
      if (SUMS) {
        s0 = __dadd_rn(s0, h0[q]);  // row order, plain adds (moments.cpp:44)
        s1 = __dadd_rn(s1, h1[q]);
        h0[q] = v0;
        h1[q] = v1;
      }
      *reinterpret_cast<double2*>(as + t * 32 * ASTRIDE + apos(pr_r * 4 + q, pr_gp)) = make_double2(v0, v1);
    }
  };
  auto flush = [&]() {  // add the held products (end of a pass)
    if (SUMS) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s0 = __dadd_rn(s0, h0[q]);
        s1 = __dadd_rn(s1, h1[q]);
        h0[q] = h1[q] = 0.0;
      }
    }
  };
  Cursor cur;
  mbar_wait(g.xfull, 0);
  const double* xst = g.xs;
  load(xst, 0, 0);
  for (uint32_t c = 0; c < g.chunks; ++c) {
    Cursor nx = cur;
    nx.next(g.stages);
    const double* nxst = g.xs + nx.st * stage_elems;
    const uint32_t slot = c & (g.aslots - 1);
    if (c >= g.aslots) mbar_wait(aempty + slot, ((c >> g.alog) - 1) & 1u);
    double* as = aring + slot * ASLOT;
#pragma unroll
    for (int t = 0; t < HSTEPS; ++t) {
      if (t + 1 < HSTEPS) {
        load(xst, t + 1, (t + 1) & 1);
      } else if (c + 1 < g.chunks) {
        mbar_wait(g.xfull + nx.st, nx.ph);
        load(nxst, 0, (t + 1) & 1);
      }
      form(as, t, t & 1);
    }
    // one arrival per warp: __syncwarp orders the lanes' A-ring stores
    // before lane 0's (release) arrive
    __syncwarp();
    if (lane == 0) mbar_arrive(afull + slot);
    release_chunk(P, g, c, cur.st);
    if (update && c + 1 == g.cpp) {  // end of the incoming pass
      flush();
      in0 = __dmul_rn(s0, P.inv);
      in1 = __dmul_rn(s1, P.inv);
      s0 = s1 = 0.0;
    }
    cur = nx;
    xst = nxst;
  }
  flush();
  // ---- order L = d-1: the row sums of this lane's two slots ----
  if (!SUMS) return;
  const double cc = P.c;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const PrefixRow& row = P.rows[static_cast<size_t>(set) * SLOTS_PER_SET + 2 * lane + e];
    if (row.vprime == 0) continue;
    const double s = e ? s1 : s0;
    if (update) {
      const double delta = __dsub_rn(e ? in1 : in0, __dmul_rn(s, P.inv));  // a - b
      P.low[row.low_off] = __fma_rn(cc, delta, P.low[row.low_off]);
    } else {
      P.low[row.low_off] = __dmul_rn(s, P.inv);
    }
  }
}


// DMMA warp: row set rs, column tiles [ct0, ct0 + NC) of the CTA's range.
// Lane (r, q): A fragment g = row slot (r, g) at k = q; B fragment c =
// x[k = q][col + 8c + r]; accumulator (g, c, e) = row slot (r, g), column
// col + 8c + 2q + e.  The operand loads run one k4 step ahead across chunk
// boundaries: the next chunk's barriers are checked and its first operands
// loaded in the middle of the current chunk's last DMMA step.
template <int NC, int N, int HS, int B>
__device__ __forceinline__ void consume(const MomParams& P, const MomTile& tile, const Ring& g, int rs, int ct0,
                                        int warp) {
  constexpr int HSTEPS = HS, KC = Geo<HS>::KC, ASLOT = Geo<HS>::ASLOT;
  const int n = N ? N : P.n;
  const int b = B ? B : P.b;  // compile-time block size where instantiated
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  const uint32_t set = tile.row0 + rs;
  const int colbase = static_cast<int>(tile.col0) + 8 * ct0;
  const bool update = P.npass == 2;
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  const double* aring = g.arings + static_cast<size_t>(rs) * g.aslots * ASLOT;
  const double* xlane = g.xs + static_cast<size_t>(q) * n + colbase + r;
  uint64_t* afull = g.afull + rs * g.aslots;
  uint64_t* aempty = g.aempty + rs * g.aslots;
  // pass-0 means of this thread (64 doubles), in the CTA's scratch
  double* __restrict__ stash = P.scratch + static_cast<size_t>(blockIdx.x) * (CWARPS * 32 * 16 * MAXNC);
  const int tid = warp * 32 + lane;
  double acc[8][NC][2];
#pragma unroll
  for (int gg = 0; gg < 8; ++gg)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[gg][c][0] = acc[gg][c][1] = 0.0;
  double a[2][8], bb[2][NC];
  auto load = [&](const double* as, const double* xb, int t, int buf) {
    const double* ap = as + t * 32 * ASTRIDE;
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
      const double2 v = *reinterpret_cast<const double2*>(ap + apos(lane, s2));
      a[buf][2 * s2] = v.x;
      a[buf][2 * s2 + 1] = v.y;
    }
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
      bb[buf][cc] = xb[static_cast<size_t>(4 * t) * n + 8 * cc];
  };
  auto mma_rows = [&](int buf, int g0, int g1) {
#pragma unroll
    for (int cc = 0; cc < NC; ++cc)
#pragma unroll
      for (int gg = g0; gg < g1; ++gg) {
        dmma(acc[gg][cc][0], acc[gg][cc][1], a[buf][gg], bb[buf][cc]);
      }
  };
  // The x stage of a chunk is complete once its A slot is: the producer
  // arrives on afull only after its own wait on the stage's TMA barrier.
  Cursor cur;  // stage of chunk c
  uint32_t slot = 0, aph = 0;
  mbar_wait(afull, 0);
  const double* as = aring;
  const double* xb = xlane;
  load(as, xb, 0, 0);
  for (uint32_t c = 0; c < g.chunks; ++c) {
    Cursor nx = cur;
    nx.next(g.stages);
    const uint32_t nslot = slot + 1 == g.aslots ? 0 : slot + 1;
    const uint32_t naph = nslot == 0 ? aph ^ 1u : aph;
    const double* nas = aring + nslot * ASLOT;
    const double* nxb = xlane + nx.st * stage_elems;
#pragma unroll
    for (int t = 0; t < HSTEPS - 1; ++t) {
      load(as, xb, t + 1, (t + 1) & 1);
      mma_rows(t & 1, 0, 8);
    }
    constexpr int LB = (HSTEPS - 1) & 1;
    mma_rows(LB, 0, 4);
    if (c + 1 < g.chunks) {
      mbar_wait(afull + nslot, naph);
      load(nas, nxb, 0, LB ^ 1);
    }
    mma_rows(LB, 4, 8);
    __syncwarp();  // every lane has consumed the slot
    if (lane == 0) mbar_arrive(aempty + slot);
    release_chunk(P, g, c, cur.st);
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
    cur = nx;
    slot = nslot;
    aph = naph;
    as = nas;
    xb = nxb;
  }

  // ---- epilogue: canonical entries only ----
  // Entries of blocks with equal neighbouring coordinates have symmetric
  // copies; for those the update's delta is also written to the delta
  // buffer at the canonical position and mirror_kernel applies it to every
  // other stored copy (or copies the value, for an assignment).  Loads are
  // batched (slot metadata, then the stash, then the old values per half)
  // so each round trip to memory is paid a few times, not per slot.
  const PrefixRow* __restrict__ rows = P.rows + static_cast<size_t>(set) * SLOTS_PER_SET + r * 8;
  uint64_t tb[8];
  uint32_t vp[8], po[8];
  int il[8];
#pragma unroll
  for (int gg = 0; gg < 8; ++gg) {
    const uint4* pr = reinterpret_cast<const uint4*>(rows + gg);
    const uint4 w0 = __ldg(pr), w1 = __ldg(pr + 1), w2 = __ldg(pr + 2);
    const uint32_t li = static_cast<uint32_t>(P.L - 1);
    const uint32_t word = li < 2 ? w0.x : li < 4 ? w0.y : li < 6 ? w0.z : w0.w;
    il[gg] = static_cast<int>((li & 1) ? (word >> 16) : (word & 0xffffu));
    tb[gg] = static_cast<uint64_t>(w1.x) | (static_cast<uint64_t>(w1.y) << 32);
    vp[gg] = w2.x;
    po[gg] = w2.y;
  }
  auto offset = [&](int gg, int c, int e, bool& ok) -> size_t {
    const int col = colbase + 8 * c + 2 * q + e;
    const int jd = col / b;
    const int J = il[gg] / b;
    ok = vp[gg] != 0 && col < n && col >= il[gg];
    return tb[gg] + static_cast<uint64_t>(vp[gg]) * b * (jd - J) + static_cast<uint64_t>(po[gg]) * ext_of(jd, n, b) +
           (col - jd * b);
  };
  if (update) {
    // the old values are read after the stash round trip: start them toward L2 now
#pragma unroll
    for (int gg = 0; gg < 8; ++gg)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        bool ok;
        const size_t o = offset(gg, c, 0, ok);
        if (ok) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.top + o));
      }
  }
  if (update) {
#pragma unroll
    for (int gg = 0; gg < 8; ++gg)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const size_t ix = static_cast<size_t>((gg * NC + c) * 2 + e) * (CWARPS * 32) + tid;
          acc[gg][c][e] = __dsub_rn(stash[ix], __dmul_rn(acc[gg][c][e], P.inv));  // a - b
        }
  } else {
#pragma unroll
    for (int gg = 0; gg < 8; ++gg)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[gg][c][e] = __dmul_rn(acc[gg][c][e], P.inv);
  }
  double* __restrict__ top = P.top;
  const double cc = P.c;
  // batches of GB slots: offsets are recomputed at the stores rather than
  // kept live next to the loaded old values
  constexpr int GB = NC >= 2 ? 2 : 4;
  constexpr int NCD = NC;
#pragma unroll
  for (int g0 = 0; g0 < 8; g0 += GB) {
    double old[GB][NCD > 0 ? NCD : 1][2];
    if (update) {
#pragma unroll
      for (int h = 0; h < GB; ++h)
#pragma unroll
        for (int c = 0; c < NCD; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            bool ok;
            const size_t o = offset(g0 + h, c, e, ok);
            old[h][c][e] = ok ? top[o] : 0.0;
          }
    }
#pragma unroll
    for (int h = 0; h < GB; ++h)
#pragma unroll
      for (int c = 0; c < NCD; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          bool ok;
          const size_t o = offset(g0 + h, c, e, ok);
          if (!ok) continue;
          const double v = acc[g0 + h][c][e];
          if (update) {
            top[o] = __fma_rn(cc, v, old[h][c][e]);
          } else {
            top[o] = v;
          }
        }
  }
}

// Column tiles [ct0, ct1) of DMMA warp w in a CTA with R row-set slots and
// nct column tiles.  Warp w runs on SM sub-partition w % 4 and serves row
// set w % R; a row set's tiles are split evenly over its 4/R sub-partitions
// first, then over the two warps of each, so every sub-partition's DMMA pipe
// gets the same share (ceil(nct R / 4) tiles at most).
__device__ __forceinline__ void warp_tiles(int w, int R, int nct, int& ct0, int& ct1) {
  const int ns = 4 / R;             // sub-partitions per row set
  const int si = (w & 3) / R;       // this warp's among them
  const int s0 = nct * si / ns, s1 = nct * (si + 1) / ns;
  const int h = w >> 2;             // first or second warp of the sub-partition
  ct0 = s0 + (s1 - s0) * h / 2;
  ct1 = s0 + (s1 - s0) * (h + 1) / 2;
}

// N: compile-time row length (0: runtime P.n) -- with it every shared-memory
// address of the inner loops is a register plus an immediate
template <int N, int HS, int B>
__global__ void __launch_bounds__(THREADS, 1) moment_top_dmma_kernel(const MomParams P) {
  constexpr int KC = Geo<HS>::KC;
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[MAX_STAGES + 2 * PWARPS * ASLOTS];
  __shared__ uint32_t rel[MAX_STAGES];
  const MomTile tile = P.tiles[blockIdx.x];
  const int R = static_cast<int>(tile.pad0);    // row-set slots of this CTA: 1, 2, 4
  const int nrs = static_cast<int>(tile.nrows); // live row sets (<= R)
  const int nct0 = static_cast<int>(tile.ncols);
  const bool sums = P.low != nullptr && tile.low;
  const int nct = nct0;
  Ring g;
  g.stages = static_cast<uint32_t>(P.stages);
  g.xs = smem;
  // reads past row n of the last stage (B fragments of the last column
  // tile) land in this padding and only feed outputs that are never stored
  g.arings = smem + static_cast<size_t>(g.stages) * KC * P.n + 64;
  g.aslots = static_cast<uint32_t>(ASLOTS * PWARPS / R);
  g.alog = 31 - __clz(g.aslots);
  g.xfull = bars;
  g.rel = rel;
  g.afull = bars + MAX_STAGES;
  g.aempty = g.afull + PWARPS * ASLOTS;  // aslots x (live row sets <= R) <= PWARPS x ASLOTS
  g.kc = KC;
  g.cpp = (P.K + KC - 1) / KC;
  g.chunks = g.cpp * P.npass;  // incoming pass, then outgoing pass
  const int warp = threadIdx.x >> 5;
  // active warps: DMMA warps whose row set is live, one producer per live row set
  int active = nrs;
  int cparts = 0;  // DMMA warps with tiles per row set (the same for every row set)
  for (int w = 0; w < CWARPS; ++w) {
    int c0, c1;
    warp_tiles(w, R, nct, c0, c1);
    active += (w % R) < nrs && c1 > c0;
    cparts += (w % R) == 0 && c1 > c0;
  }
  g.active = static_cast<uint32_t>(active);
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < g.stages; ++s) {
      mbar_init(g.xfull + s, 1);
      rel[s] = 0;
    }
    for (int s = 0; s < PWARPS * ASLOTS; ++s) {
      mbar_init(g.afull + s, 1);
      mbar_init(g.aempty + s, cparts);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t i = 0; i < g.chunks && i < g.stages; ++i) issue_chunk(P, g, i, i);
  }
  __syncthreads();
  if (warp >= CWARPS) {
    const int rs = warp - CWARPS;
    if (rs >= nrs) return;
#define CSB_PRODUCE(LM1)                                       \
  if (sums) produce<LM1, N, HS, true>(P, tile, g, rs);        \
  else produce<LM1, N, HS, false>(P, tile, g, rs);
    switch (P.L) {
      case 2: CSB_PRODUCE(1) break;
      case 3: CSB_PRODUCE(2) break;
      case 4: CSB_PRODUCE(3) break;
      case 5: CSB_PRODUCE(4) break;
      default: break;
    }
#undef CSB_PRODUCE
    return;
  }
  const int rs = warp % R;
  if (rs >= nrs) return;
  int ct0, ct1;
  warp_tiles(warp, R, nct, ct0, ct1);
  switch (ct1 - ct0) {
    case 1: consume<1, N, HS, B>(P, tile, g, rs, ct0, warp); break;
    case 2: consume<2, N, HS, B>(P, tile, g, rs, ct0, warp); break;
    case 3: consume<3, N, HS, B>(P, tile, g, rs, ct0, warp); break;
    default: break;
  }
}

// ---------------------------------------------------------------------------
// The narrowest column windows on the CUDA cores.  The prefix rows (pi, i_L)
// of window h (8h <= i_L < 8h + 8) need the columns [i_L, n); in the last
// window that is a triangle inside one 8-wide tile, which the DMMA path
// executes about twice over while its producers set the pace (13.7 TFLOP/s
// executed at cfg2, half of it useful).  Here a thread owns one task:
//  * triangle (TAIL_TRI): a prefix pi and the run of its last indices
//    i_L in [s, e) = [max(i_{L-1}, 8h), min(8h + 8, n)), with every column
//    i_d in [i_L, e), plus the order-(d-1) sums of the run's rows;
//  * rectangle (TAIL_RECT): a sub-run [s, e) of at most 4 last indices
//    times the 8 columns [c0, c0 + 8) right of the window.
// Per data row it forms P = x[pi_1] ... x[pi_{L-1}] (moments.cpp:55, left
// to right), q = P x[i_L] for each i_L of the run, adds q to the order-(d-1)
// sum (moments.cpp:44) and chains acc = fma(q, x[i_d], acc) over its
// columns (moments.cpp:47) -- the reference's own per-element sequence, so
// M_d and M_{d-1} stay bit-exact.  Tasks are grouped on the host so the
// lanes of a warp share the kind and run length (compile-time accumulator
// shapes) and the first last index s.  Rows stream through a TMA bulk-copy
// ring like the DMMA kernel's (zero rows past the end of a pass add exact
// zeros); the incoming pass's means are stashed in shared memory.
constexpr int TAIL_THREADS = 384;  // 3 warps per SM sub-partition (one CTA per SM)
constexpr int TAIL_WARPS = TAIL_THREADS / 32;
constexpr int TAIL_KC = 32;     // data rows per chunk
constexpr int TAIL_STASH = 44;  // doubles per thread: 36 + 8 (triangle of 8), 32 (rectangle 4 x 8)
// The stash lives in global memory, one slot per SM: the kernel's shared
// memory request (> half an SM's) keeps it at one resident CTA per SM.
constexpr size_t TAIL_MIN_SMEM = 120 * 1024;

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

// acc = fma(q, x, acc) that stays where it is written.  A DFMA whose three
// operand pairs all come from the register file takes the FP64 pipe for 3
// cycles instead of 2; with one operand held in the operand-reuse cache it
// takes 2 (tools/fp64_operands.cu: 66.5% of peak with nothing shared between
// consecutive DFMAs, 88.5% for runs sharing q).  ptxas left to itself
// interleaves the rows of a tile and keeps the reuse flag on only ~40% of
// this kernel's DFMAs; volatile asm keeps each row's run of FMAs -- all on the
// same q -- together.
__device__ __forceinline__ void fma_keep(double& acc, double q, double x) {
  asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(q), "d"(x));
}

template <int N, int LM1, int RL, int W, bool TRI, bool ODD>
__device__ __forceinline__ void tail_run(const MomParams& P, const TailTask& tk, const Ring& g, double* stash) {
  // TRI: the run is the column range, W == RL; else RL run rows x W columns
  constexpr int NA = TRI ? RL * (RL + 1) / 2 : RL * W;
  constexpr int NS = TRI ? RL : 0;  // order-(d-1) sums
  const int n = N ? N : P.n;  // compile-time row length: immediate shared-memory offsets
  const int s = tk.s, c0 = TRI ? tk.s : tk.c0;
  const int tid = threadIdx.x;
  int pidx[LM1];
#pragma unroll
  for (int u = 0; u < LM1; ++u) pidx[u] = tk.pidx[u];
  double acc[NA], sum[NS > 0 ? NS : 1];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
#pragma unroll
  for (int i = 0; i < NS; ++i) sum[i] = 0.0;
  const bool update = P.npass == 2;
  const size_t stage_elems = static_cast<size_t>(TAIL_KC) * n;
  Cursor cur;
  for (uint32_t c = 0; c < g.chunks; ++c) {
    mbar_wait(g.xfull + cur.st, cur.ph);
    const double* xs = g.xs + cur.st * stage_elems;
    // The prefix product of row r + 1 is formed while row r's chains run
    // (software pipelining by hand: ptxas otherwise starts every row with
    // the dependent DMUL chain P -> q -> first fma, ~28% of the kernel's
    // stall samples with 3 warps per scheduler to hide it).
    double pn = xs[pidx[0]];
#pragma unroll
    for (int u = 1; u < LM1; ++u) pn = __dmul_rn(pn, xs[pidx[u]]);
#pragma unroll 8  // (measured: 2 -> 8 rows per iteration 7.38 -> 7.02 ms at cfg2)
    for (int r = 0; r < TAIL_KC; ++r) {
      const double* xr = xs + r * n;
      const double pv = pn;
      {
        const double* xn = xs + min(r + 1, TAIL_KC - 1) * n;
        pn = xn[pidx[0]];
#pragma unroll
        for (int u = 1; u < LM1; ++u) pn = __dmul_rn(pn, xn[pidx[u]]);
      }
      // operand loads as 16-byte pairs: every shared-memory load instruction
      // costs the FP64 pipe ~2.5 issue cycles (tools/fp64_occupancy.cu), so
      // halving their number is worth more than any latency hiding here
      double xa[RL], xc[W];
      {
        int k = 0;
        if (ODD) xa[k++] = xr[s];
#pragma unroll
        for (; k + 1 < RL; k += 2) {
          const double2 v = *reinterpret_cast<const double2*>(xr + s + k);
          xa[k] = v.x;
          xa[k + 1] = v.y;
        }
        if (k < RL) xa[k] = xr[s + k];
      }
      if (TRI) {
#pragma unroll
        for (int k = 0; k < W; ++k) xc[k] = xa[k < RL ? k : 0];
      } else {  // c0 is a multiple of 8
#pragma unroll
        for (int k = 0; k < W; k += 2) {
          const double2 v = *reinterpret_cast<const double2*>(xr + c0 + k);
          xc[k] = v.x;
          xc[k + 1] = v.y;
        }
      }
      // all of the row's q first (their DMUL latencies overlap each other),
      // then each q's run of FMAs: nothing to hide inside a run, so ptxas has
      // no reason to interleave runs and drop the operand reuse
      double q[RL];
#pragma unroll
      for (int i = 0; i < RL; ++i) q[i] = __dmul_rn(pv, xa[i]);
      if (TRI) {
#pragma unroll
        for (int i = 0; i < NS; ++i) sum[i] = __dadd_rn(sum[i], q[i]);
      }
      int a = 0;
#pragma unroll
      for (int i = 0; i < RL; ++i) {
#pragma unroll
        for (int j = TRI ? i : 0; j < W; ++j, ++a) fma_keep(acc[a], q[i], xc[j]);
      }
    }
    release_chunk(P, g, c, cur.st);
    if (update && c + 1 == g.cpp) {  // end of the incoming pass: stash its means
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        stash[a * P.stash_stride + tid] = __dmul_rn(acc[a], P.inv);
        acc[a] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        stash[(NA + i) * P.stash_stride + tid] = __dmul_rn(sum[i], P.inv);
        sum[i] = 0.0;
      }
    }
    cur.next(g.stages);
  }
  if (tk.row0 == kNoRow) return;
  // epilogue: the canonical entries (pi, i_L, i_d) of M_d and (pi, i_L) of M_{d-1}
  const int b = P.b;
  const double cc = P.c;
  double* __restrict__ top = P.top;
  double* __restrict__ low = P.low;
  int a = 0;
#pragma unroll
  for (int i = 0; i < RL; ++i) {
    const PrefixRow& row = P.rows[tk.row0 + i];
    const uint64_t tb = row.top_base;
    const uint64_t vp = row.vprime, po = row.poff;
    const int J = (s + i) / b;
#pragma unroll
    for (int j = TRI ? i : 0; j < W; ++j, ++a) {
      const int col = c0 + j;
      const int jd = col / b;
      const size_t o = tb + vp * b * (jd - J) + po * ext_of(jd, n, b) + (col - jd * b);
      const double v = __dmul_rn(acc[a], P.inv);
      top[o] = update ? __fma_rn(cc, __dsub_rn(stash[a * P.stash_stride + tid], v), top[o]) : v;  // a - b
    }
    if (NS > 0 && low) {
      const double v = __dmul_rn(sum[i < NS ? i : 0], P.inv);
      low[row.low_off] =
          update ? __fma_rn(cc, __dsub_rn(stash[(NA + i) * P.stash_stride + tid], v), low[row.low_off]) : v;
    }
  }
}

template <int N, int LM1>
__device__ __forceinline__ void tail_dispatch(const MomParams& P, const TailTask& tk, const Ring& g, double* stash) {
  const int rl = tk.e - tk.s;
  const bool odd = tk.s & 1;  // warp-uniform: a warp's tasks share s
  if (tk.kind == TAIL_TRI) {
    switch (rl) {
      case 1: if (odd) tail_run<N, LM1, 1, 1, true, true>(P, tk, g, stash); else tail_run<N, LM1, 1, 1, true, false>(P, tk, g, stash); break;
      case 2: if (odd) tail_run<N, LM1, 2, 2, true, true>(P, tk, g, stash); else tail_run<N, LM1, 2, 2, true, false>(P, tk, g, stash); break;
      case 3: if (odd) tail_run<N, LM1, 3, 3, true, true>(P, tk, g, stash); else tail_run<N, LM1, 3, 3, true, false>(P, tk, g, stash); break;
      case 4: if (odd) tail_run<N, LM1, 4, 4, true, true>(P, tk, g, stash); else tail_run<N, LM1, 4, 4, true, false>(P, tk, g, stash); break;
      case 5: if (odd) tail_run<N, LM1, 5, 5, true, true>(P, tk, g, stash); else tail_run<N, LM1, 5, 5, true, false>(P, tk, g, stash); break;
      case 6: if (odd) tail_run<N, LM1, 6, 6, true, true>(P, tk, g, stash); else tail_run<N, LM1, 6, 6, true, false>(P, tk, g, stash); break;
      case 7: if (odd) tail_run<N, LM1, 7, 7, true, true>(P, tk, g, stash); else tail_run<N, LM1, 7, 7, true, false>(P, tk, g, stash); break;
      case 8: if (odd) tail_run<N, LM1, 8, 8, true, true>(P, tk, g, stash); else tail_run<N, LM1, 8, 8, true, false>(P, tk, g, stash); break;
      default: break;
    }
  } else {
    switch (rl) {
      case 1: if (odd) tail_run<N, LM1, 1, 8, false, true>(P, tk, g, stash); else tail_run<N, LM1, 1, 8, false, false>(P, tk, g, stash); break;
      case 2: if (odd) tail_run<N, LM1, 2, 8, false, true>(P, tk, g, stash); else tail_run<N, LM1, 2, 8, false, false>(P, tk, g, stash); break;
      case 3: if (odd) tail_run<N, LM1, 3, 8, false, true>(P, tk, g, stash); else tail_run<N, LM1, 3, 8, false, false>(P, tk, g, stash); break;
      case 4: if (odd) tail_run<N, LM1, 4, 8, false, true>(P, tk, g, stash); else tail_run<N, LM1, 4, 8, false, false>(P, tk, g, stash); break;
      default: break;
    }
  }
}

template <int N, int LM1>
__global__ void __launch_bounds__(TAIL_THREADS, 1) moment_tail_kernel(const MomParams P) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t bars[MAX_STAGES];
  __shared__ uint32_t rel[MAX_STAGES];
  const int warp = threadIdx.x >> 5;
  // (the block may be launched narrower than TAIL_THREADS: few tasks are
  // spread over all SMs, one or two warps per scheduler, rather than
  // packed 12 warps deep on a few)
  const uint32_t tw = blockDim.x >> 5;
  const uint32_t live = min(tw, P.tail_warps - blockIdx.x * tw);
  Ring g;
  g.stages = static_cast<uint32_t>(P.stages);
  g.xs = smem;
  g.xfull = bars;
  g.rel = rel;
  g.kc = TAIL_KC;
  g.cpp = (P.K + TAIL_KC - 1) / TAIL_KC;
  g.chunks = g.cpp * P.npass;
  g.active = live;
  const uint32_t smid = sm_id();
  if (smid >= P.stash_slots) __trap();  // the scratch is sized by %nsmid
  double* stash = P.scratch + static_cast<size_t>(smid) * TAIL_THREADS;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < g.stages; ++s) {
      mbar_init(g.xfull + s, 1);
      rel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t i = 0; i < g.chunks && i < g.stages; ++i) issue_chunk(P, g, i, i);
  }
  __syncthreads();
  if (static_cast<uint32_t>(warp) >= live) return;
  const TailTask tk = P.tail[(static_cast<size_t>(blockIdx.x) * tw + warp) * 32 + (threadIdx.x & 31)];
  tail_dispatch<N, LM1>(P, tk, g, stash);
}

size_t tail_smem_bytes(int n, int stages) {
  return std::max(TAIL_MIN_SMEM, sizeof(double) * static_cast<size_t>(stages) * TAIL_KC * n);
}

__global__ void nsmid_kernel(uint32_t* out) {
  uint32_t v;
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
  *out = v;
}

// Symmetric copies of the canonical entries written above, one CTA per
// stored block with equal neighbouring coordinates (symten.cpp:195-220):
// entry o of block j holds the value of the entry with o sorted within each
// run of equal j.  The reference RMWs every stored copy with the same
// fma(c, a - b, old) as its canonical entry (moments.cpp:294-299); the
// copies enter every step bit-identical to the canonical entry (prime
// scatters one value into all of them), so after the update they equal the
// canonical entry's new value, and a copy is exactly that: m[dst] = m[src].
// Full blocks (every extent b) stream a host-built (dst, src) list of their
// run pattern; edge blocks sort each position's offsets in place.
template <int S>
__global__ void __launch_bounds__(256) mirror_kernel(double* __restrict__ m, LayoutDev lay,
                                                     const uint32_t* __restrict__ blocks, int n, int b,
                                                     const uint2* __restrict__ lists,
                                                     const uint32_t* __restrict__ list_off) {
  const uint32_t blk = blocks[blockIdx.x];
  int j[S], e[S];
  bool full = true;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    j[k] = lay.index[static_cast<size_t>(blk) * S + k];
    e[k] = ext_of(j[k], n, b);
    full &= e[k] == b;
  }
  const uint64_t base = lay.offset[blk];
  double* __restrict__ mb = m + base;
  if (full && lists) {
    uint32_t pat = 0;
#pragma unroll
    for (int k = 1; k < S; ++k) pat |= static_cast<uint32_t>(j[k] == j[k - 1]) << (k - 1);
    const uint32_t i0 = list_off[pat], i1 = list_off[pat + 1];
    // four independent copies in flight per thread (latency-bound otherwise)
    constexpr uint32_t U = 4;
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += U * blockDim.x) {
      uint2 pr[U];
      double v[U];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) {
        const uint32_t k = i + u * blockDim.x;
        pr[u] = k < i1 ? __ldg(lists + k) : make_uint2(0u, 0u);
      }
#pragma unroll
      for (uint32_t u = 0; u < U; ++u) v[u] = mb[pr[u].y];
#pragma unroll
      for (uint32_t u = 0; u < U; ++u)
        if (i + u * blockDim.x < i1) mb[pr[u].x] = v[u];
    }
    return;
  }
  // (32-bit positions: a block of b^S <= 2^32 entries; the 64-bit divisions
  // here were calls into a division routine -- cfg4's M_6, 26 GB, took 32 ms)
  const uint32_t vol = static_cast<uint32_t>(lay.offset[blk + 1] - base);
  for (uint32_t pos = threadIdx.x; pos < vol; pos += blockDim.x) {
    int o[S];
    uint32_t rem = pos;
#pragma unroll
    for (int k = S - 1; k >= 0; --k) {
      o[k] = static_cast<int>(rem % static_cast<uint32_t>(e[k]));
      rem /= static_cast<uint32_t>(e[k]);
    }
    bool canonical = true;
#pragma unroll
    for (int k = 1; k < S; ++k)
      if (j[k] == j[k - 1] && o[k] < o[k - 1]) canonical = false;
    if (canonical) continue;
    // sort within runs (bubble passes over a tiny array, fully unrolled)
#pragma unroll
    for (int pass = 0; pass < S - 1; ++pass)
#pragma unroll
      for (int k = 1; k < S; ++k)
        if (j[k] == j[k - 1] && o[k] < o[k - 1]) {
          const int t = o[k];
          o[k] = o[k - 1];
          o[k - 1] = t;
        }
    uint32_t src = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) src = src * static_cast<uint32_t>(e[k]) + static_cast<uint32_t>(o[k]);
    mb[pos] = mb[src];
  }
}

size_t smem_bytes(int n, int stages, int hs) {
  return sizeof(double) * (static_cast<size_t>(stages) * 4 * hs * n + 64 + static_cast<size_t>(PWARPS) * ASLOTS * hs * 32 * ASTRIDE);
}

// leaves room for a co-resident low-order CTA (1 KB reserved shared memory per CTA)
constexpr size_t kSmemLimit = 224 * 1024;

int stages_for(int n, int hs) {
  int s = MAX_STAGES;
  while (s > 0 && smem_bytes(n, s, hs) > kSmemLimit) --s;
  return s;
}

// the longest chunk that still leaves >= 5 stages (>= 2 at worst); the
// 10-step chunk (instantiated for cfg2's n = 48, b = 4 only) at >= 4 stages:
// fewer chunk hand-offs per row beat the shallower ring there (cfg2 top
// kernel 16.01 -> 15.79 ms, tools/gpu_hs10.sh)
int chunk_steps(int n, int b) {
  const bool hs10 = n == 48 && b == 4;
  if (hs10 && stages_for(n, 10) >= 4) return 10;
  for (int hs : {8, 6, 4})
    if (stages_for(n, hs) >= 5) return hs;
  return 4;
}

struct DmmaKernel {
  void (*fn)(MomParams);
  const char* name;
};

// specialised (row length, chunk, block size) of the BASELINE configs; generic otherwise
DmmaKernel pick_dmma_kernel(int n, int b) {
  const int hs = chunk_steps(n, b);
#define CSB_K(NN, HH, BB) {moment_top_dmma_kernel<NN, HH, BB>, "moment_top_dmma_kernel<" #NN "," #HH "," #BB ">"}
  if (n == 96 && hs == 6 && b == 8) return CSB_K(96, 6, 8);
  if (n == 96 && hs == 8 && b == 8) return CSB_K(96, 8, 8);
  if (n == 48 && hs == 8 && b == 4) return CSB_K(48, 8, 4);
  if (n == 48 && hs == 10 && b == 4) return CSB_K(48, 10, 4);
  if (n == 24 && hs == 8 && b == 3) return CSB_K(24, 8, 3);
  if (n == 256 && hs == 4 && b == 16) return CSB_K(256, 4, 16);
  if (hs == 8) return CSB_K(0, 8, 0);
  if (hs == 6) return CSB_K(0, 6, 0);
  return CSB_K(0, 4, 0);
#undef CSB_K
}

}  // namespace

const char* dmma_kernel_name(int n, int b) { return pick_dmma_kernel(n, b).name; }

namespace {

int tail_stages(int n) {
  int st = MAX_STAGES;
  while (st > 0 && tail_smem_bytes(n, st) > kSmemLimit) --st;
  return st;
}

uint32_t sm_id_slots() {  // %nsmid of the current device (SM ids can exceed the SM count)
  static std::mutex mu;
  static std::map<int, uint32_t> cache;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  uint32_t* d = nullptr;
  uint32_t v = 0;
  CSB_CUDA(cudaMalloc(&d, sizeof(uint32_t)));
  nsmid_kernel<<<1, 1>>>(d);
  CSB_CUDA(cudaMemcpy(&v, d, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  CSB_CUDA(cudaFree(d));
  cache[dev] = v;
  return v;
}

}  // namespace

// even rows: the operand pairs are 16-byte loads
bool tail_supported(int n, int /*b*/) { return n % 2 == 0 && tail_stages(n) >= 2; }

size_t tail_scratch_doubles() { return static_cast<size_t>(sm_id_slots()) * TAIL_THREADS * TAIL_STASH; }

int tail_windows(int S, int n, int b) {
  if (S < 3 || S > 6 || !tail_supported(n, b)) return 0;
  // one triangle task per (S-2)-prefix pi of the last window: below ~4 warps
  // per SM the CUDA-core kernel is latency-bound and the DMMA tile wins
  double tasks = 1.0;
  for (int k = 1; k <= S - 2; ++k) tasks = tasks * (n + k - 1) / k;  // C(n + S - 3, S - 2)
  // (measured at cfg1, 4656 prefixes: with the two last windows here, spread
  // one warp per scheduler over the SMs, the DMMA kernel saves 0.17 ms and
  // this kernel costs 0.20 ms)
  if (tasks < 4.0 * 148 * 32) return 0;
  // (measured at cfg2: a third window on the CUDA cores costs what it saves,
  // 1.23 + 9.34 ms against 3.60 + 7.02 ms)
  return 2;  // the last two windows (one when n is not a multiple of 8)
}

void launch_moment_tail(const MomParams& p_in, cudaStream_t st) {
  if (p_in.tail_warps == 0) return;
  MomParams p = p_in;
  p.stages = tail_stages(p.n);
  if (p.stages < 2) fail(CSB_EINVAL, "moment_tail: rows too wide for the staging ring");
  p.stash_slots = sm_id_slots();
  p.stash_stride = p.stash_slots * TAIL_THREADS;  // doubles between a thread's stashed values
  const size_t smem = tail_smem_bytes(p.n, p.stages);
  using K = void (*)(MomParams);
  K kern = nullptr;
  // specialised row lengths of the BASELINE configs (orders 4 and 6); generic otherwise
  const int lm1 = p.L - 1;
  if (p.n == 48 && lm1 == 4) kern = moment_tail_kernel<48, 4>;
  else if (p.n == 96 && lm1 == 4) kern = moment_tail_kernel<96, 4>;
  else if (p.n == 96 && lm1 == 2) kern = moment_tail_kernel<96, 2>;
  else if (p.n == 256 && lm1 == 2) kern = moment_tail_kernel<256, 2>;
  else if (lm1 == 1) kern = moment_tail_kernel<0, 1>;
  else if (lm1 == 2) kern = moment_tail_kernel<0, 2>;
  else if (lm1 == 3) kern = moment_tail_kernel<0, 3>;
  else if (lm1 == 4) kern = moment_tail_kernel<0, 4>;
  else fail(CSB_EINVAL, "moment_tail: order out of range");
  ensure_smem(kern, smem);
  // warps per CTA: 12 when there is work for every SM at that depth, else
  // as few as still cover the SMs (one CTA per SM either way)
  static int sms = 0;
  if (!sms) CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const unsigned tw = std::max(1u, std::min<unsigned>(TAIL_WARPS, (p.tail_warps + sms - 1) / sms));
  const unsigned grid = (p.tail_warps + tw - 1) / tw;
  kern<<<grid, tw * 32, smem, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

// per tile: the incoming pass's means (64 values per consumer thread)
size_t dmma_scratch_per_tile() { return static_cast<size_t>(CWARPS) * 32 * 16 * MAXNC; }

bool dmma_supported(const MomParams& p) {
  // instantiated for orders 3..6 (L = 2..5); rows must be 16-byte aligned
  // for the bulk copies (even n and 16-byte aligned segment starts: a
  // caller's pointer may be offset by one double), and at least two stages
  // must fit
  if (p.n % 2 != 0 || p.L < 2 || p.L > 5) return false;
  if (!rows_aligned16(p.src, p.npass)) return false;
  return stages_for(p.n, 4) >= 2;
}

// data rows per chunk of the launched kernel: the zero-row source of a
// pass's last chunk must hold this many rows
uint32_t dmma_chunk_rows(int n, int b) {
  return std::max<uint32_t>(4u * static_cast<uint32_t>(chunk_steps(n, b)), TAIL_KC);  // either kernel's chunk
}

void launch_mirror(int S, double* m, const LayoutDev& lay, const uint32_t* blocks, uint32_t nblocks, int n, int b,
                   const uint2* lists, const uint32_t* list_off, cudaStream_t st) {
  if (!nblocks) return;
  {
    double vol = 1.0;
    for (int k = 0; k < S; ++k) vol *= static_cast<double>(b);
    if (vol > 4294967295.0) fail(CSB_EINVAL, "mirror: a block of more than 2^32 entries");
  }
  switch (S) {
#define CSB_MIRROR(SS) \
  case SS: mirror_kernel<SS><<<nblocks, 256, 0, st>>>(m, lay, blocks, n, b, lists, list_off); break;
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
  const int hs = chunk_steps(p.n, p.b);
  p.stages = stages_for(p.n, hs);
  if (p.stages < 2) fail(CSB_EINVAL, "moment_top_dmma: rows too wide for the staging ring");
  const size_t smem = smem_bytes(p.n, p.stages, hs);
  const DmmaKernel k = pick_dmma_kernel(p.n, p.b);
  ensure_smem(k.fn, smem);
  auto kern = k.fn;
  kern<<<ntiles, THREADS, smem, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
