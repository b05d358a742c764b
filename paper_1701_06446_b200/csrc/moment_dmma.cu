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
// to 4 column groups of 8, for ONE pass (incoming or outgoing rows).  The
// two passes of a tile pair run as independent CTAs; whichever finishes
// second reads its partner's means from scratch and performs the fused
// update M = fma(p/T, a - b, M) (moments.cpp:297) -- the result does not
// depend on the order they finish.
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

constexpr int WARPS = 4;  // MMA warps; lane 0 of warp 0 also drives the TMA
constexpr int THREADS = WARPS * 32;
constexpr int STAGES = 3;
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

template <int LM1, int NC>
struct Raw {
  double p[LM1 > 0 ? LM1 : 1];  // x[pi_t] of this lane's group
  double a[8];                  // x[8h + g]
  double b[NC];                 // x[col0 + 8c + r]
};

template <int LM1, int NC>
__device__ __forceinline__ void load_raw(Raw<LM1, NC>& w, const double* __restrict__ xr, int h8, int col0,
                                         int r, const int* pidx) {
#pragma unroll
  for (int t = 0; t < LM1; ++t) w.p[t] = xr[pidx[t]];
  const double2* xa = reinterpret_cast<const double2*>(xr + h8);
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const double2 v = xa[s];
    w.a[2 * s] = v.x;
    w.a[2 * s + 1] = v.y;
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) w.b[c] = xr[col0 + 8 * c + r];
}

// A = x[pi_1] * ... * x[pi_{L-1}] * x[8h + g] in the reference's order.
// Rows with g < lo (i_L < i_{L-1}) and padding groups are computed but never
// stored, so no masking is needed; data rows past the end of the pass are
// zeroed (zero == true) so they contribute exact zeros.
template <int LM1, int NC>
__device__ __forceinline__ void finish(Raw<LM1, NC>& w, bool zero) {
  if (LM1 > 0) {
    double P = w.p[0];
#pragma unroll
    for (int t = 1; t < LM1; ++t) P = __dmul_rn(P, w.p[t]);
#pragma unroll
    for (int g = 0; g < 8; ++g) w.a[g] = __dmul_rn(P, w.a[g]);  // 1.0 * x == x: none for L == 1
  }
  if (zero) {
#pragma unroll
    for (int g = 0; g < 8; ++g) w.a[g] = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) w.b[c] = 0.0;
  }
}

template <int LM1, int NC>
__device__ __forceinline__ void run_tile(const MomParams& P, const MomTile& tile, int pass, double* xs,
                                         uint64_t* full, uint64_t* empty, double* lowbufs, uint32_t* flag_smem) {
  constexpr int L = LM1 + 1;
  const int n = P.n, b = P.b;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, r = lane >> 2;
  const int h8 = static_cast<int>(tile.J) * 8;
  const int col0 = static_cast<int>(tile.col0);
  const bool do_low = (P.low != nullptr) && tile.low;
  double* lowbuf = lowbufs + warp * (2 * 4 * 66);  // double-buffered 4 x 66
  const size_t stage_elems = static_cast<size_t>(KC) * n;
  const uint32_t K = P.K;
  const uint32_t chunks = (K + KC - 1) / KC;
  const RowSource& src = P.src[pass];

  // ---- TMA producer: lane 0 of warp 0 ----
  // Chunk c goes into stage c % STAGES once every warp has released chunk
  // c - STAGES.  The producer polls without blocking and blocks only for the
  // chunk warp 0 itself needs next.
  uint32_t next_issue = 0;
  auto pump = [&](uint32_t needed) {
    if (threadIdx.x != 0) return;
    while (next_issue < chunks) {
      const uint32_t i = next_issue;
      const uint32_t st = i % STAGES;
      if (i >= STAGES) {
        const uint32_t par = ((i / STAGES) - 1) & 1u;
        if (!mbar_test(empty + st, par)) {
          if (i > needed) break;
          mbar_wait(empty + st, par);
        }
      }
      const uint32_t a0 = i * KC;
      const uint32_t kc = min(static_cast<uint32_t>(KC), K - a0);
      double* dst = xs + st * stage_elems;
      const uint32_t rb = static_cast<uint32_t>(n) * 8u;
      mbar_expect_tx(full + st, static_cast<uint32_t>(KC) * rb);
      // rows past the end of the pass are zero rows: A = B = 0 adds exact
      // zeros, so the k loop never needs masking
      if (kc < static_cast<uint32_t>(KC))
        bulk_g2s(dst + static_cast<size_t>(kc) * n, P.zeros, (KC - kc) * rb, full + st);
      // rows [a0, a0 + kc) are contiguous except across the ring's wrap
      if (a0 + kc <= src.len0 || a0 >= src.len0) {
        bulk_g2s(dst, row_ptr(src, a0, n), kc * rb, full + st);
      } else {
        const uint32_t k1 = src.len0 - a0;
        bulk_g2s(dst, row_ptr(src, a0, n), k1 * rb, full + st);
        bulk_g2s(dst + static_cast<size_t>(k1) * n, src.seg1, (kc - k1) * rb, full + st);
      }
      ++next_issue;
    }
  };

  const int gl = warp * 8 + r;  // group slot in the tile
  const bool gvalid = gl < static_cast<int>(tile.nrows);
  const uint32_t gi = tile.row0 + (gvalid ? gl : 0);
  const DmmaGroup grp = P.groups[gi];
  int pidx[LM1 > 0 ? LM1 : 1];
#pragma unroll
  for (int t = 0; t < LM1; ++t) pidx[t] = grp.pidx[t];
  const int lo = grp.lo;

  double acc[8][NC][2];
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[g][c][0] = acc[g][c][1] = 0.0;
  double lowacc[2] = {0.0, 0.0};

  auto mma_step = [&](const Raw<LM1, NC>& op) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int g = 0; g < 8; ++g) dmma(acc[g][c][0], acc[g][c][1], op.a[g], op.b[c]);
  };
  // order L sums: the 8 x 4 block (rows g, k) of a step is transposed
  // through shared memory so lane q owns rows 2q, 2q+1 and adds their four
  // k values in row order (moments.cpp:44, plain adds).  Written at step t,
  // read (after the next __syncwarp) at step t + 1.
  auto low_put = [&](const Raw<LM1, NC>& op, int buf) {
    double2* wb = reinterpret_cast<double2*>(lowbuf + buf * 264 + q * 66 + r * 8);
#pragma unroll
    for (int u = 0; u < 4; ++u) wb[u] = make_double2(op.a[2 * u], op.a[2 * u + 1]);
  };
  auto low_get = [&](double2 (&v)[4], int buf) {
#pragma unroll
    for (int kp = 0; kp < 4; ++kp) v[kp] = *reinterpret_cast<const double2*>(lowbuf + buf * 264 + kp * 66 + r * 8 + 2 * q);
  };
  auto low_add = [&](const double2 (&v)[4], int kleft) {
#pragma unroll
    for (int kp = 0; kp < 4; ++kp)
      if (kp < kleft) {
        lowacc[0] = __dadd_rn(lowacc[0], v[kp].x);
        lowacc[1] = __dadd_rn(lowacc[1], v[kp].y);
      }
  };

  bool lowpend = false;  // previous step's A values wait in lowbuf[1 - cur]
  int lb = 0;
  // one step: loads of the next step, DMMAs of this one, row sums, products
  auto step = [&](const Raw<LM1, NC>& cur, Raw<LM1, NC>& nxt, const double* xnext, bool has_next) {
    if (has_next) load_raw<LM1, NC>(nxt, xnext, h8, col0, r, pidx);
    double2 lv[4];
    if (do_low && lowpend) {
      __syncwarp();
      low_get(lv, lb ^ 1);
    }
    mma_step(cur);
    if (do_low) {
      low_put(cur, lb);
      if (lowpend) low_add(lv, 4);
      lowpend = true;
      lb ^= 1;
    }
    if (has_next) finish<LM1, NC>(nxt, false);
  };
  // The step stream is continuous across chunks: the last step of chunk c
  // loads the first operands of chunk c + 1, so the pipeline never drains.
  auto stage_ptr = [&](uint32_t c) {
    return xs + (c % STAGES) * stage_elems + static_cast<size_t>(q) * n;
  };
  Raw<LM1, NC> o0, o1;
  if (warp == 0) pump(0);
  __syncwarp();
  mbar_wait(full + 0, 0u);
  load_raw<LM1, NC>(o0, stage_ptr(0), h8, col0, r, pidx);
  finish<LM1, NC>(o0, false);
  for (uint32_t c = 0; c < chunks; ++c) {
    const double* xst = stage_ptr(c);
#pragma unroll 1
    for (int t = 0; t < KC / 4 - 2; t += 2) {
      step(o0, o1, xst + (4 * t + 4) * n, true);
      step(o1, o0, xst + (4 * t + 8) * n, true);
    }
    step(o0, o1, xst + (KC - 4) * n, true);
    // every lane has loaded its rows of this stage: release it
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + (c % STAGES));
    const bool more = c + 1 < chunks;
    if (more) {
      if (warp == 0) pump(c + 1);
      __syncwarp();
      mbar_wait(full + ((c + 1) % STAGES), ((c + 1) / STAGES) & 1u);
    }
    step(o1, o0, more ? stage_ptr(c + 1) : xst, more);
    if (warp == 0) pump(0);  // refill without blocking
  }
  if (do_low && lowpend) {
    __syncwarp();
    double2 lv[4];
    low_get(lv, lb ^ 1);
    low_add(lv, 4);
  }

  // ---- pair fixup: the second of (incoming, outgoing) does the update ----
  const bool update = P.npass == 2;
  const size_t pair = tile.pad1;
  const int tid = threadIdx.x;
  double* mine = nullptr;
  const double* other = nullptr;
  if (update) {
    double* base = P.scratch + pair * (2 * (THREADS * 64 + THREADS * 2));
    mine = base + pass * (THREADS * 64 + THREADS * 2);
    other = base + (pass ^ 1) * (THREADS * 64 + THREADS * 2);
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          mine[static_cast<size_t>((g * NC + c) * 2 + e) * THREADS + tid] = __dmul_rn(acc[g][c][e], P.inv);
    mine[THREADS * 64 + tid] = __dmul_rn(lowacc[0], P.inv);
    mine[THREADS * 64 + THREADS + tid] = __dmul_rn(lowacc[1], P.inv);
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag_smem = atomicAdd(P.flags + pair, 1u);
    __syncthreads();
    if (*flag_smem == 0) return;  // partner still running: it finishes the pair
    __threadfence();
    if (tid == 0) P.flags[pair] = 0;  // self-resetting for the next launch
  }

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
          const size_t ix = static_cast<size_t>((g * NC + c) * 2 + e) * THREADS + tid;
          const double mv = mine[ix];
          const double ov = ok[c][e] ? __ldcg(other + ix) : 0.0;
          val[c][e] = pass == 0 ? __dsub_rn(mv, ov) : __dsub_rn(ov, mv);  // a - b
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
  if (do_low) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 2 * q + e;
      const int iL = h8 + g;
      if (g < lo || iL >= n) continue;
      const PrefixRow& pr = P.rows[static_cast<size_t>(gi) * 8 + g];
      if (update) {
        const size_t ix = THREADS * 64 + static_cast<size_t>(e) * THREADS + tid;
        const double mv = mine[ix], ov2 = __ldcg(other + ix);
        const double delta = pass == 0 ? __dsub_rn(mv, ov2) : __dsub_rn(ov2, mv);
        P.low[pr.low_off] = __fma_rn(cc, delta, P.low[pr.low_off]);
        if (pr.idx[7] & 1u) P.dlow[pr.low_off] = delta;
      } else {
        P.low[pr.low_off] = __dmul_rn(lowacc[e], P.inv);
      }
    }
  }
}

__global__ void __launch_bounds__(THREADS, 2) moment_top_dmma_kernel(const MomParams P) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ uint32_t flag_smem;
  double* xs = smem;
  // dense staging ring; reads past row n of a stage (the last 8-column
  // window / column group) only feed rows and columns that are never stored
  double* lowbufs = xs + static_cast<size_t>(STAGES) * KC * P.n + 64;  // WARPS x 2 x 4 x 66
  const int pass = static_cast<int>(blockIdx.x % P.npass);
  const MomTile tile = P.tiles[blockIdx.x / P.npass];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nc = static_cast<int>(tile.pad0);
  switch (P.L * 8 + nc) {
#define CSB_CASE(LL, NCC) \
  case (LL) * 8 + (NCC): run_tile<(LL) - 1, NCC>(P, tile, pass, xs, full, empty, lowbufs, &flag_smem); break;
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
  return sizeof(double) * (static_cast<size_t>(STAGES) * KC * n + 64 + WARPS * 2 * 4 * 66);
}

}  // namespace

int dmma_warps() { return WARPS; }

// per tile pair: both passes' stashes (64 values + 2 low sums per thread)
size_t dmma_scratch_per_tile() { return static_cast<size_t>(2) * (THREADS * 64 + THREADS * 2); }

bool dmma_supported(const MomParams& p) {
  // instantiated for orders 3..6 (L = 2..5); the staging ring must fit
  if (p.n % 2 != 0 || p.L < 2 || p.L > 5) return false;
  if (smem_bytes(p.n) > 110 * 1024) return false;  // two CTAs per SM
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
  moment_top_dmma_kernel<<<ntiles * p.npass, THREADS, smem, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
