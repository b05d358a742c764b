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
// Data flow per CTA (8 warps): rows of the window stream through a 3-stage
// shared-memory ring filled by cp.async.bulk (TMA bulk copies, one per row,
// completion on an mbarrier); every warp owns MG x 8 prefix rows and NC x 8
// columns of the tile, computes its Khatri-Rao operand fragments in
// registers straight from the staged rows, and keeps its accumulators in
// registers across both passes (incoming rows, then outgoing rows).  The
// M_{d-1} sums are formed from the same fragments (warp shuffles put the
// four k values of a row in order) and kept in shared memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace csb {

namespace {

constexpr int WARPS = 8;
constexpr int THREADS = WARPS * 32;
constexpr int STAGES = 3;
constexpr int MAX_MG = 8;
constexpr int MAX_LOW_ROWS = WARPS * 8 * MAX_MG;

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

__device__ __forceinline__ bool next_perm(int* a, int len) {
  if (len < 2) return false;
  int i = len - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) {
    for (int l = 0, r = len - 1; l < r; ++l, --r) {
      const int t = a[l];
      a[l] = a[r];
      a[r] = t;
    }
    return false;
  }
  int j = len - 1;
  while (a[j] <= a[i]) --j;
  int t = a[i];
  a[i] = a[j];
  a[j] = t;
  for (int l = i + 1, r = len - 1; l < r; ++l, --r) {
    t = a[l];
    a[l] = a[r];
    a[r] = t;
  }
  return true;
}

// RMW (update) or assign every stored copy of one canonical element
// (distinct permutations of the in-block offsets within runs of equal block
// coordinate, symten.cpp:195-220).
__device__ __noinline__ void store_copies(double* dst, int S, const int* jv, int* ov, const int* ev,
                                          uint64_t blk, bool update, double c, double delta, double v) {
  bool runs = false;
  for (int k = 1; k < S; ++k) runs |= (jv[k] == jv[k - 1]);
  int rs[kMaxOrder], re[kMaxOrder], nr = 0;
  if (runs) {
    for (int s = 0; s < S;) {
      int t = s + 1;
      while (t < S && jv[t] == jv[s]) ++t;
      rs[nr] = s;
      re[nr] = t;
      ++nr;
      s = t;
    }
  }
  for (;;) {
    uint64_t off = 0;
    for (int k = 0; k < S; ++k) off = off * static_cast<uint64_t>(ev[k]) + static_cast<uint64_t>(ov[k]);
    double* p = dst + blk + off;
    *p = update ? __fma_rn(c, delta, *p) : v;
    if (!runs) break;
    int q = nr - 1;
    while (q >= 0 && !next_perm(ov + rs[q], re[q] - rs[q])) --q;
    if (q < 0) break;
  }
}

template <int MG, int NC>
__device__ __forceinline__ void run_tile(const MomParams& P, const MomTile& tile, double* xs,
                                         uint64_t* full, double* lowacc, int XS, int KC) {
  const int n = P.n, b = P.b, L = P.L;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncg = static_cast<int>((tile.ncols + 7) / 8);
  const int nr = static_cast<int>(tile.nrows);
  const int wrow0 = warp * 8 * MG;  // first tile row of this warp
  const bool do_low = (P.low != nullptr) && tile.low;

  // prefix indices of my MG rows (row = wrow0 + 8g + lane/4), two uint16
  // per register
  uint32_t pidx[MG][4];
  bool rvalid[MG];
#pragma unroll
  for (int g = 0; g < MG; ++g) {
    const int r = wrow0 + 8 * g + (lane >> 2);
    rvalid[g] = r < nr;
    const PrefixRow& pr = P.rows[tile.row0 + (rvalid[g] ? r : 0)];
    const uint32_t* w = reinterpret_cast<const uint32_t*>(pr.idx);
#pragma unroll
    for (int h = 0; h < 4; ++h) pidx[g][h] = w[h];
  }
  auto IDX = [&](int g, int q) -> int { return static_cast<int>((pidx[g][q >> 1] >> (16 * (q & 1))) & 0xffffu); };
  double acc[MG][NC][2];
#pragma unroll
  for (int g = 0; g < MG; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[g][c][0] = acc[g][c][1] = 0.0;

  const uint32_t nch = (P.K + KC - 1) / KC;  // chunks per pass
  const uint32_t total = nch * P.npass;
  const uint32_t rowbytes = static_cast<uint32_t>(n) * 8u;
  const int kq = lane & 3;       // k offset of my A / B fragment
  const int cl = lane >> 2;      // my B column within a group
  const size_t stage_elems = static_cast<size_t>(KC) * XS;

  auto issue = [&](uint32_t i) {
    const int pass = static_cast<int>(i / nch);
    const uint32_t k0 = (i % nch) * KC;
    const uint32_t kc = min(static_cast<uint32_t>(KC), P.K - k0);
    uint64_t* bar = full + (i % STAGES);
    double* dst = xs + (i % STAGES) * stage_elems;
    mbar_expect_tx(bar, kc * rowbytes);
    for (uint32_t r = 0; r < kc; ++r) bulk_g2s(dst + r * XS, row_ptr(P.src[pass], k0 + r, n), rowbytes, bar);
  };
  if (threadIdx.x == 0)
    for (uint32_t i = 0; i < min(static_cast<uint32_t>(STAGES - 1), total); ++i) issue(i);

  for (uint32_t i = 0; i < total; ++i) {
    if (threadIdx.x == 0 && i + STAGES - 1 < total) issue(i + STAGES - 1);
    mbar_wait(full + (i % STAGES), (i / STAGES) & 1u);
    const int pass = static_cast<int>(i / nch);
    const uint32_t k0 = (i % nch) * KC;
    const int kc = static_cast<int>(min(static_cast<uint32_t>(KC), P.K - k0));
    const double* xst = xs + (i % STAGES) * stage_elems;

    for (int kk = 0; kk < KC; kk += 4) {
      if (kk >= kc) break;
      const int k = kk + kq;
      const bool kv = k < kc;
      const double* xr = xst + k * XS;
      double a[MG];
#pragma unroll
      for (int g = 0; g < MG; ++g) {
        double v = 0.0;
        if (kv && rvalid[g]) {
          v = xr[IDX(g, 0)];
#pragma unroll
          for (int q = 1; q < kMaxOrder - 1; ++q)
            if (q < L) v = __dmul_rn(v, xr[IDX(g, q)]);
        }
        a[g] = v;
      }
      if (do_low) {
        // row sums of A in row order: lane kq==0 adds its own value then the
        // three following k (moments.cpp:44, plain adds)
#pragma unroll
        for (int g = 0; g < MG; ++g) {
          const double a1 = __shfl_down_sync(0xffffffffu, a[g], 1);
          const double a2 = __shfl_down_sync(0xffffffffu, a[g], 2);
          const double a3 = __shfl_down_sync(0xffffffffu, a[g], 3);
          if (kq == 0 && rvalid[g]) {
            double* s = lowacc + (pass * MAX_LOW_ROWS + wrow0 + 8 * g + cl);
            double t = __dadd_rn(*s, a[g]);
            if (kk + 1 < kc) t = __dadd_rn(t, a1);
            if (kk + 2 < kc) t = __dadd_rn(t, a2);
            if (kk + 3 < kc) t = __dadd_rn(t, a3);
            *s = t;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (c < ncg) {
          const double bv = kv ? xr[tile.col0 + 8 * c + cl] : 0.0;
#pragma unroll
          for (int g = 0; g < MG; ++g) dmma(acc[g][c][0], acc[g][c][1], a[g], bv);
        }
      }
    }
    __syncthreads();  // stage (i % STAGES) is free for chunk i + STAGES

    if (P.npass == 2 && (i + 1) == nch) {
      // end of the incoming pass: stash its means, restart the accumulators
      double* st = P.scratch + static_cast<size_t>(blockIdx.x) * (THREADS * 48);
#pragma unroll
      for (int g = 0; g < MG; ++g)
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            st[static_cast<size_t>((g * NC + c) * 2 + e) * THREADS + threadIdx.x] = __dmul_rn(acc[g][c][e], P.inv);
            acc[g][c][e] = 0.0;
          }
    }
  }

  // ---- epilogue: order d ----
  const double* st = P.scratch + static_cast<size_t>(blockIdx.x) * (THREADS * 48);
  const bool update = P.npass == 2;
#pragma unroll
  for (int g = 0; g < MG; ++g) {
    if (!rvalid[g]) continue;
    const int r = wrow0 + 8 * g + cl;
    const PrefixRow& pr = P.rows[tile.row0 + r];
    const int lastp = IDX(g, L - 1);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c >= ncg) continue;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = static_cast<int>(tile.col0) + 8 * c + 2 * kq + e;
        if (col >= n || col < lastp) continue;
        const double v = __dmul_rn(acc[g][c][e], P.inv);
        const double delta = update ? __dsub_rn(st[static_cast<size_t>((g * NC + c) * 2 + e) * THREADS + threadIdx.x], v) : 0.0;
        int jv[kMaxOrder], ov[kMaxOrder], ev[kMaxOrder];
        for (int q = 0; q < L; ++q) {
          const int iq = IDX(g, q);
          jv[q] = iq / b;
          ov[q] = iq - jv[q] * b;
          ev[q] = ext_of(jv[q], n, b);
        }
        const int jd = col / b;
        jv[L] = jd;
        ov[L] = col - jd * b;
        ev[L] = ext_of(jd, n, b);
        const uint64_t blk = pr.top_base + static_cast<uint64_t>(pr.vprime) * b * (jd - static_cast<int>(tile.J));
        store_copies(P.top, L + 1, jv, ov, ev, blk, update, P.c, delta, v);
      }
    }
  }
  // ---- epilogue: order d-1 ----
  if (do_low && kq == 0) {
#pragma unroll
    for (int g = 0; g < MG; ++g) {
      if (!rvalid[g]) continue;
      const int r = wrow0 + 8 * g + cl;
      const PrefixRow& pr = P.rows[tile.row0 + r];
      const double v = __dmul_rn(lowacc[(P.npass - 1) * MAX_LOW_ROWS + r], P.inv);
      const double delta = update ? __dsub_rn(__dmul_rn(lowacc[r], P.inv), v) : 0.0;
      int jv[kMaxOrder], ov[kMaxOrder], ev[kMaxOrder];
      for (int q = 0; q < L; ++q) {
        const int iq = IDX(g, q);
        jv[q] = iq / b;
        ov[q] = iq - jv[q] * b;
        ev[q] = ext_of(jv[q], n, b);
      }
      store_copies(P.low, L, jv, ov, ev, pr.low_off - pr.poff, update, P.c, delta, v);
    }
  }
}

__global__ void __launch_bounds__(THREADS, 1) moment_top_dmma_kernel(const MomParams P, int XS, int KC) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  double* xs = smem;
  double* lowacc = xs + static_cast<size_t>(STAGES) * KC * XS;  // 2 x MAX_LOW_ROWS
  const MomTile tile = P.tiles[blockIdx.x];
  // zero the padding columns [n, XS) of the staging ring; bulk copies only
  // ever write [0, n), so the two proxies never touch the same bytes
  const int padw = XS - P.n;
  for (int e = threadIdx.x; e < STAGES * KC * padw; e += THREADS)
    xs[(e / padw) * XS + P.n + (e % padw)] = 0.0;
  for (int e = threadIdx.x; e < 2 * MAX_LOW_ROWS; e += THREADS) lowacc[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  switch (tile.pad0) {
    case 1: run_tile<8, 1>(P, tile, xs, full, lowacc, XS, KC); break;
    case 2: run_tile<8, 2>(P, tile, xs, full, lowacc, XS, KC); break;
    case 3: run_tile<8, 3>(P, tile, xs, full, lowacc, XS, KC); break;
    case 4: run_tile<6, 4>(P, tile, xs, full, lowacc, XS, KC); break;
    case 5: run_tile<4, 5>(P, tile, xs, full, lowacc, XS, KC); break;
    case 6: run_tile<4, 6>(P, tile, xs, full, lowacc, XS, KC); break;
    case 7: run_tile<3, 7>(P, tile, xs, full, lowacc, XS, KC); break;
    case 8: run_tile<3, 8>(P, tile, xs, full, lowacc, XS, KC); break;
    case 9: run_tile<2, 9>(P, tile, xs, full, lowacc, XS, KC); break;
    case 10: run_tile<2, 10>(P, tile, xs, full, lowacc, XS, KC); break;
    case 11: run_tile<2, 11>(P, tile, xs, full, lowacc, XS, KC); break;
    default: run_tile<2, 12>(P, tile, xs, full, lowacc, XS, KC); break;
  }
}

}  // namespace

int dmma_rows_per_warp(int nc) {
  const int mg = nc <= 3 ? 8 : nc == 4 ? 6 : nc <= 6 ? 4 : nc <= 8 ? 3 : 2;
  return 8 * mg;
}

int dmma_warps() { return WARPS; }

size_t dmma_scratch_per_tile() { return static_cast<size_t>(THREADS) * 48; }

bool dmma_supported(const MomParams& p) {
  if (p.n % 2 != 0 || p.L < 1 || p.L > kMaxOrder - 1) return false;
  for (int s = 0; s < p.npass; ++s) {
    if (reinterpret_cast<uintptr_t>(p.src[s].seg0) % 16) return false;
    if (p.src[s].len1 && reinterpret_cast<uintptr_t>(p.src[s].seg1) % 16) return false;
  }
  return true;
}

void launch_moment_top_dmma(const MomParams& p, int ntiles, cudaStream_t st) {
  if (ntiles <= 0) return;
  int XS = p.n + 8;
  while (XS % 16 != 8) ++XS;
  int KC = 32;
  while (KC > 8 && static_cast<size_t>(STAGES) * KC * XS * 8 > 160 * 1024) KC /= 2;
  const size_t smem = sizeof(double) * (static_cast<size_t>(STAGES) * KC * XS + 2 * MAX_LOW_ROWS);
  CSB_CUDA(cudaFuncSetAttribute(moment_top_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  moment_top_dmma_kernel<<<ntiles, THREADS, smem, st>>>(p, XS, KC);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
