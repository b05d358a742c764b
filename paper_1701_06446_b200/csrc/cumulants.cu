// moms2cums and the low-order moment kernel (sm_100a).
//
// moms2cums_v2 (cumulants.cpp:128-196): one CTA per stored block of C_S.
//   * the 2^S - 2 lower-order sub-blocks the block's corrections read
//     (one per proper subset of index positions) are staged in shared
//     memory when they fit, so every factor C_|P|[i_P] is an LDS;
//   * phase 1: each canonical entry (offsets non-decreasing within runs of
//     equal block coordinate) is M - partition_correction<S>(f), with the
//     partitions in the reference's RGS order and no FMA contraction, so the
//     result is bit-identical to the reference;
//   * phase 2: every stored entry is written from its canonical source
//     (non-canonical entries copy, cumulants.cpp:172-185) coalesced, and the
//     block's sum of squares (knorm, symten.cpp:257-276) is reduced in a
//     fixed order for the norm/nu report.
//
// moment_lower_kernel: orders S <= d-2 of a window update / prime, one
// thread per canonical element, rows in order: acc = acc + round(product)
// exactly as the reference's upper levels (moments.cpp:55-57).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "ptx.cuh"
#include "partitions_gen.cuh"

namespace csb {

namespace {

__device__ __forceinline__ int ext_of(int j, int n, int b) { return b < n - j * b ? b : n - j * b; }


constexpr int popcount_c(int m) { return m == 0 ? 0 : (m & 1) + popcount_c(m >> 1); }

template <int S>
__device__ __forceinline__ void decode(uint32_t pos, const int (&e)[S], int (&o)[S]) {
#pragma unroll
  for (int k = S - 1; k >= 0; --k) {
    o[k] = static_cast<int>(pos % static_cast<uint32_t>(e[k]));
    pos /= static_cast<uint32_t>(e[k]);
  }
}

template <int S>
__device__ __forceinline__ bool canonical(const int (&j)[S], const int (&o)[S]) {
  bool c = true;
#pragma unroll
  for (int k = 1; k < S; ++k)
    if (j[k] == j[k - 1] && o[k] < o[k - 1]) c = false;
  return c;
}

// In-block offset of the canonical source of entry o: o sorted within runs.
template <int S>
__device__ __forceinline__ uint32_t source_of(const int (&j)[S], int (&o)[S], const int (&e)[S]) {
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
  return src;
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}

// B: compile-time block size (0: runtime) -- full blocks then decode
// positions and address factors with constant divisions and powers
// Orders <= 4: registers capped at 64 -- four 256-thread CTAs per SM for
// the in-block pass (<= 56 KB of shared memory, so registers set the
// occupancy), or one 1024-thread CTA beside large staged sub-blocks
// (b = 16: 144 KB), whose global-memory latency then has 32 warps to hide it.
template <int S, bool STAGED, int B>
__global__ void __launch_bounds__(S <= 4 ? 1024 : 256, S <= 4 ? 1 : 2) moms2cums_v2(const M2CParams P) {
  constexpr int NM = (1 << S) - 1;  // masks 1..NM-1: proper non-empty subsets
  extern __shared__ __align__(16) double sfac[];  // staged sub-blocks (STAGED)
  __shared__ uint64_t sbase[NM];                  // global (or smem) base per subset
  __shared__ uint32_t sstride[NM][S];
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t mbar;  // TMA staging of a full block (even b)
  const uint64_t blk = P.blk0 + blockIdx.x;
  const LayoutDev& LS = P.lay[S - 1];
  const int n = P.n, b = B ? B : P.b;
  int j[S], e[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    j[k] = LS.index[blk * S + k];
    e[k] = ext_of(j[k], n, b);
  }
  const uint64_t boff = LS.offset[blk];
  const uint32_t vol = static_cast<uint32_t>(LS.offset[blk + 1] - boff);

  // sub-block geometry: one mask per thread (offsets precomputed on the
  // host, MomentPlan-style, instead of ranking them here)
  const uint64_t* subs = P.subs + blk * (NM - 1);
  for (int m = 1 + static_cast<int>(threadIdx.x); m < NM; m += blockDim.x) {
    uint32_t stride = 1;
#pragma unroll
    for (int k = S - 1; k >= 0; --k) {
      if (m >> k & 1) {
        sstride[m][k] = stride;
        stride *= static_cast<uint32_t>(e[k]);
      } else {
        sstride[m][k] = 0;
      }
    }
    if (!STAGED) sbase[m] = subs[m - 1];
  }
  bool full = true;
#pragma unroll
  for (int k = 0; k < S; ++k) full &= e[k] == b;
  // a full block is assembled in shared memory: M staged, C computed in
  // place (each canonical position by the thread that reads it), copies
  // filled from the pattern list, then written out coalesced
  const bool inblk = STAGED && full && P.canon && P.mlist && P.inblk;
  double* cblk = sfac + P.cblk;
  // full blocks of an even compile-time b: every sub-block and the M block
  // are whole 16-byte-aligned blocks -> one TMA bulk copy each
  const bool bulk = B != 0 && (B % 2) == 0 && STAGED && full && n % b == 0;
  if (STAGED && threadIdx.x == 0) {
    uint32_t soff = 0;
    for (int m = 1; m < NM; ++m) {
      uint32_t svol = 1;
      for (int k = 0; k < S; ++k)
        if (m >> k & 1) svol *= static_cast<uint32_t>(e[k]);
      sbase[m] = soff;  // offset of the staged copy in shared memory
      soff += svol;
    }
    if (bulk) {
      ptx::mbar_init(&mbar, 1);
      ptx::fence_mbar_init();
      ptx::mbar_expect_tx(&mbar, static_cast<uint32_t>((soff + (inblk ? vol : 0)) * sizeof(double)));
      if (inblk) ptx::bulk_g2s(cblk, P.m + boff, vol * sizeof(double), &mbar);
      for (int m = 1; m < NM; ++m) {
        const uint32_t svol = static_cast<uint32_t>((m + 1 < NM ? sbase[m + 1] : soff) - sbase[m]);
        ptx::bulk_g2s(sfac + sbase[m], P.lower[__popc(m) - 1] + subs[m - 1], svol * sizeof(double), &mbar);
      }
    }
  }
  __syncthreads();
  if (bulk) {
    ptx::mbar_wait(&mbar, 0);
  } else if (STAGED) {
    if (inblk)
      for (uint32_t t = threadIdx.x; t < vol; t += blockDim.x) cp_async8(cblk + t, P.m + boff + t);
    // copy every needed sub-block into shared memory (coalesced per subset;
    // asynchronous, so all subsets' loads are in flight at once)
    for (int m = 1; m < NM; ++m) {
      uint32_t svol = 1;
#pragma unroll
      for (int k = 0; k < S; ++k)
        if (m >> k & 1) svol *= static_cast<uint32_t>(e[k]);
      const double* src = P.lower[__popc(m) - 1] + subs[m - 1];
      double* dst = sfac + sbase[m];
      if (inblk)
        for (uint32_t t = threadIdx.x; t < svol; t += blockDim.x) cp_async8(dst + t, src + t);
      else
        for (uint32_t t = threadIdx.x; t < svol; t += blockDim.x) dst[t] = src[t];
    }
    if (inblk) asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  if (STAGED) {
    if (inblk && P.mfix) {
      // M's symmetric copies from the staged block (before C overwrites it)
      uint32_t pat = 0;
#pragma unroll
      for (int k = 1; k < S; ++k) pat |= static_cast<uint32_t>(j[k] == j[k - 1]) << (k - 1);
      const uint32_t i1 = P.mlist_off[pat + 1];
      for (uint32_t i = P.mlist_off[pat] + threadIdx.x; i < i1; i += blockDim.x) {
        const uint2 pr = __ldg(P.mlist + i);
        P.mfix[boff + pr.x] = cblk[pr.y];
      }
      __syncthreads();
    }
  }

  double part = 0.0;  // this thread's share of the block's sum of squares
  // phase 1: canonical entries.  Full blocks (all extents b) walk the
  // precomputed canonical positions of their run pattern -- no lane idles
  // on the non-canonical copies of diagonal blocks -- and address a factor
  // in its staged sub-block with compile-time powers of b; edge blocks test
  // every position.
  // (also without staging when b is a compile-time constant: the factors
  // then come from global memory (L1 / L2) at sub-block base + offset, but the
  // canonical list, the constant powers of b and the copy lists still apply --
  // cfg4's order 6, whose 2.1 MB of sub-blocks per block cannot be staged, ran
  // the position-by-position path at ~6100 instructions per entry before)
  if (full && P.canon && (STAGED || B != 0)) {
    uint32_t pat = 0;
#pragma unroll
    for (int k = 1; k < S; ++k) pat |= static_cast<uint32_t>(j[k] == j[k - 1]) << (k - 1);
    const uint32_t cbase = P.canon_off[pat];
    const uint32_t* list = P.canon + cbase;
    const uint32_t cnt = P.canon_off[pat + 1] - cbase;
    const bool direct = !inblk && P.cstart;  // copies + norm term written here (no second pass)
    uint32_t bp[S];  // b^0 .. b^(S-1)
    bp[0] = 1;
#pragma unroll
    for (int k = 1; k < S; ++k) bp[k] = bp[k - 1] * static_cast<uint32_t>(b);
    // staged sub-block bases in registers (32-bit shared-memory offsets)
    constexpr int NB = S <= 5 ? NM : 1;
    uint32_t sb[NB];
#pragma unroll
    for (int m = 1; m < NB; ++m) sb[m] = static_cast<uint32_t>(sbase[m]);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const uint32_t pos = __ldg(list + i);
      int o[S];
      if (B) {
        uint32_t r = pos;
#pragma unroll
        for (int k = S - 1; k >= 0; --k) {
          o[k] = static_cast<int>(r % static_cast<uint32_t>(B ? B : 1));
          r /= static_cast<uint32_t>(B ? B : 1);
        }
      } else {
        decode<S>(pos, e, o);
      }
      double f[NM];
#pragma unroll
      for (int m = 1; m < NM; ++m) {
        uint32_t a = 0;
        int after = 0;  // positions of m after k (compile-time after unrolling)
#pragma unroll
        for (int k = S - 1; k >= 0; --k)
          if (m >> k & 1) a += static_cast<uint32_t>(o[k]) * bp[after++];
        if (STAGED)
          f[m] = sfac[(S <= 5 ? sb[m < NB ? m : 0] : static_cast<uint32_t>(sbase[m])) + a];
        else
          f[m] = __ldg(P.lower[__popc(m) - 1] + sbase[m] + a);
      }
      const double corr = partition_correction<S>(f);
      if (inblk) {
        cblk[pos] = __dsub_rn(cblk[pos], corr);
      } else {
        const double v = __dsub_rn(P.m[boff + pos], corr);
        P.c[boff + pos] = v;
        if (direct) {
          const uint32_t c0 = __ldg(P.cstart + cbase + i), c1 = __ldg(P.cstart + cbase + i + 1);
          for (uint32_t q = c0; q < c1; ++q) P.c[boff + __ldg(P.cdst + q)] = v;
          part = __fma_rn(static_cast<double>(1u + c1 - c0), __dmul_rn(v, v), part);
        }
      }
    }
  } else {
    for (uint32_t pos = threadIdx.x; pos < vol; pos += blockDim.x) {
      int o[S];
      decode<S>(pos, e, o);
      if (!canonical<S>(j, o)) continue;
      double f[NM];
#pragma unroll
      for (int m = 1; m < NM; ++m) {
        uint32_t a = 0;
#pragma unroll
        for (int k = 0; k < S; ++k)
          if (m >> k & 1) a += static_cast<uint32_t>(o[k]) * sstride[m][k];
        if (STAGED)
          f[m] = sfac[sbase[m] + a];
        else
          f[m] = P.lower[__popc(m) - 1][sbase[m] + a];
      }
      const double corr = partition_correction<S>(f);
      P.c[boff + pos] = __dsub_rn(P.m[boff + pos], corr);
    }
  }
  __syncthreads();  // canonical entries of this block are visible to the CTA

  // phase 2: copies + the block's sum of squares (fixed order)
  if (inblk) {
    uint32_t pat = 0;
#pragma unroll
    for (int k = 1; k < S; ++k) pat |= static_cast<uint32_t>(j[k] == j[k - 1]) << (k - 1);
    const uint32_t i1 = P.mlist_off[pat + 1];
    for (uint32_t i = P.mlist_off[pat] + threadIdx.x; i < i1; i += blockDim.x) {
      const uint2 pr = __ldg(P.mlist + i);
      cblk[pr.x] = cblk[pr.y];
    }
    __syncthreads();
    for (uint32_t pos = threadIdx.x; pos < vol; pos += blockDim.x) {
      const double v = cblk[pos];
      P.c[boff + pos] = v;
      part = __fma_rn(v, v, part);
    }
    if (P.fold_width) {
      // the block's exact norm partial from the assembled block: knorm's own
      // sequence (symten.cpp:257-276, vectorised like the reference build:
      // fold_width-wide rounded squares added in order, then an FMA tail),
      // one thread while the others write the block out
      if (threadIdx.x == 0) {
        const uint32_t nvec = vol & ~static_cast<uint32_t>(P.fold_width - 1);
        double s = 0.0;
        uint32_t q = 0;
#pragma unroll 8
        for (; q < nvec; ++q) s = __dadd_rn(s, __dmul_rn(cblk[q], cblk[q]));
        for (; q < vol; ++q) s = __fma_rn(cblk[q], cblk[q], s);
        P.partial[blockIdx.x] = s;
      }
      return;
    }
  }
  const bool lists_ok = (STAGED || B != 0) && full && P.canon;            // phase 1 walked the canonical list
  const bool direct = !inblk && lists_ok && P.cstart;                    // copies and norm term done in phase 1
  const bool listed = !inblk && lists_ok && (P.mlist || direct);
  if (listed && !direct) {
    // copies from the canonical entries this CTA just wrote (visible to the
    // block after the barrier above), then the sum of squares in order
    uint32_t pat = 0;
#pragma unroll
    for (int k = 1; k < S; ++k) pat |= static_cast<uint32_t>(j[k] == j[k - 1]) << (k - 1);
    const uint32_t i1 = P.mlist_off[pat + 1];
    for (uint32_t i = P.mlist_off[pat] + threadIdx.x; i < i1; i += blockDim.x) {
      const uint2 pr = __ldg(P.mlist + i);
      P.c[boff + pr.x] = P.c[boff + pr.y];
    }
    __syncthreads();
    for (uint32_t pos = threadIdx.x; pos < vol; pos += blockDim.x) {
      const double v = P.c[boff + pos];
      part = __fma_rn(v, v, part);
    }
  }
  for (uint32_t pos = threadIdx.x; !inblk && !listed && pos < vol; pos += blockDim.x) {
    int o[S];
    decode<S>(pos, e, o);
    double v;
    if (canonical<S>(j, o)) {
      v = P.c[boff + pos];
    } else {
      v = P.c[boff + source_of<S>(j, o, e)];
      P.c[boff + pos] = v;
    }
    part = __fma_rn(v, v, part);
  }
  for (int s = 16; s > 0; s >>= 1) part = __dadd_rn(part, __shfl_down_sync(0xffffffffu, part, s));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s = __dadd_rn(s, red[w]);
    P.partial[blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// moms2cums of a high order over full blocks (every extent B), persistent:
// one CTA per SM, two halves of 8 warps; each half walks its share of the
// CTA's blocks with the block's 2^S - 2 lower-order sub-blocks landing by TMA
// bulk copies in the half's own buffer, and no CTA-wide barrier: each warp
// reduces its share of the block's sum of squares, the last warp of the
// half to finish a block (shared-memory counter) adds the warp sums in warp
// order, writes the block's partial and refills the buffer with the half's
// next block -- whose wait the other half's arithmetic covers.  The arithmetic per canonical
// entry is moms2cums_v2's (partition_correction<S>, the reference's order),
// written with its symmetric copies straight to global memory.
// (Measured at cfg2 order 6: 1.76 ms for moms2cums_v2 -> 1.53 ms; 1.30 ms
// double-buffered with all 16 warps on one block; 1.17 ms as two halves of
// 8 warps with a block and a buffer each -- one half computes while the other
// waits for its sub-blocks; 1.10 ms with the blocks dealt in descending
// order of canonical entries.  Earlier steps: 1.30 ms
// with the refill's stage offsets from a shared table -- the refill is the
// critical path between two blocks -- and the block bookkeeping and copy
// targets requested ahead of their use.  Timing-only experiments: without
// any store 1.46 of 1.51 ms; with 6 instead of 62 bulk copies per block
// 1.42 of 1.57 ms: neither the stores nor the copy count bound it.  A variant
// handing out 32-entry chunks of the oldest open block through a shared
// cursor, so no warp waits for a block's stragglers, measured 1.66 ms:
// the per-chunk hand-off costs more than the waits it removes.)
constexpr int M2CP_THREADS = 512;
constexpr int M2CP_WARPS = M2CP_THREADS / 32;

template <int S, int B>
struct M2cStage {
  // staged doubles of mask m's sub-block (B^|m|) and its offset in a buffer
  static constexpr uint32_t vol(int m) {
    uint32_t v = 1;
    for (int k = 0; k < S; ++k)
      if (m >> k & 1) v *= B;
    return v;
  }
  static constexpr uint32_t off(int m) {
    uint32_t o = 0;
    for (int q = 1; q < m; ++q) o += vol(q);
    return o;
  }
  static constexpr uint32_t total() { return off((1 << S) - 1); }
};

template <int S, int B>
__global__ void __launch_bounds__(M2CP_THREADS, 1) moms2cums_persist(const M2CParams P, uint32_t nblocks) {
  constexpr int NM = (1 << S) - 1;
  using G = M2cStage<S, B>;
  constexpr uint32_t STAGE = G::total();
  extern __shared__ __align__(16) double sfac[];  // 2 x STAGE
  __shared__ __align__(8) uint64_t full[2];
  __shared__ uint32_t done[2];
  __shared__ double red[2][M2CP_WARPS];
  const LayoutDev& LS = P.lay[S - 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // The CTA works as two halves of 8 warps, each on a block of its own in a
  // buffer of its own (the CTA's blocks alternate between them): while one
  // half waits for its next block's sub-blocks the other keeps the FP64 pipe
  // busy, instead of all 16 warps reaching the same hand-off together.
  constexpr int HW = M2CP_WARPS / 2, HT = M2CP_THREADS / 2;
  const int half = warp / HW, hw = warp % HW;
  const uint32_t ht = threadIdx.x % HT;
  const uint32_t ncta = blockIdx.x < nblocks ? (nblocks - 1 - blockIdx.x) / gridDim.x + 1 : 0;  // this CTA's blocks
  const uint32_t nmine = (ncta + 1 - half) / 2;                                                   // this half's
  auto block_of = [&](uint32_t k) {
    const uint64_t idx = blockIdx.x + static_cast<uint64_t>(2 * k + half) * gridDim.x;
    return P.blk0 + (P.order ? static_cast<uint64_t>(__ldg(P.order + idx)) : idx);
  };
  // one warp: TMA bulk copies of block k's sub-blocks into buffer buf, the
  // lanes' copies (and their offset loads) in parallel
  // (stage offsets and sizes per mask from a shared table: the refill sits on
  // the critical path between two blocks, and deriving them per call cost
  // the issuing warp thousands of dependent integer instructions)
  __shared__ uint32_t soff[NM], svol[NM];
  auto issue = [&](uint32_t k, int buf) {
    const uint64_t blk = block_of(k);
    const uint64_t* subs = P.subs + blk * (NM - 1);
    if (lane == 0) ptx::mbar_expect_tx(&full[buf], STAGE * static_cast<uint32_t>(sizeof(double)));
    __syncwarp();
    for (int m = 1 + lane; m < NM; m += 32)
      ptx::bulk_g2s(sfac + buf * STAGE + soff[m], P.lower[__popc(m) - 1] + subs[m - 1],
                    svol[m] * static_cast<uint32_t>(sizeof(double)), &full[buf]);
  };
  for (int m = 1 + threadIdx.x; m < NM; m += M2CP_THREADS) {
    uint32_t o = 0;
    for (int q = 1; q < m; ++q) o += G::vol(q);
    soff[m] = o;
    svol[m] = G::vol(m);
  }
  if (threadIdx.x == 0) {
    ptx::mbar_init(&full[0], 1);
    ptx::mbar_init(&full[1], 1);
    done[0] = done[1] = 0;
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (hw == 0 && nmine) issue(0, half);
  uint32_t bp[S];  // B^0 .. B^(S-1)
  bp[0] = 1;
#pragma unroll
  for (int k = 1; k < S; ++k) bp[k] = bp[k - 1] * B;
  // Block bookkeeping runs one block ahead of the arithmetic: block k + 1's
  // coordinates and offset are requested when block k starts, its canonical
  // list range and this thread's first entry (position, copy range, M value)
  // before block k's reduction, so a block starts with its operands in
  // registers instead of a chain of four dependent global loads.
  uint16_t jn[S];
  uint64_t boffn = 0;
  auto request_block = [&](uint32_t k) {
    const uint64_t blk = block_of(k);
#pragma unroll
    for (int q = 0; q < S; ++q) jn[q] = LS.index[blk * S + q];
    boffn = LS.offset[blk];
  };
  uint32_t cbase_n = 0, cnt_n = 0;  // canonical list of the requested block
  uint32_t npos = 0, nc0 = 0, nc1 = 0;
  double nm = 0.0;
  auto request_first = [&]() {
    uint32_t pat = 0;
#pragma unroll
    for (int q = 1; q < S; ++q) pat |= static_cast<uint32_t>(jn[q] == jn[q - 1]) << (q - 1);
    cbase_n = P.canon_off[pat];
    cnt_n = P.canon_off[pat + 1] - cbase_n;
    if (ht < cnt_n) {
      npos = __ldg(P.canon + cbase_n + ht);
      nc0 = __ldg(P.cstart + cbase_n + ht);
      nc1 = __ldg(P.cstart + cbase_n + ht + 1);
      nm = P.m[boffn + npos];
    }
  };
  if (nmine) {
    request_block(0);
    request_first();
  }
  for (uint32_t k = 0; k < nmine; ++k) {
    const int buf = half;
    const uint64_t blk = block_of(k);
    const uint64_t boff = boffn;
    const uint32_t cbase = cbase_n, cnt = cnt_n;
    if (k + 1 < nmine) request_block(k + 1);
    const double* sb = sfac + buf * STAGE;
    // software pipeline: the next entry's position, M value and copy range
    // are loaded before this entry's partition sum
    uint32_t i = ht;
    ptx::mbar_wait(&full[buf], k & 1u);
    double part = 0.0;
    for (; i < cnt; i += HT) {
      const uint32_t pos = npos, c0 = nc0, c1 = nc1;
      const double mv = nm;
      // this entry's first copy targets too: the stores after the partition
      // sum then find their addresses in registers (a dependent global load
      // there idled the whole CTA, whose warps reach it together)
      constexpr uint32_t NPRE = 3;
      uint32_t dpre[NPRE];
#pragma unroll
      for (uint32_t q = 0; q < NPRE; ++q) dpre[q] = c0 + q < c1 ? __ldg(P.cdst + c0 + q) : 0u;
      const uint32_t in = i + HT;
      if (in < cnt) {
        npos = __ldg(P.canon + cbase + in);
        nc0 = __ldg(P.cstart + cbase + in);
        nc1 = __ldg(P.cstart + cbase + in + 1);
        nm = P.m[boff + npos];
      }
      int o[S];
      uint32_t r = pos;
#pragma unroll
      for (int q = S - 1; q >= 0; --q) {
        o[q] = static_cast<int>(r % B);
        r /= B;
      }
      double f[NM];
#pragma unroll
      for (int m = 1; m < NM; ++m) {
        uint32_t a = 0;
        int after = 0;
#pragma unroll
        for (int q = S - 1; q >= 0; --q)
          if (m >> q & 1) a += static_cast<uint32_t>(o[q]) * bp[after++];
        f[m] = sb[G::off(m) + a];
      }
      const double v = __dsub_rn(mv, partition_correction<S>(f));
      P.c[boff + pos] = v;
      const bool fix = P.mfix != nullptr;  // the update's symmetric copies of M_6 too (deferred by run_moments)
#pragma unroll
      for (uint32_t q = 0; q < NPRE; ++q)
        if (c0 + q < c1) {
          P.c[boff + dpre[q]] = v;
          if (fix) P.mfix[boff + dpre[q]] = mv;
        }
      for (uint32_t q = c0 + NPRE; q < c1; ++q) {
        const uint32_t dst = __ldg(P.cdst + q);
        P.c[boff + dst] = v;
        if (fix) P.mfix[boff + dst] = mv;
      }
      part = __fma_rn(static_cast<double>(1u + c1 - c0), __dmul_rn(v, v), part);
    }
    if (k + 1 < nmine) request_first();  // lands under the reduction and the next buffer's wait
    for (int s = 16; s > 0; s >>= 1) part = __dadd_rn(part, __shfl_down_sync(0xffffffffu, part, s));
    __syncwarp();  // every lane's reads of the buffer precede lane 0's release below
    uint32_t last = 0;
    if (lane == 0) {
      red[buf][hw] = part;
      __threadfence_block();
      last = atomicAdd(&done[buf], 1u) == HW - 1;
    }
    if (__shfl_sync(0xffffffffu, last, 0)) {  // the last warp of this block
      __threadfence_block();
      if (lane == 0) {
        double s = 0.0;
        for (int w = 0; w < HW; ++w) s = __dadd_rn(s, red[buf][w]);
        P.partial[blk - P.blk0] = s;
        *reinterpret_cast<volatile uint32_t*>(&done[buf]) = 0;
      }
      if (k + 1 < nmine) {
        ptx::fence_proxy_async();  // every warp's generic reads of the buffer before the async-proxy refill
        issue(k + 1, buf);
      }
    }
  }
}

// Write one canonical element of order S to every stored copy in its block
// (distinct permutations of the in-block offsets within runs of equal
// block coordinates): an update applies fma(c, delta, M) to each copy's own
// value (moments.cpp:294-299), an assignment stores the value.
template <int S>
__device__ void write_copies(double* m, const LowerElem& E, int n, int b, bool update, double c, double v) {
  int j[S], o[S], e[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    j[k] = E.idx[k] / b;
    o[k] = E.idx[k] - j[k] * b;
    e[k] = ext_of(j[k], n, b);
  }
  bool runs = false;
#pragma unroll
  for (int k = 1; k < S; ++k) runs |= j[k] == j[k - 1];
  for (;;) {
    uint32_t off = 0;
#pragma unroll
    for (int k = 0; k < S; ++k) off = off * static_cast<uint32_t>(e[k]) + static_cast<uint32_t>(o[k]);
    double* p = m + E.blk_off + off;
    *p = update ? __fma_rn(c, v, *p) : v;
    if (!runs) break;
    // next distinct permutation within runs (odometer over runs, from the last)
    int k = S - 1;
    bool advanced = false;
    while (k >= 0 && !advanced) {
      int s0 = k;
      while (s0 > 0 && j[s0 - 1] == j[k]) --s0;  // run [s0, k]
      // std::next_permutation on o[s0..k]
      int i = k - 1;
      while (i >= s0 && o[i] >= o[i + 1]) --i;
      if (i >= s0) {
        int t = k;
        while (o[t] <= o[i]) --t;
        int tmp = o[i];
        o[i] = o[t];
        o[t] = tmp;
        for (int l = i + 1, r = k; l < r; ++l, --r) {
          tmp = o[l];
          o[l] = o[r];
          o[r] = tmp;
        }
        advanced = true;
      } else {
        for (int l = s0, r = k; l < r; ++l, --r) {
          const int tmp = o[l];
          o[l] = o[r];
          o[r] = tmp;
        }
        k = s0 - 1;
      }
    }
    if (!advanced) break;
  }
}

// rows in flight per thread (register double buffer)
template <int S>
constexpr int low_unroll() { return S <= 2 ? 16 : S == 3 ? 8 : 4; }

template <int S, int LOW_UNROLL = low_unroll<S>()>
__device__ __forceinline__ void low_load(const RowSource& src, uint32_t k0, uint32_t K, int n, const int (&idx)[S],
                                         double (&v)[LOW_UNROLL][S]) {
#pragma unroll
  for (int u = 0; u < LOW_UNROLL; ++u) {
    const uint32_t k = min(k0 + u, K - 1);
    const double* row = k < src.len0 ? src.seg0 + static_cast<size_t>(k) * n
                                     : src.seg1 + static_cast<size_t>(k - src.len0) * n;
#pragma unroll
    for (int t = 0; t < S; ++t) v[u][t] = __ldg(row + idx[t]);
  }
}

template <int S>
__global__ void __launch_bounds__(128) moment_lower_kernel(const LowerParams P) {
  constexpr int LOW_UNROLL = low_unroll<S>();
  const uint64_t el = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const bool live = el < P.count;
  const LowerElem E = P.elems[live ? el : 0];
  const int n = P.n;
  int idx[S];
#pragma unroll
  for (int k = 0; k < S; ++k) idx[k] = E.idx[k];
  double res[2] = {0.0, 0.0};
  for (int pass = 0; pass < P.npass; ++pass) {
    const RowSource src = P.src[pass];
    const uint32_t K = src.len0 + src.len1;
    double acc = 0.0;
    // rows in order; the next LOW_UNROLL rows are loaded while the current
    // ones are folded (plain product, then add: moments.cpp:55-57)
    double cur[LOW_UNROLL][S], nxt[LOW_UNROLL][S];
    low_load<S>(src, 0, K, n, idx, cur);
    for (uint32_t k0 = 0; k0 < K; k0 += LOW_UNROLL) {
      if (k0 + LOW_UNROLL < K) low_load<S>(src, k0 + LOW_UNROLL, K, n, idx, nxt);
#pragma unroll
      for (int u = 0; u < LOW_UNROLL; ++u) {
        double v = cur[u][0];
#pragma unroll
        for (int t = 1; t < S; ++t) v = __dmul_rn(v, cur[u][t]);
        if (k0 + u < K) acc = __dadd_rn(acc, v);
      }
#pragma unroll
      for (int u = 0; u < LOW_UNROLL; ++u)
#pragma unroll
        for (int t = 0; t < S; ++t) cur[u][t] = nxt[u][t];
    }
    res[pass] = __dmul_rn(acc, P.inv);
  }
  if (!live) return;
  const bool update = P.npass == 2;
  write_copies<S>(P.m, E, n, P.b, update, P.c, update ? __dsub_rn(res[0], res[1]) : res[0]);
}

// Orders 1..ST (ST = d-2) of a window update or assignment, with the data
// rows staged in shared memory (32-row chunks, cp.async, double buffered).
// A thread owns up to W order-ST elements (pi, t0 + w) sharing the prefix
// product P = x[pi_1] ... x[pi_{ST-1}] (left to right, moments.cpp:55,71),
// adds round(P x[t0 + w]) in row order (moments.cpp:44) and, when its pi
// represents them, the depth-s prefix products (the order-s tuples
// (pi_1..pi_s), s < ST) -- so each element is the reference's plain
// row-ordered sum of rounded products, times 1/rows.
constexpr int LOW2_KC = 32;
constexpr int LOW2_THREADS = 128;

template <int ST, int W>
__global__ void __launch_bounds__(LOW2_THREADS) moment_lower2_kernel(const Lower2Params P) {
  extern __shared__ double xs[];  // 2 x LOW2_KC x n
  constexpr int NP = ST - 1;      // prefix length
  constexpr int NR = NP > 0 ? NP : 1;
  const int n = P.n;
  const uint32_t tid = blockIdx.x * LOW2_THREADS + threadIdx.x;
  const bool live = tid < P.nthreads;
  const LowerThread T = P.threads[live ? tid : 0];
  int pidx[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) pidx[k] = NP > 0 ? T.pidx[k] : 0;
  int col[W];
#pragma unroll
  for (int w = 0; w < W; ++w) col[w] = min(static_cast<int>(T.t0) + w, n - 1);
  bool rep[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) rep[k] = NP > 0 && T.rep[k] != 0xffffffffu;
  double res[2][W + NR];
  const uint32_t K = P.K;
  const uint32_t nchunks = (K + LOW2_KC - 1) / LOW2_KC;
  for (int pass = 0; pass < P.npass; ++pass) {
    const RowSource src = P.src[pass];
    auto stage = [&](uint32_t ch, int buf) {
      const uint32_t k0 = ch * LOW2_KC;
      const uint32_t kc = min(static_cast<uint32_t>(LOW2_KC), K - k0);
      double* dst = xs + static_cast<size_t>(buf) * LOW2_KC * n;
      for (uint32_t r = 0; r < kc; ++r) {
        const uint32_t k = k0 + r;
        const double* row = k < src.len0 ? src.seg0 + static_cast<size_t>(k) * n
                                         : src.seg1 + static_cast<size_t>(k - src.len0) * n;
        for (int cI = threadIdx.x; cI < n; cI += LOW2_THREADS) cp_async8(dst + r * n + cI, row + cI);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[W + NR];
#pragma unroll
    for (int w = 0; w < W + NR; ++w) acc[w] = 0.0;
    stage(0, 0);
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nchunks) {
        stage(ch + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const double* xb = xs + static_cast<size_t>(buf) * LOW2_KC * n;
      const uint32_t kc = min(static_cast<uint32_t>(LOW2_KC), K - ch * LOW2_KC);
      if (kc == LOW2_KC) {
#pragma unroll 4
        for (uint32_t r = 0; r < LOW2_KC; ++r) {
          const double* x = xb + r * n;
          double pv = 1.0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            pv = k == 0 ? x[pidx[0]] : __dmul_rn(pv, x[pidx[k]]);
            if (rep[k]) acc[W + k] = __dadd_rn(acc[W + k], pv);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] = __dadd_rn(acc[w], NP > 0 ? __dmul_rn(pv, x[col[w]]) : x[col[w]]);
        }
      } else {
        for (uint32_t r = 0; r < kc; ++r) {
          const double* x = xb + r * n;
          double pv = 1.0;
#pragma unroll
          for (int k = 0; k < NP; ++k) {
            pv = k == 0 ? x[pidx[0]] : __dmul_rn(pv, x[pidx[k]]);
            if (rep[k]) acc[W + k] = __dadd_rn(acc[W + k], pv);
          }
#pragma unroll
          for (int w = 0; w < W; ++w) acc[w] = __dadd_rn(acc[w], NP > 0 ? __dmul_rn(pv, x[col[w]]) : x[col[w]]);
        }
      }
      __syncthreads();  // the buffer is refilled next iteration
    }
#pragma unroll
    for (int w = 0; w < W + NR; ++w) res[pass][w] = __dmul_rn(acc[w], P.inv);
  }
  if (!live) return;
  const bool update = P.npass == 2;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    if (w >= T.cnt) break;
    const double v = update ? __dsub_rn(res[0][w], res[1][w]) : res[0][w];
    write_copies<ST>(P.m[ST - 1], P.elems[ST - 1][T.e0 + w], n, P.b, update, P.c, v);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    if (!rep[k]) continue;
    const double v = update ? __dsub_rn(res[0][W + k], res[1][W + k]) : res[0][W + k];
    switch (k) {  // depth k + 1
      case 0: write_copies<1>(P.m[0], P.elems[0][T.rep[0]], n, P.b, update, P.c, v); break;
      case 1: write_copies<(ST > 2 ? 2 : 1)>(P.m[1], P.elems[1][T.rep[1]], n, P.b, update, P.c, v); break;
      case 2: write_copies<(ST > 3 ? 3 : 1)>(P.m[2], P.elems[2][T.rep[2]], n, P.b, update, P.c, v); break;
      default: break;
    }
  }
}

}  // namespace

size_t moms2cums_stage_bytes(int S, int n, int b) {
  // upper bound: all sub-blocks full (b^|m| doubles per subset)
  size_t tot = 0;
  for (int m = 1; m < (1 << S) - 1; ++m) {
    size_t v = 1;
    for (int k = 0; k < S; ++k)
      if (m >> k & 1) v *= static_cast<size_t>(b < n ? b : n);
    tot += v;
  }
  return tot * sizeof(double);
}

namespace {
constexpr size_t kM2cInblkLimit = 64 * 1024;  // staged sub-blocks + one block: >= 3 CTAs per SM
size_t m2c_block_vol(int S, int n, int b) {
  size_t vol = 1;
  for (int k = 0; k < S; ++k) vol *= static_cast<size_t>(b < n ? b : n);
  return vol;
}
}  // namespace

bool m2c_fuse_ok(int S, int n, int b) {
  if (S < 2 || S > 6 || n % b != 0) return false;  // every block full
  if ((S == 6 || S == 5) && b == 4) return true;  // moms2cums_persist writes M's copies beside C's
  const size_t sm0 = moms2cums_stage_bytes(S, n, b);
  const size_t vol = m2c_block_vol(S, n, b);
  return sm0 <= 160 * 1024 && vol <= (1u << 20) && sm0 + vol * sizeof(double) <= kM2cInblkLimit;
}

// The persistent kernel's case: order 6, every block full (n a multiple of
// b = 4), the direct canonical-list path (no in-block pass, no deferred M
// mirror) -- two buffers of the 62 staged sub-blocks (2 x 92 KB) per SM.
bool m2c_persist_ok(int S, const M2CParams& p) {
  return (S == 6 || S == 5) && p.b == 4 && p.n % 4 == 0 && p.canon && p.cstart &&
         2 * M2cStage<6, 4>::total() * sizeof(double) <= 200 * 1024;
}

template <int S>
void launch_m2c_persist(const M2CParams& p, uint64_t nblocks, cudaStream_t st) {
  static int sms = 0;
  if (!sms) CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t smem = 2 * M2cStage<S, 4>::total() * sizeof(double);
  ensure_smem(moms2cums_persist<S, 4>, smem);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(nblocks, static_cast<uint64_t>(sms)));
  moms2cums_persist<S, 4><<<grid, M2CP_THREADS, smem, st>>>(p, static_cast<uint32_t>(nblocks));
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

bool launch_moms2cums_v2(int S, const M2CParams& p, uint64_t nblocks, cudaStream_t st) {
  if (nblocks == 0) return false;
  // (order 5 only with thousands of blocks: with few, the in-block pass and its exact norm partials win)
  if (m2c_persist_ok(S, p) && (S == 6 || nblocks > 3000)) {
    if (S == 6) launch_m2c_persist<6>(p, nblocks, st);
    else launch_m2c_persist<5>(p, nblocks, st);
    return false;
  }
  const unsigned g = static_cast<unsigned>(nblocks);
  const size_t sm0 = moms2cums_stage_bytes(S, p.n, p.b);
  const bool staged = sm0 <= 160 * 1024;
  // one full block of C_S beside the staged sub-blocks, when it fits
  const size_t vol = m2c_block_vol(S, p.n, p.b);
  M2CParams q = p;
  size_t sm = sm0;
  if (staged && q.mlist && sm0 + vol * sizeof(double) <= kM2cInblkLimit) {
    q.cblk = static_cast<uint32_t>(sm0 / sizeof(double));
    q.inblk = true;
    sm = sm0 + vol * sizeof(double);
  } else {
    q.inblk = false;
    if (q.mfix) fail(CSB_ERUNTIME, "moms2cums: deferred mirror without an in-block pass");
  }
  // every block full and assembled in shared memory: its exact norm partial
  // comes out of the same pass (else finalize computes them)
  const bool exact = q.inblk && q.canon && p.n % p.b == 0 && p.fold_width > 0;
  if (!exact) q.fold_width = 0;
  const int bb = p.b < p.n ? p.b : p.n;
  // big blocks outside shared memory: one wide CTA per SM (orders <= 4)
  const unsigned threads = S <= 4 && staged && !q.inblk && vol >= 16384 ? 1024u : 256u;
  switch (S) {
#define CSB_M2C_B(SS, BB)                                                                                  \
  ensure_smem(moms2cums_v2<SS, true, BB>, sm);                                                             \
  moms2cums_v2<SS, true, BB><<<g, threads, sm, st>>>(q);
#define CSB_M2C(SS)                                                                                         \
  case SS:                                                                                                  \
    if (staged) {                                                                                           \
      if (bb == 4) {                                                                                        \
        CSB_M2C_B(SS, 4)                                                                                    \
      } else if (bb == 8) {                                                                                 \
        CSB_M2C_B(SS, 8)                                                                                    \
      } else if (bb == 16) {                                                                                \
        CSB_M2C_B(SS, 16)                                                                                   \
      } else {                                                                                              \
        CSB_M2C_B(SS, 0)                                                                                    \
      }                                                                                                     \
    } else if (bb == 8 && SS >= 5) {                                                                        \
      moms2cums_v2<SS, false, 8><<<g, 256, 0, st>>>(q);                                                     \
    } else {                                                                                                \
      moms2cums_v2<SS, false, 0><<<g, 256, 0, st>>>(q);                                                     \
    }                                                                                                       \
    break;
    CSB_M2C(2) CSB_M2C(3) CSB_M2C(4) CSB_M2C(5) CSB_M2C(6)
#undef CSB_M2C
#undef CSB_M2C_B
    default: fail(CSB_EINVAL, "moms2cums: device path supports orders <= 6");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
  return exact;
}

// The same work with the rows read through L1 instead of staged: a lean
// kernel (<= 64 registers, no shared memory) that runs beside the DMMA
// top-pair kernel on a side stream, in the registers and issue slots the
// top kernel leaves free.  One element per thread (W = 1 thread table).
template <int ST>
__global__ void __launch_bounds__(LOW2_THREADS, 8) moment_lower_side_kernel(const Lower2Params P) {
  constexpr int NP = ST - 1;
  constexpr int NR = NP > 0 ? NP : 1;
  constexpr int U = 4;  // rows in flight
  const int n = P.n;
  const uint32_t tid = blockIdx.x * LOW2_THREADS + threadIdx.x;
  const bool live = tid < P.nthreads;
  const LowerThread T = P.threads[live ? tid : 0];
  int pidx[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) pidx[k] = NP > 0 ? T.pidx[k] : 0;
  const int col = T.t0;
  bool rep[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) rep[k] = NP > 0 && T.rep[k] != 0xffffffffu;
  double res[2][1 + NR];
  const uint32_t K = P.K;
  for (int pass = 0; pass < P.npass; ++pass) {
    const RowSource src = P.src[pass];
    double acc[1 + NR];
#pragma unroll
    for (int w = 0; w < 1 + NR; ++w) acc[w] = 0.0;
    double cur[U][NR + 1];
    auto load = [&](uint32_t k0, double (&v)[U][NR + 1]) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = min(k0 + u, K - 1);
        const double* row = k < src.len0 ? src.seg0 + static_cast<size_t>(k) * n
                                         : src.seg1 + static_cast<size_t>(k - src.len0) * n;
#pragma unroll
        for (int t = 0; t < NP; ++t) v[u][t] = __ldg(row + pidx[t]);
        v[u][NR] = __ldg(row + col);
      }
    };
    load(0, cur);
    for (uint32_t k0 = 0; k0 < K; k0 += U) {
      double nxt[U][NR + 1];
      if (k0 + U < K) load(k0 + U, nxt);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (k0 + u >= K) break;
        double pv = 1.0;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
          pv = k == 0 ? cur[u][0] : __dmul_rn(pv, cur[u][k]);
          if (rep[k]) acc[1 + k] = __dadd_rn(acc[1 + k], pv);
        }
        acc[0] = __dadd_rn(acc[0], NP > 0 ? __dmul_rn(pv, cur[u][NR]) : cur[u][NR]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t <= NR; ++t) cur[u][t] = nxt[u][t];
    }
#pragma unroll
    for (int w = 0; w < 1 + NR; ++w) res[pass][w] = __dmul_rn(acc[w], P.inv);
  }
  if (!live) return;
  const bool update = P.npass == 2;
  {
    const double v = update ? __dsub_rn(res[0][0], res[1][0]) : res[0][0];
    write_copies<ST>(P.m[ST - 1], P.elems[ST - 1][T.e0], n, P.b, update, P.c, v);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    if (!rep[k]) continue;
    const double v = update ? __dsub_rn(res[0][1 + k], res[1][1 + k]) : res[0][1 + k];
    switch (k) {
      case 0: write_copies<1>(P.m[0], P.elems[0][T.rep[0]], n, P.b, update, P.c, v); break;
      case 1: write_copies<(ST > 2 ? 2 : 1)>(P.m[1], P.elems[1][T.rep[1]], n, P.b, update, P.c, v); break;
      case 2: write_copies<(ST > 3 ? 3 : 1)>(P.m[2], P.elems[2][T.rep[2]], n, P.b, update, P.c, v); break;
      default: break;
    }
  }
}

// Orders <= d-2 when they are few (cfg1: 4,656 + 96 elements): one thread
// per order-ST element (and the lower-order tuples it represents), the
// pass's rows streamed through a shared-memory ring by TMA bulk copies
// (one producer warp, full/empty mbarriers), so each thread's row-ordered
// chain of plain adds (moments.cpp:44) runs at the DADD latency instead of
// waiting on L2 for every few rows.
constexpr int LOWT_THREADS = 256;
constexpr int LOWT_MAXST = 8;

// W > 1: a thread owns the W consecutive order-ST elements (pi, t0 .. t0 +
// W - 1) of one prefix, so the prefix loads and products are shared (the
// per-element chain is unchanged: acc += round(P x[t]), row order).
template <int ST, int W>
__global__ void __launch_bounds__(LOWT_THREADS + 32) moment_lower_tma_kernel(const Lower2Params P, int stages, int kr) {
  extern __shared__ __align__(128) double xs[];  // stages x kr x n
  __shared__ __align__(8) uint64_t full[LOWT_MAXST], empty[LOWT_MAXST];
  constexpr int NP = ST - 1;
  constexpr int NR = NP > 0 ? NP : 1;
  const int n = P.n;
  const uint32_t K = P.K;
  const uint32_t cpp = (K + kr - 1) / kr;
  const uint32_t chunks = cpp * P.npass;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(empty + s, LOWT_THREADS / 32);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= LOWT_THREADS) {  // producer warp: one lane issues the copies
    if (threadIdx.x != LOWT_THREADS) return;
    const uint32_t rb = static_cast<uint32_t>(n) * 8u;
    for (uint32_t c = 0; c < chunks; ++c) {
      const uint32_t st = c % stages;
      if (c >= static_cast<uint32_t>(stages)) ptx::mbar_wait(empty + st, ((c / stages) - 1) & 1u);
      const uint32_t pass = c >= cpp ? 1u : 0u;
      const RowSource src = P.src[pass];
      const uint32_t a0 = (c - pass * cpp) * kr;
      const uint32_t kc = min(static_cast<uint32_t>(kr), K - a0);
      double* dst = xs + static_cast<size_t>(st) * kr * n;
      ptx::mbar_expect_tx(full + st, kc * rb);
      auto rowp = [&](uint32_t k) {
        return k < src.len0 ? src.seg0 + static_cast<size_t>(k) * n : src.seg1 + static_cast<size_t>(k - src.len0) * n;
      };
      if (a0 + kc <= src.len0 || a0 >= src.len0) {
        ptx::bulk_g2s(dst, rowp(a0), kc * rb, full + st);
      } else {  // across the ring's wrap
        const uint32_t k1 = src.len0 - a0;
        ptx::bulk_g2s(dst, rowp(a0), k1 * rb, full + st);
        ptx::bulk_g2s(dst + static_cast<size_t>(k1) * n, src.seg1, (kc - k1) * rb, full + st);
      }
    }
    return;
  }
  const uint32_t tid = blockIdx.x * LOWT_THREADS + threadIdx.x;
  const bool live = tid < P.nthreads;
  const LowerThread T = P.threads[live ? tid : 0];
  int pidx[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) pidx[k] = NP > 0 ? T.pidx[k] : 0;
  const int col = T.t0;
  const int cnt = live ? T.cnt : 0;
  const int stride = T.pad ? static_cast<int>(T.pad) : 1;  // strided tables: elements t0 + k * stride
  int cw[W];  // element columns, clamped to the row (entries w >= cnt are dropped)
#pragma unroll
  for (int w = 0; w < W; ++w) cw[w] = min(col + w * stride, n - 1);
  bool rep[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) rep[k] = NP > 0 && T.rep[k] != 0xffffffffu;
  constexpr int NA = W + NR;  // acc[0 .. W): the order-ST elements; acc[W + k]: prefix depth k + 1
  double res[2][NA];
  double acc[NA];
#pragma unroll
  for (int w = 0; w < NA; ++w) acc[w] = 0.0;
  for (uint32_t c = 0; c < chunks; ++c) {
    const uint32_t st = c % stages;
    ptx::mbar_wait(full + st, (c / stages) & 1u);
    const uint32_t pass = c >= cpp ? 1u : 0u;
    const uint32_t kc = min(static_cast<uint32_t>(kr), K - (c - pass * cpp) * kr);
    const double* xb = xs + static_cast<size_t>(st) * kr * n;
#pragma unroll 8
    for (uint32_t r = 0; r < kc; ++r) {
      const double* x = xb + r * n;
      double pv = 1.0;
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        pv = k == 0 ? x[pidx[0]] : __dmul_rn(pv, x[pidx[k]]);
        if (rep[k]) acc[W + k] = __dadd_rn(acc[W + k], pv);
      }
#pragma unroll
      for (int w = 0; w < W; ++w) acc[w] = __dadd_rn(acc[w], NP > 0 ? __dmul_rn(pv, x[cw[w]]) : x[cw[w]]);
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(empty + st);
    if (c + 1 == cpp || c + 1 == chunks) {  // end of a pass
#pragma unroll
      for (int w = 0; w < NA; ++w) {
        res[pass][w] = __dmul_rn(acc[w], P.inv);
        acc[w] = 0.0;
      }
    }
  }
  if (!live) return;
  const bool update = P.npass == 2;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    if (w >= cnt) break;
    const double v = update ? __dsub_rn(res[0][w], res[1][w]) : res[0][w];
    write_copies<ST>(P.m[ST - 1], P.elems[ST - 1][T.e0 + w * stride], n, P.b, update, P.c, v);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    if (!rep[k]) continue;
    const double v = update ? __dsub_rn(res[0][W + k], res[1][W + k]) : res[0][W + k];
    switch (k) {
      case 0: write_copies<1>(P.m[0], P.elems[0][T.rep[0]], n, P.b, update, P.c, v); break;
      case 1: write_copies<(ST > 2 ? 2 : 1)>(P.m[1], P.elems[1][T.rep[1]], n, P.b, update, P.c, v); break;
      case 2: write_copies<(ST > 3 ? 3 : 1)>(P.m[2], P.elems[2][T.rep[2]], n, P.b, update, P.c, v); break;
      default: break;
    }
  }
}

bool lower_tma_supported(const Lower2Params& p) {
  return p.n % 2 == 0 && p.n <= 4096 && rows_aligned16(p.src, p.npass);
}

void launch_moment_lower_tma(int ST, int W, const Lower2Params& p, cudaStream_t st) {
  if (!p.nthreads) return;
  const unsigned g = (p.nthreads + LOWT_THREADS - 1) / LOWT_THREADS;
  const int kr = 32;
  const size_t stage_bytes = static_cast<size_t>(kr) * p.n * sizeof(double);
  // deep ring (up to 200 KB) unless the grid needs more than one CTA per SM
  // to fit in one wave: then the stages that many CTAs per SM leave room for
  static int sms = 0;
  if (!sms) CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t per_sm = std::max<size_t>(1, (g + sms - 1) / static_cast<unsigned>(sms));
  const size_t budget = std::min<size_t>(200u << 10, (220u << 10) / std::min<size_t>(per_sm, 4));
  int stages = static_cast<int>(std::min<size_t>(LOWT_MAXST, budget / stage_bytes));
  if (stages < 2) fail(CSB_EINVAL, "moment_lower_tma: rows too wide");
  const size_t sm = stages * stage_bytes;
  switch (ST * 8 + W) {
#define CSB_LOWT(SS, WW)                                                                                      \
  case SS * 8 + WW:                                                                                           \
    ensure_smem(moment_lower_tma_kernel<SS, WW>, sm);                                                         \
    moment_lower_tma_kernel<SS, WW><<<g, LOWT_THREADS + 32, sm, st>>>(p, stages, kr);                         \
    break;
    CSB_LOWT(1, 1) CSB_LOWT(2, 1) CSB_LOWT(3, 1) CSB_LOWT(4, 1) CSB_LOWT(2, 4) CSB_LOWT(3, 4) CSB_LOWT(4, 4)
#undef CSB_LOWT
    default: fail(CSB_EINVAL, "moment_lower_tma: order or width out of range");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

void launch_moment_lower_side(int ST, const Lower2Params& p, cudaStream_t st) {
  if (!p.nthreads) return;
  const unsigned g = (p.nthreads + LOW2_THREADS - 1) / LOW2_THREADS;
  switch (ST) {
    case 1: moment_lower_side_kernel<1><<<g, LOW2_THREADS, 0, st>>>(p); break;
    case 2: moment_lower_side_kernel<2><<<g, LOW2_THREADS, 0, st>>>(p); break;
    case 3: moment_lower_side_kernel<3><<<g, LOW2_THREADS, 0, st>>>(p); break;
    case 4: moment_lower_side_kernel<4><<<g, LOW2_THREADS, 0, st>>>(p); break;
    default: fail(CSB_EINVAL, "moment_lower_side: order out of range");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

void launch_moment_lower2(int ST, int W, const Lower2Params& p, cudaStream_t st) {
  if (!p.nthreads) return;
  const unsigned g = (p.nthreads + LOW2_THREADS - 1) / LOW2_THREADS;
  const size_t sm = 2ull * LOW2_KC * p.n * sizeof(double);
  switch (ST * 8 + W) {
#define CSB_LOW2(SS, WW)                                                                                  \
  case SS * 8 + WW:                                                                                       \
    ensure_smem(moment_lower2_kernel<SS, WW>, sm);                                                      \
    moment_lower2_kernel<SS, WW><<<g, LOW2_THREADS, sm, st>>>(p);                                         \
    break;
    CSB_LOW2(1, 1) CSB_LOW2(1, 4) CSB_LOW2(2, 1) CSB_LOW2(2, 4) CSB_LOW2(3, 1) CSB_LOW2(3, 4) CSB_LOW2(4, 1)
    CSB_LOW2(4, 4)
#undef CSB_LOW2
    default: fail(CSB_EINVAL, "moment_lower2: order out of range");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

void launch_moment_lower(int S, const LowerParams& p, cudaStream_t st) {
  if (!p.count) return;
  const unsigned g = static_cast<unsigned>((p.count + 127) / 128);
  switch (S) {
#define CSB_LOW(SS) \
  case SS: moment_lower_kernel<SS><<<g, 128, 0, st>>>(p); break;
    CSB_LOW(1) CSB_LOW(2) CSB_LOW(3) CSB_LOW(4) CSB_LOW(5) CSB_LOW(6)
#undef CSB_LOW
    default: fail(CSB_EINVAL, "moment_lower: order out of range");
  }
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
