// sm_100a kernels of the sliding-window moment/cumulant hot path.
//
// Arithmetic follows the reference's evaluation order exactly
// so results are bit-identical to it:
//   * moment products: left-to-right chain starting at x[i_1]
//     (moments.cpp:55,71);
//   * top order d: acc = fma(A, x[i_d], acc) in row order (moments.cpp:47);
//   * every lower order: acc = acc + round(product) (moments.cpp:44,57);
//   * means: acc * (1.0 / rows) (moments.cpp:148-150);
//   * update: M = fma(p/T, a - b, M) for every stored copy (moments.cpp:297);
//   * cumulants: partition sum in RGS order, no FMA (cumulants.cpp:64-82).
// The file is compiled with -fmad=false; every intended FMA is an explicit
// __fma_rn and every unfused product/sum an explicit __dmul_rn/__dadd_rn.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.cuh"
#include "partitions_gen.cuh"

namespace csb {

namespace {

constexpr int KC = 8;        // data rows per smem chunk
constexpr int MAXROWS = 1024;  // prefix rows per tile
constexpr int T = kMomThreads;

__device__ __forceinline__ const double* row_ptr(const RowSource& s, uint32_t k, int n) {
  return k < s.len0 ? s.seg0 + static_cast<size_t>(k) * n
                    : s.seg1 + static_cast<size_t>(k - s.len0) * n;
}

__device__ __forceinline__ bool next_perm(int* a, int len) {
  // std::next_permutation on a short int range
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

// Calls f(offset) for every stored copy of a canonical element: all
// distinct permutations of the in-block offsets o within runs of equal
// block coordinate j (symten.cpp:195-220).  o must be sorted within runs.
// Returns the number of copies.
template <class F>
__device__ __forceinline__ int for_each_copy(int S, const int* j, int* o, const int* e,
                                             uint64_t blk_off, F&& f) {
  bool runs = false;
  for (int k = 1; k < S; ++k) runs |= (j[k] == j[k - 1]);
  if (!runs) {
    uint64_t off = 0;
    for (int k = 0; k < S; ++k) off = off * e[k] + o[k];
    f(blk_off + off);
    return 1;
  }
  int rs[kMaxOrder], re[kMaxOrder], nr = 0;
  for (int s = 0; s < S;) {
    int t = s + 1;
    while (t < S && j[t] == j[s]) ++t;
    rs[nr] = s;
    re[nr] = t;
    ++nr;
    s = t;
  }
  int count = 0;
  for (;;) {
    uint64_t off = 0;
    for (int k = 0; k < S; ++k) off = off * e[k] + o[k];
    f(blk_off + off);
    ++count;
    int q = nr - 1;
    while (q >= 0 && !next_perm(o + rs[q], re[q] - rs[q])) --q;
    if (q < 0) break;
  }
  return count;
}

__device__ __forceinline__ int ext_of(int j, int n, int b) { return b < n - j * b ? b : n - j * b; }

// Epilogue of one order-S element: RMW (update) or assign every stored copy.
__device__ __noinline__ void store_top(const MomParams& P, const MomTile& tile, int r, int col,
                                       const uint16_t* id, double a, double v) {
  const int n = P.n, b = P.b, L = P.L;
  if (L > 0 && col < static_cast<int>(id[L - 1])) return;  // below the diagonal: a copy
  const PrefixRow& pr = P.rows[tile.row0 + r];
  const int jd = col / b;
  int jv[kMaxOrder], ov[kMaxOrder], ev[kMaxOrder];
  for (int q = 0; q < L; ++q) {
    jv[q] = id[q] / b;
    ov[q] = id[q] - jv[q] * b;
    ev[q] = ext_of(jv[q], n, b);
  }
  jv[L] = jd;
  ov[L] = col - jd * b;
  ev[L] = ext_of(jd, n, b);
  const uint64_t blk = pr.top_base + static_cast<uint64_t>(pr.vprime) * b * (jd - static_cast<int>(tile.J));
  double* top = P.top;
  if (P.npass == 2) {
    const double delta = __dsub_rn(a, v);
    const double c = P.c;
    for_each_copy(L + 1, jv, ov, ev, blk, [&](uint64_t off) { top[off] = __fma_rn(c, delta, top[off]); });
  } else {
    for_each_copy(L + 1, jv, ov, ev, blk, [&](uint64_t off) { top[off] = v; });
  }
}

// ---------------------------------------------------------------------------
// Moment pair kernel: orders S (GEMM over prefix rows x columns) and S-1
// (row sums of the Khatri-Rao operand) for one tile of prefix rows.
template <bool TOP_FMA>
__global__ void __launch_bounds__(T, 1) moment_pair_kernel(const MomParams P) {
  extern __shared__ __align__(16) double smem[];
  const MomTile tile = P.tiles[blockIdx.x];
  const int n = P.n, b = P.b, L = P.L;
  const int N = static_cast<int>(tile.ncols);
  const int CG = (N + 7) / 8;
  const int nr = static_cast<int>(tile.nrows);
  const int RG = (nr + 7) / 8;
  const int XS = (n + 1) & ~1;
  const int BS = CG * 8;
  const int AS = RG * 8;
  double* xs = smem;
  double* bs = xs + KC * XS;
  double* as = bs + KC * BS;
  double* lowstash = as + KC * AS;
  uint16_t* ridx = reinterpret_cast<uint16_t*>(lowstash + AS);  // AS x 8

  const int t = threadIdx.x;
  const int rg = t / CG, cg = t % CG;
  const bool active = rg < RG;

  for (int e = t; e < AS; e += T) {
    if (e < nr) {
      const PrefixRow& pr = P.rows[tile.row0 + e];
      for (int k = 0; k < 8; ++k) ridx[e * 8 + k] = pr.idx[k];
    } else {
      for (int k = 0; k < 8; ++k) ridx[e * 8 + k] = 0;
    }
  }

  for (int pass = 0; pass < P.npass; ++pass) {
    const RowSource src = P.src[pass];
    double acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
    double lacc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) lacc[i] = 0.0;

    for (uint32_t k0 = 0; k0 < P.K; k0 += KC) {
      const int kc = static_cast<int>(min(static_cast<uint32_t>(KC), P.K - k0));
      __syncthreads();
      for (int e = t; e < KC * XS; e += T) {
        const int k = e / XS, c = e % XS;
        xs[e] = (k < kc && c < n) ? row_ptr(src, k0 + k, n)[c] : 0.0;
      }
      for (int e = t; e < KC * BS; e += T) {
        const int k = e / BS, c = e % BS;
        bs[e] = (k < kc && c < N) ? row_ptr(src, k0 + k, n)[tile.col0 + c] : 0.0;
      }
      __syncthreads();
      if (t < RG) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = 8 * t + i;
          const uint16_t* id = ridx + r * 8;
          for (int k = 0; k < KC; ++k) {
            double a;
            if (r >= nr || k >= kc) {
              a = 0.0;
            } else if (L == 0) {
              a = 1.0;
            } else {
              const double* xr = xs + k * XS;
              a = xr[id[0]];
              for (int q = 1; q < L; ++q) a = __dmul_rn(a, xr[id[q]]);
              lacc[i] = __dadd_rn(lacc[i], a);
            }
            as[k * AS + r] = a;
          }
        }
      }
      __syncthreads();
      if (active) {
        for (int k = 0; k < kc; ++k) {
          double av[8], bv[8];
          const double2* ap = reinterpret_cast<const double2*>(as + k * AS + 8 * rg);
          const double2* bp = reinterpret_cast<const double2*>(bs + k * BS + 8 * cg);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 x = ap[q];
            av[2 * q] = x.x;
            av[2 * q + 1] = x.y;
            const double2 y = bp[q];
            bv[2 * q] = y.x;
            bv[2 * q + 1] = y.y;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (TOP_FMA)
                acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
              else
                acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(av[i], bv[j]));
            }
        }
      }
    }

    const bool final_pass = (pass == P.npass - 1);
    const size_t sbase = static_cast<size_t>(blockIdx.x) * 64 * T;
    if (!final_pass) {
      // stash the incoming means for the fused update epilogue
      if (active) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            P.scratch[sbase + static_cast<size_t>(i * 8 + j) * T + t] = __dmul_rn(acc[i][j], P.inv);
      }
      if (t < RG) {
#pragma unroll
        for (int i = 0; i < 8; ++i) lowstash[8 * t + i] = __dmul_rn(lacc[i], P.inv);
      }
      continue;
    }

    // ---- epilogue: order S ----
    if (active) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 8 * rg + i;
        if (r >= nr) continue;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int cc = 8 * cg + jj;
          if (cc >= N) continue;
          const double v = __dmul_rn(acc[i][jj], P.inv);
          const double a = (P.npass == 2) ? P.scratch[sbase + static_cast<size_t>(i * 8 + jj) * T + t] : 0.0;
          store_top(P, tile, r, static_cast<int>(tile.col0) + cc, ridx + r * 8, a, v);
        }
      }
    }
    // ---- epilogue: order S-1 ----
    if (P.low != nullptr && tile.low && L > 0 && t < RG) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 8 * t + i;
        if (r >= nr) continue;
        const PrefixRow& pr = P.rows[tile.row0 + r];
        const uint16_t* id = ridx + r * 8;
        const double v = __dmul_rn(lacc[i], P.inv);
        double delta = 0.0;
        if (P.npass == 2) delta = __dsub_rn(lowstash[r], v);
        int jv[kMaxOrder], ov[kMaxOrder], ev[kMaxOrder];
        for (int q = 0; q < L; ++q) {
          jv[q] = id[q] / b;
          ov[q] = id[q] - jv[q] * b;
          ev[q] = ext_of(jv[q], n, b);
        }
        const uint64_t blk = pr.low_off - pr.poff;
        double* low = P.low;
        const double cc_ = P.c;
        if (P.npass == 2) {
          for_each_copy(L, jv, ov, ev, blk, [&](uint64_t off) { low[off] = __fma_rn(cc_, delta, low[off]); });
        } else {
          for_each_copy(L, jv, ov, ev, blk, [&](uint64_t off) { low[off] = v; });
        }
      }
    }
  }
}

__global__ void copy_c1_kernel(const double* m1, double* c1, double* partial, LayoutDev lay,
                               uint64_t nblocks) {
  // C_1 = M_1 (cumulants.cpp:139), one CTA per block; the block's sum of
  // squares is reduced exactly as knorm_partials_kernel does (same element
  // order and association), so stream reports and knorm() agree bitwise
  const uint64_t blk = blockIdx.x;
  if (blk >= nblocks) return;
  __shared__ double red[8];
  double s = 0.0;
  for (uint64_t i = lay.offset[blk] + threadIdx.x; i < lay.offset[blk + 1]; i += blockDim.x) {
    const double v = m1[i];
    c1[i] = v;
    s = __fma_rn(v, v, s);
  }
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) a = __dadd_rn(a, red[w]);
    partial[blk] = a;
  }
}

// Per-block sums of |e|^k in the reference's exact order (knorm,
// symten.cpp:257-276): each block's entries folded one by one in storage
// order.  The reference build vectorises the k = 2 fold without
// reassociating it: `width`-wide rounded squares added one by one, then a
// fused multiply-add tail for the last vol mod width entries (width = 4 for
// an AVX2 build, 8 for AVX-512; the oracle documents both).
//
// One warp takes 32 consecutive blocks and lane g runs block g's
// sequential chain, so one add instruction advances 32 chains.  The
// entries arrive by coalesced loads, a 32 x 32 tile per chunk (lane l
// loads entry l of every block's chunk, the next chunk's loads in flight
// while this one is chained), transposed through shared memory: slot
// [e][(g + e) mod 32] holds entry e of block g, so the stores (fixed g)
// and the chain reads (fixed e) both hit distinct banks.
constexpr int KN_CHUNK = 32;  // entries per block and chunk (one per lane)
constexpr int KN_WARPS = 4;   // warps (x 32 blocks) per CTA
__global__ void __launch_bounds__(KN_WARPS * 32) knorm_exact_kernel(const double* __restrict__ t, LayoutDev lay,
                                                                    uint64_t blk0, uint64_t nblk, double k, int width,
                                                                    double* __restrict__ partial) {
  __shared__ double tile[KN_WARPS][KN_CHUNK][32];
  __shared__ uint64_t boff[KN_WARPS][32];
  __shared__ uint32_t bvol[KN_WARPS][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * KN_WARPS + w) * 32 + lane;
  const bool live = i < nblk;
  const uint64_t blk = blk0 + (live ? i : 0);
  const uint64_t off = lay.offset[blk];
  const uint32_t vol = live ? static_cast<uint32_t>(lay.offset[blk + 1] - off) : 0;
  boff[w][lane] = off;
  bvol[w][lane] = vol;
  uint32_t maxvol = vol;
  for (int o = 16; o > 0; o >>= 1) maxvol = max(maxvol, __shfl_xor_sync(0xffffffffu, maxvol, o));
  __syncwarp();
  const uint32_t nchunk = (maxvol + KN_CHUNK - 1) / KN_CHUNK;
  double (*tl)[32] = tile[w];
  // entry `lane` of each block's chunks c and c + 1: two chunks of loads in
  // flight (the tensor was just written, so mostly L2 hits)
  double x[2][32];
  auto load = [&](uint32_t c, int buf) {
    const uint32_t q = c * KN_CHUNK + lane;
#pragma unroll
    for (int g = 0; g < 32; ++g) x[buf][g] = q < bvol[w][g] ? t[boff[w][g] + q] : 0.0;
  };
  const uint32_t nvec = vol & ~static_cast<uint32_t>(width - 1);
  double s = 0.0;
  if (nchunk) load(0, 0);
  if (nchunk > 1) load(1, 1);
  for (uint32_t c = 0; c < nchunk; ++c) {
    if (c & 1) {
#pragma unroll
      for (int g = 0; g < 32; ++g) tl[lane][(g + lane) & 31] = x[1][g];
    } else {
#pragma unroll
      for (int g = 0; g < 32; ++g) tl[lane][(g + lane) & 31] = x[0][g];
    }
    __syncwarp();
    if (c + 2 < nchunk) {  // refill the buffer just stored: in flight during the next two chains
      if (c & 1) load(c + 2, 1);
      else load(c + 2, 0);
    }
    const uint32_t q0 = c * KN_CHUNK;
    const uint32_t e1 = vol > q0 ? min(vol - q0, static_cast<uint32_t>(KN_CHUNK)) : 0;
    auto at = [&](uint32_t e) { return tl[e][(lane + e) & 31]; };
    if (k == 2.0) {
      const uint32_t ev = nvec > q0 ? min(nvec - q0, e1) : 0;  // rounded squares, then the FMA tail
      if (ev == KN_CHUNK) {
        // whole chunk of rounded squares: form all 32 first (independent),
        // so only the adds wait on one another
        double sq[KN_CHUNK];
#pragma unroll
        for (int e = 0; e < KN_CHUNK; ++e) {
          const double y = at(e);
          sq[e] = __dmul_rn(y, y);
        }
#pragma unroll
        for (int e = 0; e < KN_CHUNK; ++e) s = __dadd_rn(s, sq[e]);
      } else {
        uint32_t e = 0;
        for (; e < ev; ++e) {
          const double y = at(e);
          s = __dadd_rn(s, __dmul_rn(y, y));
        }
        for (; e < e1; ++e) {
          const double y = at(e);
          s = __fma_rn(y, y, s);
        }
      }
    } else if (k == 1.0) {
      for (uint32_t e = 0; e < e1; ++e) s = __dadd_rn(s, fabs(at(e)));
    } else {
      for (uint32_t e = 0; e < e1; ++e) s = __dadd_rn(s, pow(fabs(at(e)), k));
    }
    __syncwarp();  // the tile is rewritten by the next chunk
  }
  if (live) partial[blk] = s;
}

// The blocks' partial sums folded in block order, acc = acc + mult * s
// (symten.cpp:268; the product is rounded, the reference build does not
// contract it).  One CTA per order: the threads form the rounded products
// of a slice of blocks in shared memory (coalesced, in parallel), thread 0
// adds them in block order -- the reference's sequence bit for bit, with
// only the adds on the sequential path.  CTA 0 also gathers the diagonals.
constexpr int NF_THREADS = 256;
constexpr int NF_SLICE = 2048;
__global__ void __launch_bounds__(NF_THREADS) norm_finalize_kernel(const NormParams P) {
  __shared__ double prod[2][NF_SLICE];
  const int s = static_cast<int>(blockIdx.x);
  if (P.fold && s < P.norders) {
    const double* __restrict__ mult = P.mult[s];
    const double* __restrict__ part = P.partial[s];
    const uint64_t nb = P.nblocks[s];
    double a = 0.0;
    for (uint64_t base = 0, it = 0; base < nb; base += NF_SLICE, ++it) {
      double* pr = prod[it & 1];  // double buffer: slice it + 1 forms while thread 0 adds slice it
      const uint64_t cnt = nb - base < NF_SLICE ? nb - base : NF_SLICE;
      for (uint64_t i = threadIdx.x; i < cnt; i += NF_THREADS) pr[i] = __dmul_rn(mult[base + i], part[base + i]);
      __syncthreads();
      if (threadIdx.x == 0) {
#pragma unroll 8
        for (uint64_t i = 0; i < cnt; ++i) a = __dadd_rn(a, pr[i]);
      }
    }
    if (threadIdx.x == 0) P.out[s] = a;
  }
  if (s != 0) return;
  for (int q = 0; q < 3; ++q) {
    if (!P.diag_src[q]) continue;
    for (int i = threadIdx.x; i < P.n; i += blockDim.x)
      P.out[P.norders + q * P.n + i] = P.diag_src[q][P.diag_off[q][i]];
  }
}

// Diagonal entries of a sharded tensor: the owner's value, zero elsewhere
// (summed over ranks this reproduces the full diagonal exactly).
__global__ void diag_pick_kernel(const double* c, const uint64_t* off, uint64_t lo, uint64_t hi, int n,
                                 double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = (off[i] >= lo && off[i] < hi) ? c[off[i]] : 0.0;
}

__global__ void combine_kernel(const double* a, const double* b, double w1, double w2, double* out,
                               uint64_t count) {
  // combine (moments.cpp:258-262): z = w1 * z + w2 * b, contracted to
  // fma(w1, z, w2 * b) by the reference build
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = __fma_rn(w1, a[i], __dmul_rn(w2, b[i]));
}

std::atomic<uint64_t> g_launches{0};

}  // namespace

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }  // a replayed graph's kernels

void launch_moment_pair(const MomParams& p, int ntiles, bool top_fma, cudaStream_t st) {
  if (ntiles <= 0) return;
  const int XS = (p.n + 1) & ~1;
  const int BS = ((p.n + 7) / 8) * 8;
  const size_t smem = sizeof(double) * (KC * XS + KC * BS + KC * MAXROWS + MAXROWS) +
                      sizeof(uint16_t) * MAXROWS * 8;
  if (top_fma) {
    ensure_smem(moment_pair_kernel<true>, smem);
    moment_pair_kernel<true><<<ntiles, T, smem, st>>>(p);
  } else {
    ensure_smem(moment_pair_kernel<false>, smem);
    moment_pair_kernel<false><<<ntiles, T, smem, st>>>(p);
  }
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

// out[i] = t[off[i]]: sampled elements of a stored tensor (parity checks
// at full size, dumps of selected entries)
__global__ void gather_kernel(const double* __restrict__ t, const uint64_t* __restrict__ off, uint64_t count,
                              double* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = t[off[i]];
}

void launch_gather(const double* t, const uint64_t* off, uint64_t count, double* out, cudaStream_t st) {
  if (!count) return;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((count + 255) / 256, 4096));
  gather_kernel<<<g, 256, 0, st>>>(t, off, count, out);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_copy_c1(const double* m1, double* c1, double* partial, const LayoutDev& lay,
                    uint64_t nblocks, uint64_t, cudaStream_t st) {
  copy_c1_kernel<<<static_cast<unsigned>(nblocks), 256, 0, st>>>(m1, c1, partial, lay, nblocks);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_norm_finalize(const NormParams& p, cudaStream_t st) {
  norm_finalize_kernel<<<p.fold ? std::max(1, p.norders) : 1, NF_THREADS, 0, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_knorm_exact(const double* t, const LayoutDev& lay, uint64_t blk0, uint64_t nblk, double k, int width,
                        double* partial, cudaStream_t st) {
  if (!nblk) return;
  const unsigned grid = static_cast<unsigned>((nblk + 32 * KN_WARPS - 1) / (32 * KN_WARPS));
  knorm_exact_kernel<<<grid, KN_WARPS * 32, 0, st>>>(t, lay, blk0, nblk, k, width, partial);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_diag_pick(const double* c, const uint64_t* off, uint64_t lo, uint64_t hi, int n, double* out,
                      cudaStream_t st) {
  diag_pick_kernel<<<(n + 255) / 256, 256, 0, st>>>(c, off, lo, hi, n, out);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

void launch_combine(const double* a, const double* b, double w1, double w2, double* out,
                    uint64_t count, cudaStream_t st) {
  if (!count) return;
  combine_kernel<<<592, 256, 0, st>>>(a, b, w1, w2, out, count);
  CSB_CUDA(cudaGetLastError());
  g_launches.fetch_add(1, std::memory_order_relaxed);
}

}  // namespace csb
