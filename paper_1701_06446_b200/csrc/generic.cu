// Any-order kernels: moments of orders above 8 and cumulants of orders 7..16
// (the reference allows tensors up to order 20, symten.hpp:87, and set
// partitions up to s = 16, cumulants.hpp:24).  The specialised kernels
// (DMMA top pair, staged moms2cums, generated partition code) stop at order
// 8 / 6; these run the same arithmetic for any order with one thread per
// stored element and no pyramid or scatter tables: a thread decodes its
// entry, and if the entry is canonical (offsets non-decreasing within runs
// of equal block coordinate, cumulants.cpp:163-168) evaluates the
// reference's own sequence on its sorted index; a second pass copies every
// other entry from its canonical source (cumulants.cpp:172-185; for the
// moments the copies enter an update bit-identical to their source, so
// copying the source's new value equals the reference's RMW of each copy).
//
//  * moments (moments.cpp:32-60,140-150,287-299): q = x[i_1], q = q x[i_k]
//    left to right; the top order chains acc = fma(q_{d-1}, x[i_d], acc)
//    over the rows, every other order acc = acc + q_s; mean = acc (1/rows);
//    update M = fma(p/T, a - b, M).
//  * cumulants (cumulants.cpp:64-82,128-196): C = M - sum over the set
//    partitions with >= 2 parts, in lexicographic order of their restricted
//    growth strings, of the product (starting at 1.0) of C_|P|[i_P] over the
//    parts in order of their smallest member; products then sums, no FMA.
//
// They are not tuned: an order-9+ tensor is small in any dimension that
// fits a GPU, and the partition count (Bell numbers) bounds the cumulants.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.cuh"

namespace csb {

namespace {

constexpr int GEN_THREADS = 128;

__device__ __forceinline__ int gen_ext(int j, int n, int b) { return b < n - j * b ? b : n - j * b; }

// Stored element e of `lay`: its sorted global index, whether it is the
// canonical copy, and the stored offset of that canonical copy (src).
__device__ bool decode_entry(const LayoutDev& lay, uint64_t e, int n, int b, int* idx, uint64_t* src) {
  const int S = lay.order;
  // the block holding e: last r with offset[r] <= e
  uint64_t lo = 0, hi = lay.nblocks;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (lay.offset[mid] <= e) lo = mid;
    else hi = mid;
  }
  uint64_t rem = e - lay.offset[lo];
  const uint16_t* j = lay.index + lo * S;
  for (int k = S - 1; k >= 0; --k) {
    const int ext = gen_ext(j[k], n, b);
    idx[k] = static_cast<int>(rem % ext);  // in-block offsets first
    rem /= ext;
  }
  // blocks are non-decreasing, so only offsets inside runs of equal block
  // coordinate can be out of order: insertion sort within the runs
  bool canonical = true;
  for (int k = 1; k < S; ++k) {
    if (j[k] != j[k - 1]) continue;
    const int v = idx[k];
    int l = k - 1;
    while (l >= 0 && j[l] == j[k] && idx[l] > v) {
      idx[l + 1] = idx[l];
      --l;
      canonical = false;
    }
    idx[l + 1] = v;
  }
  uint64_t off = 0;
  for (int k = 0; k < S; ++k) {
    off = off * static_cast<uint64_t>(gen_ext(j[k], n, b)) + static_cast<uint64_t>(idx[k]);
    idx[k] += j[k] * b;
  }
  *src = lay.offset[lo] + off;
  return canonical;
}

// every non-canonical entry takes its canonical source's value
__global__ void __launch_bounds__(GEN_THREADS) copy_generic_kernel(double* t, LayoutDev lay, uint64_t stored, int n,
                                                                    int b) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(GEN_THREADS) + threadIdx.x; e < stored;
       e += static_cast<uint64_t>(gridDim.x) * GEN_THREADS) {
    int idx[kMaxOrderAny];
    uint64_t src;
    if (!decode_entry(lay, e, n, b, idx, &src)) t[e] = t[src];
  }
}

__device__ __forceinline__ const double* gen_row(const RowSource& s, uint32_t k, int n) {
  return k < s.len0 ? s.seg0 + static_cast<size_t>(k) * n : s.seg1 + static_cast<size_t>(k - s.len0) * n;
}

__global__ void __launch_bounds__(GEN_THREADS) moment_generic_kernel(const GenMomParams P) {
  const int S = P.lay.order;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(GEN_THREADS) + threadIdx.x; e < P.stored;
       e += static_cast<uint64_t>(gridDim.x) * GEN_THREADS) {
    int idx[kMaxOrderAny];
    uint64_t src;
    if (!decode_entry(P.lay, e, P.n, P.b, idx, &src)) continue;  // copied afterwards
    double mean[2] = {0.0, 0.0};
    for (int pass = 0; pass < P.npass; ++pass) {
      double acc = 0.0;
      for (uint32_t k = 0; k < P.K; ++k) {
        const double* row = gen_row(P.src[pass], k, P.n);
        double q = row[idx[0]];
        const int nf = P.top ? S - 1 : S;  // factors of q
        for (int t = 1; t < nf; ++t) q = __dmul_rn(q, row[idx[t]]);
        if (P.top && S >= 2) acc = __fma_rn(q, row[idx[S - 1]], acc);
        else acc = __dadd_rn(acc, q);
      }
      mean[pass] = __dmul_rn(acc, P.inv);
    }
    if (P.npass == 2) P.m[e] = __fma_rn(P.c, __dsub_rn(mean[0], mean[1]), P.m[e]);
    else P.m[e] = mean[0];
  }
}

// C_len[sub] for a sorted index (at_sorted_unchecked, symten.cpp:171-181).
__device__ double gen_at_sorted(const LayoutDev& lay, const double* data, const int* sub, int n, int b) {
  const int len = lay.order;
  uint64_t r = 0, off = 0;
  int prev = 0;
  for (int i = 0; i < len; ++i) {
    const int j = sub[i] / b;
    const uint64_t* pf = lay.prefix + static_cast<size_t>(len - 1 - i) * (lay.grid + 1);
    r += pf[j] - pf[prev];
    prev = j;
    off = off * static_cast<uint64_t>(gen_ext(j, n, b)) + static_cast<uint64_t>(sub[i] - j * b);
  }
  return data[lay.offset[r] + off];
}

__global__ void __launch_bounds__(GEN_THREADS) moms2cums_generic_kernel(const GenM2CParams P) {
  const int S = P.s;
  const LayoutDev& L = P.lay[S - 1];
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(GEN_THREADS) + threadIdx.x; e < P.stored;
       e += static_cast<uint64_t>(gridDim.x) * GEN_THREADS) {
    int idx[kMaxCumOrderAny];
    uint64_t src;
    if (!decode_entry(L, e, P.n, P.b, idx, &src)) continue;  // copied afterwards
    // restricted growth strings in lexicographic order; a = 0...0 (one part) is skipped
    int a[kMaxCumOrderAny], mx[kMaxCumOrderAny];  // mx[i] = max(a[0..i])
    for (int i = 0; i < S; ++i) a[i] = mx[i] = 0;
    double acc = 0.0;
    for (;;) {
      // successor: rightmost position that can grow (a[i] <= max of the prefix before it)
      int i = S - 1;
      while (i >= 1 && a[i] > mx[i - 1]) --i;
      if (i < 1) break;
      ++a[i];
      mx[i] = a[i] > mx[i - 1] ? a[i] : mx[i - 1];
      for (int k = i + 1; k < S; ++k) {
        a[k] = 0;
        mx[k] = mx[i];
      }
      const int parts = mx[S - 1] + 1;  // >= 2 here
      double prod = 1.0;
      for (int q = 0; q < parts; ++q) {
        int sub[kMaxCumOrderAny], len = 0;
        for (int k = 0; k < S; ++k)
          if (a[k] == q) sub[len++] = idx[k];
        prod = __dmul_rn(prod, gen_at_sorted(P.lay[len - 1], P.lower[len - 1], sub, P.n, P.b));
      }
      acc = __dadd_rn(acc, prod);
    }
    P.c[e] = __dsub_rn(P.m[e], acc);
  }
}

unsigned gen_grid(uint64_t stored) {
  const uint64_t want = (stored + GEN_THREADS - 1) / GEN_THREADS;
  return static_cast<unsigned>(want < 148ull * 64 ? (want ? want : 1) : 148ull * 64);
}

}  // namespace

void launch_moment_generic(const GenMomParams& p, cudaStream_t st) {
  moment_generic_kernel<<<gen_grid(p.stored), GEN_THREADS, 0, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
  copy_generic_kernel<<<gen_grid(p.stored), GEN_THREADS, 0, st>>>(p.m, p.lay, p.stored, p.n, p.b);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

void launch_moms2cums_generic(const GenM2CParams& p, cudaStream_t st) {
  moms2cums_generic_kernel<<<gen_grid(p.stored), GEN_THREADS, 0, st>>>(p);
  CSB_CUDA(cudaGetLastError());
  count_launch();
  copy_generic_kernel<<<gen_grid(p.stored), GEN_THREADS, 0, st>>>(p.c, p.lay[p.s - 1], p.stored, p.n, p.b);
  CSB_CUDA(cudaGetLastError());
  count_launch();
}

}  // namespace csb
