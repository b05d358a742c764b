// Per-column-window timing of the top-pair DMMA kernel (experiments): the
// launch plan of one shape is filtered to the tiles of one window h (the
// prefix rows whose last index lies in [8h, 8h + 8)) and launched alone on
// random rows in update mode, so the cost of each window can be set against
// its share of the algorithmic work.  Links the library's objects.
//   make -C paper_1701_06446_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//     -I include -I paper_1701_06446_b200/csrc tools/window_bench.cu paper_1701_06446_b200/build/*.o \
//     -o tools/window_bench -ldl
//   tools/window_bench d n b p [reps] [tail windows]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "kernels.cuh"
#include "layout.hpp"

using namespace csb;

int main(int argc, char** argv) {
  const int d = argc > 1 ? atoi(argv[1]) : 6;
  const int n = argc > 2 ? atoi(argv[2]) : 48;
  const int b = argc > 3 ? atoi(argv[3]) : 4;
  const int p = argc > 4 ? atoi(argv[4]) : 2000;
  const int reps = argc > 5 ? atoi(argv[5]) : 5;
  Layout top(d, n, b), low(d - 1, n, b);
  MomentPlan plan;
  const int tail = argc > 6 ? atoi(argv[6]) : tail_windows(d, n, b);
  plan.build_dmma(d, n, b, top, &low, dmma_scratch_per_tile(), tail);
  plan.upload();
  std::vector<double> x(2ull * p * n);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  for (auto& v : x) v = nd(rng);
  double *xd, *mt, *ml, *scratch, *zeros;
  cudaMalloc(&xd, x.size() * 8);
  cudaMemcpy(xd, x.data(), x.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&mt, top.stored * 8);
  cudaMalloc(&ml, low.stored * 8);
  cudaMemset(mt, 0, top.stored * 8);
  cudaMemset(ml, 0, low.stored * 8);
  const size_t ntiles = plan.tiles.size();
  cudaMalloc(&scratch, ntiles * plan.scratch_per_tile * 8);
  const size_t zc = static_cast<size_t>(dmma_chunk_rows(n, b)) * n;
  cudaMalloc(&zeros, zc * 8);
  cudaMemset(zeros, 0, zc * 8);
  MomParams P;
  P.src[0].seg0 = xd;
  P.src[0].len0 = p;
  P.src[1].seg0 = xd + static_cast<size_t>(p) * n;
  P.src[1].len0 = p;
  P.npass = 2;
  P.K = p;
  P.n = n;
  P.b = b;
  P.L = d - 1;
  P.rows = plan.d_rows.ptr;
  P.pairs = plan.d_pairs.ptr;
  P.top = mt;
  P.low = ml;
  P.scratch = scratch;
  P.zeros = zeros;
  P.c = 0.1;
  P.inv = 1.0 / p;
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int maxh = 0;
  for (const auto& t : plan.tiles) maxh = std::max<int>(maxh, t.J);
  printf("{\"kernel\": \"%s\", \"d\": %d, \"n\": %d, \"b\": %d, \"p\": %d, \"windows\": [", dmma_kernel_name(n, b), d, n,
         b, p);
  double total = 0.0;
  for (int h = -1; h <= maxh; ++h) {
    std::vector<MomTile> sel;
    uint64_t rowsets = 0, coltiles = 0;
    for (const auto& t : plan.tiles)
      if (h < 0 || static_cast<int>(t.J) == h) {
        sel.push_back(t);
        rowsets += t.nrows;
        coltiles += static_cast<uint64_t>(t.nrows) * t.ncols;
      }
    if (sel.empty()) continue;
    MomTile* dt;
    cudaMalloc(&dt, sel.size() * sizeof(MomTile));
    cudaMemcpy(dt, sel.data(), sel.size() * sizeof(MomTile), cudaMemcpyHostToDevice);
    P.tiles = dt;
    launch_moment_top_dmma(P, static_cast<int>(sel.size()), st);  // warm-up
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) launch_moment_top_dmma(P, static_cast<int>(sel.size()), st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    if (h >= 0) total += ms;
    // executed DMMA MACs per data row: row sets x 64 rows x column tiles x 8
    const double exec_macs = 64.0 * 8.0 * static_cast<double>(coltiles);
    printf("%s{\"h\": %d, \"ctas\": %zu, \"rowsets\": %llu, \"tile_rowsets\": %llu, \"ms\": %.4f, "
           "\"exec_tflops\": %.2f}",
           h < 0 ? "" : ", ", h, sel.size(), (unsigned long long)rowsets, (unsigned long long)coltiles, ms,
           2.0 * exec_macs * 2.0 * p / (ms * 1e-3) / 1e12);
    cudaFree(dt);
  }
  double tail_ms = 0.0;
  if (!plan.tail.empty()) {
    MomParams pt = P;
    pt.rows = plan.d_tail_rows.ptr;
    pt.tail = plan.d_tail.ptr;
    pt.tail_warps = static_cast<uint32_t>(plan.tail.size() / 32);
    double* ts;
    cudaMalloc(&ts, tail_scratch_doubles() * 8);
    pt.scratch = ts;
    launch_moment_tail(pt, st);
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) launch_moment_tail(pt, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    tail_ms = ms / reps;
  }
  cudaError_t err = cudaGetLastError();
  printf("], \"sum_windows_ms\": %.4f, \"tail_tasks\": %zu, \"tail_ms\": %.4f, \"err\": \"%s\"}\n", total,
         plan.tail.size(), tail_ms, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
