// Dependent-chain latencies of FP64 ops on one warp (standalone, no other
// load): DADD, DMUL, DFMA, and an LDS -> DADD chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = out[0] + threadIdx.x * 1e-12, b = 1.0000001, s = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) a = __fma_rn(a, b, b);
  long long t3 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    const double v = sm[idx & 1023];
    s = __dadd_rn(s, v);
    idx = idx + static_cast<int>(s) + 1;  // address depends on the sum: LDS -> DADD -> LDS
  }
  long long t4 = clock64();
  for (int i = 0; i < iters; ++i) s = __dadd_rn(s, sm[(threadIdx.x + i) & 1023]);  // independent LDS, dependent DADD
  long long t5 = clock64();
  out[1 + threadIdx.x] = a + s;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 64); cudaMalloc(&c, 8 * 8);
  cudaMemset(o, 0, 8 * 64);
  const int iters = 4096;
  k<<<1, 32>>>(o, c, iters);
  k<<<1, 32>>>(o, c, iters);
  long long h[5];
  cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"dadd_lat\": %.2f, \"dmul_lat\": %.2f, \"dfma_lat\": %.2f, \"lds_dadd_chain\": %.2f, \"dadd_chain_lds_indep\": %.2f}\n",
         h[0] / (double)iters, h[1] / (double)iters, h[2] / (double)iters, h[3] / (double)iters, h[4] / (double)iters);
  return 0;
}
