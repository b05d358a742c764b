// How busy can the FP64 pipe get with few resident warps?  One CTA per SM
// (forced by the shared-memory request) of W warps per scheduler, each thread
// running CH independent DFMA chains (optionally with one broadcast LDS.64
// per LDS_EVERY DFMAs, like the tail kernel's operand loads).  Prints the
// fraction of 64 DFMA/clk/SM reached.  Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o tools/fp64_occupancy tools/fp64_occupancy.cu
#include <cuda_runtime.h>

#include <cstdio>

// MODE 0: broadcast LDS.64; 1: broadcast LDS.128 (both halves used, one per
// 2 * LDS_EVERY DFMAs); 2: lane-varying conflict-free LDS.64; 3: lane-varying LDS.128
template <int CH, int LDS_EVERY, int MODE = 0>
__global__ void k(double* out, int iters, double a) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  double x = a, x2 = a;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (LDS_EVERY > 0) {
        if (MODE == 0 && c % LDS_EVERY == 0) x = sm[(it + c) & 63];
        if (MODE == 2 && c % LDS_EVERY == 0) x = sm[((it + c) & 31) * 32 + lane];
        if ((MODE == 1 || MODE == 3) && c % (2 * LDS_EVERY) == 0) {
          const int idx = MODE == 1 ? ((it + c) & 31) * 2 : ((it + c) & 15) * 64 + lane * 2;
          const double2 v = *reinterpret_cast<const double2*>(sm + idx);
          x = v.x;
          x2 = v.y;
        }
        if ((MODE == 1 || MODE == 3) && c % (2 * LDS_EVERY) == LDS_EVERY) x = x2;
      }
      acc[c] = __fma_rn(acc[c], x, a);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH, int LDS_EVERY, int MODE = 0>
void run(int sms, int wps, double* out, double mhz) {
  const int threads = 128 * wps, iters = 20000;
  const size_t smem = 120 * 1024;
  cudaFuncSetAttribute(k<CH, LDS_EVERY, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<CH, LDS_EVERY, MODE><<<sms, threads, smem>>>(out, 100, 1.0000001);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<CH, LDS_EVERY, MODE><<<sms, threads, smem>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = (double)sms * threads * CH * iters;
  const double per_clk_sm = dfma / (best * 1e-3) / (mhz * 1e6) / sms;
  printf("{\"mode\": %d, \"chains\": %d, \"lds_every\": %d, \"warps_per_scheduler\": %d, \"ms\": %.3f, \"dfma_per_clk_sm\": %.2f, \"frac_of_64\": %.3f}\n",
         MODE, CH, LDS_EVERY, wps, best, per_clk_sm, per_clk_sm / 64.0);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  const double mhz = khz / 1000.0;
  double* out;
  cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 1024);
  const int sms = p.multiProcessorCount;
  for (int w : {1, 2, 3, 4, 6}) run<32, 0>(sms, w, out, mhz);
  for (int w : {3, 4}) {
    run<32, 4, 0>(sms, w, out, mhz);
    run<32, 4, 1>(sms, w, out, mhz);
    run<32, 4, 2>(sms, w, out, mhz);
    run<32, 4, 3>(sms, w, out, mhz);
    run<32, 2, 0>(sms, w, out, mhz);
    run<32, 2, 1>(sms, w, out, mhz);
    run<32, 8, 0>(sms, w, out, mhz);
    run<32, 8, 1>(sms, w, out, mhz);
  }
  return cudaDeviceSynchronize() != cudaSuccess;
}
