// Does the FP64 pipe keep its rate when every DFMA reads three distinct
// register pairs (acc[i][j] = fma(q[i], x[j], acc[i][j]), the register-tile
// pattern of the tail kernel) instead of a chain with shared operands?
// One CTA per SM, 3 warps per scheduler.  Build like tools/fp64_occupancy.cu.
#include <cuda_runtime.h>
#include <cstdio>

// ORDER 0: column-major (x shared by consecutive DFMAs), 1: row-major (q
// shared), 2: diagonal sweeps (consecutive DFMAs share no operand)
template <int RI, int CJ, int ROWMAJOR>
__global__ void __launch_bounds__(384, 1) k(double* out, int iters, double a) {
  extern __shared__ double sm[];
  double acc[RI][CJ], q[RI], x[CJ];
#pragma unroll
  for (int i = 0; i < RI; ++i) q[i] = 1.0 + 1e-9 * (threadIdx.x + i);
#pragma unroll
  for (int j = 0; j < CJ; ++j) x[j] = 1.0 - 1e-9 * (threadIdx.x + j);
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int j = 0; j < CJ; ++j) acc[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
    if (ROWMAJOR == 2) {
#pragma unroll
      for (int t = 0; t < CJ; ++t)
#pragma unroll
        for (int i = 0; i < RI; ++i) {
          asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[i][(i + t) % CJ]) : "d"(q[i]), "d"(x[(i + t) % CJ]));
        }
    } else if (ROWMAJOR == 3) {  // row-major through volatile asm (order kept at the PTX level)
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) {
          asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc[i][j]) : "d"(q[i]), "d"(x[j]));
        }
    } else if (ROWMAJOR == 1) {
#pragma unroll
      for (int i = 0; i < RI; ++i)
#pragma unroll
        for (int j = 0; j < CJ; ++j) acc[i][j] = __fma_rn(q[i], x[j], acc[i][j]);
    } else {
#pragma unroll
      for (int j = 0; j < CJ; ++j)
#pragma unroll
        for (int i = 0; i < RI; ++i) acc[i][j] = __fma_rn(q[i], x[j], acc[i][j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int j = 0; j < CJ; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int RI, int CJ, int ROWMAJOR>
void run(int sms, double* out, double mhz) {
  const int threads = 384, iters = 20000;
  const size_t smem = 120 * 1024;
  cudaFuncSetAttribute(k<RI, CJ, ROWMAJOR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<RI, CJ, ROWMAJOR><<<sms, threads, smem>>>(out, 100, 1.0000001);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<RI, CJ, ROWMAJOR><<<sms, threads, smem>>>(out, iters, 1.0000001);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dfma = (double)sms * threads * RI * CJ * iters;
  const double per = dfma / (best * 1e-3) / (mhz * 1e6) / sms;
  printf("{\"tile\": \"%dx%d\", \"order\": \"%s\", \"dfma_per_clk_sm\": %.2f, \"frac_of_64\": %.3f}\n", RI, CJ,
         ROWMAJOR == 1 ? "row-major (q shared by consecutive DFMAs)"
         : ROWMAJOR == 0 ? "column-major (x shared)"
         : ROWMAJOR == 2 ? "diagonal sweeps via volatile asm (nothing shared)"
                         : "row-major via volatile asm",
         per, per / 64.0);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 1024);
  const int sms = p.multiProcessorCount;
  const double mhz = khz / 1000.0;
  run<4, 8, 1>(sms, out, mhz);
  run<4, 8, 0>(sms, out, mhz);
  run<4, 8, 2>(sms, out, mhz);
  run<4, 8, 3>(sms, out, mhz);
  run<8, 8, 1>(sms, out, mhz);
  run<8, 8, 2>(sms, out, mhz);
  run<8, 8, 3>(sms, out, mhz);
  run<6, 6, 1>(sms, out, mhz);
  return cudaDeviceSynchronize() != cudaSuccess;
}
