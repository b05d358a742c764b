// FP64 microbenchmarks for the roofline denominator (MEASURED_PEAKS.json has
// no FP64 entry):
//   1. DFMA throughput (CUDA-core FP64), register-resident independent chains;
//   2. DMMA throughput: mma.sync.aligned.m8n8k4.row.col.f64 (the only FP64
//      tensor-core path on sm_100a; tcgen05 has no f64 kind);
//   3. whether one DMMA equals the sequential FMA chain over k = 0..3
//      bit for bit (decides whether a DMMA kernel can stay bitwise with the
//      reference's row-ordered FMA accumulation).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));              \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

constexpr int CHAINS = 16;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = __fma_rn(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int MMA_ACC = 8;

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double d[MMA_ACC][2];
#pragma unroll
  for (int c = 0; c < MMA_ACC; ++c) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < MMA_ACC; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < MMA_ACC; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA interleaved: does the FP64 tensor path overlap with the
// FP64 FMA pipe?  Same DMMA count as dmma_kernel plus `nf` DFMA per DMMA.
template <int NF>
__global__ void mixed_kernel(double* out, int iters, double a, double b) {
  double d[MMA_ACC][2];
  double f[MMA_ACC][NF > 0 ? NF : 1];
#pragma unroll
  for (int c = 0; c < MMA_ACC; ++c) {
    d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
#pragma unroll
    for (int q = 0; q < (NF > 0 ? NF : 1); ++q) f[c][q] = c + q;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < MMA_ACC; ++c) {
      dmma(d[c][0], d[c][1], a, b);
#pragma unroll
      for (int q = 0; q < NF; ++q) f[c][q] = __fma_rn(f[c][q], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < MMA_ACC; ++c) {
    s += d[c][0] + d[c][1];
#pragma unroll
    for (int q = 0; q < (NF > 0 ? NF : 1); ++q) s += f[c][q];
  }
  if (s == 12345.678) out[0] = s;
}

// One m8n8k4 on given A (8x4 row-major), B (4x8), C (8x8); writes D (8x8).
__global__ void dmma_once(const double* A, const double* B, const double* Cm, double* D) {
  const int l = threadIdx.x;
  const int r = l >> 2, k = l & 3;
  double a = A[r * 4 + k];          // A fragment: row l/4, col l%4
  double b = B[k * 8 + r];          // B fragment: row l%4, col l/4
  double d0 = Cm[r * 8 + 2 * k], d1 = Cm[r * 8 + 2 * k + 1];
  dmma(d0, d1, a, b);
  D[r * 8 + 2 * k] = d0;
  D[r * 8 + 2 * k + 1] = d1;
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  auto run = [&](auto kern, int blocks, int threads, int iters, double flop_per_iter_thread,
                 const char* name) {
    kern<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      CK(cudaEventRecord(e0));
      kern<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
    }
    const double flops = (double)blocks * threads * iters * flop_per_iter_thread;
    printf("  \"%s_tflops\": %.3f,\n", name, flops / (best * 1e-3) / 1e12);
    return flops / (best * 1e-3) / 1e12;
  };
  printf("{\n  \"sms\": %d,\n", sms);
  // DFMA: 2 flops per FMA
  run(dfma_kernel, sms * 8, 256, 20000, 2.0 * CHAINS, "dfma");
  // DMMA: per warp per mma 2*8*8*4 = 512 flops -> 16 per thread
  run(dmma_kernel, sms * 8, 256, 20000, 16.0 * MMA_ACC, "dmma");

  // DMMA issue rate vs warps per SMSP: 148*m CTAs of 128 threads (m warps
  // per SMSP when spread evenly), 8 independent accumulators per warp
  for (int m : {1, 2, 3, 4, 8}) {
    char name[64];
    snprintf(name, sizeof name, "dmma_%dwarp_per_smsp", m);
    run(dmma_kernel, sms * m, 128, 20000, 16.0 * MMA_ACC, name);
  }

  // mixed: report the time ratio against DMMA alone (1.0 = DFMA fully hidden)
  {
    auto time_it = [&](auto kern) {
      kern<<<sms * 8, 256>>>(out, 10, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        kern<<<sms * 8, 256>>>(out, 20000, 1.0000001, 1e-9);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
      }
      return best;
    };
    const float t0 = time_it(mixed_kernel<0>);
    const float t1 = time_it(mixed_kernel<1>);
    const float t2 = time_it(mixed_kernel<2>);
    const float t4 = time_it(mixed_kernel<4>);
    printf("  \"mixed_dmma_plus_1dfma_ratio\": %.3f,\n  \"mixed_dmma_plus_2dfma_ratio\": %.3f,\n"
           "  \"mixed_dmma_plus_4dfma_ratio\": %.3f,\n", t1 / t0, t2 / t0, t4 / t0);
  }

  // bitwise check of one DMMA against the sequential FMA chain
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  int diff_seq = 0, diff_rev = 0, trials = 200;
  std::vector<double> A(32), B(32), Cm(64), D(64);
  double *dA, *dB, *dC, *dD;
  CK(cudaMalloc(&dA, 32 * 8));
  CK(cudaMalloc(&dB, 32 * 8));
  CK(cudaMalloc(&dC, 64 * 8));
  CK(cudaMalloc(&dD, 64 * 8));
  for (int t = 0; t < trials; ++t) {
    for (auto& v : A) v = nd(rng) * 3;
    for (auto& v : B) v = nd(rng) * 3;
    for (auto& v : Cm) v = nd(rng) * 10;
    CK(cudaMemcpy(dA, A.data(), 32 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), 32 * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dC, Cm.data(), 64 * 8, cudaMemcpyHostToDevice));
    dmma_once<<<1, 32>>>(dA, dB, dC, dD);
    CK(cudaMemcpy(D.data(), dD, 64 * 8, cudaMemcpyDeviceToHost));
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) {
        double s = Cm[r * 8 + c];
        for (int k = 0; k < 4; ++k) s = std::fma(A[r * 4 + k], B[k * 8 + c], s);
        double q = Cm[r * 8 + c];
        for (int k = 3; k >= 0; --k) q = std::fma(A[r * 4 + k], B[k * 8 + c], q);
        diff_seq += s != D[r * 8 + c];
        diff_rev += q != D[r * 8 + c];
      }
  }
  printf("  \"dmma_vs_seq_fma_mismatches\": %d,\n  \"dmma_vs_rev_fma_mismatches\": %d,\n"
         "  \"dmma_bit_trials\": %d,\n",
         diff_seq, diff_rev, trials * 64);
  printf("  \"gpu\": \"%s\",\n  \"clock_mhz\": %d\n}\n", prop.name, prop.clockRate / 1000);
  return 0;
}
