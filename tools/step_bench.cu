// Microbenchmark of the DMMA moment kernel's inner k-step in isolation
// (operands from a fixed shared-memory row buffer, no TMA / epilogue), to
// separate the step's own DMMA-pipe efficiency from pipeline and tail
// effects.  Variants: NC column groups, low-order sums on/off, warps/SMSP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/step_bench tools/step_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                         \
  do {                                                                \
    cudaError_t e = (x);                                              \
    if (e != cudaSuccess) {                                           \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));         \
      exit(1);                                                        \
    }                                                                 \
  } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int N = 96;
constexpr int KROWS = 16;

template <int NC, bool LOW, int LM1, bool SPEC = false>
__global__ void step_kernel(double* out, int steps) {
  __shared__ __align__(16) double xs[KROWS * N + 64];
  __shared__ __align__(16) double lowbufs[4][2 * 264];
  for (int i = threadIdx.x; i < KROWS * N + 64; i += blockDim.x) xs[i] = 1.0 + 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane & 3, r = lane >> 2;
  double* lowbuf = lowbufs[warp];
  int pidx[LM1 > 0 ? LM1 : 1];
  for (int t = 0; t < LM1; ++t) pidx[t] = (r * 7 + t * 13) % N;
  const int h8 = 40, col0 = 40;
  double acc[8][NC][2] = {};
  double lowacc[2] = {0, 0};
  int lb = 0;
  if (SPEC && (warp & 1)) {
    // pure DMMA stream: operands straight from smem (A pre-formed)
    for (int s = 0; s < steps; ++s) {
      const double* xr = xs + ((4 * s + q) % KROWS) * N;
      double a[8], b[NC];
#pragma unroll
      for (int g = 0; g < 8; ++g) a[g] = xr[h8 + g];
#pragma unroll
      for (int c = 0; c < NC; ++c) b[c] = xr[col0 + 8 * c + r];
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int g = 0; g < 8; ++g) dmma(acc[g][c][0], acc[g][c][1], a[g], b[c]);
    }
  } else if (SPEC) {
    // producer-like stream: products + in-lane row sums, no DMMA
    for (int s = 0; s < steps; ++s) {
      const double* xr = xs + ((4 * s + q) % KROWS) * N;
      double p = 1.0;
      for (int t = 0; t < LM1; ++t) p = __dmul_rn(p, xr[pidx[t]]);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        const double v = __dmul_rn(p, xr[h8 + g]);
        lowacc[g & 1] = __dadd_rn(lowacc[g & 1], v);
        lowbuf[(g * 32 + lane) % 528] = v;
      }
    }
  } else
  for (int s = 0; s < steps; ++s) {
    const double* xr = xs + ((4 * s + q) % KROWS) * N;
    double p = 1.0;
    for (int t = 0; t < LM1; ++t) p = __dmul_rn(p, xr[pidx[t]]);
    double a[8], b[NC];
    const double2* xa = reinterpret_cast<const double2*>(xr + h8);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double2 v = xa[u];
      a[2 * u] = __dmul_rn(p, v.x);
      a[2 * u + 1] = __dmul_rn(p, v.y);
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) b[c] = xr[col0 + 8 * c + r];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int g = 0; g < 8; ++g) dmma(acc[g][c][0], acc[g][c][1], a[g], b[c]);
    if (LOW) {
      double2* wb = reinterpret_cast<double2*>(lowbuf + lb * 264 + q * 66 + r * 8);
#pragma unroll
      for (int u = 0; u < 4; ++u) wb[u] = make_double2(a[2 * u], a[2 * u + 1]);
      __syncwarp();
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        const double2 v = *reinterpret_cast<const double2*>(lowbuf + lb * 264 + kp * 66 + r * 8 + 2 * q);
        lowacc[0] = __dadd_rn(lowacc[0], v.x);
        lowacc[1] = __dadd_rn(lowacc[1], v.y);
      }
      lb ^= 1;
    }
  }
  double sum = lowacc[0] + lowacc[1];
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) sum += acc[g][c][0] + acc[g][c][1];
  if (sum == 1234.5) out[0] = sum;
}

template <int NC, bool LOW, int LM1, bool SPEC = false>
void run(const char* name, int ctas_per_sm, int warps_per_cta, int sms, double* out, cudaEvent_t e0, cudaEvent_t e1) {
  const int steps = 4000;
  auto k = step_kernel<NC, LOW, LM1, SPEC>;
  k<<<sms * ctas_per_sm, warps_per_cta * 32>>>(out, 10);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0));
    k<<<sms * ctas_per_sm, warps_per_cta * 32>>>(out, steps);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  const double flops = 512.0 * 8 * NC * steps * (double)sms * ctas_per_sm * warps_per_cta / (SPEC ? 2 : 1);
  printf("  \"%s_w%d\": %.2f,\n", name, ctas_per_sm * warps_per_cta / 4, flops / (best * 1e-3) / 1e12);
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  double* out;
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("{\n");
  for (int w : {2, 4}) {
    run<3, false, 2>("nc3_nolow", w, 4, sms, out, e0, e1);
    run<3, true, 2>("nc3_low", w, 4, sms, out, e0, e1);
    run<1, true, 2>("nc1_low", w, 4, sms, out, e0, e1);
    run<1, true, 2, true>("nc1_spec", w, 4, sms, out, e0, e1);
    run<2, true, 2, true>("nc2_spec", w, 4, sms, out, e0, e1);
    run<3, true, 2, true>("nc3_spec", w, 4, sms, out, e0, e1);
    run<4, true, 2, true>("nc4_spec", w, 4, sms, out, e0, e1);
  }
  printf("  \"unit\": \"TFLOP/s executed DMMA\"\n}\n");
  return 0;
}
