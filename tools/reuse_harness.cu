// Offline harness for tools/sass_reuse.py: the tail kernel's triangle and
// rectangle row loops in isolation (seconds to compile), to see how source
// shape and ptxas options change the operand-reuse fraction.
//   nvcc -cubin -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -DVARIANT=0 -o /tmp/t.cubin tools/reuse_harness.cu
//   python tools/sass_reuse.py /tmp/t.cubin
#include <cstdint>
#ifndef VARIANT
#define VARIANT 0
#endif
__device__ __forceinline__ void fma_keep(double& acc, double q, double x) {
  asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(q), "d"(x));
}
template <int RL, int W, bool TRI>
__global__ void __launch_bounds__(384, 1) k(const double* __restrict__ g, double* out, const int* pid, int s, int c0, int chunks) {
  extern __shared__ __align__(16) double xs[];
  constexpr int n = 48, KC = 32, LM1 = 4;
  constexpr int NA = TRI ? RL * (RL + 1) / 2 : RL * W;
  for (int i = threadIdx.x; i < KC * n; i += blockDim.x) xs[i] = g[i];
  __syncthreads();
  int pidx[LM1];
  for (int u = 0; u < LM1; ++u) pidx[u] = pid[threadIdx.x * LM1 + u];
  double acc[NA], sum[RL];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = 0.0;
#pragma unroll
  for (int i = 0; i < RL; ++i) sum[i] = 0.0;
  for (int c = 0; c < chunks; ++c) {
    double pn = xs[pidx[0]];
#pragma unroll
    for (int u = 1; u < LM1; ++u) pn = __dmul_rn(pn, xs[pidx[u]]);
#pragma unroll 8
    for (int r = 0; r < KC; ++r) {
      const double* xr = xs + r * n;
      const double pv = pn;
      {
        const double* xn = xs + min(r + 1, KC - 1) * n;
        pn = xn[pidx[0]];
#pragma unroll
        for (int u = 1; u < LM1; ++u) pn = __dmul_rn(pn, xn[pidx[u]]);
      }
      double xa[RL], xc[W];
#pragma unroll
      for (int k = 0; k + 1 < RL; k += 2) {
        const double2 v = *reinterpret_cast<const double2*>(xr + s + k);
        xa[k] = v.x; xa[k + 1] = v.y;
      }
      if (RL & 1) xa[RL - 1] = xr[s + RL - 1];
      if (TRI) {
#pragma unroll
        for (int k = 0; k < W; ++k) xc[k] = xa[k < RL ? k : 0];
      } else {
#pragma unroll
        for (int k = 0; k < W; k += 2) {
          const double2 v = *reinterpret_cast<const double2*>(xr + c0 + k);
          xc[k] = v.x; xc[k + 1] = v.y;
        }
      }
      double q[RL];
#pragma unroll
      for (int i = 0; i < RL; ++i) q[i] = __dmul_rn(pv, xa[i]);
      if (TRI) {
#pragma unroll
        for (int i = 0; i < RL; ++i) sum[i] = __dadd_rn(sum[i], q[i]);
      }
      int a = 0;
#if VARIANT == 0
#pragma unroll
      for (int i = 0; i < RL; ++i)
#pragma unroll
        for (int j = TRI ? i : 0; j < W; ++j, ++a) fma_keep(acc[a], q[i], xc[j]);
#elif VARIANT == 1  // column-major: x shared
#pragma unroll
      for (int j = 0; j < W; ++j)
#pragma unroll
        for (int i = 0; i < RL; ++i)
          if (!TRI || i <= j) {
            const int aa = TRI ? (i * W - i * (i - 1) / 2 + (j - i)) : i * W + j;
            fma_keep(acc[aa], q[i], xc[j]);
          }
#endif
    }
  }
  double t = 0;
#pragma unroll
  for (int a = 0; a < NA; ++a) t += acc[a];
#pragma unroll
  for (int i = 0; i < RL; ++i) t += sum[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template __global__ void k<8, 8, true>(const double*, double*, const int*, int, int, int);
template __global__ void k<4, 8, false>(const double*, double*, const int*, int, int, int);
