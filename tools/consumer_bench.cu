// Microbenchmark of the DMMA consumer loop of moment_top_dmma_kernel in
// isolation: A fragments from a shared-memory ring in the kernel's layout
// (ASTRIDE = 10 doubles per lane entry, 4 x LDS.128 per k4 step), B
// fragments from staged rows (n = 96), software-pipelined one k4 step
// ahead, NC column tiles.  No producer, no TMA, no epilogue: measures the
// DMMA issue efficiency of the loop itself vs warps per SM sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/consumer_bench tools/consumer_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstdio>

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e = (x);                                        \
    if (e != cudaSuccess) {                                     \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));   \
      exit(1);                                                  \
    }                                                           \
  } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int N = 96;
constexpr int HSTEPS = 4;
constexpr int ASTRIDE = 10;
constexpr int ASLOT = HSTEPS * 32 * ASTRIDE;
constexpr int KC = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// MODE 0: loads + DMMA (the kernel's loop); 1: DMMA only on register
// operands.  SPIN: one more warp per SM sub-partition spins on an mbarrier
// try_wait (like an idle producer) while the DMMA warps run.
template <int NC, int MODE, int SPIN = 0>
__global__ void __launch_bounds__(256, 1) consumer_kernel(double* out, int chunks) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ volatile int done;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    done = 0;
  }
  double* xs = sm;                       // 2 stages x KC x N
  double* ar = sm + 2 * KC * N + 64;     // 2 slots x ASLOT
  for (int i = threadIdx.x; i < 2 * KC * N + 64 + 2 * ASLOT; i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
  __syncthreads();
  if (SPIN >= 5 && threadIdx.x >= blockDim.x - 128) {
    // dependent DADD chains (2 per lane) beside the DMMA warps: report the
    // chain latency per add in cycles
    double s0 = 0.0, s1 = 0.0, v = 1e-9 * threadIdx.x;
    const int iters = 20000;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      s0 = __dadd_rn(s0, v);
      s1 = __dadd_rn(s1, v);
    }
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0)
      printf("{\"dadd_chain_cycles_per_add\": %.2f, \"with_dmma\": %d}\n", double(t1 - t0) / iters, SPIN == 5);
    if (s0 + s1 == 12345.678) out[1] = s0;
    if (SPIN == 5) return;
  }
  if (SPIN >= 3 && SPIN < 5 && threadIdx.x >= blockDim.x - 128) {
    // FP64 (non-tensor) warp: independent DMUL/DADD chains, like a producer
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 1.0 + 1e-9 * (threadIdx.x + i);
    const int iters = chunks * (SPIN == 3 ? 16 : 4);  // 8 DMUL per iteration
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __dmul_rn(v[i], 0.9999999999);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 12345.678) out[1] = s;
    return;
  }
  if (SPIN && threadIdx.x >= blockDim.x - 128) {
    // spinning waiter: try_wait on a phase that completes only at the end
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(0u)
          : "memory");
      if (SPIN == 2) __nanosleep(200);
    }
    return;
  }
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, q = lane & 3;
  double acc[8][NC][2];
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[g][c][0] = acc[g][c][1] = 0.0;
  const int col0 = 8;
  for (int c = 0; c < chunks; ++c) {
    const double* as = ar + (c & 1) * ASLOT + (r * 4 + q) * ASTRIDE;
    const double* xb = xs + (c & 1) * KC * N + q * N + col0 + r;
    double a[2][8], bb[2][NC];
    auto load = [&](int t, int buf) {
      const double2* ap = reinterpret_cast<const double2*>(as + t * 32 * ASTRIDE);
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        const double2 v = ap[s2];
        a[buf][2 * s2] = v.x;
        a[buf][2 * s2 + 1] = v.y;
      }
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) bb[buf][cc] = xb[(4 * t) * N + 8 * cc];
    };
    if (MODE == 2) {
      // per-chunk protocol of the real kernel: wait on a (ready) full
      // barrier, arrive on an empty barrier after the chunk
      __shared__ __align__(8) uint64_t fullb[8], emptyb[8];
      const int w = threadIdx.x >> 5;
      if (c == 0 && lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&fullb[w])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&emptyb[w])), "r"(1));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fullb[w])) : "memory");
      }
      __syncwarp();
      {
        uint32_t ok = 0;
        while (!ok)
          asm volatile(
              "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
              : "=r"(ok)
              : "r"(smem_u32(&fullb[w])), "r"((uint32_t)(c & 1))
              : "memory");
      }
      load(0, 0);
#pragma unroll
      for (int t = 0; t < HSTEPS; ++t) {
        if (t + 1 < HSTEPS) load(t + 1, (t + 1) & 1);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int g = 0; g < 8; ++g) dmma(acc[g][cc][0], acc[g][cc][1], a[t & 1][g], bb[t & 1][cc]);
      }
      __syncwarp();
      if (lane == 0) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&emptyb[w])) : "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&fullb[w])) : "memory");
      }
    } else if (MODE == 1) {
      if (c == 0) load(0, 0);
#pragma unroll
      for (int t = 0; t < HSTEPS; ++t)
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int g = 0; g < 8; ++g) dmma(acc[g][cc][0], acc[g][cc][1], a[0][g], bb[0][cc]);
    } else {
      load(0, 0);
#pragma unroll
      for (int t = 0; t < HSTEPS; ++t) {
        if (t + 1 < HSTEPS) load(t + 1, (t + 1) & 1);
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
          for (int g = 0; g < 8; ++g) dmma(acc[g][cc][0], acc[g][cc][1], a[t & 1][g], bb[t & 1][cc]);
      }
    }
  }
  if (SPIN && SPIN < 3) {
    __syncwarp();
    if (lane == 0 && atomicAdd((int*)&done, 1) == (int)(blockDim.x / 32 - 4) - 1)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  double s = 0;
#pragma unroll
  for (int g = 0; g < 8; ++g)
#pragma unroll
    for (int c = 0; c < NC; ++c) s += acc[g][c][0] + acc[g][c][1];
  if (s == 12345.678) out[0] = s;
}

template <int NC, int MODE, int SPIN = 0>
void run(int wps, double* out, int sms) {
  const int threads = 128 * wps + (SPIN ? 128 : 0);
  const size_t smem = sizeof(double) * (2 * KC * N + 64 + 2 * ASLOT);
  CK(cudaFuncSetAttribute(consumer_kernel<NC, MODE, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int chunks = 4000;
  consumer_kernel<NC, MODE, SPIN><<<sms, threads, smem>>>(out, 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    consumer_kernel<NC, MODE, SPIN><<<sms, threads, smem>>>(out, chunks);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double dmmas = double(sms) * (128 * wps) / 32 * chunks * HSTEPS * 8 * NC;
  printf("{\"nc\": %d, \"mode\": %d, \"spin\": %d, \"warps_per_smsp\": %d, \"tflops\": %.2f, \"cycles_per_dmma_per_smsp\": %.2f}\n", NC,
         MODE, SPIN, wps, dmmas * 512 / (best * 1e-3) / 1e12,
         (best * 1e-3) * 1.965e9 / (dmmas / (sms * 4)));
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out;
  CK(cudaMalloc(&out, 64));
  for (int w : {1, 2}) {
    run<1, 0>(w, out, sms);
    run<2, 0>(w, out, sms);
    run<4, 0>(w, out, sms);
    run<1, 1>(w, out, sms);
    run<2, 1>(w, out, sms);
    run<2, 2>(w, out, sms);
    run<2, 0, 3>(w, out, sms);
    run<2, 0, 4>(w, out, sms);
    run<2, 0, 1>(w, out, sms);
  }
  return 0;
}
