// Shared host-side helpers: error classes (mirroring the reference's
// exception types), CUDA error checks, device buffers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "cumstream_b200.h"

namespace csb {

// Status-carrying exception; the C ABI maps it back to CSB_* codes.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
  if (!ok) fail(CSB_EINVAL, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(CSB_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CSB_CUDA(call) ::csb::cuda_check((call), #call)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel, device
// and size (it costs microseconds of host time per call on the step path)
void set_smem_attr(const void* kern, size_t bytes);
template <class K>
inline void ensure_smem(K kern, size_t bytes) {
  set_smem_attr(reinterpret_cast<const void*>(kern), bytes);
}

// Owning device allocation (value-less; copying is explicit).
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  std::size_t count = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(std::exchange(o.ptr, nullptr)), count(std::exchange(o.count, 0)) {}
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = std::exchange(o.ptr, nullptr);
      count = std::exchange(o.count, 0);
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(std::size_t n) {
    release();
    if (n) CSB_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
    count = n;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
  }
  std::size_t bytes() const { return count * sizeof(T); }
};

inline uint64_t binom(int n, int k) {
  if (k < 0 || k > n) return 0;
  if (k > n - k) k = n - k;
  uint64_t r = 1;
  for (int i = 1; i <= k; ++i) r = r * static_cast<uint64_t>(n - k + i) / static_cast<uint64_t>(i);
  return r;
}
inline uint64_t multiset_count(int a, int r) { return binom(a + r - 1, r); }

void ensure_device();  // throws CSB_ERUNTIME without a usable CUDA device

// Host -> device upload of metadata / user data that is COMPLETE when this
// returns.  A plain cudaMemcpy from pageable memory may return before its DMA
// lands, and the library's non-blocking streams do not order against the
// legacy stream, so every such upload is followed by a device sync.
inline void h2d_sync(void* dst, const void* src, std::size_t bytes) {
  if (!bytes) return;
  CSB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  CSB_CUDA(cudaDeviceSynchronize());
}
inline void memset_sync(void* dst, int v, std::size_t bytes) {
  if (!bytes) return;
  CSB_CUDA(cudaMemset(dst, v, bytes));
  CSB_CUDA(cudaDeviceSynchronize());
}

}  // namespace csb
