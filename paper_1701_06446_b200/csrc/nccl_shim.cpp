#include "nccl_shim.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace csb {
namespace nccl {

namespace {

// ABI of the few NCCL entry points used (nccl.h, stable since NCCL 2.0)
typedef int ncclResult_t;
typedef struct {
  char internal[kUniqueIdBytes];
} ncclUniqueId;
typedef void* ncclComm_t;
constexpr int ncclDouble = 8;  // ncclFloat64
constexpr int ncclSum = 0;

struct Api {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    // an NCCL the process already holds (e.g. the one PyTorch bundles) first;
    // else the system's, loaded RTLD_LOCAL so its symbols do not shadow a
    // different NCCL that a later import brings along
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.h = dlopen(name, RTLD_NOW | RTLD_NOLOAD);
      if (a.h) break;
    }
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      if (a.h) break;
      a.h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
    }
    if (!a.h) return;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(a.h, "ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(a.h, "ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.h, "ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.h, "ncclGetErrorString"));
  });
  return a;
}

void check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* msg = api().GetErrorString ? api().GetErrorString(r) : "?";
    fail(CSB_ERUNTIME, std::string(what) + ": " + msg);
  }
}

Api& need() {
  Api& a = api();
  if (!a.h || !a.GetUniqueId || !a.CommInitRank || !a.Broadcast || !a.AllReduce)
    fail(CSB_ERUNTIME, "NCCL (libnccl.so.2) is not available");
  return a;
}

}  // namespace

bool available() { return api().h != nullptr; }

void get_unique_id(unsigned char out[kUniqueIdBytes]) {
  ncclUniqueId id;
  check(need().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, kUniqueIdBytes);
}

void* comm_init(int nranks, int rank, const unsigned char idb[kUniqueIdBytes]) {
  ncclUniqueId id;
  std::memcpy(id.internal, idb, kUniqueIdBytes);
  ncclComm_t c = nullptr;
  check(need().CommInitRank(&c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void comm_destroy(void* comm) {
  if (comm && api().CommDestroy) api().CommDestroy(static_cast<ncclComm_t>(comm));
}

void allgather_ranges(void* comm, double* buf, const uint64_t* off, const uint64_t* cnt, int nranks,
                      cudaStream_t st) {
  Api& a = need();
  check(a.GroupStart(), "ncclGroupStart");
  for (int r = 0; r < nranks; ++r)
    if (cnt[r])
      check(a.Broadcast(buf + off[r], buf + off[r], cnt[r], ncclDouble, r, static_cast<ncclComm_t>(comm), st),
            "ncclBroadcast");
  check(a.GroupEnd(), "ncclGroupEnd");
}

void allreduce_sum(void* comm, double* buf, uint64_t count, cudaStream_t st) {
  if (!count) return;
  check(need().AllReduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), st),
        "ncclAllReduce");
}

}  // namespace nccl

namespace {

class NcclComm final : public Comm {
 public:
  NcclComm(int nranks, int rank, const unsigned char* id) : Comm(nranks, rank), c_(nccl::comm_init(nranks, rank, id)) {}
  ~NcclComm() override { nccl::comm_destroy(c_); }
  void allgather_ranges(double* buf, const uint64_t* off, const uint64_t* cnt, cudaStream_t st) override {
    nccl::allgather_ranges(c_, buf, off, cnt, nranks, st);
  }
  void allreduce_sum(double* buf, uint64_t count, cudaStream_t st) override {
    nccl::allreduce_sum(c_, buf, count, st);
  }

 private:
  void* c_;
};

// Caller-supplied collectives.  host_staged: the engine drains its stream,
// copies the span to a pinned host buffer, calls back on host memory and
// copies the result back (a CPU transport such as gloo); otherwise the
// callback gets the device pointer and the cudaStream_t to order on.
class OpsComm final : public Comm {
 public:
  OpsComm(int nranks, int rank, const csb_comm_ops& ops) : Comm(nranks, rank), ops_(ops) {}
  ~OpsComm() override {
    if (host_) cudaFreeHost(host_);
  }
  void allgather_ranges(double* buf, const uint64_t* off, const uint64_t* cnt, cudaStream_t st) override {
    if (!ops_.allgather_ranges) fail(CSB_ERUNTIME, "comm: allgather_ranges callback missing");
    if (!ops_.host_staged) {
      if (ops_.allgather_ranges(ops_.ctx, buf, off, cnt, nranks, st) != 0)
        fail(CSB_ERUNTIME, "comm: allgather_ranges callback failed");
      return;
    }
    uint64_t lo = UINT64_MAX, hi = 0;
    for (int r = 0; r < nranks; ++r)
      if (cnt[r]) {
        lo = std::min(lo, off[r]);
        hi = std::max(hi, off[r] + cnt[r]);
      }
    if (hi <= lo) return;
    double* h = stage(buf + lo, hi - lo, st);
    std::vector<uint64_t> rel(off, off + nranks);
    for (auto& o : rel) o = o >= lo ? o - lo : 0;
    if (ops_.allgather_ranges(ops_.ctx, h, rel.data(), cnt, nranks, nullptr) != 0)
      fail(CSB_ERUNTIME, "comm: allgather_ranges callback failed");
    unstage(buf + lo, hi - lo, st);
  }
  void allreduce_sum(double* buf, uint64_t count, cudaStream_t st) override {
    if (!ops_.allreduce_sum) fail(CSB_ERUNTIME, "comm: allreduce_sum callback missing");
    if (!count) return;
    if (!ops_.host_staged) {
      if (ops_.allreduce_sum(ops_.ctx, buf, count, st) != 0) fail(CSB_ERUNTIME, "comm: allreduce_sum callback failed");
      return;
    }
    double* h = stage(buf, count, st);
    if (ops_.allreduce_sum(ops_.ctx, h, count, nullptr) != 0) fail(CSB_ERUNTIME, "comm: allreduce_sum callback failed");
    unstage(buf, count, st);
  }

 private:
  double* stage(const double* dev, uint64_t count, cudaStream_t st) {
    if (cap_ < count) {
      if (host_) cudaFreeHost(host_);
      host_ = nullptr;
      cap_ = 0;
      CSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&host_), count * sizeof(double)));
      cap_ = count;
    }
    CSB_CUDA(cudaMemcpyAsync(host_, dev, count * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    return host_;
  }
  void unstage(double* dev, uint64_t count, cudaStream_t st) {
    CSB_CUDA(cudaMemcpyAsync(dev, host_, count * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaStreamSynchronize(st));  // the host buffer is reused by the next call
  }
  csb_comm_ops ops_;
  double* host_ = nullptr;
  uint64_t cap_ = 0;
};

}  // namespace

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char* id) {
  return std::make_shared<NcclComm>(nranks, rank, id);
}

std::shared_ptr<Comm> make_ops_comm(int nranks, int rank, const csb_comm_ops& ops) {
  return std::make_shared<OpsComm>(nranks, rank, ops);
}

}  // namespace csb
