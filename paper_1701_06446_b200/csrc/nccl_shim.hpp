// NCCL, resolved at run time (dlopen "libnccl.so.2"): the library has no
// link-time NCCL dependency for single-GPU use, and in a process that
// already loaded torch's NCCL the same library instance is reused.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>

#include "cumstream_b200.h"

namespace csb {

// The exchange the sharded engine needs: an in-place allgather
// of per-rank contiguous ranges (collective C2, M_{d-1}) and a sum
// allreduce (collective C3, norm partials and the C_d diagonal), both on
// device buffers ordered on the engine's stream.  Implementations: NCCL
// (the product path over NVLink) and caller-supplied callbacks
// (csb_comm_init_ops: e.g. torch.distributed/gloo in the tests).  Streams
// hold a shared_ptr, so destroying or replacing the process communicator
// never pulls it from under a live stream.
class Comm {
 public:
  Comm(int nranks, int rank) : nranks(nranks), rank(rank) {}
  virtual ~Comm() = default;
  virtual void allgather_ranges(double* buf, const uint64_t* off, const uint64_t* cnt, cudaStream_t st) = 0;
  virtual void allreduce_sum(double* buf, uint64_t count, cudaStream_t st) = 0;
  const int nranks, rank;
};

std::shared_ptr<Comm> make_nccl_comm(int nranks, int rank, const unsigned char* id);
std::shared_ptr<Comm> make_ops_comm(int nranks, int rank, const csb_comm_ops& ops);

namespace nccl {

constexpr int kUniqueIdBytes = 128;

bool available();                                   // libnccl.so.2 could be loaded
void get_unique_id(unsigned char out[kUniqueIdBytes]);
void* comm_init(int nranks, int rank, const unsigned char id[kUniqueIdBytes]);
void comm_destroy(void* comm);
// in-place allgather of variable-size contiguous ranges: rank r owns
// [off[r], off[r] + cnt[r]) doubles of buf (one broadcast per rank, grouped)
void allgather_ranges(void* comm, double* buf, const uint64_t* off, const uint64_t* cnt, int nranks,
                      cudaStream_t st);
void allreduce_sum(void* comm, double* buf, uint64_t count, cudaStream_t st);

}  // namespace nccl
}  // namespace csb
