// NCCL, resolved at run time (dlopen "libnccl.so.2"): the library has no
// link-time NCCL dependency for single-GPU use, and in a process that
// already loaded torch's NCCL the same library instance is reused.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace csb {
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
