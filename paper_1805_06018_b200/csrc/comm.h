// NCCL binding of the shard-by-k reduce (comm.cpp).  Every function returns "" on success or an
// error message.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>

#define PCB_COMM_ID_BYTES 128

namespace pcb {
bool comm_available(std::string* why);
int comm_version();
std::string comm_unique_id(void* out128);
std::string comm_init(const void* id128, int nranks, int rank, void** out);
void comm_destroy(void* comm);
std::string comm_sum(void* comm, double* buf, size_t count, int root, cudaStream_t st);
}  // namespace pcb
