// comm.cuh — NCCL-backed communicator used by the row-sharded driver.
#pragma once
#include "internal.cuh"

namespace rpca {

struct NcclUniqueId {
  char internal[128];
};

struct Comm {
  void* handle = nullptr;  // ncclComm_t
  int nranks = 1;
  int rank = 0;
};

rpca_status comm_unique_id(void* id, size_t bytes);
void comm_init(Ctx& c, int nranks, int rank, const void* id);
void comm_destroy(Ctx& c);
// in-place fp64 sum over ranks on the context stream (no-op on one rank)
void allreduce_sum(Ctx& c, double* buf, size_t count);
// recv = concat over ranks of `bytes_per_rank` bytes from each rank's send
void allgather_bytes(Ctx& c, const void* send, void* recv, size_t bytes_per_rank);

}  // namespace rpca
