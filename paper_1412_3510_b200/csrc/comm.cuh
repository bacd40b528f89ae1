// comm.cuh — communicators for the row-sharded driver.
#pragma once
#include "internal.cuh"

namespace rpca {

struct NcclUniqueId {
  char internal[128];
};

// A communicator over the ranks that hold row shards of A.  Collectives are
// enqueued on (or, for the virtual communicator, synchronised with) the
// context stream; sums run in a fixed rank order.
struct Comm {
  int nranks = 1;
  int rank = 0;
  virtual ~Comm() = default;
  virtual bool graphable() const = 0;  // may the collectives be captured in a CUDA graph?
  virtual void allreduce_sum(Ctx& c, double* buf, size_t count) = 0;
  // recv = concat over ranks (rank order) of bytes_per_rank bytes from each rank's send
  virtual void allgather(Ctx& c, const void* send, void* recv, size_t bytes_per_rank) = 0;
};

rpca_status comm_unique_id(void* id, size_t bytes);
void comm_init(Ctx& c, int nranks, int rank, const void* id);
void comm_init_virtual(Ctx& c, void* group, int rank);
void* virtual_group_create(int nranks);
void virtual_group_destroy(void* group);
void comm_destroy(Ctx& c);

inline int comm_size(const Ctx& c) { return c.comm ? c.comm->nranks : 1; }
// With a communicator attached the collectives always run (a 1-rank NCCL
// communicator exercises the same calls as P ranks).
inline void allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (c.comm && count) c.comm->allreduce_sum(c, buf, count);
}
void allgather_bytes(Ctx& c, const void* send, void* recv, size_t bytes_per_rank);

}  // namespace rpca
