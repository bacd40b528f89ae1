// comm.cu — the multi-GPU plumbing of SURVEY.md §8(e): rows of A are sharded
// across ranks (one process per GPU), A·X stays local, Aᵀ·Y and the small
// l×l reductions are summed with NCCL all-reduce over NVLink/NVSwitch and the
// TSLU/TSQR candidates are exchanged with all-gather.  NCCL is loaded at run
// time (dlopen of the libnccl.so.2 PyTorch already brings), so the library
// has no link-time NCCL dependency and single-GPU users never load it.
#include <dlfcn.h>

#include <cstring>

#include "comm.cuh"

namespace rpca {
namespace {

typedef int (*fn_getid)(void*);
typedef int (*fn_init)(void**, int, NcclUniqueId, int);
typedef int (*fn_destroy)(void*);
typedef int (*fn_allreduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*fn_allgather)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef const char* (*fn_errstr)(int);

struct Nccl {
  void* h = nullptr;
  fn_getid getid = nullptr;
  fn_init init = nullptr;
  fn_destroy destroy = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_allgather allgather = nullptr;
  fn_errstr errstr = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  if (!n.h) {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!n.h) n.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.h) break;
    }
    if (!n.h) {
      const char* env = getenv("RPCA_NCCL_PATH");
      if (env) n.h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    }
    RPCA_REQUIRE(n.h, RPCA_E_NCCL, "cannot load libnccl.so.2 (import torch first or set RPCA_NCCL_PATH)");
    n.getid = (fn_getid)dlsym(n.h, "ncclGetUniqueId");
    n.init = (fn_init)dlsym(n.h, "ncclCommInitRank");
    n.destroy = (fn_destroy)dlsym(n.h, "ncclCommDestroy");
    n.allreduce = (fn_allreduce)dlsym(n.h, "ncclAllReduce");
    n.allgather = (fn_allgather)dlsym(n.h, "ncclAllGather");
    n.errstr = (fn_errstr)dlsym(n.h, "ncclGetErrorString");
    RPCA_REQUIRE(n.getid && n.init && n.destroy && n.allreduce && n.allgather, RPCA_E_NCCL, "NCCL symbols missing");
  }
  return n;
}

void check(int r, const char* what) {
  if (r != 0) {
    set_last_error("%s failed: %s", what, nccl().errstr ? nccl().errstr(r) : "?");
    throw Error{RPCA_E_NCCL};
  }
}

constexpr int kNcclFloat64 = 8;  // ncclFloat64
constexpr int kNcclInt8 = 0;     // ncclInt8 (bytes)
constexpr int kNcclSum = 0;      // ncclSum

}  // namespace

rpca_status comm_unique_id(void* id, size_t bytes) {
  RPCA_REQUIRE(id && bytes >= sizeof(NcclUniqueId), RPCA_E_ARG, "unique id buffer must hold 128 bytes");
  NcclUniqueId u;
  check(nccl().getid(&u), "ncclGetUniqueId");
  memcpy(id, &u, sizeof(u));
  return RPCA_OK;
}

void comm_init(Ctx& c, int nranks, int rank, const void* id) {
  RPCA_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks && id, RPCA_E_ARG, "bad rank/nranks/id");
  if (c.comm) comm_destroy(c);
  Comm* cm = new Comm();
  cm->nranks = nranks;
  cm->rank = rank;
  NcclUniqueId u;
  memcpy(&u, id, sizeof(u));
  check(nccl().init(&cm->handle, nranks, u, rank), "ncclCommInitRank");
  c.comm = cm;
}

void comm_destroy(Ctx& c) {
  if (!c.comm) return;
  if (c.comm->handle) nccl().destroy(c.comm->handle);
  delete c.comm;
  c.comm = nullptr;
}

void allreduce_sum(Ctx& c, double* buf, size_t count) {
  if (!c.comm || c.comm->nranks == 1 || count == 0) return;
  check(nccl().allreduce(buf, buf, count, kNcclFloat64, kNcclSum, c.comm->handle, c.stream), "ncclAllReduce");
}

void allgather_bytes(Ctx& c, const void* send, void* recv, size_t bytes_per_rank) {
  if (!c.comm || c.comm->nranks == 1) {
    if (send != recv) RPCA_CUDA(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  check(nccl().allgather(send, recv, bytes_per_rank, kNcclInt8, c.comm->handle, c.stream), "ncclAllGather");
}

}  // namespace rpca
