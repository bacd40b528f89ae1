// comm.cu — the multi-GPU plumbing of SURVEY.md §8(e): rows of A are sharded
// across ranks (one process per GPU), A·X stays local, Aᵀ·Y and the small
// l×l Grams are summed with NCCL all-reduce over NVLink/NVSwitch and the
// TSLU candidates are exchanged with all-gather.  NCCL is loaded at run time
// (dlopen of the libnccl.so.2 PyTorch brings), so single-GPU users never load it.
//
// VirtualComm runs P ranks as P contexts (one host thread each) on ONE GPU
// for testing the sharded algorithms: every collective synchronises the
// caller's stream, meets the other ranks at a host barrier, and moves data
// with device copies / a fixed-order sum kernel.  No kernel ever waits on
// another rank's kernel (B200_PROFILING.md: ranks must not spin on each other
// on one device).
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

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

struct NcclComm : Comm {
  void* handle = nullptr;
  // NCCL collectives are stream-captured into the driver call's CUDA graph
  // (one graph launch per PCA at N > 1 too); RPCA_NCCL_GRAPH=0 launches the
  // call eagerly instead.  A 1-rank communicator exercises the captured path
  // on one GPU (tests/test_gpu_sharded.py).
  bool graph = true;
  bool graphable() const override { return graph; }
  void allreduce_sum(Ctx& c, double* buf, size_t count) override {
    check(nccl().allreduce(buf, buf, count, kNcclFloat64, kNcclSum, handle, c.stream), "ncclAllReduce");
  }
  void allgather(Ctx& c, const void* send, void* recv, size_t bytes) override {
    check(nccl().allgather(send, recv, bytes, kNcclInt8, handle, c.stream), "ncclAllGather");
  }
  ~NcclComm() override {
    if (handle) nccl().destroy(handle);
  }
};

// ------------------------------------------------------------------ virtual
struct Group {
  int n;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptrs;
  double* scratch = nullptr;
  size_t scratch_count = 0;
  explicit Group(int n_) : n(n_), ptrs(n_, nullptr) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

__global__ void sum_ranks_kernel(const double* const* __restrict__ src, int n, size_t count, double* __restrict__ dst) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += src[r][i];  // fixed rank order
    dst[i] = s;
  }
}

struct VirtualComm : Comm {
  Group* g = nullptr;
  bool graphable() const override { return false; }
  void allreduce_sum(Ctx& c, double* buf, size_t count) override {
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    g->ptrs[rank] = buf;
    g->barrier();
    if (rank == 0) {
      if (g->scratch_count < count) {
        if (g->scratch) RPCA_CUDA(cudaFree(g->scratch));
        RPCA_CUDA(cudaMalloc(&g->scratch, count * sizeof(double) + g->n * sizeof(double*)));
        g->scratch_count = count;
      }
      const double** table = reinterpret_cast<const double**>(g->scratch + g->scratch_count);
      RPCA_CUDA(cudaMemcpyAsync(table, g->ptrs.data(), g->n * sizeof(double*), cudaMemcpyHostToDevice, c.stream));
      sum_ranks_kernel<<<(unsigned)std::min<size_t>(cdiv(count, 256), 1024), 256, 0, c.stream>>>(table, g->n, count,
                                                                                                 g->scratch);
      RPCA_CHECK_LAUNCH();
      RPCA_CUDA(cudaStreamSynchronize(c.stream));
    }
    g->barrier();
    RPCA_CUDA(cudaMemcpyAsync(buf, g->scratch, count * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    g->barrier();
  }
  void allgather(Ctx& c, const void* send, void* recv, size_t bytes) override {
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    g->ptrs[rank] = send;
    g->barrier();
    for (int r = 0; r < g->n; ++r)
      RPCA_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + r * bytes, g->ptrs[r], bytes, cudaMemcpyDeviceToDevice,
                                c.stream));
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    g->barrier();
  }
};

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
  NcclComm* cm = new NcclComm();
  const char* g = getenv("RPCA_NCCL_GRAPH");
  cm->graph = !(g && g[0] == '0');  // captured by default; RPCA_NCCL_GRAPH=0 opts out
  cm->nranks = nranks;
  cm->rank = rank;
  NcclUniqueId u;
  memcpy(&u, id, sizeof(u));
  const int r = nccl().init(&cm->handle, nranks, u, rank);
  if (r != 0) {
    delete cm;
    check(r, "ncclCommInitRank");
  }
  c.comm = cm;
}

void* virtual_group_create(int nranks) {
  RPCA_REQUIRE(nranks >= 1 && nranks <= 64, RPCA_E_ARG, "virtual group size %d", nranks);
  return new Group(nranks);
}

void virtual_group_destroy(void* group) {
  Group* g = static_cast<Group*>(group);
  if (g && g->scratch) cudaFree(g->scratch);
  delete g;
}

void comm_init_virtual(Ctx& c, void* group, int rank) {
  Group* g = static_cast<Group*>(group);
  RPCA_REQUIRE(g && rank >= 0 && rank < g->n, RPCA_E_ARG, "bad virtual group / rank");
  if (c.comm) comm_destroy(c);
  VirtualComm* vc = new VirtualComm();
  vc->g = g;
  vc->nranks = g->n;
  vc->rank = rank;
  c.comm = vc;
}

void comm_destroy(Ctx& c) {
  delete c.comm;
  c.comm = nullptr;
}

void allgather_bytes(Ctx& c, const void* send, void* recv, size_t bytes_per_rank) {
  if (!c.comm) {
    if (send != recv) RPCA_CUDA(cudaMemcpyAsync(recv, send, bytes_per_rank, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  c.comm->allgather(c, send, recv, bytes_per_rank);
}

}  // namespace rpca
