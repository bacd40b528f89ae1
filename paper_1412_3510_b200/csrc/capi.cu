// capi.cu — the extern "C" entry points of include/rpca.h.  Each one maps
// C++ exceptions of the driver to an rpca_status; no arithmetic here.
#include <cstring>
#include <new>
#include <string>

#include "comm.cuh"
#include "internal.cuh"

struct rpca_ctx : rpca::Ctx {};

namespace rpca {
void pca(Ctx&, const rpca_mat*, int64_t, int, int, int64_t, uint64_t, void*, int64_t, void*, void*, int64_t);
void eigens(Ctx&, const rpca_mat*, int64_t, int, int64_t, uint64_t, int, void*, int64_t, void*);
void diffsnorm(Ctx&, const rpca_mat*, int, const double*, int64_t, const double*, const double*, int64_t, int64_t,
               int, uint64_t, double*);
const char* last_error_cstr();
void apply_step(Ctx&, const rpca_mat*, const double*, int, const double*, int64_t, double*);
void apply_emu_step(Ctx&, const rpca_mat*, const double*, int64_t, double*);
void colmeans_step(Ctx&, const rpca_mat*, double*);
void clear_cache(Ctx&);
size_t workspace_query(Ctx&, int, const rpca_mat*, int64_t, int64_t, int);
void set_workspace(Ctx&, void*, size_t);
}  // namespace rpca

namespace {

template <class F>
rpca_status guard(F&& f) {
  try {
    f();
    return RPCA_OK;
  } catch (const rpca::Error& e) {
    return e.code;
  } catch (const std::bad_alloc&) {
    rpca::set_last_error("host allocation failed");
    return RPCA_E_NOMEM;
  } catch (...) {
    rpca::set_last_error("unknown exception");
    return RPCA_E_CUDA;
  }
}

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};


}  // namespace

extern "C" {

rpca_status rpca_ctx_create(rpca_ctx** out, int device, void* stream, uint32_t flags) {
  if (!out) return RPCA_E_ARG;
  return guard([&] {
    int ndev = 0;
    RPCA_CUDA(cudaGetDeviceCount(&ndev));
    RPCA_REQUIRE(device >= 0 && device < ndev, RPCA_E_ARG, "device %d out of range (%d devices)", device, ndev);
    DeviceScope ds(device);
    cudaDeviceProp prop;
    RPCA_CUDA(cudaGetDeviceProperties(&prop, device));
    RPCA_REQUIRE(prop.major == 10, RPCA_E_ARG, "device %d is sm_%d%d; this library is built for sm_100a", device,
                 prop.major, prop.minor);
    rpca_ctx* c = new rpca_ctx();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    c->flags = flags;
    c->num_sms = prop.multiProcessorCount;
    if (cudaMallocHost(&c->status_host, 64) != cudaSuccess || cudaMalloc(&c->dscratch, 256) != cudaSuccess) {
      (void)cudaGetLastError();
      if (c->status_host) cudaFreeHost(c->status_host);
      delete c;
      rpca::set_last_error("context scratch allocation failed");
      throw rpca::Error{RPCA_E_NOMEM};
    }
    *out = c;
  });
}

rpca_status rpca_ctx_destroy(rpca_ctx* c) {
  if (!c) return RPCA_OK;
  return guard([&] {
    DeviceScope ds(c->device);
    if (c->comm) rpca::comm_destroy(*c);
    cudaStreamSynchronize(c->stream);
    for (auto& g : c->graphs) cudaGraphExecDestroy(g.second.exec);
    for (auto e : c->prof_pool) cudaEventDestroy(e);
    if (c->status_host) cudaFreeHost(c->status_host);
    if (c->side) {
      cudaStreamSynchronize(c->side);
      cudaStreamDestroy(c->side);
    }
    for (auto e : c->side_ev) cudaEventDestroy(e);
    if (c->h2d) {
      cudaStreamSynchronize(c->h2d);
      cudaStreamDestroy(c->h2d);
      for (auto e : c->h2d_ev) cudaEventDestroy(e);
    }
    if (c->work) {
      cudaStreamSynchronize(c->work);
      cudaStreamDestroy(c->work);
      cudaEventDestroy(c->fence_in);
      cudaEventDestroy(c->fence_out);
    }
    if (c->ws && !c->ws_user) cudaFree(c->ws);
    if (c->dscratch) cudaFree(c->dscratch);
    delete c;
  });
}

rpca_status rpca_ctx_set_stream(rpca_ctx* c, void* stream) {
  if (!c) return RPCA_E_ARG;
  c->stream = static_cast<cudaStream_t>(stream);
  return RPCA_OK;
}

rpca_status rpca_ctx_set_flags(rpca_ctx* c, uint32_t flags) {
  if (!c) return RPCA_E_ARG;
  if (flags & ~(uint32_t)(RPCA_FLAG_UNIFORM_OMEGA | RPCA_FLAG_OUTPUTS_HOST | RPCA_FLAG_CHECK_FINITE | RPCA_FLAG_NO_GRAPH |
                          RPCA_FLAG_RENORM_ODD | RPCA_FLAG_STREAM_A))
    return RPCA_E_ARG;
  c->flags = flags;
  return RPCA_OK;
}

rpca_status rpca_ctx_sync(rpca_ctx* c) {
  if (!c) return RPCA_E_ARG;
  return guard([&] { RPCA_CUDA(cudaStreamSynchronize(c->stream)); });
}

rpca_status rpca_workspace_size(rpca_ctx* c, size_t* bytes) {
  if (!c || !bytes) return RPCA_E_ARG;
  *bytes = c->ws_cap;
  return RPCA_OK;
}

rpca_status rpca_workspace_query(rpca_ctx* c, int op, const rpca_mat* A, int64_t k, int64_t l, int its,
                                 size_t* bytes) {
  if (!c || !A || !bytes) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    *bytes = rpca::workspace_query(*c, op, A, k, l, its);
  });
}

rpca_status rpca_set_workspace(rpca_ctx* c, void* dptr, size_t bytes) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::set_workspace(*c, dptr, bytes);
  });
}

rpca_status rpca_launch_count(rpca_ctx* c, int64_t* count) {
  if (!c || !count) return RPCA_E_ARG;
  *count = c->launches;
  return RPCA_OK;
}

rpca_status rpca_profile_begin(rpca_ctx* c) { return rpca_profile_begin_mode(c, RPCA_PROFILE_ALL); }

rpca_status rpca_profile_begin_mode(rpca_ctx* c, int mode) {
  if (!c || (mode != RPCA_PROFILE_ALL && mode != RPCA_PROFILE_PASSES)) return RPCA_E_ARG;
  return guard([&] {
    c->prof_out.clear();
    c->prof = mode;
  });
}

rpca_status rpca_profile_end(rpca_ctx* c, char* buf, size_t cap, size_t* needed) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    c->prof = 0;
    RPCA_CUDA(cudaStreamSynchronize(c->stream));
    std::string out;
    char line[160];
    for (auto& r : c->prof_out) {
      snprintf(line, sizeof(line), "%s\t%.6f\n", r.first, r.second);
      out += line;
    }
    if (needed) *needed = out.size() + 1;
    if (buf && cap) {
      const size_t n = std::min(cap - 1, out.size());
      memcpy(buf, out.data(), n);
      buf[n] = 0;
    }
  });
}

const char* rpca_strerror(rpca_status s) {
  switch (s) {
    case RPCA_OK: return "ok";
    case RPCA_E_ARG: return "invalid argument";
    case RPCA_E_SHAPE: return "invalid shape";
    case RPCA_E_NONFINITE: return "non-finite input";
    case RPCA_E_NOTPSD: return "matrix is not positive semidefinite";
    case RPCA_E_CUDA: return "CUDA error";
    case RPCA_E_NCCL: return "NCCL error";
    case RPCA_E_WORKSPACE: return "workspace too small";
    case RPCA_E_NOTIMPL: return "not implemented";
    case RPCA_E_NOMEM: return "out of memory";
  }
  return "unknown status";
}

const char* rpca_last_error(void) { return rpca::last_error_cstr(); }

rpca_status rpca_comm_unique_id(void* id, size_t bytes) {
  return guard([&] {
    rpca_status s = rpca::comm_unique_id(id, bytes);
    if (s != RPCA_OK) throw rpca::Error{s};
  });
}

rpca_status rpca_comm_init(rpca_ctx* c, int nranks, int rank, const void* id) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::comm_init(*c, nranks, rank, id);
  });
}

rpca_status rpca_virtual_group_create(int nranks, void** group) {
  return guard([&] {
    RPCA_REQUIRE(group, RPCA_E_ARG, "group is NULL");
    *group = rpca::virtual_group_create(nranks);
  });
}

rpca_status rpca_virtual_group_destroy(void* group) {
  return guard([&] { rpca::virtual_group_destroy(group); });
}

rpca_status rpca_comm_init_virtual(rpca_ctx* c, void* group, int rank) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::comm_init_virtual(*c, group, rank);
  });
}

rpca_status rpca_omega(rpca_ctx* c, uint64_t seed, uint32_t stream_id, int64_t rows, int64_t cols, int dist,
                       int round_f32, double* out) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    RPCA_REQUIRE(rows >= 0 && cols >= 0, RPCA_E_SHAPE, "negative shape");
    RPCA_REQUIRE(dist == RPCA_GAUSSIAN || dist == RPCA_UNIFORM, RPCA_E_ARG, "bad dist");
    RPCA_REQUIRE(out || rows * cols == 0, RPCA_E_ARG, "out is NULL");
    DeviceScope ds(c->device);
    rpca::omega(*c, seed, stream_id, rows, cols, dist, round_f32, out);
  });
}

rpca_status rpca_colmeans(rpca_ctx* c, const rpca_mat* A, double* cm) {
  if (!c || !A || !cm) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::colmeans_step(*c, A, cm);
  });
}

rpca_status rpca_apply(rpca_ctx* c, const rpca_mat* A, const double* cm, int adjoint, const double* X, int64_t l,
                       double* Y) {
  if (!c || !A || !X || !Y) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::apply_step(*c, A, cm, adjoint, X, l, Y);
  });
}

rpca_status rpca_apply_int8emu(rpca_ctx* c, const rpca_mat* A, const double* X, int64_t l, double* Y) {
  if (!c || !A || !X || !Y) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::apply_emu_step(*c, A, X, l, Y);
  });
}

rpca_status rpca_ctx_clear_cache(rpca_ctx* c) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::clear_cache(*c);
  });
}

rpca_status rpca_lu_renorm(rpca_ctx* c, double* Y, int64_t m, int64_t l, double* U, int64_t* piv) {
  if (!c || !Y) return RPCA_E_ARG;
  return guard([&] {
    RPCA_REQUIRE(l >= 1 && l <= rpca::kMaxL && m >= l, RPCA_E_SHAPE, "need 1 ≤ l ≤ 64, m ≥ l");
    DeviceScope ds(c->device);
    rpca::Arena ar = c->arena(rpca::lu_ws_bytes(m, (int)l) + 65536);
    rpca::profiled_step(*c, [&] { rpca::lu_renorm(*c, Y, m, (int)l, U, piv, ar); });
  });
}

rpca_status rpca_qr(rpca_ctx* c, double* Y, int64_t m, int64_t l, double* R) {
  if (!c || !Y) return RPCA_E_ARG;
  return guard([&] {
    RPCA_REQUIRE(l >= 1 && l <= rpca::kMaxL && m >= l, RPCA_E_SHAPE, "need 1 ≤ l ≤ 64, m ≥ l");
    DeviceScope ds(c->device);
    rpca::Arena ar = c->arena(rpca::qr_ws_bytes(m, (int)l) + 65536);
    rpca::profiled_step(*c, [&] { rpca::qr(*c, Y, m, (int)l, R, ar); });
  });
}

rpca_status rpca_orthonormalize(rpca_ctx* c, double* Y, int64_t m, int64_t l, double* R, int* used_householder) {
  if (!c || !Y) return RPCA_E_ARG;
  return guard([&] {
    RPCA_REQUIRE(l >= 1 && l <= rpca::kMaxL && m >= l, RPCA_E_SHAPE, "need 1 ≤ l ≤ 64, m ≥ l");
    DeviceScope ds(c->device);
    const size_t need = std::max(rpca::orth_ws_bytes(*c, m, (int)l), rpca::orth_house_ws_bytes(m, (int)l, 1));
    rpca::Arena ar = c->arena(need + (size_t)m * l * 8 + 65536);
    double* Yin = ar.get<double>((size_t)m * l);  // the input, for the fallback
    RPCA_CUDA(cudaMemcpyAsync(Yin, Y, (size_t)m * l * 8, cudaMemcpyDeviceToDevice, c->stream));
    RPCA_CUDA(cudaMemsetAsync(rpca::breakdown_flag(*c), 0, 4, c->stream));
    rpca::profiled_step(*c, [&] { rpca::orthonormalize(*c, Y, m, (int)l, R, ar); });
    RPCA_CUDA(cudaMemcpyAsync(c->status_host, rpca::breakdown_flag(*c), 4, cudaMemcpyDeviceToHost, c->stream));
    RPCA_CUDA(cudaStreamSynchronize(c->stream));
    const int broke = c->status_host[0];
    if (used_householder) *used_householder = broke;
    if (broke) {
      RPCA_CUDA(cudaMemcpyAsync(Y, Yin, (size_t)m * l * 8, cudaMemcpyDeviceToDevice, c->stream));
      rpca::profiled_step(*c, [&] { rpca::orthonormalize_house(*c, Y, m, (int)l, R, ar); });
      RPCA_CUDA(cudaStreamSynchronize(c->stream));
    }
  });
}

rpca_status rpca_small_svd(rpca_ctx* c, const double* G, int64_t n, int64_t l, double* Vt, double* sigma,
                           double* W) {
  if (!c || !G || !Vt || !sigma || !W) return RPCA_E_ARG;
  return guard([&] {
    RPCA_REQUIRE(l >= 1 && l <= rpca::kMaxL && n >= l, RPCA_E_SHAPE, "need 1 ≤ l ≤ 64, n ≥ l");
    DeviceScope ds(c->device);
    rpca::Sizer s;
    s.add<double>(n * l);
    s.add<double>(2 * l * l);
    rpca::Arena ar = c->arena(s.total + std::max(rpca::orth_ws_bytes(*c, n, (int)l),
                                                 rpca::thin_gemm_ws_bytes(n, (int)l, (int)l)) + 65536);
    double* Qb = ar.get<double>(n * l);
    double* R = ar.get<double>(l * l);
    double* Vr = ar.get<double>(l * l);
    RPCA_CUDA(cudaMemcpyAsync(Qb, G, sizeof(double) * n * l, cudaMemcpyDeviceToDevice, c->stream));
    rpca::orthonormalize(*c, Qb, n, (int)l, R, ar);
    rpca::jacobi_svd_small(*c, R, (int)l, sigma, W, Vr);
    rpca::thin_gemm(*c, Qb, n, (int)l, Vr, (int)l, nullptr, Vt, l, RPCA_F64, ar);
  });
}

rpca_status rpca_pca(rpca_ctx* c, const rpca_mat* A, int64_t k, int raw, int its, int64_t l, uint64_t seed, void* U,
                     int64_t ldu, void* S, void* V, int64_t ldv) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::pca(*c, A, k, raw, its, l, seed, U, ldu, S, V, ldv);
  });
}

rpca_status rpca_eigens(rpca_ctx* c, const rpca_mat* A, int64_t k, int its, int64_t l, uint64_t seed, int variant,
                        void* U, int64_t ldu, void* lam) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::eigens(*c, A, k, its, l, seed, variant, U, ldu, lam);
  });
}

rpca_status rpca_reig(rpca_ctx* c, const rpca_mat* A, int64_t k, int its, int64_t l, uint64_t seed, void* U,
                      int64_t ldu, void* lam) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::eigens(*c, A, k, its, l, seed, 2 /* kReig */, U, ldu, lam);
  });
}

rpca_status rpca_diffsnorm(rpca_ctx* c, const rpca_mat* A, int raw, const double* U, int64_t ldu, const double* S,
                           const double* V, int64_t ldv, int64_t k, int its, uint64_t seed, double* out) {
  if (!c) return RPCA_E_ARG;
  return guard([&] {
    DeviceScope ds(c->device);
    rpca::diffsnorm(*c, A, raw, U, ldu, S, V, ldv, k, its, seed, out);
  });
}

}  // extern "C"
