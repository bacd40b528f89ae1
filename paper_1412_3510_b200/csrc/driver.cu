// driver.cu — host orchestration of the randomized PCA path and the C ABI
// (include/rpca.h).  Every arithmetic step runs in the kernels of this
// library; this file only validates arguments, plans the workspace and
// enqueues launches on the context's stream.
//
//   rpca_pca      — PAPER.md §2 eqs. (i1)-(i4) l.116-149, power iterations
//                   l.186-204, LU inside / QR last §5 l.382-425, centring and
//                   adjoint l.427-435.
//   rpca_eigens   — PAPER.md §3 l.214-282 (stabilised Nyström), self-adjoint
//                   loop l.386-412.
//   rpca_diffsnorm— PAPER.md §4 l.362-371.
#include <cstdarg>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>

#include "comm.cuh"

namespace rpca {

static thread_local std::string g_last_error;

void set_last_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

const char* last_error_cstr() { return g_last_error.c_str(); }

void prof_mark(Ctx& c, const char* name) {
  if (c.prof_used == c.prof_pool.size()) {
    cudaEvent_t e;
    RPCA_CUDA(cudaEventCreate(&e));
    c.prof_pool.push_back(e);
  }
  cudaEvent_t e = c.prof_pool[c.prof_used++];
  if (c.capturing) RPCA_CUDA(cudaEventRecordWithFlags(e, c.stream, cudaEventRecordExternal));
  else RPCA_CUDA(cudaEventRecord(e, c.stream));
  c.prof_recs.push_back(ProfRec{name, e});
}

void ensure_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> done;
  int dev = 0;
  RPCA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  auto key = std::make_pair(dev, kernel);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return;
  RPCA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done[key] = bytes;
}

namespace {

void harvest(Ctx& c, const std::vector<ProfRec>& marks) {
  for (size_t i = 1; i < marks.size(); ++i) {
    float ms = 0.f;
    RPCA_CUDA(cudaEventElapsedTime(&ms, marks[i - 1].ev, marks[i].ev));
    c.prof_out.emplace_back(marks[i].name, ms);
  }
}

struct KeyHasher {
  uint64_t h = 1469598103934665603ull;
  template <class T>
  KeyHasher& operator<<(const T& v) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
    for (size_t i = 0; i < sizeof(T); ++i) { h ^= p[i]; h *= 1099511628211ull; }
    return *this;
  }
};

}  // namespace

// A step API call (rpca_lu_renorm, rpca_qr, …) enqueued directly on the
// caller's stream: with profiling on, its launch marks are harvested here.
void profiled_step(Ctx& c, const std::function<void()>& body) {
  if (!c.prof) {
    body();
    return;
  }
  c.prof_recs.clear();
  c.prof_used = 0;
  prof_mark(c, "start");
  body();
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  harvest(c, c.prof_recs);
}

// Run `body` (which only enqueues work on c.stream) either directly or as a
// cached CUDA graph; then synchronise the stream and harvest profile marks.
template <class F>
void execute_on(Ctx& c, uint64_t key, bool graphable, F&& body) {
  const bool use_graph = graphable && c.use_graphs && !(c.flags & RPCA_FLAG_NO_GRAPH);
  key ^= (uint64_t)c.prof * 0x9E3779B97F4A7C15ull;
  if (use_graph) {
    for (auto& g : c.graphs)
      if (g.first == key) {
        RPCA_CUDA(cudaGraphLaunch(g.second.exec, c.stream));
        c.launches += g.second.nlaunch;
        RPCA_CUDA(cudaStreamSynchronize(c.stream));
        if (c.prof) harvest(c, g.second.marks);
        return;
      }
  }
  c.prof_recs.clear();
  c.prof_used = 0;
  const int64_t l0 = c.launches;
  if (use_graph) {
    RPCA_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
    c.capturing = true;
    cudaGraph_t graph = nullptr;
    try {
      if (c.prof) prof_mark(c, "start");
      body();
    } catch (...) {
      c.capturing = false;
      cudaStreamEndCapture(c.stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();
      throw;
    }
    c.capturing = false;
    RPCA_CUDA(cudaStreamEndCapture(c.stream, &graph));
    CachedGraph cg;
    RPCA_CUDA(cudaGraphInstantiate(&cg.exec, graph, 0));
    RPCA_CUDA(cudaGraphDestroy(graph));
    cg.marks = c.prof_recs;
    cg.nlaunch = c.launches - l0;
    if (c.graphs.size() >= 16) {
      for (auto& g : c.graphs) cudaGraphExecDestroy(g.second.exec);
      c.graphs.clear();
    }
    c.graphs.emplace_back(key, cg);
    RPCA_CUDA(cudaGraphLaunch(cg.exec, c.stream));
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    if (c.prof) harvest(c, cg.marks);
  } else {
    if (c.prof) prof_mark(c, "start");
    body();
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    if (c.prof) harvest(c, c.prof_recs);
  }
}

// Run `body` (which only enqueues work on c.stream) on the context's private
// non-blocking stream — fenced by events against the caller's stream, which
// may be the legacy default stream that cannot be captured — either directly
// or as a cached CUDA graph; then synchronise and harvest profile marks.
template <class F>
void execute(Ctx& c, uint64_t key, bool graphable, F&& body) {
  if (!c.work) {
    RPCA_CUDA(cudaStreamCreateWithFlags(&c.work, cudaStreamNonBlocking));
    RPCA_CUDA(cudaEventCreateWithFlags(&c.fence_in, cudaEventDisableTiming));
    RPCA_CUDA(cudaEventCreateWithFlags(&c.fence_out, cudaEventDisableTiming));
  }
  cudaStream_t user = c.stream;
  RPCA_CUDA(cudaEventRecord(c.fence_in, user));
  RPCA_CUDA(cudaStreamWaitEvent(c.work, c.fence_in, 0));
  c.stream = c.work;
  try {
    execute_on(c, key, graphable, body);
  } catch (...) {
    c.stream = user;
    throw;
  }
  c.stream = user;
  RPCA_CUDA(cudaEventRecord(c.fence_out, c.work));
  RPCA_CUDA(cudaStreamWaitEvent(user, c.fence_out, 0));
}

void drop_graphs(Ctx& c) {
  for (auto& g : c.graphs) cudaGraphExecDestroy(g.second.exec);
  c.graphs.clear();
}

void Ctx::rebase(char* old_base, char* new_base) {
  auto mv = [&](auto& p) {
    if (p) p = reinterpret_cast<std::remove_reference_t<decltype(p)>>(
               new_base + (reinterpret_cast<const char*>(p) - old_base));
  };
  for (CsrA* a : {&tcache.A, &tcache.T}) {
    mv(a->hc);
    mv(a->hr);
    mv(a->hpart);
  }
  mv(tcache.T.ptr);
  mv(tcache.T.idx);
  mv(tcache.T.vals);
}

void Ctx::reserve(size_t total) {
  if (total <= ws_cap) return;
  RPCA_REQUIRE(!ws_user, RPCA_E_WORKSPACE,
               "caller workspace too small: %zu bytes needed, %zu given (rpca_workspace_query)", total, ws_cap);
  const size_t want = total + (total >> 4) + (1 << 20);
  char* nws = nullptr;
  RPCA_CUDA(cudaStreamSynchronize(stream));
  for (auto& g : graphs) cudaGraphExecDestroy(g.second.exec);
  graphs.clear();
  const cudaError_t e = cudaMalloc(&nws, want);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    set_last_error("workspace cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
    throw Error{RPCA_E_NOMEM};
  }
  if (ws) {
    if (persist) RPCA_CUDA(cudaMemcpy(nws, ws, persist, cudaMemcpyDeviceToDevice));
    rebase(ws, nws);
    RPCA_CUDA(cudaFree(ws));
  }
  ws = nws;
  ws_cap = want;
}

Arena Ctx::arena(size_t bytes) {
  reserve(persist + bytes);
  Arena a;
  a.base = ws + persist;
  a.cap = ws_cap - persist;
  a.off = 0;
  return a;
}

namespace {

int elem_size(int dtype) { return dtype == RPCA_F64 ? 8 : 4; }

void validate_mat(const rpca_mat* A) {
  RPCA_REQUIRE(A, RPCA_E_ARG, "A is NULL");
  RPCA_REQUIRE(A->kind == RPCA_DENSE || A->kind == RPCA_CSR, RPCA_E_ARG, "bad kind %d", A->kind);
  RPCA_REQUIRE(A->dtype == RPCA_F64 || A->dtype == RPCA_F32, RPCA_E_ARG, "bad dtype %d", A->dtype);
  RPCA_REQUIRE(A->location == RPCA_DEVICE || A->location == RPCA_HOST, RPCA_E_ARG, "bad location");
  RPCA_REQUIRE(A->m >= 1 && A->n >= 1, RPCA_E_SHAPE, "m=%lld n=%lld", (long long)A->m, (long long)A->n);
  RPCA_REQUIRE(A->row0 >= 0 && A->m_local >= 0 && A->row0 + A->m_local <= A->m, RPCA_E_SHAPE, "bad row shard");
  if (A->kind == RPCA_DENSE) {
    RPCA_REQUIRE(A->a || A->m_local == 0, RPCA_E_ARG, "A.a is NULL");
    RPCA_REQUIRE(A->lda >= A->n, RPCA_E_SHAPE, "lda < n");
  } else {
    RPCA_REQUIRE(A->rowptr && (A->nnz == 0 || (A->colind && A->vals)), RPCA_E_ARG, "CSR arrays are NULL");
    RPCA_REQUIRE(A->nnz >= 0 && A->n <= INT32_MAX, RPCA_E_SHAPE, "bad nnz / n > 2^31-1");
  }
}

// Out-of-core A (§8(f) N4, RPCA_FLAG_STREAM_A; "a matrix A
// stored on disk"): a host dense A is streamed through two device buffers of
// `chunk` rows per pass.  stage() issues the H2D copy of a chunk on the copy
// stream once the buffer's previous user has finished (event `freed`) and
// makes the compute stream wait for it (event `ready`); release() marks the
// buffer free after the kernels enqueued on it.  Because the copy of chunk
// c+1 is enqueued before the compute stream reaches it, it overlaps the pass
// kernels on chunk c.
struct Streamer {
  const char* host = nullptr;
  int es = 8, dtype = RPCA_F64;
  int64_t lda = 0, m = 0, n = 0, chunk = 0;
  char* buf[2] = {nullptr, nullptr};
  int64_t q = 0;  // chunks staged so far in this call
  int64_t nchunks() const { return cdiv(m, chunk); }
  DenseA stage(Ctx& c, int64_t ci, int64_t* r0_out) {
    const int b = (int)(q & 1);
    if (q >= 2) RPCA_CUDA(cudaStreamWaitEvent(c.h2d, c.h2d_ev[2 + b], 0));
    const int64_t r0 = ci * chunk, rows = std::min(chunk, m - r0);
    RPCA_CUDA(cudaMemcpyAsync(buf[b], host + r0 * lda * es, (size_t)rows * lda * es, cudaMemcpyHostToDevice, c.h2d));
    RPCA_CUDA(cudaEventRecord(c.h2d_ev[b], c.h2d));
    RPCA_CUDA(cudaStreamWaitEvent(c.stream, c.h2d_ev[b], 0));
    if (c.prof == 1) prof_mark(c, "h2d_chunk");  // (profiling only: one record per staged chunk)
    *r0_out = r0;
    return DenseA{buf[b], dtype, rows, n, lda};
  }
  void release(Ctx& c) {
    RPCA_CUDA(cudaEventRecord(c.h2d_ev[2 + (q & 1)], c.stream));
    ++q;
  }
};

int64_t stream_chunk_rows(const rpca_mat* A) {
  const char* e = getenv("RPCA_STREAM_CHUNK_MB");
  const int64_t mb = e ? std::max<int64_t>(1, atoll(e)) : int64_t(256);
  const int64_t row_bytes = A->lda * (A->dtype == RPCA_F64 ? 8 : 4);
  return std::max<int64_t>(128, (mb << 20) / std::max<int64_t>(1, row_bytes) / 128 * 128);
}

bool streamed(const Ctx& c, const rpca_mat* A) {
  return (c.flags & RPCA_FLAG_STREAM_A) && A->location == RPCA_HOST && A->kind == RPCA_DENSE && A->m_local > 0;
}

// Device view of A's local shard (dense or CSR + cached CSR(Aᵀ), or a
// streamed host dense A).
struct MatV {
  bool csr = false;
  DenseA d{};
  CsrA a{}, at{};
  int64_t m = 0, n = 0;  // local rows, columns
  int dtype = RPCA_F64;
  Streamer* st = nullptr;
};

MatV probe_of(const rpca_mat* A) {
  MatV v;
  v.csr = A->kind == RPCA_CSR;
  v.m = A->m_local;
  v.n = A->n;
  v.dtype = A->dtype;
  v.d = DenseA{A->a, A->dtype, A->m_local, A->n, A->lda};
  v.a = CsrA{A->rowptr, A->colind, A->vals, A->dtype, A->m_local, A->nnz};
  return v;
}

// Device bytes of CSR(Aᵀ) (n+1 row pointers, nnz indices and values) plus the
// heavy-row plans of A and Aᵀ: the persistent prefix a sparse A keeps in the
// workspace, and the scratch its construction needs (above the prefix).
struct CsrLayout {
  size_t b_ptr, b_idx, b_val, b_plan_a, b_plan_t;
  size_t persist() const { return b_ptr + b_idx + b_val + b_plan_a + b_plan_t; }
};
CsrLayout csr_layout(const rpca_mat* A) {
  const CsrA probe{nullptr, nullptr, nullptr, A->dtype, A->m_local, A->nnz};
  return CsrLayout{Arena::align((A->n + 1) * 8), Arena::align(A->nnz * 4 + 4),
                   Arena::align(A->nnz * elem_size(A->dtype) + 8), csr_heavy_plan_bytes(probe),
                   csr_heavy_plan_bytes(probe)};
}
size_t csr_build_scratch(const rpca_mat* A) {
  const CsrA probe{nullptr, nullptr, nullptr, A->dtype, A->m_local, A->nnz};
  return csr_transpose_ws_bytes(probe) + 65536;
}

// Lay CSR(Aᵀ) and both plans out in `mem` (a CsrLayout's worth of bytes) and
// build them, using `scratch` for the transpose.  host_ptr: A's row pointers
// on the host when A was copied from there.
void build_transpose(Ctx& c, CsrA& src, int64_t n, char* mem, Arena& scratch, CsrA& T, const int64_t* host_ptr,
                     const CsrLayout& L) {
  T = CsrA{reinterpret_cast<int64_t*>(mem), reinterpret_cast<int32_t*>(mem + L.b_ptr), mem + L.b_ptr + L.b_idx,
           src.dtype, n, src.nnz};
  csr_transpose(c, src, n, T, scratch);
  char* plans = mem + L.b_ptr + L.b_idx + L.b_val;
  csr_build_heavy_plan(c, src, plans, host_ptr);
  csr_build_heavy_plan(c, T, plans + L.b_plan_a);
}

// A device CSR A's transpose is built once per matrix (before any graph
// capture) and cached at the start of the workspace, keyed by the pointers,
// shape and a fingerprint of the contents (pointers alone are
// recycled by allocators).  Host CSR inputs are copied and transposed inside
// each call instead (device_view).  Returns the fingerprint (0 for dense A).
uint64_t ensure_transpose(Ctx& c, const rpca_mat* A) {
  if (A->kind != RPCA_CSR || A->location != RPCA_DEVICE) return 0;
  CsrA src{A->rowptr, A->colind, A->vals, A->dtype, A->m_local, A->nnz};
  const uint64_t fp = csr_fingerprint(c, src);
  KeyHasher kh;
  kh << A->rowptr << A->colind << A->vals << A->m_local << A->n << A->nnz << A->dtype << fp;
  if (c.tcache.valid && c.tcache.key == kh.h) return fp;
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  drop_graphs(c);
  c.tcache.valid = false;
  c.persist = 0;
  const CsrLayout L = csr_layout(A);
  c.reserve(L.persist() + csr_build_scratch(A));
  Arena scratch{c.ws + L.persist(), c.ws_cap - L.persist(), 0};
  build_transpose(c, src, A->n, c.ws, scratch, c.tcache.T, nullptr, L);
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  c.tcache.A = src;
  c.tcache.key = kh.h;
  c.tcache.valid = true;
  c.persist = L.persist();
  return fp;
}

// A device dense A whose row stride (or base) the TMA pass kernels cannot
// address — lda·s not a multiple of 16 bytes, e.g. an odd n in fp64 — would
// fall to the CUDA-core fallback kernels (≈ 4× slower): the
// drivers copy it once per call into a padded layout instead (one read and
// one write of A at HBM speed, inside the call's graph).
int64_t padded_lda(const rpca_mat* A) {
  const int per16 = 16 / elem_size(A->dtype);
  return (A->lda + per16 - 1) / per16 * per16;
}
bool needs_pad(const rpca_mat* A) {
  if (A->kind != RPCA_DENSE || A->location != RPCA_DEVICE || A->m_local == 0) return false;
  static const bool off = getenv("RPCA_NO_PAD") != nullptr;  // ablation: the CUDA-core fallback
  return !off && (((A->lda * elem_size(A->dtype)) % 16) != 0 || (reinterpret_cast<uintptr_t>(A->a) & 15u) != 0);
}

MatV device_view(Ctx& c, const rpca_mat* A, Arena& ar, Streamer* st = nullptr, bool pad = true) {
  MatV v = probe_of(A);
  if (pad && needs_pad(A)) {
    const int es = elem_size(A->dtype);
    const int64_t ld = padded_lda(A);
    char* dev = ar.get<char>((size_t)A->m_local * ld * es);
    copy_rows(c, A->a, A->lda, dev, ld, A->m_local, A->n, es);  // (cudaMemcpy2D: 1.9 ms for C2's 3.2 GB)
    v.d.a = dev;
    v.d.lda = ld;
    return v;
  }
  if (st && streamed(c, A)) {
    if (!c.h2d) {
      RPCA_CUDA(cudaStreamCreateWithFlags(&c.h2d, cudaStreamNonBlocking));
      for (auto& e : c.h2d_ev) RPCA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const int es = elem_size(A->dtype);
    st->host = static_cast<const char*>(A->a);
    st->es = es;
    st->dtype = A->dtype;
    st->lda = A->lda;
    st->m = A->m_local;
    st->n = A->n;
    st->chunk = std::min<int64_t>(A->m_local, stream_chunk_rows(A));
    st->q = 0;
    for (auto& b : st->buf) b = ar.get<char>((size_t)st->chunk * A->lda * es);
    v.st = st;
    v.d.a = nullptr;
    return v;
  }
  if (v.csr && A->location == RPCA_DEVICE) {
    v.a = c.tcache.A;
    v.at = c.tcache.T;
    return v;
  }
  if (v.csr) {  // host CSR: copy the three arrays, then transpose and plan in the arena
    const int es = elem_size(A->dtype);
    int64_t* ptr = ar.get<int64_t>(A->m_local + 1);
    int32_t* idx = ar.get<int32_t>(A->nnz + 1);
    char* vals = ar.get<char>((size_t)A->nnz * es + 8);
    RPCA_CUDA(cudaMemcpyAsync(ptr, A->rowptr, (A->m_local + 1) * 8, cudaMemcpyHostToDevice, c.stream));
    RPCA_CUDA(cudaMemcpyAsync(idx, A->colind, (size_t)A->nnz * 4, cudaMemcpyHostToDevice, c.stream));
    RPCA_CUDA(cudaMemcpyAsync(vals, A->vals, (size_t)A->nnz * es, cudaMemcpyHostToDevice, c.stream));
    const CsrLayout L = csr_layout(A);
    char* mem = ar.get<char>(L.persist());
    const size_t mark = ar.off;
    v.a = CsrA{ptr, idx, vals, A->dtype, A->m_local, A->nnz};
    build_transpose(c, v.a, A->n, mem, ar, v.at, A->rowptr, L);
    ar.off = mark;
    return v;
  }
  if (A->location == RPCA_HOST && A->m_local > 0) {
    const size_t bytes = (size_t)A->m_local * A->lda * elem_size(A->dtype);
    void* dev = ar.get<char>(bytes);
    RPCA_CUDA(cudaMemcpyAsync(dev, A->a, bytes, cudaMemcpyHostToDevice, c.stream));
    v.d.a = dev;
  }
  return v;
}

// arena bytes device_view takes for a host A (+ the transpose scratch of a host CSR)
size_t host_copy_bytes(const Ctx& c, const rpca_mat* A) {
  if (needs_pad(A)) return (size_t)A->m_local * padded_lda(A) * elem_size(A->dtype) + 256;
  if (A->location != RPCA_HOST) return 0;
  if (streamed(c, A))
    return 2 * Arena::align((size_t)std::min<int64_t>(A->m_local, stream_chunk_rows(A)) * A->lda *
                            elem_size(A->dtype)) + 512;
  if (A->kind == RPCA_DENSE) return (size_t)A->m_local * A->lda * elem_size(A->dtype) + 256;
  Sizer s;
  s.add<int64_t>(A->m_local + 1);
  s.add<int32_t>(A->nnz + 1);
  s.add<char>((size_t)A->nnz * elem_size(A->dtype) + 8);
  s.add<char>(csr_layout(A).persist());
  return s.total + csr_build_scratch(A);
}

// The operator the range finder sketches (reading Q6): F = A, or Aᵀ if m < n.
// With a multi-rank communicator A's rows are sharded: vectors of length m
// are row shards, vectors of length n are replicated, and every Aᵀ·(·) —
// a sum over rows — is all-reduced.
// Implicit column centring as the projector P = I − 11ᵀ/m
// on the m-long side: (A − 1c)·X = P·(A·X) and (A − 1c)ᵀ·Y = Aᵀ·(P·Y), since
// c·X = 1ᵀ(A·X)/m.  Equal to the paper's rank-1 corrections in exact
// arithmetic (reading Q8) and it needs no column-means pass over A.
struct Op {
  MatV A;
  bool centered;
  int64_t m_total;  // global rows of A (the mean is over all ranks' rows)
  bool trans;
  bool sharded;
};

// mu = the column means of an m-long block over the global rows (this shard's
// sums, all-reduced, ÷ m_total).  P·Y = Y − 1·muᵀ is never formed: the mean
// is subtracted on load by the block's consumer (the LU renormalisation, the
// Aᵀ·Y operand preparation).
void column_mean(Ctx& c, const double* Y, int64_t rows, int l, int64_t m_total, bool sharded, double* mu, Arena& ar) {
  const size_t mark = ar.off;
  weighted_colsum(c, nullptr, Y, rows, l, mu, ar, 0, 1.0 / (double)m_total);
  if (sharded) allreduce_sum(c, mu, (size_t)l);
  ar.off = mark;
}

// Y = A·X [− 1·(c·X)]
void apply_ax(Ctx& c, const MatV& A, const double* cmean, const double* X, int l, double* Y, Arena& ar) {
  NvtxRange nv("pass A·X");
  const size_t mark = ar.off;
  double* cx = nullptr;
  if (cmean) {
    cx = ar.get<double>(kMaxL);
    weighted_colsum(c, cmean, X, A.n, l, cx, ar);
  }
  if (A.st) {  // out-of-core: row chunks are independent
    for (int64_t ci = 0; ci < A.st->nchunks(); ++ci) {
      int64_t r0 = 0;
      const DenseA Ac = A.st->stage(c, ci, &r0);
      const size_t m2 = ar.off;
      dense_ax(c, Ac, X, l, Y + r0 * l, ar, cx);
      ar.off = m2;
      A.st->release(c);
    }
  } else if (A.csr) {
    csr_spmm(c, A.a, X, l, Y);
    if (cx) sub_rank1(c, Y, A.m, l, nullptr, cx);
  } else {
    dense_ax(c, A.d, X, l, Y, ar, cx);
  }
  ar.off = mark;
}

// Z = Aᵀ·(Y − 1·ymeanᵀ) [− cᵀ·(1ᵀY)] — this shard's rows only
void apply_aty(Ctx& c, const MatV& A, const double* cmean, const double* Y, int l, double* Z, Arena& ar,
               const double* ymean = nullptr) {
  NvtxRange nv("pass Aᵀ·Y");
  const size_t mark = ar.off;
  if (A.st) {  // out-of-core: Z = Σ_chunks A_cᵀ·Y_c, added in chunk order
    double* Zc = ar.get<double>((size_t)A.n * l);
    for (int64_t ci = 0; ci < A.st->nchunks(); ++ci) {
      int64_t r0 = 0;
      const DenseA Ac = A.st->stage(c, ci, &r0);
      const size_t m2 = ar.off;
      dense_aty(c, Ac, Y + r0 * l, l, cmean, ci == 0 ? Z : Zc, ar, ymean);
      ar.off = m2;
      A.st->release(c);
      if (ci > 0) add_into(c, Z, Zc, A.n * l);
    }
  } else if (A.csr) {
    csr_spmm(c, A.at, Y, l, Z, ymean);
    if (cmean) {
      double* sy = ar.get<double>(kMaxL);
      weighted_colsum(c, nullptr, Y, A.m, l, sy, ar);
      sub_rank1(c, Z, A.n, l, cmean, sy);
    }
  } else {
    dense_aty(c, A.d, Y, l, cmean, Z, ar, ymean);
  }
  ar.off = mark;
}

// cmean = column means of the whole A (local sums ÷ m_total, all-reduced)
void colmeans(Ctx& c, const MatV& A, int64_t m_total, double* cmean, Arena& ar, bool sharded = false) {
  const size_t mark = ar.off;
  if (A.st) {
    double* cc = ar.get<double>(A.n);
    for (int64_t ci = 0; ci < A.st->nchunks(); ++ci) {
      int64_t r0 = 0;
      const DenseA Ac = A.st->stage(c, ci, &r0);
      const size_t m2 = ar.off;
      colmeans_dense(c, Ac.a, Ac.dtype, Ac.m, Ac.n, Ac.lda, m_total, ci == 0 ? cmean : cc, ar);
      ar.off = m2;
      A.st->release(c);
      if (ci > 0) add_into(c, cmean, cc, A.n);
    }
  } else if (A.csr) {
    csr_colmeans(c, A.at, m_total, cmean);
  } else {
    colmeans_dense(c, A.d.a, A.d.dtype, A.d.m, A.d.n, A.d.lda, m_total, cmean, ar);
  }
  ar.off = mark;
  if (sharded) allreduce_sum(c, cmean, A.n);
}

// F·X and F*·Y with the centring projector on the m-long side.  An m-long
// OUTPUT is returned uncentred together with its pending column means (in
// `mu`, the return value; NULL when nothing is pending) for the renormalisation
// that consumes it; an m-long INPUT is centred on load (its means are taken
// into `tmp`).
// Y = A·X (this shard's rows) and, centred, Y's column means over the global
// rows: from the pass epilogue's column sums where the pass writes them (the
// fp32 tcgen05 pass), else from one more read of Y
const double* ax_and_mean(Ctx& c, const Op& F, const double* X, int l, double* Y, double* mu, Arena& ar) {
  const size_t mark = ar.off;
  struct Reset {  // the request never outlives this pass, error or not
    Ctx& c;
    ~Reset() { c.ax_colpart = nullptr; c.ax_colpart_n = 0; }
  } reset{c};
  c.ax_colpart_n = 0;
  c.ax_colpart = (F.centered && !F.A.csr && !F.A.st) ? ar.get<double>(ax_colpart_elems(F.A.m, l)) : nullptr;
  apply_ax(c, F.A, nullptr, X, l, Y, ar);
  const double* part = c.ax_colpart;
  const int64_t np = c.ax_colpart_n;
  c.ax_colpart = nullptr;
  c.ax_colpart_n = 0;
  if (F.centered) {
    if (np > 0) {
      // the partials are an np × l row-major block: its column sums, fixed order
      weighted_colsum(c, nullptr, part, np, l, mu, ar, 0, 1.0 / (double)F.m_total);
      if (F.sharded) allreduce_sum(c, mu, (size_t)l);
    } else {
      column_mean(c, Y, F.A.m, l, F.m_total, F.sharded, mu, ar);
    }
  }
  ar.off = mark;
  return F.centered ? mu : nullptr;
}

// What the driver knows about an m-long INPUT block's column means: compute
// them (one read of the block), the block is exactly centred (P is the
// identity on it), or they are given (a block left unrenormalised, whose
// pending means its producer computed).
struct InMean {
  bool centred = false;
  const double* given = nullptr;
};

const double* input_mean(Ctx& c, const Op& F, const double* X, int l, double* tmp, Arena& ar, const InMean& im) {
  if (!F.centered || im.centred) return nullptr;
  if (im.given) return im.given;
  column_mean(c, X, F.A.m, l, F.m_total, F.sharded, tmp, ar);
  return tmp;
}

const double* fwd(Ctx& c, const Op& F, const double* X, int l, double* Y, double* mu, double* tmp, Arena& ar,
                  const InMean& im = InMean{}) {
  if (F.trans) {  // F = A_cᵀ: Y = Aᵀ·(P·X)
    const double* xm = input_mean(c, F, X, l, tmp, ar, im);
    apply_aty(c, F.A, nullptr, X, l, Y, ar, xm);
    if (F.sharded) allreduce_sum(c, Y, (size_t)F.A.n * l);
    return nullptr;
  }
  return ax_and_mean(c, F, X, l, Y, mu, ar);  // Y = P·(A·X), P pending
}
// Sharded sparse Z = Aᵀ·(P·Y) with its all-reduce (C5's n×l
// reduction is 256 MB, comparable to the SpMM itself): the heavy rows of
// CSR(Aᵀ) first, then the light rows in tiles of n/kTiles output rows, each
// tile's all-reduce issued on the context's second stream as soon as the tile
// is written, so the NCCL transfer of tile t overlaps the SpMM of tile t+1.
// Inside a captured call the fork/join events become graph edges.
constexpr int kAllreduceTiles = 8;

void csr_aty_allreduce_overlapped(Ctx& c, const CsrA& T, const double* Y, int l, double* Z, const double* ymean) {
  const int64_t n = T.rows;
  if (!c.side) RPCA_CUDA(cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking));
  while ((int)c.side_ev.size() < kAllreduceTiles + 1) {
    cudaEvent_t e;
    RPCA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.side_ev.push_back(e);
  }
  csr_spmm_heavy(c, T, Y, l, Z, ymean);
  const cudaStream_t main = c.stream;
  for (int t = 0; t < kAllreduceTiles; ++t) {
    const int64_t j0 = n * t / kAllreduceTiles, j1 = n * (t + 1) / kAllreduceTiles;
    csr_spmm_rows(c, T, j0, j1, Y, l, Z, ymean);
    RPCA_CUDA(cudaEventRecord(c.side_ev[t], main));
    RPCA_CUDA(cudaStreamWaitEvent(c.side, c.side_ev[t], 0));
    c.stream = c.side;
    try {
      allreduce_sum(c, Z + j0 * l, (size_t)(j1 - j0) * l);
    } catch (...) {
      c.stream = main;
      throw;
    }
    c.stream = main;
  }
  RPCA_CUDA(cudaEventRecord(c.side_ev[kAllreduceTiles], c.side));
  RPCA_CUDA(cudaStreamWaitEvent(main, c.side_ev[kAllreduceTiles], 0));
}

const double* adj(Ctx& c, const Op& F, const double* Y, int l, double* Z, double* mu, double* tmp, Arena& ar,
                  const InMean& im = InMean{}) {
  if (F.trans) return ax_and_mean(c, F, Y, l, Z, mu, ar);  // Z = P·(A·Y), P pending
  const double* ym = input_mean(c, F, Y, l, tmp, ar, im);  // Z = Aᵀ·(P·Y)
  if (F.sharded && F.A.csr && (size_t)F.A.n * l * 8 >= ((size_t)32 << 20)) {
    csr_aty_allreduce_overlapped(c, F.A.at, Y, l, Z, ym);
    return nullptr;
  }
  apply_aty(c, F.A, nullptr, Y, l, Z, ar, ym);
  if (F.sharded) allreduce_sum(c, Z, (size_t)F.A.n * l);
  return nullptr;
}

// §8(f) N2 on an out-of-core A: one interior power round of the
// RENORM_ODD schedule, Y = A·Z and Z' = Aᵀ·(P·Y), from ONE stream of A — the
// "halve the number of disk accesses" of PAPER.md:442-449: every chunk's
// Y_c = A_c·Z is followed at once by Z' += A_cᵀ·Y_c while A_c is resident.
// Centred, P·Y needs Y's global column means μ, known only after the last
// chunk, so the correction is applied in the paper's rank-1 form (PAPER.md:
// 430-435): Z' −= (Aᵀ1)·μᵀ = m·c_A·μᵀ, with A's column means c_A summed
// from the resident chunks of the first fused round.  Single-rank only.
void fused_round(Ctx& c, const Op& F, const double* Z, int l, double* Y, double* Zn, double* cA, bool have_cA,
                 double* mu, Arena& ar) {
  NvtxRange nv("fused pass Aᵀ(A·Z)");
  const MatV& A = F.A;
  const size_t mark = ar.off;
  double* Zc = ar.get<double>((size_t)A.n * l);
  double* cc = ar.get<double>(A.n);
  double* Zacc = Zn == Z ? ar.get<double>((size_t)A.n * l) : Zn;  // Z is read by every chunk's A·Z
  for (int64_t ci = 0; ci < A.st->nchunks(); ++ci) {
    int64_t r0 = 0;
    const DenseA Ac = A.st->stage(c, ci, &r0);
    const size_t m2 = ar.off;
    dense_ax(c, Ac, Z, l, Y + r0 * l, ar, nullptr);
    ar.off = m2;
    dense_aty(c, Ac, Y + r0 * l, l, nullptr, ci == 0 ? Zacc : Zc, ar, nullptr);
    ar.off = m2;
    if (F.centered && !have_cA) {
      colmeans_dense(c, Ac.a, Ac.dtype, Ac.m, Ac.n, Ac.lda, F.m_total, ci == 0 ? cA : cc, ar);
      ar.off = m2;
    }
    A.st->release(c);
    if (ci > 0) {
      add_into(c, Zacc, Zc, A.n * l);
      if (F.centered && !have_cA) add_into(c, cA, cc, A.n);
    }
  }
  if (F.centered) {
    column_mean(c, Y, A.m, l, F.m_total, false, mu, ar);
    sub_rank1(c, Zacc, A.n, l, cA, mu, (double)F.m_total);
  }
  if (Zacc != Zn) RPCA_CUDA(cudaMemcpyAsync(Zn, Zacc, sizeof(double) * A.n * l, cudaMemcpyDeviceToDevice, c.stream));
  ar.off = mark;
}

// The int8-digit emulation of a driver call's A·X passes (dense_ax_emu.cu):
// decided BEFORE the call's graph runs, from one read of A that yields the
// row exponents and the dynamic-range guard (row_exp_kernel; a synchronising
// read of one flag) — worth it from two A·X passes on.  A row whose largest
// |a| exceeds 1/8 of its Σ|a| keeps the call on the fp64 DMMA passes (ADVICE
// r1).  Device-resident dense fp64 A only (a host A is staged
// inside the call).  RPCA_NO_EMU=1 disables it.
struct EmuPlan {
  const int* E = nullptr;
  const void* A = nullptr;
  bool on() const { return E != nullptr; }
};

EmuPlan emu_prepare(Ctx& c, const rpca_mat* Am, int l, int ax_passes, Arena& ar) {
  static const bool off = getenv("RPCA_NO_EMU") != nullptr;
  EmuPlan p;
  const MatV A = probe_of(Am);
  if (off || A.csr || Am->location != RPCA_DEVICE || ax_passes < 2 || !emu_eligible(A.d, l)) return p;
  int* E = ar.get<int>(A.d.m);
  int* wide = reinterpret_cast<int*>(c.dscratch + 8);
  RPCA_CUDA(cudaMemsetAsync(wide, 0, 4, c.stream));
  row_exponents(c, A.d, E, wide);
  RPCA_CUDA(cudaMemcpyAsync(c.status_host + 2, wide, 4, cudaMemcpyDeviceToHost, c.stream));
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  if (c.status_host[2]) return p;
  p.E = E;
  p.A = A.d.a;
  return p;
}

// For the duration of a driver call's body: the emulation's row exponents
struct EmuScope {
  Ctx& c;
  EmuScope(Ctx& c_, const EmuPlan& p) : c(c_) {
    c.emu_E = p.E;
    c.emu_A = p.A;
  }
  ~EmuScope() {
    c.emu_E = nullptr;
    c.emu_A = nullptr;
  }
};

size_t op_ws(Ctx& c, const MatV& A, int l) {
  const size_t small = (size_t)(cdiv(std::max(A.m, A.n), 2048) + 4) * kMaxL * 8 * 2 + 65536;
  if (A.csr) return small;
  const size_t colpart = (size_t)ax_colpart_elems(A.m, kMaxL) * 8 + 256;  // centred A·X epilogue sums
  return std::max(ax_ws_bytes(A.d, l) + 4096 * 4 + colpart, aty_ws_bytes(c, A.d, l)) + small;
}

// A block of `rows` rows that is either whole (replicated) or this rank's
// shard starting at global row `row0` of a row-sharded block.
struct Blk {
  double* p;
  int64_t rows;
  bool sharded;
  int64_t row0;
};

// (mu: the block's pending column means, or NULL)
void renorm_lu(Ctx& c, const Blk& Y, int l, Arena& ar, const double* mu = nullptr) {
  NvtxRange nv("LU renormalisation");
  const size_t mark = ar.off;
  if (Y.sharded) lu_renorm_sharded(c, Y.p, Y.rows, Y.row0, l, nullptr, ar, mu);
  else lu_renorm(c, Y.p, Y.rows, l, nullptr, nullptr, ar, mu);
  ar.off = mark;
}
// the last renormalisation and the QR of Bᵀ: LU-Cholesky-QR
// (Householder TSQR instead when the call is re-run after a breakdown)
void renorm_qr(Ctx& c, const Blk& Y, int l, double* R, Arena& ar, const double* mu = nullptr) {
  NvtxRange nv("orthonormalisation");
  const size_t mark = ar.off;
  if (c.force_house) {
    if (Y.sharded) orthonormalize_house_sharded(c, Y.p, Y.rows, l, R, ar, mu);
    else orthonormalize_house(c, Y.p, Y.rows, l, R, ar, mu);
  } else if (Y.sharded) {
    orthonormalize_sharded(c, Y.p, Y.rows, Y.row0, l, R, ar, mu);
  } else {
    orthonormalize(c, Y.p, Y.rows, l, R, ar, mu);
  }
  ar.off = mark;
}

// Run a driver body (execute()) with the device status words reset, then read
// them: RPCA_FLAG_CHECK_FINITE + a non-finite value seen ⇒ RPCA_E_NONFINITE;
// a Cholesky-QR breakdown (cholqr.cu) ⇒ the whole call runs once more with
// Householder TSQR for its final orthonormalisations.  The body must carve its
// buffers from `ar` (rewound for the second run).
template <class F>
void run_checked(Ctx& c, uint64_t key, bool graphable, Arena& ar, F&& body) {
  const size_t mark = ar.off;
  for (int attempt = 0; attempt < 2; ++attempt) {
    ar.off = mark;
    c.force_house = attempt == 1;
    try {
      execute(c, key ^ (attempt ? 0x5BD1E9955BD1E995ull : 0ull), graphable, [&] {
        RPCA_CUDA(cudaMemsetAsync(c.dscratch, 0, 8, c.stream));
        body();
      });
    } catch (...) {
      c.force_house = false;
      throw;
    }
    c.force_house = false;
    RPCA_CUDA(cudaMemcpyAsync(c.status_host, c.dscratch, 8, cudaMemcpyDeviceToHost, c.work));
    RPCA_CUDA(cudaStreamSynchronize(c.work));
    RPCA_REQUIRE(!((c.flags & RPCA_FLAG_CHECK_FINITE) && c.status_host[0]), RPCA_E_NONFINITE,
                 "non-finite value in A (or an overflow in A·Ω) — RPCA_FLAG_CHECK_FINITE");
    if (!c.status_host[1]) return;
  }
}

// Without a communicator A must be whole; with one (any size), every rank
// holds a non-empty row shard and the sharded schedule runs.  Returns whether
// the call runs sharded.
bool check_shard(Ctx& c, const rpca_mat* A) {
  if (!c.comm) {
    RPCA_REQUIRE(A->row0 == 0 && A->m_local == A->m, RPCA_E_SHAPE,
                 "row shard given but no communicator (rpca_comm_init)");
    return false;
  }
  RPCA_REQUIRE(A->m_local >= 1, RPCA_E_SHAPE, "sharded call: every rank needs ≥ 1 row (m_local = 0)");
  return true;
}

bool graphable_comm(const Ctx& c) { return !c.comm || c.comm->graphable(); }

void sync_status(Ctx& c) { RPCA_CUDA(cudaStreamSynchronize(c.stream)); }

}  // namespace

// ============================================================ step APIs
void apply_step(Ctx& c, const rpca_mat* Am, const double* cm, int adjoint, const double* X, int64_t l, double* Y) {
  validate_mat(Am);
  RPCA_REQUIRE(Am->location == RPCA_DEVICE, RPCA_E_ARG, "apply: device A only");
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && X && Y, RPCA_E_SHAPE, "apply: bad l / NULL X, Y");
  ensure_transpose(c, Am);
  const MatV probe = probe_of(Am);
  Arena ar = c.arena(op_ws(c, probe, (int)l) + host_copy_bytes(c, Am) + 65536);
  const MatV A = device_view(c, Am, ar);
  const bool sh = check_shard(c, Am);
  profiled_step(c, [&] {
    if (adjoint) {
      apply_aty(c, A, cm, X, (int)l, Y, ar);
      if (sh) allreduce_sum(c, Y, (size_t)A.n * l);
    } else {
      apply_ax(c, A, cm, X, (int)l, Y, ar);
    }
  });
}

// Y = A·X through the int8-digit emulation (dense fp64 A, 24 < l ≤ 48): the
// path rpca_pca / rpca_eigens take for such A, exposed for tests and benches
void apply_emu_step(Ctx& c, const rpca_mat* Am, const double* X, int64_t l, double* Y) {
  validate_mat(Am);
  RPCA_REQUIRE(Am->location == RPCA_DEVICE, RPCA_E_ARG, "apply_int8emu: device A only");
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && X && Y, RPCA_E_SHAPE, "apply_int8emu: bad l / NULL X, Y");
  const MatV probe = probe_of(Am);
  RPCA_REQUIRE(!probe.csr && emu_eligible(probe.d, (int)l), RPCA_E_NOTIMPL,
               "apply_int8emu: needs a dense fp64 A (m ≥ 128, n ≥ 32) and 24 < l ≤ 48");
  Arena ar = c.arena(op_ws(c, probe, (int)l) + (size_t)probe.m * 4 + host_copy_bytes(c, Am) + 65536);
  const MatV A = device_view(c, Am, ar);
  int* E = ar.get<int>(A.d.m);
  profiled_step(c, [&] {
    row_exponents(c, A.d, E);  // the caller asked for the emulation: no dynamic-range guard
    EmuScope emu(c, EmuPlan{E, A.d.a});
    dense_ax(c, A.d, X, (int)l, Y, ar, nullptr);
  });
}

void colmeans_step(Ctx& c, const rpca_mat* Am, double* cm) {
  validate_mat(Am);
  RPCA_REQUIRE(Am->location == RPCA_DEVICE && cm, RPCA_E_ARG, "colmeans: device A and c only");
  ensure_transpose(c, Am);
  const MatV probe = probe_of(Am);
  Arena ar = c.arena((size_t)(cdiv(probe.m, 8192) + 2) * probe.n * 8 + host_copy_bytes(c, Am) + 65536);
  const MatV A = device_view(c, Am, ar);
  colmeans(c, A, Am->m, cm, ar, check_shard(c, Am));
}

void clear_cache(Ctx& c) {
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  c.tcache.valid = false;
  c.tcache.key = 0;
  c.persist = 0;
  drop_graphs(c);
}

// Arena bytes of one rpca_pca call (the workspace plan; vectors of length m are
// this rank's rows).  Used by the driver and by rpca_workspace_query.
size_t pca_arena_bytes(Ctx& c, const rpca_mat* Am, int64_t k, int64_t l, int64_t ldu, int64_t ldv) {
  const bool out_host = (c.flags & RPCA_FLAG_OUTPUTS_HOST) != 0;
  const int osz = elem_size(Am->dtype);
  const int64_t m = Am->m, n = Am->n, ml = Am->m_local;
  const int L = (int)l, K = (int)k;
  const MatV probe = probe_of(Am);
  const bool trans = m < n;
  const int64_t nin = trans ? ml : n, nout = trans ? n : ml;
  Sizer sz;
  sz.add<char>(host_copy_bytes(c, Am));
  sz.add<double>(nin * l);   // Zb
  sz.add<double>(nout * l);  // Yb
  sz.add<double>(4 * l * l + 4 * l);
  sz.add<double>(2 * kMaxL);  // column means
  sz.add<double>(std::max(nin, nout) * k);  // V-side temp
  sz.add<double>(k);                        // signs
  sz.add<int>(ml + 16);                     // row exponents (EmuScope)
  if (out_host) {
    sz.add<char>((size_t)ml * ldu * osz);
    sz.add<char>((size_t)n * ldv * osz);
    sz.add<char>((size_t)k * osz);
  }
  if (streamed(c, Am)) {  // chunk accumulators, A's column means, the fused round's buffers
    sz.add<double>(n);
    sz.add<double>(3 * n * l + 2 * n);
  }
  size_t scratch = op_ws(c, probe, L);
  scratch = std::max(scratch, lu_ws_bytes(std::max(nin, nout), L));
  scratch = std::max(scratch, orth_ws_bytes(c, std::max(nin, nout), L));
  scratch = std::max(scratch, qr_ws_bytes(std::max(nin, nout), L) + (size_t)4 * l * l * 8);  // Householder fallback
  scratch = std::max(scratch, (size_t)(cdiv(std::max(ml, n), 2048) + 2) * (n + 2 * k) * 8 + 65536);
  scratch = std::max(scratch, thin_gemm_ws_bytes(std::max(nin, nout), L, K) + 65536);
  return sz.total + scratch + 65536;
}

// ============================================================ rpca_pca
void pca(Ctx& c, const rpca_mat* Am, int64_t k, int raw, int its, int64_t l, uint64_t seed, void* U, int64_t ldu,
         void* S, void* V, int64_t ldv) {
  NvtxRange nv("rpca_pca");
  validate_mat(Am);
  const bool sh = check_shard(c, Am);
  if (l <= 0) l = k + 2;
  const int64_t mn = std::min(Am->m, Am->n);
  RPCA_REQUIRE(k >= 1 && l >= k && l <= mn && its >= 0, RPCA_E_SHAPE, "need 1 ≤ k ≤ l ≤ min(m,n), its ≥ 0");
  RPCA_REQUIRE(l <= kMaxL, RPCA_E_SHAPE, "l=%lld > %d not supported", (long long)l, kMaxL);
  RPCA_REQUIRE(U && S && V, RPCA_E_ARG, "U, S, V must not be NULL");
  RPCA_REQUIRE(ldu >= k && ldv >= k, RPCA_E_SHAPE, "ldu, ldv must be ≥ k");
  const int L = (int)l, K = (int)k;
  const bool out_host = (c.flags & RPCA_FLAG_OUTPUTS_HOST) != 0;
  const bool renorm_odd = (c.flags & RPCA_FLAG_RENORM_ODD) != 0;
  const int dist = (c.flags & RPCA_FLAG_UNIFORM_OMEGA) ? RPCA_UNIFORM : RPCA_GAUSSIAN;
  const int odt = Am->dtype, osz = elem_size(odt);
  const int64_t m = Am->m, n = Am->n, ml = Am->m_local, r0 = Am->row0;

  const bool trans = m < n;
  const int64_t nin = trans ? ml : n, nout = trans ? n : ml;
  const size_t need = pca_arena_bytes(c, Am, k, l, ldu, ldv);  // allocation happens before any capture
  const uint64_t fp = ensure_transpose(c, Am);
  Arena ar = c.arena(need);

  const EmuPlan ep = emu_prepare(c, Am, L, trans ? its + 2 : its + 1, ar);
  KeyHasher kh;
  kh << 1 << *Am << k << raw << its << l << seed << U << ldu << S << V << ldv << c.flags << c.ws << c.persist << fp
     << c.comm << ep.on();
  const bool graphable = Am->location == RPCA_DEVICE && !out_host && graphable_comm(c);

  Streamer stm;
  run_checked(c, kh.h, graphable, ar, [&] {
    const MatV dA = device_view(c, Am, ar, &stm);
    EmuScope emu(c, ep);
    double* Zb = ar.get<double>(nin * l);
    double* Yb = ar.get<double>(nout * l);
    double* R = ar.get<double>(l * l);
    double* W = ar.get<double>(l * l);
    double* Vr = ar.get<double>(l * l);
    double* sig = ar.get<double>(l);
    double* side = ar.get<double>(std::max(nin, nout) * k);
    double* sign = ar.get<double>(k);
    void *Ud = U, *Vd = V, *Sd = S;
    if (out_host) {
      Ud = ar.get<char>((size_t)ml * ldu * osz);
      Vd = ar.get<char>((size_t)n * ldv * osz);
      Sd = ar.get<char>((size_t)k * osz);
    }
    double* mub = ar.get<double>(2 * kMaxL);  // pending column means / input means
    // the m-long block is the sharded one
    const Blk Y{Yb, nout, sh && !trans, r0}, Z{Zb, nin, sh && trans, r0};
    Op F{dA, !raw, m, trans, sh};
    // Ω (nin×l; for the sketched Aᵀ, this rank's rows of the m×l Ω); the fp32
    // path consumes fl32(Ω) exactly as the oracle does
    omega(c, seed, 0u, nin, l, dist, odt == RPCA_F32, Zb, trans ? r0 : 0);
    const double* mu = fwd(c, F, Zb, L, Yb, mub, mub + kMaxL, ar);  // mu: Y's pending centring
    // a non-finite entry of A makes its row of A·Ω non-finite (Ω is finite and
    // nonzero): the check reads Y, not A
    if (c.flags & RPCA_FLAG_CHECK_FINITE) finite_check(c, Yb, nout * l, finite_flag(c));
    if (its == 0) renorm_qr(c, Y, L, nullptr, ar, mu);
    else renorm_lu(c, Y, L, ar, mu);
    // A renormalised m-long block is centred only up to the cancellation in
    // L = Y·M − 1·(μM) (|Y·M| ≫ |L| when A's column means dominate), and Aᵀ
    // amplifies a residual mean by m·c: its consumer re-derives the means
    // (skipping that read cost 1.8e-7 in σ on a centred parity case).
    const InMean cent{};
    // RENORM_ODD on an out-of-core A, one rank, m ≥ n: the interior rounds
    // are fused into one stream of A each (fused_round)
    const bool fuse = renorm_odd && dA.st && !trans && !sh && its >= 2;
    double* cA = fuse && F.centered ? ar.get<double>(n) : nullptr;
    for (int it = 1; it <= its; ++it) {
      if (fuse && it >= 2) {
        // the previous round's Y = A·Z was not formed separately: this pass
        // forms it and Z = Aᵀ·(P·Y) together
        fused_round(c, F, Zb, L, Yb, Zb, cA, it > 2, mub, ar);
        renorm_lu(c, Z, L, ar, nullptr);
      } else {
        const bool y_left = it > 1 && renorm_odd;  // Y skipped its LU: its means are pending in mu
        mu = adj(c, F, Yb, L, Zb, mub, mub + kMaxL, ar, y_left ? InMean{false, mu} : cent);
        renorm_lu(c, Z, L, ar, mu);
      }
      if (fuse && it < its) continue;  // Y = A·Z happens inside the next fused pass
      mu = fwd(c, F, Zb, L, Yb, mub, mub + kMaxL, ar, cent);
      // RPCA_FLAG_RENORM_ODD: the long-side block of an
      // interior round goes into the next F*·Y unrenormalised — the schedule
      // that lets F*(F·Z) stream in one pass; its pending centring travels
      // with it to the next adj()
      if (it < its && renorm_odd) continue;
      if (it < its) renorm_lu(c, Y, L, ar, mu);
      else renorm_qr(c, Y, L, nullptr, ar, mu);
    }
    // Bᵀ = F*·Q (eq. i2), Bᵀ = Q_B·R, R = Vr·Σ·Wᵀ ⇒ B = W Σ (Q_B Vr)ᵀ (eq. i3)
    mu = adj(c, F, Yb, L, Zb, mub, mub + kMaxL, ar, cent);
    renorm_qr(c, Z, L, R, ar, mu);
    jacobi_svd_small(c, R, L, sig, W, Vr);
    {
      const size_t mark = ar.off;
      // V (n×k, replicated) fixes the column signs; U is this rank's rows
      if (!trans) {
        // V = Q_B·Vr[:, :k] (n×k), U = Q·W[:, :k] (m×k)  (eq. i4)
        thin_gemm(c, Zb, nin, L, Vr, K, nullptr, side, k, RPCA_F64, ar);
        column_signs(c, side, n, K, k, sign, ar);
        scale_cast(c, side, n, K, sign, Vd, ldv, odt);
        thin_gemm(c, Yb, nout, L, W, K, sign, Ud, ldu, odt, ar);
      } else {
        // sketched Aᵀ: its "U" = Q·W is A's V (n×k); its "V" = Q_B·Vr is A's U
        thin_gemm(c, Yb, nout, L, W, K, nullptr, side, k, RPCA_F64, ar);
        column_signs(c, side, n, K, k, sign, ar);
        scale_cast(c, side, n, K, sign, Vd, ldv, odt);
        thin_gemm(c, Zb, nin, L, Vr, K, sign, Ud, ldu, odt, ar);
      }
      copy_cast(c, sig, Sd, k, odt);
      ar.off = mark;
    }
    if (out_host) {
      RPCA_CUDA(cudaMemcpyAsync(U, Ud, (size_t)ml * ldu * osz, cudaMemcpyDeviceToHost, c.stream));
      RPCA_CUDA(cudaMemcpyAsync(V, Vd, (size_t)n * ldv * osz, cudaMemcpyDeviceToHost, c.stream));
      RPCA_CUDA(cudaMemcpyAsync(S, Sd, (size_t)k * osz, cudaMemcpyDeviceToHost, c.stream));
    }
  });
}

// the self-adjoint indefinite eigendecomposition (rpca_reig) runs the eigens
// driver up to B2 = QᵀAQ, then a Jacobi eigendecomposition of it
constexpr int kReig = 2;

size_t eigens_arena_bytes(Ctx& c, const rpca_mat* Am, int64_t k, int64_t l, int64_t ldu) {
  const bool out_host = (c.flags & RPCA_FLAG_OUTPUTS_HOST) != 0;
  const int osz = elem_size(Am->dtype);
  const int64_t n = Am->n, ml = Am->m_local;
  const int P = comm_size(c);
  const int64_t pad = c.comm ? cdiv(n, P) : n;
  const int L = (int)l, K = (int)k;
  const MatV probe = probe_of(Am);
  Sizer sz;
  sz.add<char>(host_copy_bytes(c, Am));
  sz.add<double>(2 * P * pad * l + 2 * ml * l);
  sz.add<double>(6 * l * l + 8 * l + 16);
  sz.add<double>(ml * k + k);
  sz.add<int>(ml + 16);  // row exponents (EmuScope)
  if (out_host) {
    sz.add<char>((size_t)ml * ldu * osz);
    sz.add<char>((size_t)k * osz);
  }
  size_t scratch = op_ws(c, probe, L);
  scratch = std::max(scratch, lu_ws_bytes(ml, L));
  scratch = std::max(scratch, orth_ws_bytes(c, ml, L));
  scratch = std::max(scratch, qr_ws_bytes(ml, L) + (size_t)4 * l * l * 8);  // Householder fallback
  scratch = std::max(scratch, (size_t)(cdiv(n, 2048) + 2) * l * l * 8 + 65536 + (size_t)P * 3 * l * 8);
  scratch = std::max(scratch, thin_gemm_ws_bytes(ml, L, K) + gram_ws_bytes(c, ml, L) + 65536);
  return sz.total + scratch + 65536;
}

// ============================================================ rpca_eigens
// Row-sharded: the shards must be the uniform partition
// (rank r holds rows [r·⌈n/P⌉, min(n, (r+1)·⌈n/P⌉))) so that Q can be
// all-gathered into one n×l block for A_r·Q; B2 = Σ_r Q_rᵀB1_r and ‖B1‖_F²
// are all-reduced; U is returned for this rank's rows.
void eigens(Ctx& c, const rpca_mat* Am, int64_t k, int its, int64_t l, uint64_t seed, int variant, void* U,
            int64_t ldu, void* lam) {
  NvtxRange nv("rpca_eigens");
  validate_mat(Am);
  const bool sh = check_shard(c, Am);
  RPCA_REQUIRE(Am->m == Am->n, RPCA_E_SHAPE, "eigens needs a square A");
  RPCA_REQUIRE(variant == RPCA_SHIFT_CHOL || variant == RPCA_SQRT || variant == kReig, RPCA_E_ARG, "bad variant");
  if (l <= 0) l = k + 2;
  const int64_t n = Am->n, ml = Am->m_local, r0 = Am->row0;
  RPCA_REQUIRE(k >= 1 && l >= k && l <= n && its >= 0 && l <= kMaxL, RPCA_E_SHAPE, "bad k/l/its");
  RPCA_REQUIRE(U && lam && ldu >= k, RPCA_E_ARG, "bad outputs");
  const int P = comm_size(c), rank = c.comm ? c.comm->rank : 0;
  const int64_t pad = sh ? cdiv(n, P) : n;  // rows per gathered slot
  if (sh)
    RPCA_REQUIRE(r0 == rank * pad && ml == std::min(pad, n - r0), RPCA_E_SHAPE,
                 "sharded eigens: rank %d must hold rows [%lld, %lld) (uniform partition)", rank,
                 (long long)(rank * pad), (long long)std::min(n, (rank + 1) * pad));
  const int L = (int)l, K = (int)k;
  const bool out_host = (c.flags & RPCA_FLAG_OUTPUTS_HOST) != 0;
  const int dist = (c.flags & RPCA_FLAG_UNIFORM_OMEGA) ? RPCA_UNIFORM : RPCA_GAUSSIAN;
  const int odt = Am->dtype, osz = elem_size(odt);

  const size_t need = eigens_arena_bytes(c, Am, k, l, ldu);
  const uint64_t fp = ensure_transpose(c, Am);
  Arena ar = c.arena(need);

  const EmuPlan ep = emu_prepare(c, Am, L, its + 2, ar);
  KeyHasher kh;
  kh << 2 << *Am << k << its << l << seed << variant << U << ldu << lam << c.flags << c.ws << c.persist << fp
     << c.comm << ep.on();
  const bool graphable = Am->location == RPCA_DEVICE && !out_host && graphable_comm(c);
  // fixed buffers are carved before execute() so that graph replays (which do
  // not run the lambda) see the same pointers
  double* Qa = ar.get<double>(P * pad * l);  // gathered n×l Q (this rank's rows at slot `rank`)
  double* Qb = ar.get<double>(P * pad * l);
  double* B1 = ar.get<double>(ml * l);
  double* Fm = ar.get<double>(ml * l);
  double* G = ar.get<double>(l * l);
  double* Minv = ar.get<double>(l * l);
  double* R = ar.get<double>(l * l);
  double* W = ar.get<double>(l * l);
  double* Vr = ar.get<double>(l * l);
  double* sig = ar.get<double>(l);
  double* scal = ar.get<double>(8);  // [0] = ‖B1‖_F², [1] = ν
  int* status = ar.get<int>(4);
  void* Ud = U;
  void* Ld = lam;
  if (out_host) {
    Ud = ar.get<char>((size_t)ml * ldu * osz);
    Ld = ar.get<char>((size_t)k * osz);
  }
  const int64_t slot = (int64_t)rank * pad * l;
  auto signs = [&](const double* X, double* sign) {
    if (sh) column_signs_sharded(c, X, ml, r0, K, k, sign, ar);
    else column_signs(c, X, ml, K, k, sign, ar);
  };
  double* Qfin = ((its & 1) ? Qb : Qa) + slot;  // this rank's final Q after the loop's swaps
  Streamer stm;
  run_checked(c, kh.h, graphable, ar, [&] {
    const MatV dA = device_view(c, Am, ar, &stm);
    EmuScope emu(c, ep);
    double* Qf = Qa;  // gathered Q
    double* Qo = Qb;  // the other gather buffer
    double* side = ar.get<double>(ml * k);
    double* sign = ar.get<double>(k);
    auto gather = [&] { allgather_bytes(c, Qf + slot, Qf, sizeof(double) * pad * l); };
    RPCA_CUDA(cudaMemsetAsync(status, 0, sizeof(int), c.stream));
    // self-adjoint loop: Y = AΩ, then its × (Q = A·Q)
    omega(c, seed, 0u, n, l, dist, odt == RPCA_F32, Qo);  // the whole n×l Ω on every rank
    apply_ax(c, dA, nullptr, Qo, L, Qf + slot, ar);
    if (c.flags & RPCA_FLAG_CHECK_FINITE) finite_check(c, Qf + slot, ml * l, finite_flag(c));
    const Blk Q0{Qf + slot, ml, sh, r0};
    if (its == 0) renorm_qr(c, Q0, L, nullptr, ar);
    else renorm_lu(c, Q0, L, ar);
    for (int it = 1; it <= its; ++it) {
      gather();
      apply_ax(c, dA, nullptr, Qf, L, Qo + slot, ar);
      std::swap(Qf, Qo);
      const Blk Qi{Qf + slot, ml, sh, r0};
      if (it < its) renorm_lu(c, Qi, L, ar);
      else renorm_qr(c, Qi, L, nullptr, ar);
    }
    gather();
    apply_ax(c, dA, nullptr, Qf, L, B1, ar);  // (start) B1 = A·Q (this rank's rows)
    {
      const size_t mark = ar.off;
      // (second) B2 = QᵀB1 (symmetrised in the kernels below) on the fp64
      // tensor-core Gram kernel
      gram(c, Qf + slot, B1, ml, L, G, ar);
      if (sh) allreduce_sum(c, G, (size_t)l * l);
      if (variant == kReig) {
        // reig: T = sym(QᵀAQ) = E·Λ·Eᵀ,
        // U = Q·E[:, :k], λ signed, ordered by |λ| — Rayleigh–Ritz, no shift
        sym_eig_abs(c, G, L, sig, W);
        thin_gemm(c, Qf + slot, ml, L, W, K, nullptr, side, k, RPCA_F64, ar);
        signs(side, sign);
        scale_cast(c, side, ml, K, sign, Ud, ldu, odt);
        copy_cast(c, sig, Ld, k, odt);
        ar.off = mark;
        return;
      }
      if (variant == RPCA_SHIFT_CHOL) {
        weighted_colsum(c, B1, B1, ml * l, 1, scal, ar);  // ‖B1‖_F²
        if (sh) allreduce_sum(c, scal, 1);
        nystrom_shift_chol(c, G, scal, L, n, odt == RPCA_F32 ? 0x1p-23 : 0x1p-52, Minv, scal + 1, status);
        right_mult(c, B1, Qf + slot, scal + 1, Minv, ml, L, Fm);  // F = (B1 + νQ)·C⁻¹ (eq. pseudo)
      } else {
        nystrom_sqrt(c, G, L, Minv, scal + 1, status);
        right_mult(c, B1, nullptr, nullptr, Minv, ml, L, Fm);  // F = B1·C⁺
      }
      ar.off = mark;
    }
    // F = U S Wᵀ: Q_F R_F = F, R_F = Vr Σ Wᵀ ⇒ U = Q_F·Vr; Σ = S² (eq. finish)
    renorm_qr(c, Blk{Fm, ml, sh, r0}, L, R, ar);
    jacobi_svd_small(c, R, L, sig, W, Vr);
    {
      const size_t mark = ar.off;
      thin_gemm(c, Fm, ml, L, Vr, K, nullptr, side, k, RPCA_F64, ar);
      signs(side, sign);
      scale_cast(c, side, ml, K, sign, Ud, ldu, odt);
      nystrom_lambda(c, sig, scal + 1, K, Ld, odt);
      ar.off = mark;
    }
  });
  RPCA_CUDA(cudaMemcpyAsync(c.status_host, status, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  sync_status(c);
  const int st = *c.status_host;
  RPCA_REQUIRE(st != 1, RPCA_E_NOTPSD, "Nyström: B2 is not positive definite after the shifts (PAPER.md:262-273)");
  if (st == 2) {  // A·Q = 0: λ = 0, U = Q[:, :k] (DESIGN.md reading)
    const size_t mark = ar.off;
    double* sign = ar.get<double>(k);
    double* side = ar.get<double>(ml * k);
    RPCA_CUDA(cudaMemcpy2DAsync(side, k * 8, Qfin, l * 8, k * 8, ml, cudaMemcpyDeviceToDevice, c.stream));
    signs(side, sign);
    scale_cast(c, side, ml, K, sign, Ud, ldu, odt);
    RPCA_CUDA(cudaMemsetAsync(Ld, 0, (size_t)k * osz, c.stream));
    ar.off = mark;
  }
  if (out_host) {
    RPCA_CUDA(cudaMemcpyAsync(U, Ud, (size_t)ml * ldu * osz, cudaMemcpyDeviceToHost, c.stream));
    RPCA_CUDA(cudaMemcpyAsync(lam, Ld, (size_t)k * osz, cudaMemcpyDeviceToHost, c.stream));
  }
  sync_status(c);
}

// ============================================================ rpca_diffsnorm
// Row-sharded: x, z (length n) are replicated, y (length m) and U are this
// rank's rows; z — linear in y — is all-reduced once per iteration.
size_t diffsnorm_arena_bytes(Ctx& c, const rpca_mat* Am, int64_t k) {
  const int64_t n = Am->n, ml = Am->m_local;
  Sizer sz;
  sz.add<char>(host_copy_bytes(c, Am));
  sz.add<double>(2 * n + ml + n + k + 64);
  const size_t scratch = op_ws(c, probe_of(Am), 1) + (size_t)(cdiv(std::max(ml, n), 2048) + 2) * (n + 64) * 8;
  return sz.total + scratch + 65536;
}

void diffsnorm(Ctx& c, const rpca_mat* Am, int raw, const double* U, int64_t ldu, const double* S, const double* V,
               int64_t ldv, int64_t k, int its, uint64_t seed, double* out) {
  NvtxRange nv("rpca_diffsnorm");
  validate_mat(Am);
  const bool sh = check_shard(c, Am);
  RPCA_REQUIRE(k >= 0 && its >= 1 && out, RPCA_E_SHAPE, "bad k/its/out");
  RPCA_REQUIRE(k == 0 || (U && S && V && ldu >= k && ldv >= k), RPCA_E_ARG, "bad factors");
  const int64_t m = Am->m, n = Am->n, ml = Am->m_local;
  const size_t need = diffsnorm_arena_bytes(c, Am, k);
  const uint64_t fp = ensure_transpose(c, Am);
  Arena ar = c.arena(need);
  KeyHasher kh;
  kh << 3 << *Am << raw << U << ldu << S << V << ldv << k << its << seed << c.ws << c.persist << fp << c.comm;
  double* x = ar.get<double>(n);
  double* z = ar.get<double>(n);
  double* y = ar.get<double>(ml);
  double* cmean = ar.get<double>(n);
  double* t = ar.get<double>(std::max<int64_t>(k, 1));
  double* sc = ar.get<double>(8);  // [0] nz2, [1] est, [2] scratch
  int* done = ar.get<int>(4);
  kh << c.flags;
  Streamer stm;
  run_checked(c, kh.h, Am->location == RPCA_DEVICE && graphable_comm(c), ar, [&] {
    const MatV dA = device_view(c, Am, ar, &stm);
    if (!raw) {
      const size_t mark = ar.off;
      colmeans(c, dA, m, cmean, ar, sh);
      ar.off = mark;
    }
    const double* cm = raw ? nullptr : cmean;
    RPCA_CUDA(cudaMemsetAsync(done, 0, 4 * sizeof(int), c.stream));
    RPCA_CUDA(cudaMemsetAsync(sc, 0, 8 * sizeof(double), c.stream));
    omega(c, seed, 1u, n, 1, RPCA_GAUSSIAN, 0, z);
    {
      const size_t mark = ar.off;
      weighted_colsum(c, z, z, n, 1, sc, ar);
      ar.off = mark;
    }
    // normalise the start vector (est/done of this call go to scratch slots)
    power_step(c, sc, z, x, n, sc + 2, done + 1);
    for (int it = 0; it < its; ++it) {
      const size_t mark = ar.off;
      apply_ax(c, dA, cm, x, 1, y, ar);  // y = A x [− 1 (c·x)]
      if (k > 0) {                       // y −= U (S ⊙ (Vᵀx))
        weighted_colsum(c, x, V, n, (int)k, t, ar, ldv);
        hadamard(c, t, S, (int)k);
        rank_k_sub(c, y, U, ldu, t, ml, (int)k);
      }
      if (it == 0 && (c.flags & RPCA_FLAG_CHECK_FINITE)) finite_check(c, y, ml, finite_flag(c));
      apply_aty(c, dA, cm, y, 1, z, ar);  // z = Aᵀ y [− cᵀ (1ᵀy)]
      if (k > 0) {                        // z −= V (S ⊙ (Uᵀy))
        weighted_colsum(c, y, U, ml, (int)k, t, ar, ldu);
        hadamard(c, t, S, (int)k);
        rank_k_sub(c, z, V, ldv, t, n, (int)k);
      }
      if (sh) allreduce_sum(c, z, n);
      weighted_colsum(c, z, z, n, 1, sc, ar);  // ‖z‖²
      power_step(c, sc, z, x, n, sc + 1, done);
      ar.off = mark;
    }
  });
  RPCA_CUDA(cudaMemcpyAsync(c.status_host, sc + 1, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  sync_status(c);
  memcpy(out, c.status_host, sizeof(double));
}

// ============================================================ workspace API
// Bytes a call needs: a device CSR's persistent CSR(Aᵀ) prefix plus the larger
// of its construction scratch and the call's arena (include/rpca.h).
size_t workspace_query(Ctx& c, int op, const rpca_mat* Am, int64_t k, int64_t l, int its) {
  validate_mat(Am);
  RPCA_REQUIRE(its >= 0, RPCA_E_SHAPE, "its < 0");
  if (l <= 0) l = k + 2;
  size_t arena = 0;
  switch (op) {
    case RPCA_OP_PCA:
      RPCA_REQUIRE(k >= 1 && l >= k && l <= kMaxL, RPCA_E_SHAPE, "bad k / l");
      arena = pca_arena_bytes(c, Am, k, l, k, k);
      break;
    case RPCA_OP_EIGENS:
    case RPCA_OP_REIG:
      RPCA_REQUIRE(k >= 1 && l >= k && l <= kMaxL, RPCA_E_SHAPE, "bad k / l");
      arena = eigens_arena_bytes(c, Am, k, l, k);
      break;
    case RPCA_OP_DIFFSNORM:
      RPCA_REQUIRE(k >= 0, RPCA_E_SHAPE, "bad k");
      arena = diffsnorm_arena_bytes(c, Am, k);
      break;
    case RPCA_OP_APPLY:
      RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "bad l");
      arena = std::max(op_ws(c, probe_of(Am), (int)l) + (size_t)Am->m_local * 4,
                       (size_t)(cdiv(Am->m_local, 8192) + 2) * Am->n * 8) + host_copy_bytes(c, Am) + 65536;
      break;
    default: RPCA_REQUIRE(false, RPCA_E_ARG, "bad op %d", op);
  }
  if (Am->kind == RPCA_CSR && Am->location == RPCA_DEVICE)
    return csr_layout(Am).persist() + std::max(csr_build_scratch(Am), arena);
  return arena;
}

void set_workspace(Ctx& c, void* ptr, size_t bytes) {
  RPCA_REQUIRE(!ptr || (reinterpret_cast<uintptr_t>(ptr) & 255) == 0, RPCA_E_ARG,
               "workspace must be 256-byte aligned");
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  drop_graphs(c);
  c.tcache.valid = false;
  c.persist = 0;
  if (c.ws && !c.ws_user) RPCA_CUDA(cudaFree(c.ws));
  c.ws = static_cast<char*>(ptr);
  c.ws_cap = ptr ? bytes : 0;
  c.ws_user = ptr != nullptr;
}

}  // namespace rpca
