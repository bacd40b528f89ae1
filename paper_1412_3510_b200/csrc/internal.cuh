// internal.cuh — host-side interfaces between the driver and the kernel
// launchers of the randomized-PCA path.  Not part of the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace rpca {

// NVTX range over a host scope (one range per pass / step, for
// nsys or any NVTX tool; header-only NVTX3, inert without a tool attached).
// Inside a captured driver call the ranges mark the capture; with
// RPCA_FLAG_NO_GRAPH they bracket every launch sequence.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

constexpr int kMaxL = 64;  // widest sketch the l×l kernels (one CTA) support

// ---------------------------------------------------------------- workspace
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  size_t off = 0;
  static size_t align(size_t b) { return (b + 255) & ~size_t(255); }
  template <class T>
  T* get(size_t count) {
    size_t bytes = align(count * sizeof(T));
    RPCA_REQUIRE(off + bytes <= cap, RPCA_E_WORKSPACE, "workspace overflow (%zu + %zu > %zu)", off, bytes, cap);
    T* p = reinterpret_cast<T*>(base + off);
    off += bytes;
    return p;
  }
};

// Bytes a sequence of get<T>(count) calls needs (same rounding as Arena).
struct Sizer {
  size_t total = 0;
  template <class T>
  void add(size_t count) { total += Arena::align(count * sizeof(T)); }
};

struct Comm;  // multi-GPU communicator (comm.cu)

// sparse A (row-major CSR, int64 row pointers, int32 sorted column indices)
struct CsrA {
  const int64_t* ptr;
  const int32_t* idx;
  const void* vals;
  int dtype;
  int64_t rows, nnz;
  // heavy-row plan (csr.cu, built once per matrix and cached): rows with more
  // than kHeavyNnz nonzeros are cut into chunks, one warp each, whose partial
  // rows are summed in ascending chunk order.  hc[c] = (row, t0, t1);
  // hr[k] = (row, first chunk), hr[nhr] = (−1, nhc); hpart: nhc × kMaxL doubles
  const int64_t* hc = nullptr;
  int64_t nhc = 0;
  const int64_t* hr = nullptr;
  int64_t nhr = 0;
  double* hpart = nullptr;
};
constexpr int64_t kHeavyNnz = 4096;


// Optional per-launch timing (rpca_profile): an event is recorded on the
// context stream after every launch; a launch's duration is the gap to the
// previous event (launches are stream-serialised).
struct ProfRec {
  const char* name;
  cudaEvent_t ev;
};

// A captured driver call: replayed with cudaGraphLaunch when the same call
// (same pointers, shapes, flags) comes again — one launch instead of ~50.
struct CachedGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<ProfRec> marks;
  int64_t nlaunch = 0;
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t flags = 0;
  int num_sms = 148;
  // Workspace: context-owned (grown by cudaMalloc before a call when needed)
  // or caller-owned (rpca_set_workspace: never reallocated; too small ⇒
  // RPCA_E_WORKSPACE).  Its first `persist` bytes hold the cached CSR(Aᵀ)
  // and heavy-row plans of the last sparse A; call arenas start after them.
  char* ws = nullptr;
  size_t ws_cap = 0;
  bool ws_user = false;
  size_t persist = 0;
  // 256 bytes of device scratch allocated with the context: status words
  // (finite check, QR breakdown) and the CSR fingerprint
  char* dscratch = nullptr;
  int64_t launches = 0;
  Comm* comm = nullptr;
  int prof = 0;  // 0 off, 1 every launch, 2 the A-streaming pass kernels only
  const char* tag = nullptr;  // profile name for the pass kernels when used on thin blocks
  bool capturing = false;
  bool use_graphs = true;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  std::vector<std::pair<const char*, float>> prof_out;
  std::vector<std::pair<uint64_t, CachedGraph>> graphs;
  int* status_host = nullptr;  // pinned scratch for device status words
  cudaStream_t work = nullptr;   // private stream the drivers run (and capture) on
  // cached CSR(Aᵀ) of the last sparse A, at the start of the workspace; keyed
  // by the CSR pointers, shape AND a fingerprint of the arrays' contents
  // (csr_fingerprint, one read of the CSR per call), so a different matrix
  // at recycled addresses — or an in-place edit — rebuilds it
  struct TransposeCache {
    bool valid = false;
    uint64_t key = 0;
    CsrA T{};
    CsrA A{};                   // the cached matrix itself, with its heavy-row plan
  } tcache;
  // pointers into [ws, ws + persist) move with the workspace
  void rebase(char* old_base, char* new_base);
  // the workspace holds ≥ total bytes (keeping the persistent prefix)
  void reserve(size_t total);
  cudaEvent_t fence_in = nullptr, fence_out = nullptr;
  // second stream + events for collectives overlapped with compute (the tiled
  // sparse Aᵀ·Y all-reduce of driver.cu)
  cudaStream_t side = nullptr;
  std::vector<cudaEvent_t> side_ev;
  // out-of-core A (RPCA_FLAG_STREAM_A): host→device copy stream and the
  // ready / freed events of its two chunk buffers
  cudaStream_t h2d = nullptr;
  cudaEvent_t h2d_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // fp64 A·X on the int8 tensor cores (dense_ax_emu.cu): the row exponents of
  // the driver call's A, valid while that call runs (EmuScope)
  const int* emu_E = nullptr;
  const void* emu_A = nullptr;
  // centred A·X: where the pass kernel can, its epilogue writes the column
  // sums of Y per (128-row tile, 32-row quarter) here (the driver sets the
  // buffer, the fp32 pass sets the count) — no second read of Y for its mean
  double* ax_colpart = nullptr;
  int64_t ax_colpart_n = 0;
  // set by the driver when a call is re-run after a Cholesky-QR breakdown:
  // the final orthonormalisations use Householder TSQR (tsqr.cu)
  bool force_house = false;
  Arena arena(size_t bytes);  // ensures capacity, returns an arena over the workspace
};

// device status words in the context's scratch (reset by the drivers)
inline int* finite_flag(Ctx& c) { return reinterpret_cast<int*>(c.dscratch); }        // non-finite seen
inline int* breakdown_flag(Ctx& c) { return reinterpret_cast<int*>(c.dscratch + 4); }  // Cholesky-QR breakdown

void prof_mark(Ctx& c, const char* name);
// run a step-API body; with profiling on, harvest its launch marks
void profiled_step(Ctx& c, const std::function<void()>& body);
struct TagScope {
  Ctx& c;
  const char* prev;
  TagScope(Ctx& c_, const char* t) : c(c_), prev(c_.tag) { c.tag = t; }
  ~TagScope() { c.tag = prev; }
};

// the pass kernels over A (dense A·X / Aᵀ·Y on A itself, CSR SpMM) — the
// ones profile mode 2 brackets with events
inline bool is_pass_kernel(const char* name) {
  return (name[0] == 'a' && name[1] == 'x' && name[2] == '_') ||
         (name[0] == 'a' && name[1] == 't' && name[2] == 'y' && name[3] == '_' && name[4] != 'r') ||
         (name[0] == 'c' && name[1] == 's' && name[2] == 'r' && name[3] == '_' && name[4] == 's');
}
inline void count_launch(Ctx& c, int n = 1, const char* name = "misc") {
  c.launches += n;
  if (c.prof == 1 || (c.prof == 2 && !c.tag && is_pass_kernel(name))) prof_mark(c, name);
}
// before a pass-kernel launch: in mode 2 close the preceding interval ("gap")
inline void prof_pre(Ctx& c) {
  if (c.prof == 2 && !c.tag) prof_mark(c, "gap");
}

// ---------------------------------------------------------------- kernels
// omega.cu
// rows [row0, row0+rows) of the rows×cols Ω of PAPER.md (eq. i1), row-major
void omega(Ctx& c, uint64_t seed, uint32_t sid, int64_t rows, int64_t cols, int dist, int round32, double* out,
           int64_t row0 = 0);

// thin.cu — small kernels on thin blocks
// Packed operand layouts for the DMMA kernels (see dense_ax.cu / dense_aty.cu)
int64_t packx_elems(int64_t n, int l);   // doubles in the packed X of an n×l block
int64_t packy_elems(int64_t m, int l);   // doubles in the packed Y of an m×l block
void pack_x(Ctx& c, const double* X, int64_t n, int l, double* Xp);
void pack_y(Ctx& c, const double* Y, int64_t m, int l, double* Yp, const double* ymean = nullptr);
// v[j] = Σ_k a[k]·X[k][j] (a may be NULL ⇒ all-ones), fixed-order reduction
void weighted_colsum(Ctx& c, const double* a, const double* X, int64_t rows, int l, double* v, Arena& ar,
                     int64_t ldx = 0, double scale = 1.0);
// Y −= α·u·vᵀ (u = NULL ⇒ ones)
void sub_rank1(Ctx& c, double* Y, int64_t rows, int l, const double* u /*rows or NULL=ones*/, const double* v,
               double alpha = 1.0);
void colmeans_dense(Ctx& c, const void* A, int dtype, int64_t m, int64_t n, int64_t lda, int64_t m_total,
                    double* cmean, Arena& ar);
// Out (rows×k, ld ldo, dtype out_dtype) = In (rows×l) · W[:, :k] (W l×l) · diag(sign)
void thin_gemm(Ctx& c, const double* In, int64_t rows, int l, const double* W, int k, const double* sign,
               void* Out, int64_t ldo, int out_dtype, Arena& ar);
size_t thin_gemm_ws_bytes(int64_t rows, int l, int k);
// sign[j] = sign of the largest-|·| entry of column j of V (rows×k), lowest index on ties
void column_signs(Ctx& c, const double* V, int64_t rows, int k, int64_t ldv, double* sign, Arena& ar);
// same rule over a V whose rows [row0, row0+rows) are this rank's shard
void column_signs_sharded(Ctx& c, const double* V, int64_t rows, int64_t row0, int k, int64_t ldv, double* sign,
                          Arena& ar);
void copy_cast(Ctx& c, const double* src, void* dst, int64_t count, int dtype);
// dst (rows×k, ld ldd, dtype) = src (rows×k, ld k) · diag(sign)   (sign may be NULL)
void scale_cast(Ctx& c, const double* src, int64_t rows, int k, const double* sign, void* dst, int64_t ldd, int dtype);
// G (l×l) = Xᵀ·Y over rows (gram.cu: fp64 tensor cores, per-CTA partials summed in CTA order)
void gram(Ctx& c, const double* X, const double* Y, int64_t rows, int l, double* G, Arena& ar);
size_t gram_ws_bytes(Ctx& c, int64_t rows, int l);
// Out (rows×l) = (In + ν·Q)·M, ν read from device (Q may be NULL ⇒ Out = In·M)
void right_mult(Ctx& c, const double* In, const double* Q, const double* nu, const double* M, int64_t rows, int l,
                double* Out);
// y −= U·t  (U rows×k, ld ldu)
void rank_k_sub(Ctx& c, double* y, const double* U, int64_t ldu, const double* t, int64_t rows, int k);
// t ← t ⊙ S
void hadamard(Ctx& c, double* t, const double* S, int k);
// dst (rows × cols, ld ldd) ← src (ld lds), elements of es bytes (4 or 8)
void copy_rows(Ctx& c, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols, int es);
// Z[i] += W[i]
void add_into(Ctx& c, double* Z, const double* W, int64_t count);
// *flag = 1 if any of x[0..count) is NaN or ±Inf (flag untouched otherwise)
void finite_check(Ctx& c, const double* x, int64_t count, int* flag);

// dense_ax.cu / dense_aty.cu
struct DenseA {
  const void* a;
  int dtype;
  int64_t m, n, lda;  // m = local rows
};
size_t ax_ws_bytes(const DenseA& A, int l);
// Y = A·X [− 1·cxᵀ]  (cx = c·X, the centring correction of PAPER.md:430; may be NULL)
// upper: X is upper triangular (the DMMA path skips its zero blocks)
void dense_ax(Ctx& c, const DenseA& A, const double* X, int l, double* Y, Arena& ar, const double* cx = nullptr,
              bool upper = false);
// dense_ax_emu.cu — fp64 A·X as int8-digit products on tcgen05 (Ozaki scheme I)
bool emu_eligible(const DenseA& A, int l);
// E[i] = row i's exponent; wide (may be NULL, not cleared here) set to 1 if a
// row's largest |a| exceeds 1/8 of its Σ|a| (the emulation guard)
void row_exponents(Ctx& c, const DenseA& A, int* E, int* wide = nullptr);
size_t emu_ws_bytes(const DenseA& A, int l);
void dense_ax_emu(Ctx& c, const DenseA& A, const int* E, const double* X, int l, double* Y, Arena& ar);
size_t aty_ws_bytes(Ctx& c, const DenseA& A, int l);
// Z (n×l) = Aᵀ·(Y − 1·ymeanᵀ) [− cmean ⊗ colsum(Y)] (cmean, ymean may be NULL)
void dense_aty(Ctx& c, const DenseA& A, const double* Y, int l, const double* cmean, double* Z, Arena& ar,
               const double* ymean = nullptr);

// csr.cu — sparse A (row-major CSR, int64 row pointers, int32 sorted column indices)
// Y (rows×l) = A·(X − 1·xmeanᵀ)   (X has as many rows as A has columns; xmean may be NULL)
void csr_spmm(Ctx& c, const CsrA& A, const double* X, int l, double* Y, const double* xmean = nullptr);
// the two halves of csr_spmm: rows [r0, r1) except heavy ones, and the heavy rows
void csr_spmm_rows(Ctx& c, const CsrA& A, int64_t r0, int64_t r1, const double* X, int l, double* Y,
                   const double* xmean = nullptr);
void csr_spmm_heavy(Ctx& c, const CsrA& A, const double* X, int l, double* Y, const double* xmean = nullptr);
size_t csr_transpose_ws_bytes(const CsrA& A);
// upper bound of the device bytes csr_build_heavy_plan writes for A
size_t csr_heavy_plan_bytes(const CsrA& A);
// A's heavy-row plan built into mem (≥ csr_heavy_plan_bytes(A)); sets the plan
// fields of A.  host_ptr: A's row pointers on the host (else read from the
// device — synchronises the stream)
void csr_build_heavy_plan(Ctx& c, CsrA& A, char* mem, const int64_t* host_ptr = nullptr);
// order-independent 64-bit hash of A's row pointers, column indices and
// values (one read of the CSR; synchronises the stream)
uint64_t csr_fingerprint(Ctx& c, const CsrA& A);
// T = CSR(Aᵀ) (n rows) into caller buffers T.ptr (n+1), T.idx, T.vals (nnz); stable in rows
void csr_transpose(Ctx& c, const CsrA& A, int64_t n, CsrA& T, Arena& scratch);
// cmean[j] = (Σ_i A_ij)/m_total from CSR(Aᵀ), rows ascending
void csr_colmeans(Ctx& c, const CsrA& T, int64_t m_total, double* cmean);

// dense_f32_tc.cu — fp32 A on tcgen05 (3×TF32)
bool f32_tc_ok(const DenseA& A);
size_t ax_f32_ws_bytes(const DenseA& A, int l);
// Y = A·X [− 1·cxᵀ] (cx may be NULL)
void dense_ax_f32(Ctx& c, const DenseA& A, const double* X, int l, const double* cx, double* Y, Arena& ar);
inline int64_t ax_colpart_elems(int64_t m, int l) { return ((m + 127) / 128) * 4 * (int64_t)l; }

size_t aty_f32_ws_bytes(Ctx& c, const DenseA& A, int l);
// Z = Aᵀ·Y [− cmean·syᵀ]
void dense_aty_f32(Ctx& c, const DenseA& A, const double* Y, int l, const double* cmean, const double* sy,
                   double* Z, Arena& ar, const double* ymean = nullptr);
void aty_reduce_partials(Ctx& c, const double* part, int64_t U, int64_t P, int64_t cpc, int maxslots, int64_t n,
                         int l, int LP, const double* cmean, const double* sy, double* Z);

// tslu.cu
size_t lu_ws_bytes(int64_t m, int l);
// LU renormalisation of (Y − 1·muᵀ) when mu ≠ NULL (a pending centring, reading Q8)
void lu_renorm(Ctx& c, double* Y, int64_t m, int l, double* U_out, int64_t* piv_out, Arena& ar,
               const double* mu = nullptr);
// row shard [row0, row0+m) of a matrix distributed over the context's communicator
void lu_renorm_sharded(Ctx& c, double* Y, int64_t m, int64_t row0, int l, double* U_out, Arena& ar,
                       const double* mu = nullptr);

// tsqr.cu
size_t qr_ws_bytes(int64_t m, int l);
void qr(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar);

// cholqr.cu — LU-Cholesky-QR: Y ← Q (orthonormal, span Y), R (l×l upper, diag ≥ 0, Y = Q·R)
size_t orth_ws_bytes(int64_t m, int l);
size_t orth_ws_bytes(Ctx& c, int64_t m, int l);
void orthonormalize(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar, const double* mu = nullptr);
void orthonormalize_sharded(Ctx& c, double* Y, int64_t m, int64_t row0, int l, double* R_out, Arena& ar,
                            const double* mu = nullptr);
// the Householder fallback of the two above (Y − 1·muᵀ when mu ≠ NULL); the
// sharded form factors the local block, all-gathers the l×l R's, factors the
// stack redundantly and applies this rank's slice of its Q
size_t orth_house_ws_bytes(int64_t m, int l, int nranks);
void orthonormalize_house(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar, const double* mu = nullptr);
void orthonormalize_house_sharded(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar,
                                  const double* mu = nullptr);

// small.cu — one-CTA l×l kernels
// R (l×l) → Jacobi: R·W = Vr·diag(sigma); sigma sorted, Vr completed.
void jacobi_svd_small(Ctx& c, const double* R, int l, double* sigma, double* W, double* Vr);
// Nyström SHIFT_CHOL: from G = QᵀB1 (l×l) and fro2 = ‖B1‖_F²:
// B2 = sym(G), ν = u·√n·‖B1‖_F, C = chol(B2 + νI) with ν ×10 on failure (≤ 5
// retries); writes Minv = C⁻¹ (upper), nu, status (0 ok, 1 not PSD, 2 zero B1).
void nystrom_shift_chol(Ctx& c, const double* G, const double* fro2, int l, int64_t n, double unit_roundoff,
                        double* Minv, double* nu, int* status);
// Nyström SQRT: B2 = sym(G) = E·diag(μ)·Eᵀ (Jacobi), Minv =
// E·diag(μ^-1/2 or 0)·Eᵀ (cut-off 1e-12·sqrt(max μ)); status 1 if min μ < -1e-6·max|μ|.
void nystrom_sqrt(Ctx& c, const double* G, int l, double* Minv, double* nu, int* status);
// reig: sym(G) = E·diag(λ)·Eᵀ by Jacobi; lam (l) ordered by |λ| descending, signed; E (l×l) its columns
void sym_eig_abs(Ctx& c, const double* G, int l, double* lam, double* E);
// lam[j] = max(σ_j² − ν, 0)   (eq. finish), cast to dtype
void nystrom_lambda(Ctx& c, const double* sigma, const double* nu, int k, void* lam, int dtype);
// power-method scalar step: nz = sqrt(nz2); est = done ? est : (nz == 0 ? 0 : sqrt(nz));
// x = nz > 0 ? z/nz : 0
void power_step(Ctx& c, const double* nz2, double* z, double* x, int64_t n, double* est, int* done);

}  // namespace rpca
