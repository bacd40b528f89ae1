/*
 * rpca.h — C ABI of the B200-native randomized PCA / SVD hot path of
 * Szlam, Kluger & Tygert, "An implementation of a randomized algorithm for
 * principal component analysis", arXiv:1412.3510 (PAPER.md in the survey).
 *
 * Every entry point takes plain pointers and sizes.  Unless a field says
 * otherwise, matrices are ROW-MAJOR, thin blocks (m×l, n×l, l×l) are fp64
 * with leading dimension = number of columns, and all buffers are DEVICE
 * memory of the context's GPU owned by the caller.  The library keeps no
 * pointer to caller data past the return of a call, except the workspace
 * given to rpca_set_workspace (the cached CSR(Aᵀ) lives in the workspace).
 * Calls enqueue on the context's stream; calls that return host scalars or
 * statuses computed on the device synchronise that stream (noted per call).
 *
 * Errors: every call returns an rpca_status; RPCA_OK = 0.  On error the
 * outputs are unspecified, and rpca_last_error() gives a message.  Invalid
 * shapes never launch a kernel.  A context is not thread-safe.
 */
#ifndef RPCA_H_
#define RPCA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RPCA_OK = 0,
  RPCA_E_ARG = 1,       /* null pointer, bad enum, bad flags, misaligned pointer */
  RPCA_E_SHAPE = 2,     /* k<1, l<k, l>min(m,n), its<0, m,n<1, bad shard, non-square for eigens */
  RPCA_E_NONFINITE = 3, /* non-finite input seen (only with RPCA_FLAG_CHECK_FINITE) */
  RPCA_E_NOTPSD = 4,    /* Nyström: shifted Cholesky failed after all retries / SQRT found a
                           negative eigenvalue of B2 below -1e-6·‖B2‖ */
  RPCA_E_CUDA = 5,
  RPCA_E_NCCL = 6,
  RPCA_E_WORKSPACE = 7,
  RPCA_E_NOTIMPL = 8,
  RPCA_E_NOMEM = 9
} rpca_status;

/* matrix kinds / dtypes / locations */
enum { RPCA_DENSE = 0, RPCA_CSR = 1 };
enum { RPCA_F64 = 0, RPCA_F32 = 1 };
enum { RPCA_DEVICE = 0, RPCA_HOST = 1 };

/* Ω distributions (PAPER.md:163-168 normal; PAPER.md:437-440 uniform [-1,1]) */
enum { RPCA_GAUSSIAN = 0, RPCA_UNIFORM = 1 };

/* Nyström stabilisations (§3, l.257-282) */
enum { RPCA_SHIFT_CHOL = 0, RPCA_SQRT = 1 };

/* flags for rpca_ctx_create / the drivers */
#define RPCA_FLAG_UNIFORM_OMEGA 0x1u  /* draw Ω from U[-1,1] instead of N(0,1) */
#define RPCA_FLAG_OUTPUTS_HOST 0x2u   /* U, S, V / lam are HOST buffers (copied back inside the call) */
#define RPCA_FLAG_CHECK_FINITE 0x4u   /* non-finite input → RPCA_E_NONFINITE: detected from the
                                         first thin block (A·Ω; a NaN/Inf entry of A makes its row
                                         non-finite since Ω is finite and nonzero; an overflow in A·Ω
                                         reports the same), no extra pass over A; diffsnorm also
                                         checks the factors through y = A·x − U·(S⊙Vᵀx) */
#define RPCA_FLAG_NO_GRAPH 0x8u       /* do not capture/replay driver calls as CUDA graphs */
#define RPCA_FLAG_STREAM_A 0x20u     /* out-of-core A (§8(f) N4): a HOST dense A is not
                                         staged whole; every pass streams it through two device
                                         buffers of $RPCA_STREAM_CHUNK_MB (default 256) MB, the
                                         H2D copy of chunk c+1 overlapping the pass on chunk c
                                         (pin the host A for overlap).  With RPCA_FLAG_RENORM_ODD
                                         each interior round F*(F·Z) streams A ONCE (its + 2 streams
                                         instead of 2·its + 2) */
#define RPCA_FLAG_RENORM_ODD 0x10u    /* rpca_pca: renormalise only after the odd applications
                                         (§8(f) N2) — the long-side block of each
                                         interior power round enters the next adjoint application
                                         unrenormalised (its LU skipped); faster, less accurate */

/* ops for rpca_workspace_query */
enum { RPCA_OP_PCA = 1, RPCA_OP_EIGENS = 2, RPCA_OP_DIFFSNORM = 3, RPCA_OP_APPLY = 4, RPCA_OP_REIG = 5 };

/*
 * The matrix A (§2 l.107-114: m×n, k ≪ min(m,n)).
 *   kind = RPCA_DENSE: `a` points at row i*lda (elements), lda ≥ n.
 *   kind = RPCA_CSR:   rowptr[m_local+1] (int64, rowptr[0] = 0), colind[nnz]
 *                      (int32, sorted within a row, < n), vals[nnz].
 *   dtype: element type of a / vals (fp64 or fp32).  fp32 inputs are computed
 *   with fp32 products (dense: 3×TF32 tensor-core split) and fp64 reductions.
 *   m, n: GLOBAL shape.  row0, m_local: the rows [row0, row0+m_local) this
 *   rank holds (single GPU: 0, m).  location: RPCA_DEVICE or RPCA_HOST (host
 *   A — dense, or all three CSR arrays — is copied to the device inside each
 *   call, the end-to-end mode; a host CSR's transpose is rebuilt per call).
 *   A device CSR's transpose CSR(Aᵀ) is
 *   cached in the workspace across calls, keyed by the pointers, the shape
 *   and a 64-bit fingerprint of the three arrays' contents recomputed on
 *   every call (one read of the CSR, ≈ 0.5% of a C5 PCA), so a different
 *   matrix at recycled addresses or an in-place edit rebuilds it.
 */
typedef struct {
  int32_t kind;
  int32_t dtype;
  int64_t m, n;
  int64_t row0, m_local;
  const void* a;
  int64_t lda;
  const int64_t* rowptr;
  const int32_t* colind;
  const void* vals;
  int64_t nnz;
  int32_t location;
  int32_t reserved;
} rpca_mat;

typedef struct rpca_ctx rpca_ctx;

/* ---- context ------------------------------------------------------------
 * rpca_ctx_create: binds to CUDA `device` and `stream` (a cudaStream_t; NULL
 * = the legacy default stream).  flags: default driver flags (RPCA_FLAG_*).
 * Allocates 64 bytes of pinned host and 256 bytes of device scratch.  By
 * default the context owns a growable device workspace: the first call of a
 * given size allocates (cudaMalloc, outside any capture), later calls of the
 * same or smaller size do not, so steady-state calls are CUDA-graph captured
 * and replayed.  See rpca_set_workspace for a caller-owned workspace.      */
rpca_status rpca_ctx_create(rpca_ctx** ctx, int device, void* stream, uint32_t flags);
rpca_status rpca_ctx_destroy(rpca_ctx* ctx);
rpca_status rpca_ctx_set_stream(rpca_ctx* ctx, void* stream);
rpca_status rpca_ctx_set_flags(rpca_ctx* ctx, uint32_t flags);
rpca_status rpca_ctx_sync(rpca_ctx* ctx);
/* drop cached state: captured CUDA graphs and the cached CSR(Aᵀ) of a sparse A
 * (the transpose is keyed by the CSR pointers and shape — call this after
 * modifying a sparse A in place).                                          */
rpca_status rpca_ctx_clear_cache(rpca_ctx* ctx);
/* bytes of workspace currently held by the context */
rpca_status rpca_workspace_size(rpca_ctx* ctx, size_t* bytes);
/* Caller-owned workspace.
 * rpca_workspace_query: *bytes = device workspace one call of `op` needs for
 * A (RPCA_OP_PCA / _EIGENS: k, l (≤ 0 ⇒ k+2), its; RPCA_OP_DIFFSNORM: k = the
 * factors' rank; RPCA_OP_APPLY: l = the thin block's width, covers
 * rpca_apply / rpca_apply_int8emu / rpca_colmeans), with the context's
 * current flags (RPCA_FLAG_OUTPUTS_HOST adds staging) and communicator, and
 * outputs with ld = k.  For a device CSR A it includes the cached CSR(Aᵀ) and
 * the heavy-row plans.  Reads no matrix data; RPCA_E_SHAPE / RPCA_E_ARG as the
 * op would.
 * rpca_set_workspace: the context uses [dptr, dptr + bytes) (device memory of
 * its GPU, 256-byte aligned, owned by the caller, not touched after the
 * context is destroyed or another workspace is set) and never calls
 * cudaMalloc for calls again; a call needing more returns RPCA_E_WORKSPACE
 * before launching anything.  dptr = NULL returns to a context-owned
 * workspace.  Either way the cached CSR(Aᵀ) and captured graphs are dropped.
 * Synchronises the context stream.                                         */
rpca_status rpca_workspace_query(rpca_ctx* ctx, int op, const rpca_mat* A, int64_t k, int64_t l, int its,
                                 size_t* bytes);
rpca_status rpca_set_workspace(rpca_ctx* ctx, void* dptr, size_t bytes);
const char* rpca_strerror(rpca_status s);
const char* rpca_last_error(void);
/* number of kernels this library launched since the context was created */
rpca_status rpca_launch_count(rpca_ctx* ctx, int64_t* count);
/* per-launch timing: after rpca_profile_begin, an event is recorded on the
 * context stream behind every kernel launch; rpca_profile_end synchronises the
 * stream, stops recording and writes "name<TAB>milliseconds\n" per launch
 * (duration = gap to the previous event; launches are stream-serialised) into
 * buf (NUL-terminated, truncated to cap); *needed = full length.            */
rpca_status rpca_profile_begin(rpca_ctx* ctx);
/* mode RPCA_PROFILE_ALL (= rpca_profile_begin) or RPCA_PROFILE_PASSES: events
 * only around the pass kernels that stream A (the other intervals are reported
 * as "gap"), which keeps event overhead out of a timed region; RPCA_E_ARG for
 * any other mode */
#define RPCA_PROFILE_ALL 1
#define RPCA_PROFILE_PASSES 2
rpca_status rpca_profile_begin_mode(rpca_ctx* ctx, int mode);
rpca_status rpca_profile_end(rpca_ctx* ctx, char* buf, size_t cap, size_t* needed);

/* ---- multi-GPU (rows of A sharded across ranks) ---------
 * rpca_comm_unique_id: writes an ncclUniqueId (128 bytes) into `id` (host).
 * rpca_comm_init: ncclCommInitRank(nranks, id, rank) on the context's device
 * (NCCL is dlopen'ed: libnccl.so.2 as loaded by the process, else
 * $RPCA_NCCL_PATH; RPCA_E_NCCL if none).  With nranks > 1 the drivers treat
 * A as this rank's row shard [row0, row0+m_local) (m_local ≥ 1 on every
 * rank): vectors of length m are row shards, vectors of length n are
 * replicated, Aᵀ·(·) and the l×l Grams are all-reduced (fp64 sum), the LU's
 * tournament candidates are all-gathered.  Every rank must make the same
 * sequence of calls with the same scalar arguments.
 * rpca_virtual_group_create / rpca_comm_init_virtual: a test communicator —
 * P contexts on ONE device, each driven by its own host thread, meeting at
 * host barriers; collectives are device copies and a fixed-order sum kernel
 * (no kernel ever waits on another rank's kernel).  Not CUDA-graph captured.
 * The group must outlive the contexts attached to it.                     */
rpca_status rpca_comm_unique_id(void* id, size_t bytes);
rpca_status rpca_comm_init(rpca_ctx* ctx, int nranks, int rank, const void* id);
rpca_status rpca_virtual_group_create(int nranks, void** group);
rpca_status rpca_virtual_group_destroy(void* group);
rpca_status rpca_comm_init_virtual(rpca_ctx* ctx, void* group, int rank);

/* ---- §8(a) step a1: Ω ------------------------------------------------------
 * out (rows×cols, row-major, fp64, device) = the test block of PAPER.md:163-168
 * (dist RPCA_GAUSSIAN) or PAPER.md:437-440 (RPCA_UNIFORM).  Element e =
 * i·cols + j takes Philox4x32-10 call p = e>>1 with counter (lo32 p, hi32 p,
 * 0, stream_id) and key (lo32 seed, hi32 seed); a, b = the two 53-bit
 * uniforms of the call; Gaussian: r = sqrt(-2 ln(1-a)), e even → r cos 2πb,
 * e odd → r sin 2πb; uniform: 2a-1 / 2b-1 (reading Q7).
 * round_f32 != 0 rounds every value to fp32 (the fp32 path's Ω).            */
rpca_status rpca_omega(rpca_ctx* ctx, uint64_t seed, uint32_t stream_id, int64_t rows, int64_t cols,
                       int dist, int round_f32, double* out);

/* ---- column means: c[j] = (1/m)·Σ_i A_ij over the global
 * rows (sharded: local sums ÷ m, all-reduced).                              */
rpca_status rpca_colmeans(rpca_ctx* ctx, const rpca_mat* A, double* c);

/* ---- §8(a) steps a2, a4, a6: applications of A --------
 * adjoint = 0: Y (m_local×l) = A·X (X n×l) [ − 1·(c·X) if c != NULL ]
 * adjoint = 1: Y (n×l)       = Aᵀ·X (X m_local×l) [ − cᵀ·(1ᵀX) if c != NULL ]
 *   (with a communicator, the adjoint result is all-reduced over ranks.)
 * c: column means (n, fp64, device) or NULL (no centring).
 * Dense fp64 A uses the fp64 tensor cores (DMMA); fp32 A uses 3×TF32
 * products; every sum across K-chunks, CTAs and ranks is fp64 and runs in a
 * fixed order, so results are bitwise reproducible for a fixed device/grid. */
rpca_status rpca_apply(rpca_ctx* ctx, const rpca_mat* A, const double* c, int adjoint, const double* X,
                       int64_t l, double* Y);

/* ---- step a2 on the int8 tensor cores: Y (m_local×l) = A·X for a dense fp64
 * A whose A·X passes rpca_pca / rpca_eigens emulate (24 < l ≤ 48, m ≥ 128,
 * n ≥ 32): A and X split into 7 balanced base-256 digit planes with per-row /
 * per-column exponents, 28 exact int8 products (Ozaki scheme I); error
 * ≲ 2^-55·2^E_i·2^G_j per term, relative to the row / column maxima of A and
 * X.  Reads A twice (row exponents, then the pass).  Non-finite
 * entries give NaN rows / columns.  RPCA_E_NOTIMPL for other A or l.        */
rpca_status rpca_apply_int8emu(rpca_ctx* ctx, const rpca_mat* A, const double* X, int64_t l, double* Y);

/* ---- §8(a) step a3: LU renormalisation ("[Q,R]=lu(Q)") ---
 * In place: Y (m×l, m ≥ l) ← L with Y = L·U, L in the ORIGINAL row order
 * (unit lower triangular in the pivot rows, reading Q3).  Pivot rows are
 * chosen by tournament pivoting (GEPP on row blocks, then on stacked
 * candidates; lowest row index on ties); a pivot that is exactly 0 makes
 * L's column the unit vector at its row.  U (l×l, device) and piv (l int64,
 * device) may be NULL.                                                     */
rpca_status rpca_lu_renorm(rpca_ctx* ctx, double* Y, int64_t m, int64_t l, double* U, int64_t* piv);

/* ---- §8(a) step a5: the pipeline's orthonormalisation --
 * In place: Y (m×l, m ≥ l) ← Q, Y = Q·R, R upper (l×l, device, may be NULL),
 * diag(R) ≥ 0 — exactly the kernels rpca_pca / rpca_eigens run for their last
 * renormalisation and the QR of Bᵀ: tournament LU (Y = L·U), then two
 * Cholesky-QR steps on L (LU-Cholesky-QR2).  A Cholesky pivot of LᵀL below
 * 2^-40 of its largest (κ(L) ≳ 1e6) is a breakdown: the call then redoes the
 * block with Householder TSQR (as rpca_qr) — the drivers re-run the whole
 * call that way.  *used_householder (host, may be NULL) reports it.
 * Synchronises the stream.                                                 */
rpca_status rpca_orthonormalize(rpca_ctx* ctx, double* Y, int64_t m, int64_t l, double* R, int* used_householder);

/* ---- §8(a) steps a5/a7: Householder QR --------
 * In place: Y (m×l, m ≥ l) ← Q with orthonormal columns, Y = Q·R, R upper
 * triangular with diag(R) ≥ 0 (R: l×l device, may be NULL).  Tall-skinny
 * Householder (TSQR tree); rank-deficient Y still yields orthonormal Q.   */
rpca_status rpca_qr(rpca_ctx* ctx, double* Y, int64_t m, int64_t l, double* R);

/* ---- §8(a) step a7: small SVD (eq. i3) ------------------
 * G (n×l, n ≥ l) = Vt · diag(sigma) · Wᵀ: Vt (n×l) orthonormal, sigma (l)
 * non-increasing ≥ 0, W (l×l) orthogonal.  TSQR of G, then one-sided Jacobi
 * on the l×l R in one CTA (threshold 2^-52, ≤ 30 sweeps).  All device.      */
rpca_status rpca_small_svd(rpca_ctx* ctx, const double* G, int64_t n, int64_t l, double* Vt, double* sigma,
                           double* W);

/* ---- the whole path: rank-k PCA (§2 eqs. i1-i4, §5) -------------
 *   Y = A·Ω [centred]; Q = its==0 ? qr(Y) : lu(Y)
 *   for it = 1..its: Z = lu(Aᵀ·Q); Y = A·Z; Q = it<its ? lu(Y) : qr(Y)
 *   Bᵀ = Aᵀ·Q; Bᵀ = V·Σ·Wᵀ; U = Q·W; truncate to k.
 * raw != 0: no centring; raw == 0: implicit column centring.
 * its ≥ 0 extra power rounds: 2·its+2 passes over A.
 * l ≤ 0 means l = k+2.  When m < n the path sketches Aᵀ and swaps U and V.
 * Outputs in A's dtype: U (m_local×k, ld ldu ≥ k), S (k, non-increasing),
 * V (n×k, ld ldv ≥ k, replicated on every rank).  Sign convention: the
 * largest-|·| entry of every column of V is positive (lowest index on ties).
 * Synchronises the stream (reads the device status word).                  */
rpca_status rpca_pca(rpca_ctx* ctx, const rpca_mat* A, int64_t k, int raw, int its, int64_t l, uint64_t seed,
                     void* U, int64_t ldu, void* S, void* V, int64_t ldv);

/* ---- the stabilised Nyström path (§3, l.214-282) -----------------
 * A square, self-adjoint, nonnegative definite (not checked).  Q from the
 * self-adjoint loop of PAPER.md:386-412 (its+1 applications, LU inside, QR
 * last); B1 = A·Q; B2 = sym(QᵀB1); variant RPCA_SHIFT_CHOL: ν = u·√n·‖B1‖_F,
 * C = chol(B2 + νI) (ν ×10 up to 5 retries), F = (B1 + νQ)·C⁻¹;
 * RPCA_SQRT: C = B2^{1/2} with a 1e-12-regularised pseudo-inverse.  F = U·S·Wᵀ,
 * lam = max(S² − ν, 0).  Outputs in A's dtype: U (m_local×k, ld ldu), lam (k).
 * Sharded: the shards must be the uniform partition, rank r holding rows
 * [r·⌈n/P⌉, min(n, (r+1)·⌈n/P⌉)) (Q is all-gathered for A_r·Q), else
 * RPCA_E_SHAPE.  Synchronises the stream.                                   */
rpca_status rpca_eigens(rpca_ctx* ctx, const rpca_mat* A, int64_t k, int its, int64_t l, uint64_t seed,
                        int variant, void* U, int64_t ldu, void* lam);

/* ---- self-adjoint, possibly indefinite A (§8(f) N1) ------------------------
 * PAPER.md:183-184 ("Further accelerations are possible when A is
 * self-adjoint").  A square and symmetric (the caller's
 * promise, not checked).  Q from the self-adjoint loop of PAPER.md:386-412
 * (as rpca_eigens: its+1 applications, LU inside, QR last); B1 = A·Q (one
 * more pass); T = (QᵀB1 + B1ᵀQ)/2 = E·Λ·Eᵀ by Jacobi; U = Q·E truncated to
 * the k eigenvalues of largest |λ| (ties: the larger λ, then the lower index).
 * its + 2 passes over A.  Outputs in A's dtype: U (m_local×k, ld ldu; the
 * largest-|·| entry of each column positive), lam (k, signed, |lam|
 * non-increasing).  Sharding as rpca_eigens (uniform row partition).
 * Synchronises the stream.                                                 */
rpca_status rpca_reig(rpca_ctx* ctx, const rpca_mat* A, int64_t k, int its, int64_t l, uint64_t seed, void* U,
                      int64_t ldu, void* lam);

/* ---- accuracy: ‖A − U·diag(S)·Vᵀ‖ by the randomized power method ----------
 * PAPER.md §4 l.362-371.  x = stream-1 Gaussian n-vector (seed), normalised;
 * its times: y = E·x, z = Eᵀ·y, est = sqrt(‖z‖), x = z/‖z‖.  E = A [centred
 * if raw == 0] − U·diag(S)·Vᵀ, never formed.  U (m_local×k, ld ldu), S (k),
 * V (n×k, ld ldv), fp64 device (k = 0 allowed: estimates ‖A‖).  For eigens
 * factors pass V = U and S = lam.  *out (host) gets the estimate; synchronises. */
rpca_status rpca_diffsnorm(rpca_ctx* ctx, const rpca_mat* A, int raw, const double* U, int64_t ldu,
                           const double* S, const double* V, int64_t ldv, int64_t k, int its, uint64_t seed,
                           double* out);

#ifdef __cplusplus
}
#endif
#endif /* RPCA_H_ */
