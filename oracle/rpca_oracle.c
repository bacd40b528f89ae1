/*
 * rpca_oracle.c — the CPU ORACLE for the randomized PCA hot path of
 * Szlam, Kluger & Tygert, "An implementation of a randomized algorithm for
 * principal component analysis" (arXiv 1412.3510; /root/reference/PAPER.md).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It shares no code, header, table or constant generator
 * with the CUDA path (paper_1412_3510_b200/csrc); neither includes the other.
 *
 * Rules (DESIGN.md §3 "Oracle"):
 *   - plain C99, naive loops, no BLAS/LAPACK; fp64 everywhere (fp32 inputs are
 *     upcast exactly on read);
 *   - every sum runs in a fixed order that does not depend on the thread
 *     count: ascending index, or, for the long reductions over m, fixed
 *     2048-row chunks whose partials are added in ascending chunk order;
 *     OpenMP loops only split over outputs they own;
 *   - each function cites the PAPER.md passage (line numbers, section,
 *     equation label) it follows; where the paper is silent the DESIGN.md
 *     reading (SURVEY.md §8(c) Q-numbers) is named.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): Philox vs the cuRAND header's
 * host path; Gaussian/uniform moments and KS; LU/QR/Jacobi vs LAPACK via
 * numpy/scipy and their defining identities; PROPACK diagonals (PAPER.md
 * 460-491); exact-rank and l = min(m,n) special cases; centering ≡ explicit
 * centering; Nyström exact-rank; diffsnorm vs full SVD.  Every function below
 * has at least one pin; none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_E_ARG 1
#define ORC_E_SHAPE 2
#define ORC_E_NOTPSD 4
#define ORC_E_NOMEM 9

#define CHUNK 2048 /* fixed reduction chunk over rows (thread-count independent) */

/* ------------------------------------------------------------------------
 * Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11), the counter-based
 * generator behind Ω.  PAPER.md:163-168 asks for i.i.d. normal test vectors,
 * PAPER.md:437-440 allows uniform [-1,1] ("robust to the quality of the
 * random numbers").  Counter layout = DESIGN.md reading Q7.
 * ---------------------------------------------------------------------- */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  uint32_t n0 = hi1 ^ c[1] ^ k[0], n1 = lo1, n2 = hi0 ^ c[3] ^ k[1], n3 = lo0;
  c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
    philox_round(c, k);
  }
  memcpy(out, c, sizeof(c));
}

/* Ω (rows × cols, row-major).  Element e = i·cols + j uses Philox call
 * p = e >> 1 with ctr = (lo32 p, hi32 p, 0, stream), key = (lo32 seed, hi32
 * seed); a = ((x0<<32 | x1) >> 11)·2^-53, b likewise from (x2, x3).
 * dist 0 (Gaussian, Box–Muller): r = sqrt(-2 ln(1-a)); e even → r cos 2πb,
 * e odd → r sin 2πb.  dist 1 (uniform [-1,1]): e even →
 * 2a-1, e odd → 2b-1.  Reading Q7. */
void oracle_omega(uint64_t seed, uint32_t stream, int64_t rows, int64_t cols, int dist, double* out) {
  const int64_t total = rows * cols;
  const int64_t calls = (total + 1) / 2;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < calls; ++p) {
    uint32_t ctr[4] = {(uint32_t)p, (uint32_t)((uint64_t)p >> 32), 0u, stream};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t x[4];
    oracle_philox4x32_10(ctr, key, x);
    uint64_t ua = (((uint64_t)x[0] << 32) | x[1]) >> 11;
    uint64_t ub = (((uint64_t)x[2] << 32) | x[3]) >> 11;
    double a = (double)ua * 0x1p-53, b = (double)ub * 0x1p-53;
    double v0, v1;
    if (dist == 0) {
      double r = sqrt(-2.0 * log(1.0 - a));
      v0 = r * cos(2.0 * M_PI * b);
      v1 = r * sin(2.0 * M_PI * b);
    } else {
      v0 = 2.0 * a - 1.0;
      v1 = 2.0 * b - 1.0;
    }
    int64_t e = 2 * p;
    out[e] = v0;
    if (e + 1 < total) out[e + 1] = v1;
  }
}

/* ------------------------------------------------------------------------
 * The matrix A and its two applications.  PAPER.md:427-435 (§5): A is
 * applied to a block as A*Q, its adjoint as (Q'*A)' without forming A*, and
 * the mean-centred matrix as A*Q - ones(m,1)*(c*Q) without forming it, where
 * c is the 1×n vector of column means.
 * ---------------------------------------------------------------------- */
typedef struct {
  int kind;   /* 0 dense row-major, 1 CSR */
  int dtype;  /* 0 f64, 1 f32 */
  int64_t m, n, lda;
  const void* a;
  const int64_t* rowptr;
  const int32_t* colind;
  const void* vals;
} omat;

static inline double dense_at(const omat* A, int64_t i, int64_t j) {
  if (A->dtype == 0) return ((const double*)A->a)[i * A->lda + j];
  return (double)((const float*)A->a)[i * A->lda + j];
}
static inline double csr_val(const omat* A, int64_t t) {
  if (A->dtype == 0) return ((const double*)A->vals)[t];
  return (double)((const float*)A->vals)[t];
}

/* c_j = (Σ_i A_ij)/m, i ascending. */
static void colmeans(const omat* A, double* c) {
  const int64_t m = A->m, n = A->n;
  if (A->kind == 0) {
#pragma omp parallel for schedule(static)
    for (int64_t j0 = 0; j0 < n; j0 += 64) {
      int64_t j1 = j0 + 64 < n ? j0 + 64 : n;
      double acc[64] = {0};
      for (int64_t i = 0; i < m; ++i)
        for (int64_t j = j0; j < j1; ++j) acc[j - j0] += dense_at(A, i, j);
      for (int64_t j = j0; j < j1; ++j) c[j] = acc[j - j0] / (double)m;
    }
  } else {
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0;
    for (int64_t i = 0; i < m; ++i)
      for (int64_t t = A->rowptr[i]; t < A->rowptr[i + 1]; ++t) c[A->colind[t]] += csr_val(A, t);
    for (int64_t j = 0; j < n; ++j) c[j] /= (double)m;
  }
}

/* Y (m×l) = A·X (X n×l), then, if c != NULL, Y -= 1·(c·X). */
static void apply_A(const omat* A, const double* c, const double* X, int64_t l, double* Y) {
  const int64_t m = A->m, n = A->n;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    double* y = Y + i * l;
    for (int64_t j = 0; j < l; ++j) y[j] = 0.0;
    if (A->kind == 0) {
      for (int64_t k = 0; k < n; ++k) {
        double a = dense_at(A, i, k);
        const double* x = X + k * l;
        for (int64_t j = 0; j < l; ++j) y[j] += a * x[j];
      }
    } else {
      for (int64_t t = A->rowptr[i]; t < A->rowptr[i + 1]; ++t) {
        double a = csr_val(A, t);
        const double* x = X + (int64_t)A->colind[t] * l;
        for (int64_t j = 0; j < l; ++j) y[j] += a * x[j];
      }
    }
  }
  if (c) {
    double* cx = (double*)calloc((size_t)l, sizeof(double));
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = 0; j < l; ++j) cx[j] += c[k] * X[k * l + j];
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < l; ++j) Y[i * l + j] -= cx[j];
    free(cx);
  }
}

/* Z (n×l) = Aᵀ·Y (Y m×l) — the "(Q'*A)'" of PAPER.md:432-435 — then, if
 * c != NULL, Z -= cᵀ·(1ᵀY) (the adjoint of the centring, reading Q8).
 * Each Z_kj sums over i ascending. */
static void apply_At(const omat* A, const double* c, const double* Y, int64_t l, double* Z) {
  const int64_t m = A->m, n = A->n;
  if (A->kind == 0) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
      int64_t k1 = k0 + 32 < n ? k0 + 32 : n;
      for (int64_t k = k0; k < k1; ++k)
        for (int64_t j = 0; j < l; ++j) Z[k * l + j] = 0.0;
      for (int64_t i = 0; i < m; ++i) {
        const double* y = Y + i * l;
        for (int64_t k = k0; k < k1; ++k) {
          double a = dense_at(A, i, k);
          double* z = Z + k * l;
          for (int64_t j = 0; j < l; ++j) z[j] += a * y[j];
        }
      }
    }
  } else {
    for (int64_t k = 0; k < n * l; ++k) Z[k] = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      const double* y = Y + i * l;
      for (int64_t t = A->rowptr[i]; t < A->rowptr[i + 1]; ++t) {
        double a = csr_val(A, t);
        double* z = Z + (int64_t)A->colind[t] * l;
        for (int64_t j = 0; j < l; ++j) z[j] += a * y[j];
      }
    }
  }
  if (c) {
    double* sy = (double*)calloc((size_t)l, sizeof(double));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < l; ++j) sy[j] += Y[i * l + j];
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = 0; j < l; ++j) Z[k * l + j] -= c[k] * sy[j];
    free(sy);
  }
}

/* Orientation (reading Q6): the pipeline sketches the operator F with
 * fwd_in ≤ fwd_out; for m < n, F = Aᵀ and the outputs are swapped. */
typedef struct { const omat* A; const double* c; int trans; } oop;
static void op_fwd(const oop* o, const double* X, int64_t l, double* Y) {
  if (o->trans) apply_At(o->A, o->c, X, l, Y); else apply_A(o->A, o->c, X, l, Y);
}
static void op_adj(const oop* o, const double* Y, int64_t l, double* Z) {
  if (o->trans) apply_A(o->A, o->c, Y, l, Z); else apply_At(o->A, o->c, Y, l, Z);
}

/* ------------------------------------------------------------------------
 * Renormalisation ("we renormalize after each application
 * of A or A*"; §5: "[Q,R] = lu(Q)").
 * LU with partial pivoting, in place: Y (m×l) ← L in the ORIGINAL row order
 * (MATLAB's two-output lu returns the permuted lower factor, reading Q3).
 * Pivot of column j = unpivoted row of largest |·|, lowest index on ties.
 * Exact zero maximum: U_jj = 0, no elimination, L column j = unit vector at
 * the chosen row.  U (l×l, may be NULL) and piv (l, may be NULL) returned.
 * ---------------------------------------------------------------------- */
int oracle_lu_renorm(double* Y, int64_t m, int64_t l, double* U, int64_t* piv) {
  if (m < l || l < 1) return ORC_E_SHAPE;
  int64_t* pos = (int64_t*)malloc((size_t)m * sizeof(int64_t)); /* pivot position or -1 */
  double* Uw = (double*)calloc((size_t)(l * l), sizeof(double));
  if (!pos || !Uw) { free(pos); free(Uw); return ORC_E_NOMEM; }
  for (int64_t i = 0; i < m; ++i) pos[i] = -1;
  for (int64_t j = 0; j < l; ++j) {
    int64_t p = -1;
    double best = -1.0;
    for (int64_t i = 0; i < m; ++i) {
      if (pos[i] >= 0) continue;
      double v = fabs(Y[i * l + j]);
      if (v > best) { best = v; p = i; }
    }
    pos[p] = j;
    for (int64_t t = j; t < l; ++t) Uw[j * l + t] = Y[p * l + t];
    double ujj = Uw[j * l + j];
    if (ujj == 0.0) {
      for (int64_t i = 0; i < m; ++i)
        if (pos[i] < 0) Y[i * l + j] = 0.0;
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < m; ++i) {
        if (pos[i] >= 0) continue;
        double mult = Y[i * l + j] / ujj;
        Y[i * l + j] = mult;
        for (int64_t t = j + 1; t < l; ++t) Y[i * l + t] -= mult * Uw[j * l + t];
      }
    }
  }
  /* pivot rows: multipliers left of the diagonal, 1 on it, 0 right of it */
  for (int64_t i = 0; i < m; ++i) {
    int64_t t = pos[i];
    if (t < 0) continue;
    Y[i * l + t] = 1.0;
    for (int64_t s = t + 1; s < l; ++s) Y[i * l + s] = 0.0;
    if (piv) piv[t] = i;
  }
  if (U) memcpy(U, Uw, (size_t)(l * l) * sizeof(double));
  free(pos); free(Uw);
  return ORC_OK;
}

/* Householder QR ("Gram-Schmidt ... or other methods for
 * constructing QR decompositions"; §5, unpivoted per
 * PAPER.md:422-425, reading Q4).  v = x + sign(x1)‖x‖e1 with sign(0) = +1;
 * explicit thin Q by back-application to I[:, :l]; signs flipped so that
 * diag(R) ≥ 0.  In place: Y (m×l) ← Q.  R (l×l, may be NULL). */
static double dot_rows(const double* a, int64_t lda, const double* b, int64_t ldb, int64_t r0, int64_t r1) {
  /* Σ_{i=r0}^{r1-1} a[i*lda]·b[i*ldb], fixed 2048-row chunks, ascending */
  double total = 0.0;
  int64_t nch = (r1 - r0 + CHUNK - 1) / CHUNK;
  if (nch <= 1) {
    for (int64_t i = r0; i < r1; ++i) total += a[i * lda] * b[i * ldb];
    return total;
  }
  double* part = (double*)malloc((size_t)nch * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nch; ++q) {
    int64_t i0 = r0 + q * CHUNK, i1 = i0 + CHUNK < r1 ? i0 + CHUNK : r1;
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) s += a[i * lda] * b[i * ldb];
    part[q] = s;
  }
  for (int64_t q = 0; q < nch; ++q) total += part[q];
  free(part);
  return total;
}

int oracle_house_qr(double* Y, int64_t m, int64_t l, double* R) {
  if (m < l || l < 1) return ORC_E_SHAPE;
  double* V = (double*)calloc((size_t)(m * l), sizeof(double)); /* reflectors, column-wise */
  double* vv = (double*)calloc((size_t)l, sizeof(double));      /* vᵀv (0 ⇒ identity) */
  double* Rw = (double*)calloc((size_t)(l * l), sizeof(double));
  if (!V || !vv || !Rw) { free(V); free(vv); free(Rw); return ORC_E_NOMEM; }
  for (int64_t j = 0; j < l; ++j) {
    double nx2 = dot_rows(Y + j, l, Y + j, l, j, m);
    double nx = sqrt(nx2);
    double x1 = Y[j * l + j];
    if (nx == 0.0) { /* nothing to annihilate */
      vv[j] = 0.0;
      for (int64_t t = j; t < l; ++t) Rw[j * l + t] = Y[j * l + t];
      continue;
    }
    double sg = (x1 >= 0.0) ? 1.0 : -1.0;
    for (int64_t i = j; i < m; ++i) V[i * l + j] = Y[i * l + j];
    V[j * l + j] = x1 + sg * nx;
    vv[j] = dot_rows(V + j, l, V + j, l, j, m);
    /* apply H = I - 2 v vᵀ/(vᵀv) to columns j..l-1 */
    for (int64_t t = j; t < l; ++t) {
      double w = dot_rows(V + j, l, Y + t, l, j, m);
      double f = 2.0 * w / vv[j];
#pragma omp parallel for schedule(static)
      for (int64_t i = j; i < m; ++i) Y[i * l + t] -= f * V[i * l + j];
    }
    for (int64_t t = j; t < l; ++t) Rw[j * l + t] = Y[j * l + t];
  }
  /* explicit Q = H_0 ⋯ H_{l-1} I[:, :l] */
  memset(Y, 0, (size_t)(m * l) * sizeof(double));
  for (int64_t j = 0; j < l; ++j) Y[j * l + j] = 1.0;
  for (int64_t j = l - 1; j >= 0; --j) {
    if (vv[j] == 0.0) continue;
    for (int64_t t = j; t < l; ++t) {
      double w = dot_rows(V + j, l, Y + t, l, j, m);
      double f = 2.0 * w / vv[j];
#pragma omp parallel for schedule(static)
      for (int64_t i = j; i < m; ++i) Y[i * l + t] -= f * V[i * l + j];
    }
  }
  /* diag(R) ≥ 0 */
  for (int64_t j = 0; j < l; ++j) {
    if (Rw[j * l + j] < 0.0) {
      for (int64_t t = j; t < l; ++t) Rw[j * l + t] = -Rw[j * l + t];
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < m; ++i) Y[i * l + j] = -Y[i * l + j];
    }
  }
  if (R) memcpy(R, Rw, (size_t)(l * l) * sizeof(double));
  free(V); free(vv); free(Rw);
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * The small SVD (eq. i3 "W Σ V* = B"; LAPACK's svd in the
 * paper).  Reading Q9/Q18: cyclic one-sided Hestenes
 * Jacobi on the n×l matrix G = Bᵀ: pairs (p,q), p<q, row-cyclic; rotate iff
 * |γ| > 2^-52·sqrt(αβ); stop after a sweep without rotation or 30 sweeps.
 * Result: G·W = Ṽ·diag(σ), σ non-increasing, so G = Ṽ Σ Wᵀ and
 * B = Gᵀ = W Σ Ṽᵀ.  In place: G ← Ṽ (unit columns; zero-σ columns completed
 * to an orthonormal set by Gram–Schmidt of e_1, e_2, …).  W is l×l.
 * ---------------------------------------------------------------------- */
static void colpair_dots(const double* G, int64_t n, int64_t l, int64_t p, int64_t q,
                         double* alpha, double* beta, double* gamma) {
  int64_t nch = (n + CHUNK - 1) / CHUNK;
  double a = 0, b = 0, g = 0;
  if (nch <= 1) {
    for (int64_t i = 0; i < n; ++i) {
      double x = G[i * l + p], y = G[i * l + q];
      a += x * x; b += y * y; g += x * y;
    }
  } else {
    double* part = (double*)malloc((size_t)(3 * nch) * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; ++c) {
      int64_t i0 = c * CHUNK, i1 = i0 + CHUNK < n ? i0 + CHUNK : n;
      double sa = 0, sb = 0, sg = 0;
      for (int64_t i = i0; i < i1; ++i) {
        double x = G[i * l + p], y = G[i * l + q];
        sa += x * x; sb += y * y; sg += x * y;
      }
      part[3 * c] = sa; part[3 * c + 1] = sb; part[3 * c + 2] = sg;
    }
    for (int64_t c = 0; c < nch; ++c) { a += part[3 * c]; b += part[3 * c + 1]; g += part[3 * c + 2]; }
    free(part);
  }
  *alpha = a; *beta = b; *gamma = g;
}

static void complete_orthonormal(double* G, int64_t n, int64_t l, int64_t col) {
  /* G[:, col] ← first (else largest-residual) e_t orthogonalised (twice)
     against columns 0..col-1 */
  double* v = (double*)malloc((size_t)n * sizeof(double));
  double* best = (double*)malloc((size_t)n * sizeof(double));
  double bestn = -1.0;
  for (int64_t t = 0; t < n; ++t) {
    for (int64_t i = 0; i < n; ++i) v[i] = (i == t) ? 1.0 : 0.0;
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t s = 0; s < col; ++s) {
        double d = 0.0;
        for (int64_t i = 0; i < n; ++i) d += G[i * l + s] * v[i];
        for (int64_t i = 0; i < n; ++i) v[i] -= d * G[i * l + s];
      }
    double nv = 0.0;
    for (int64_t i = 0; i < n; ++i) nv += v[i] * v[i];
    nv = sqrt(nv);
    if (nv > bestn) { bestn = nv; memcpy(best, v, (size_t)n * sizeof(double)); }
    if (nv >= 0.5) break;
  }
  for (int64_t i = 0; i < n; ++i) G[i * l + col] = best[i] / bestn;
  free(v); free(best);
}

int oracle_jacobi_svd(double* G, int64_t n, int64_t l, double* sigma, double* W) {
  if (n < l || l < 1) return ORC_E_SHAPE;
  double* Wk = (double*)calloc((size_t)(l * l), sizeof(double));
  for (int64_t j = 0; j < l; ++j) Wk[j * l + j] = 1.0;
  const double eps = 0x1p-52;
  for (int sweep = 0; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int64_t p = 0; p < l - 1; ++p)
      for (int64_t q = p + 1; q < l; ++q) {
        double a, b, g;
        colpair_dots(G, n, l, p, q, &a, &b, &g);
        /* √a·√b and hypot(1, ζ), not √(ab) and √(1+ζ²): the products
           overflow for columns of norm above 2^256 (a rotation test that is
           never true there would return the column norms of G as σ) */
        if (!(fabs(g) > eps * sqrt(a) * sqrt(b))) continue;
        rotated = 1;
        double zeta = (b - a) / (2.0 * g);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; ++i) {
          double x = G[i * l + p], y = G[i * l + q];
          G[i * l + p] = cs * x - sn * y;
          G[i * l + q] = sn * x + cs * y;
        }
        for (int64_t i = 0; i < l; ++i) {
          double x = Wk[i * l + p], y = Wk[i * l + q];
          Wk[i * l + p] = cs * x - sn * y;
          Wk[i * l + q] = sn * x + cs * y;
        }
      }
    if (!rotated) break;
  }
  /* σ_j = ‖g_j‖, sorted non-increasing (stable) */
  double* s = (double*)malloc((size_t)l * sizeof(double));
  int64_t* ord = (int64_t*)malloc((size_t)l * sizeof(int64_t));
  for (int64_t j = 0; j < l; ++j) {
    double a, b, g;
    colpair_dots(G, n, l, j, j, &a, &b, &g);
    s[j] = sqrt(a);
    ord[j] = j;
  }
  for (int64_t i = 1; i < l; ++i) { /* insertion sort, stable */
    int64_t o = ord[i], j = i;
    while (j > 0 && s[ord[j - 1]] < s[o]) { ord[j] = ord[j - 1]; --j; }
    ord[j] = o;
  }
  double* Gs = (double*)malloc((size_t)(n * l) * sizeof(double));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < l; ++j) Gs[i * l + j] = G[i * l + ord[j]];
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < l; ++j) W[i * l + j] = Wk[i * l + ord[j]];
  for (int64_t j = 0; j < l; ++j) sigma[j] = s[ord[j]];
  memcpy(G, Gs, (size_t)(n * l) * sizeof(double));
  for (int64_t j = 0; j < l; ++j) {
    if (sigma[j] > 0.0) {
      double inv = 1.0 / sigma[j];
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) G[i * l + j] *= inv;
    } else {
      complete_orthonormal(G, n, l, j);
    }
  }
  free(Wk); free(s); free(ord); free(Gs);
  return ORC_OK;
}

/* Symmetric cyclic Jacobi eigen-decomposition of the l×l S (for the SQRT
 * Nyström variant, "The SVD of B2 provides a convenient
 * means for computing the self-adjoint square-root").  S = E diag(mu) Eᵀ,
 * mu non-increasing.  S is destroyed. */
int oracle_jacobi_eig(double* S, int64_t l, double* mu, double* E) {
  double* Ek = (double*)calloc((size_t)(l * l), sizeof(double));
  for (int64_t j = 0; j < l; ++j) Ek[j * l + j] = 1.0;
  const double eps = 0x1p-52;
  for (int sweep = 0; sweep < 30; ++sweep) {
    int rotated = 0;
    for (int64_t p = 0; p < l - 1; ++p)
      for (int64_t q = p + 1; q < l; ++q) {
        double apq = S[p * l + q], app = S[p * l + p], aqq = S[q * l + q];
        if (!(fabs(apq) > eps * sqrt(fabs(app)) * sqrt(fabs(aqq)))) continue; /* no overflow of app·aqq */
        rotated = 1;
        double zeta = (aqq - app) / (2.0 * apq);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
        double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int64_t r = 0; r < l; ++r) { /* S ← S J (columns p,q) */
          double x = S[r * l + p], y = S[r * l + q];
          S[r * l + p] = c * x - s * y;
          S[r * l + q] = s * x + c * y;
        }
        for (int64_t r = 0; r < l; ++r) { /* S ← Jᵀ S (rows p,q) */
          double x = S[p * l + r], y = S[q * l + r];
          S[p * l + r] = c * x - s * y;
          S[q * l + r] = s * x + c * y;
        }
        S[p * l + q] = S[q * l + p] = 0.0;
        for (int64_t r = 0; r < l; ++r) {
          double x = Ek[r * l + p], y = Ek[r * l + q];
          Ek[r * l + p] = c * x - s * y;
          Ek[r * l + q] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  int64_t* ord = (int64_t*)malloc((size_t)l * sizeof(int64_t));
  for (int64_t j = 0; j < l; ++j) ord[j] = j;
  for (int64_t i = 1; i < l; ++i) {
    int64_t o = ord[i], j = i;
    while (j > 0 && S[ord[j - 1] * l + ord[j - 1]] < S[o * l + o]) { ord[j] = ord[j - 1]; --j; }
    ord[j] = o;
  }
  for (int64_t j = 0; j < l; ++j) mu[j] = S[ord[j] * l + ord[j]];
  for (int64_t i = 0; i < l; ++i)
    for (int64_t j = 0; j < l; ++j) E[i * l + j] = Ek[i * l + ord[j]];
  free(Ek); free(ord);
  return ORC_OK;
}

/* Sign convention for the non-unique factors (reading Q10): the entry of
 * largest |·| of each column of Vout is made positive (lowest index on
 * ties); the same flip is applied to Uout. */
static void sign_normalize(double* Uo, int64_t mu, double* Vo, int64_t nv, int64_t k) {
  for (int64_t j = 0; j < k; ++j) {
    int64_t arg = 0;
    double best = -1.0;
    for (int64_t i = 0; i < nv; ++i) {
      double a = fabs(Vo[i * k + j]);
      if (a > best) { best = a; arg = i; }
    }
    if (Vo[arg * k + j] < 0.0) {
      for (int64_t i = 0; i < nv; ++i) Vo[i * k + j] = -Vo[i * k + j];
      if (Uo)
        for (int64_t i = 0; i < mu; ++i) Uo[i * k + j] = -Uo[i * k + j];
    }
  }
}

static int make_omat(omat* A, int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
                     const int64_t* rowptr, const int32_t* colind, const void* vals) {
  if (kind != 0 && kind != 1) return ORC_E_ARG;
  if (dtype != 0 && dtype != 1) return ORC_E_ARG;
  if (m < 1 || n < 1) return ORC_E_SHAPE;
  A->kind = kind; A->dtype = dtype; A->m = m; A->n = n; A->lda = lda;
  A->a = a; A->rowptr = rowptr; A->colind = colind; A->vals = vals;
  if (kind == 0 && (!a || lda < n)) return ORC_E_ARG;
  if (kind == 1 && (!rowptr || !colind || !vals)) return ORC_E_ARG;
  return ORC_OK;
}

static void round_to_f32(double* x, int64_t count) {
  for (int64_t i = 0; i < count; ++i) x[i] = (double)(float)x[i];
}

/* ------------------------------------------------------------------------
 * oracle_pca — PAPER.md §2 (i1)–(i4), (approx) l.116-149; the range finder
 * l.157-172; power iterations l.186-198 with renormalisation after each
 * application l.200-204; LU in interior steps, QR at the last, §5
 * l.382-425; centring and adjoint l.427-435.  its = number of EXTRA power
 * rounds (reading Q1): 2·its+2 applications of A or A*.
 *
 *   Y = F·Ω [centred]; Q = its==0 ? qr(Y) : lu(Y)
 *   for it = 1..its: Z = lu(F*·Q); Y = F·Z; Q = it<its ? lu(Y) : qr(Y)
 *   Bᵀ = F*·Q;  Bᵀ = Ṽ Σ Wᵀ (Jacobi);  U = Q·W;  truncate to k.
 *
 * Outputs (row-major): U m×k, S k, V n×k; sign convention Q10.
 * raw != 0: no centring; raw == 0: implicit column centring.
 * renorm_odd != 0 (oracle_pca_ex; §8(f) N2, "renormalize
 * only in the odd-numbered iterations"): the interior rounds' Y = F·Z is
 * passed to the next F* unrenormalised (the first lu and the last qr stay).
 * ---------------------------------------------------------------------- */
int oracle_pca_ex(int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
                  const int64_t* rowptr, const int32_t* colind, const void* vals,
                  int64_t k, int raw, int its, int64_t l, uint64_t seed, int dist, int renorm_odd,
                  double* U, double* S, double* V) {
  omat A;
  int st = make_omat(&A, kind, dtype, m, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  if (l <= 0) l = k + 2;
  int64_t mn = m < n ? m : n;
  if (k < 1 || l < k || l > mn || its < 0) return ORC_E_SHAPE;
  if (!U || !S || !V) return ORC_E_ARG;
  double* c = NULL;
  if (!raw) { c = (double*)malloc((size_t)n * sizeof(double)); colmeans(&A, c); }
  oop F = {&A, c, m < n};
  int64_t nin = F.trans ? m : n, nout = F.trans ? n : m;
  double* Om = (double*)malloc((size_t)(nin * l) * sizeof(double));
  double* Y = (double*)malloc((size_t)(nout * l) * sizeof(double));
  double* Z = (double*)malloc((size_t)(nin * l) * sizeof(double));
  double* Wm = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* sg = (double*)malloc((size_t)l * sizeof(double));
  if (!Om || !Y || !Z || !Wm || !sg) { st = ORC_E_NOMEM; goto done; }
  oracle_omega(seed, 0u, nin, l, dist, Om);
  if (dtype == 1) round_to_f32(Om, nin * l); /* both sides consume fl32(Ω), §8(c) */
  op_fwd(&F, Om, l, Y);
  st = (its == 0) ? oracle_house_qr(Y, nout, l, NULL) : oracle_lu_renorm(Y, nout, l, NULL, NULL);
  if (st) goto done;
  for (int it = 1; it <= its; ++it) {
    op_adj(&F, Y, l, Z);
    if ((st = oracle_lu_renorm(Z, nin, l, NULL, NULL))) goto done;
    op_fwd(&F, Z, l, Y);
    if (it < its && renorm_odd) continue;
    st = (it < its) ? oracle_lu_renorm(Y, nout, l, NULL, NULL) : oracle_house_qr(Y, nout, l, NULL);
    if (st) goto done;
  }
  /* Y holds Q (nout×l); Bᵀ = F*·Q (nin×l) — eq. (i2) B = Q*A */
  op_adj(&F, Y, l, Z);
  if ((st = oracle_jacobi_svd(Z, nin, l, sg, Wm))) goto done; /* Z ← Ṽ, B = W Σ Ṽᵀ */
  {
    /* eq. (i4) U = Q·W, truncated to k */
    double* Ulift = (double*)malloc((size_t)(nout * k) * sizeof(double));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nout; ++i)
      for (int64_t j = 0; j < k; ++j) {
        double s = 0.0;
        for (int64_t t = 0; t < l; ++t) s += Y[i * l + t] * Wm[t * l + j];
        Ulift[i * k + j] = s;
      }
    double* Vt = (double*)malloc((size_t)(nin * k) * sizeof(double));
    for (int64_t i = 0; i < nin; ++i)
      for (int64_t j = 0; j < k; ++j) Vt[i * k + j] = Z[i * l + j];
    if (!F.trans) { /* U (m×k) = Ulift, V (n×k) = Ṽ */
      memcpy(U, Ulift, (size_t)(m * k) * sizeof(double));
      memcpy(V, Vt, (size_t)(n * k) * sizeof(double));
    } else {        /* sketched Aᵀ: swap (reading Q6) */
      memcpy(U, Vt, (size_t)(m * k) * sizeof(double));
      memcpy(V, Ulift, (size_t)(n * k) * sizeof(double));
    }
    free(Ulift); free(Vt);
    for (int64_t j = 0; j < k; ++j) S[j] = sg[j];
    sign_normalize(U, m, V, n, k);
  }
done:
  free(c); free(Om); free(Y); free(Z); free(Wm); free(sg);
  return st;
}

int oracle_pca(int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
               const int64_t* rowptr, const int32_t* colind, const void* vals,
               int64_t k, int raw, int its, int64_t l, uint64_t seed, int dist,
               double* U, double* S, double* V) {
  return oracle_pca_ex(kind, dtype, m, n, a, lda, rowptr, colind, vals, k, raw, its, l, seed, dist, 0, U, S, V);
}

/* Upper Cholesky C with CᵀC = B (l×l) — eq. (Cholesky).
 * Returns 0 on success, 1 if a pivot is not strictly positive. */
static int chol_upper(const double* B, int64_t l, double* C) {
  memset(C, 0, (size_t)(l * l) * sizeof(double));
  for (int64_t j = 0; j < l; ++j) {
    double d = B[j * l + j];
    for (int64_t t = 0; t < j; ++t) d -= C[t * l + j] * C[t * l + j];
    if (!(d > 0.0)) return 1;
    double cjj = sqrt(d);
    C[j * l + j] = cjj;
    for (int64_t i = j + 1; i < l; ++i) {
      double s = B[j * l + i];
      for (int64_t t = 0; t < j; ++t) s -= C[t * l + j] * C[t * l + i];
      C[j * l + i] = s / cjj;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------
 * oracle_eigens — the stabilised Nyström method, §3 l.214-282:
 * (start) B1 = AQ; (second) B2 = Q*B1; (Cholesky) C*C = B2; (pseudo)
 * F = B1 C^-1; USV* = F; (finish) Σ = S².  Q comes from the self-adjoint
 * loop of §5: Y = AΩ, then its rounds of Q = A·Q with LU
 * in interior rounds and QR at the last (its + 2 applications of A, reading
 * Q1).  variant 0 = SHIFT_CHOL (the authors' code; shift
 * ν = u·√n·‖B1‖_F, ×10 up to 5 retries, reading Q11); variant 1 = SQRT
 * (self-adjoint square root from the eigen-decomposition
 * of B2, pseudo-inverse cutoff 1e-12).
 * Outputs: U n×k, lam k (non-increasing, ≥ 0).
 * ---------------------------------------------------------------------- */
int oracle_eigens(int kind, int dtype, int64_t n, const void* a, int64_t lda,
                  const int64_t* rowptr, const int32_t* colind, const void* vals,
                  int64_t k, int its, int64_t l, uint64_t seed, int dist, int variant,
                  double* U, double* lam) {
  omat A;
  int st = make_omat(&A, kind, dtype, n, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  if (l <= 0) l = k + 2;
  if (k < 1 || l < k || l > n || l > 512 || its < 0) return ORC_E_SHAPE;
  if (variant != 0 && variant != 1) return ORC_E_ARG;
  double* Om = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* Q = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* B1 = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* B2 = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* C = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* Wm = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* sg = (double*)malloc((size_t)l * sizeof(double));
  oracle_omega(seed, 0u, n, l, dist, Om);
  if (dtype == 1) round_to_f32(Om, n * l);
  apply_A(&A, NULL, Om, l, Q);
  st = (its == 0) ? oracle_house_qr(Q, n, l, NULL) : oracle_lu_renorm(Q, n, l, NULL, NULL);
  if (st) goto done;
  for (int it = 1; it <= its; ++it) {
    apply_A(&A, NULL, Q, l, B1);
    memcpy(Q, B1, (size_t)(n * l) * sizeof(double));
    st = (it < its) ? oracle_lu_renorm(Q, n, l, NULL, NULL) : oracle_house_qr(Q, n, l, NULL);
    if (st) goto done;
  }
  apply_A(&A, NULL, Q, l, B1); /* (start) */
  for (int64_t p = 0; p < l; ++p) /* (second), symmetrised (reading Q19) */
    for (int64_t q = 0; q < l; ++q) B2[p * l + q] = dot_rows(Q + p, l, B1 + q, l, 0, n);
  for (int64_t p = 0; p < l; ++p)
    for (int64_t q = p + 1; q < l; ++q) {
      double s = 0.5 * (B2[p * l + q] + B2[q * l + p]);
      B2[p * l + q] = B2[q * l + p] = s;
    }
  double nu = 0.0;
  if (variant == 0) {
    double f2 = 0.0;
    for (int64_t q = 0; q < l; ++q) f2 += dot_rows(B1 + q, l, B1 + q, l, 0, n);
    double fro = sqrt(f2);
    if (fro == 0.0) { /* A·Q = 0: nothing to approximate (DESIGN.md reading) */
      for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < k; ++j) U[i * k + j] = Q[i * l + j];
      for (int64_t j = 0; j < k; ++j) lam[j] = 0.0;
      sign_normalize(NULL, 0, U, n, k);
      goto done;
    }
    double u = (dtype == 1) ? 0x1p-23 : 0x1p-52;
    nu = u * sqrt((double)n) * fro;
    double* B2s = (double*)malloc((size_t)(l * l) * sizeof(double));
    int ok = 0;
    for (int attempt = 0; attempt <= 5; ++attempt) {
      memcpy(B2s, B2, (size_t)(l * l) * sizeof(double));
      for (int64_t j = 0; j < l; ++j) B2s[j * l + j] += nu;
      if (chol_upper(B2s, l, C) == 0) { ok = 1; break; }
      nu *= 10.0;
    }
    free(B2s);
    if (!ok) { st = ORC_E_NOTPSD; goto done; }
    /* F = (B1 + νQ)·C^-1, forward substitution per row (eq. pseudo) */
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double* f = B1 + i * l;
      for (int64_t j = 0; j < l; ++j) f[j] += nu * Q[i * l + j];
      for (int64_t j = 0; j < l; ++j) {
        double s = f[j];
        for (int64_t t = 0; t < j; ++t) s -= f[t] * C[t * l + j];
        f[j] = s / C[j * l + j];
      }
    }
  } else {
    double* mu = (double*)malloc((size_t)l * sizeof(double));
    double* E = (double*)malloc((size_t)(l * l) * sizeof(double));
    double* B2c = (double*)malloc((size_t)(l * l) * sizeof(double));
    memcpy(B2c, B2, (size_t)(l * l) * sizeof(double));
    oracle_jacobi_eig(B2c, l, mu, E);
    double mx = 0.0;
    for (int64_t j = 0; j < l; ++j) mx = fabs(mu[j]) > mx ? fabs(mu[j]) : mx;
    if (mu[l - 1] < -1e-6 * mx) { free(mu); free(E); free(B2c); st = ORC_E_NOTPSD; goto done; }
    double smax = sqrt(mu[0] > 0 ? mu[0] : 0.0);
    double* d = (double*)malloc((size_t)l * sizeof(double));
    for (int64_t j = 0; j < l; ++j) {
      double sj = sqrt(mu[j] > 0.0 ? mu[j] : 0.0);
      d[j] = (sj > 1e-12 * smax && sj > 0.0) ? 1.0 / sj : 0.0;
    }
    /* C+ = E diag(d) Eᵀ, F = B1·C+ */
    for (int64_t p = 0; p < l; ++p)
      for (int64_t q = 0; q < l; ++q) {
        double s = 0.0;
        for (int64_t t = 0; t < l; ++t) s += E[p * l + t] * d[t] * E[q * l + t];
        C[p * l + q] = s;
      }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double row[512];
      for (int64_t j = 0; j < l; ++j) {
        double s = 0.0;
        for (int64_t t = 0; t < l; ++t) s += B1[i * l + t] * C[t * l + j];
        row[j] = s;
      }
      for (int64_t j = 0; j < l; ++j) B1[i * l + j] = row[j];
    }
    free(mu); free(E); free(B2c); free(d);
  }
  /* USV* = F (one-sided Jacobi on F gives its LEFT singular vectors as the
     normalised columns), (finish) Σ = S², minus the shift */
  if ((st = oracle_jacobi_svd(B1, n, l, sg, Wm))) goto done;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < k; ++j) U[i * k + j] = B1[i * l + j];
  for (int64_t j = 0; j < k; ++j) {
    double v = sg[j] * sg[j] - nu;
    lam[j] = v > 0.0 ? v : 0.0;
  }
  sign_normalize(NULL, 0, U, n, k);
done:
  free(Om); free(Q); free(B1); free(B2); free(C); free(Wm); free(sg);
  return st;
}

/* ------------------------------------------------------------------------
 * oracle_reig — the self-adjoint (possibly indefinite) eigendecomposition:
 * PAPER.md:183-184 (§2, "Further accelerations are possible when A is
 * self-adjoint"), the self-adjoint range finder of §5 PAPER.md:386-416 (the
 * loop of oracle_eigens: LU in interior rounds, QR at the last), then
 * T = QᵀAQ (one more application of A: B1 = A·Q,
 * T = QᵀB1), symmetrised (T + Tᵀ)/2, its dense eigendecomposition (the
 * cyclic Jacobi of oracle_jacobi_eig), U = Q·E, truncated to the k
 * eigenvalues of largest |λ| (ties: the larger λ, then the lower index;
 * SPEC.md "Open Questions": truncation by |λ|).  its + 2 applications of A.
 * Outputs: U n×k (largest-|·| entry of each column positive), lam k (signed,
 * |lam| non-increasing).
 * ---------------------------------------------------------------------- */
int oracle_reig(int kind, int dtype, int64_t n, const void* a, int64_t lda,
                const int64_t* rowptr, const int32_t* colind, const void* vals,
                int64_t k, int its, int64_t l, uint64_t seed, int dist, double* U, double* lam) {
  omat A;
  int st = make_omat(&A, kind, dtype, n, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  if (l <= 0) l = k + 2;
  if (k < 1 || l < k || l > n || l > 512 || its < 0) return ORC_E_SHAPE;
  double* Om = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* Q = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* B1 = (double*)malloc((size_t)(n * l) * sizeof(double));
  double* T = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* E = (double*)malloc((size_t)(l * l) * sizeof(double));
  double* mu = (double*)malloc((size_t)l * sizeof(double));
  int64_t* ord = (int64_t*)malloc((size_t)l * sizeof(int64_t));
  oracle_omega(seed, 0u, n, l, dist, Om);
  if (dtype == 1) round_to_f32(Om, n * l);
  apply_A(&A, NULL, Om, l, Q);
  st = (its == 0) ? oracle_house_qr(Q, n, l, NULL) : oracle_lu_renorm(Q, n, l, NULL, NULL);
  if (st) goto done;
  for (int it = 1; it <= its; ++it) {
    apply_A(&A, NULL, Q, l, B1);
    memcpy(Q, B1, (size_t)(n * l) * sizeof(double));
    st = (it < its) ? oracle_lu_renorm(Q, n, l, NULL, NULL) : oracle_house_qr(Q, n, l, NULL);
    if (st) goto done;
  }
  apply_A(&A, NULL, Q, l, B1);
  for (int64_t p = 0; p < l; ++p) /* T = QᵀAQ */
    for (int64_t q = 0; q < l; ++q) T[p * l + q] = dot_rows(Q + p, l, B1 + q, l, 0, n);
  for (int64_t p = 0; p < l; ++p) /* (T + Tᵀ)/2 */
    for (int64_t q = p + 1; q < l; ++q) {
      double s = 0.5 * (T[p * l + q] + T[q * l + p]);
      T[p * l + q] = T[q * l + p] = s;
    }
  oracle_jacobi_eig(T, l, mu, E); /* mu non-increasing, E's columns the eigenvectors */
  for (int64_t j = 0; j < l; ++j) ord[j] = j; /* stable insertion sort by |mu| desc, ties: larger mu first */
  for (int64_t i = 1; i < l; ++i) {
    int64_t o = ord[i], j = i;
    while (j > 0 && (fabs(mu[ord[j - 1]]) < fabs(mu[o]) ||
                     (fabs(mu[ord[j - 1]]) == fabs(mu[o]) && mu[ord[j - 1]] < mu[o]))) {
      ord[j] = ord[j - 1];
      --j;
    }
    ord[j] = o;
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) /* U = Q·E[:, ord[:k]] */
    for (int64_t j = 0; j < k; ++j) {
      double s = 0.0;
      for (int64_t t = 0; t < l; ++t) s += Q[i * l + t] * E[t * l + ord[j]];
      U[i * k + j] = s;
    }
  for (int64_t j = 0; j < k; ++j) lam[j] = mu[ord[j]];
  sign_normalize(NULL, 0, U, n, k);
done:
  free(Om); free(Q); free(B1); free(T); free(E); free(mu); free(ord);
  return st;
}

/* ------------------------------------------------------------------------
 * oracle_diffsnorm — §4: the spectral norm of the
 * discrepancy ‖A − UΣV*‖ by the power method with a random start
 * (Kuczyński–Woźniakowski, within a factor of two w.h.p.).  Reading Q13:
 * x = Gaussian stream-1 n-vector (seed), normalised; its times:
 *   y = E x, z = E* y, est = sqrt(‖z‖), x = z/‖z‖ (‖z‖ = 0 ⇒ 0),
 * with E = A [centred] − U diag(S) Vᵀ applied implicitly.
 * U m×k, S k, V n×k (row-major).  For eigens factors pass V = U, S = λ.
 * ---------------------------------------------------------------------- */
int oracle_diffsnorm(int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
                     const int64_t* rowptr, const int32_t* colind, const void* vals, int raw,
                     const double* U, const double* S, const double* V, int64_t k, int its,
                     uint64_t seed, double* out) {
  omat A;
  int st = make_omat(&A, kind, dtype, m, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  if (k < 0 || its < 1 || !out) return ORC_E_SHAPE;
  double* c = NULL;
  if (!raw) { c = (double*)malloc((size_t)n * sizeof(double)); colmeans(&A, c); }
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* y = (double*)malloc((size_t)m * sizeof(double));
  double* z = (double*)malloc((size_t)n * sizeof(double));
  double* t = (double*)malloc((size_t)(k > 0 ? k : 1) * sizeof(double));
  oracle_omega(seed, 1u, n, 1, 0, x);
  double nx = sqrt(dot_rows(x, 1, x, 1, 0, n));
  for (int64_t i = 0; i < n; ++i) x[i] /= nx;
  double est = 0.0;
  for (int it = 0; it < its; ++it) {
    apply_A(&A, c, x, 1, y);
    for (int64_t j = 0; j < k; ++j) t[j] = S[j] * dot_rows(V + j, k, x, 1, 0, n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < k; ++j) s += U[i * k + j] * t[j];
      y[i] -= s;
    }
    apply_At(&A, c, y, 1, z);
    for (int64_t j = 0; j < k; ++j) t[j] = S[j] * dot_rows(U + j, k, y, 1, 0, m);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < k; ++j) s += V[i * k + j] * t[j];
      z[i] -= s;
    }
    double nz = sqrt(dot_rows(z, 1, z, 1, 0, n));
    if (nz == 0.0) { est = 0.0; break; }
    est = sqrt(nz);
    for (int64_t i = 0; i < n; ++i) x[i] = z[i] / nz;
  }
  *out = est;
  free(c); free(x); free(y); free(z); free(t);
  return ORC_OK;
}

/* Thin wrappers so tests can pin the two applications on their own. */
int oracle_apply(int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
                 const int64_t* rowptr, const int32_t* colind, const void* vals, int raw, int adjoint,
                 const double* X, int64_t l, double* Y) {
  omat A;
  int st = make_omat(&A, kind, dtype, m, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  double* c = NULL;
  if (!raw) { c = (double*)malloc((size_t)n * sizeof(double)); colmeans(&A, c); }
  if (adjoint) apply_At(&A, c, X, l, Y); else apply_A(&A, c, X, l, Y);
  free(c);
  return ORC_OK;
}

int oracle_colmeans(int kind, int dtype, int64_t m, int64_t n, const void* a, int64_t lda,
                    const int64_t* rowptr, const int32_t* colind, const void* vals, double* c) {
  omat A;
  int st = make_omat(&A, kind, dtype, m, n, a, lda, rowptr, colind, vals);
  if (st) return st;
  colmeans(&A, c);
  return ORC_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
