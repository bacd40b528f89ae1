// cholqr.cu — orthonormalisation of a tall-skinny block by LU-Cholesky-QR:
//   Y = L·U (tournament LU, tslu.cu) → L = Q1·R1 (Cholesky of LᵀL) →
//   Q1 = Q·R2 (Cholesky of Q1ᵀQ1) ⇒ Y = Q·(R2·R1·U), diag(R) ≥ 0 by a final
//   column sign fix.
// PAPER.md:406-425 asks for a QR of the last block ("[Q,R,E] = qr(Q,0)",
// pivoting unnecessary) — any backward-stable QR gives the same span and the
// same final factors up to rounding ("what differs from the
// paper").  LU with partial pivoting makes L well conditioned (its pivot rows
// are unit lower triangular with |multipliers| ≤ 1), which is what Cholesky-QR
// needs; LU is backward stable, so R = R2·R1·U keeps the small singular values
// as accurately as Householder (Terao, Ozaki, Ogita 2020, "LU-Cholesky QR").
// Exact zero pivots (rank-deficient Y) make L's column a unit vector, so L —
// and hence Q — stays full rank and orthonormal.
// The two Grams (LᵀL, Q1ᵀQ1) run on the fp64 tensor-core adjoint pass
// (gram.cu) and the two triangular products on the A·X pass
// (dense_ax, in place); only the l×l Cholesky/inverse is a one-CTA kernel.
#include "comm.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

// One CTA: R = chol(G) (upper, RᵀR = G, G full l×l) → X = R⁻¹ (upper);
// Rtot = R·Rprev (Rprev upper or NULL); if `signfix`, D = sign(diag(Rtot)):
// Minv = X·D, Rtot ← D·Rtot.
__global__ void __launch_bounds__(kThreads) chol_kernel(const double* __restrict__ Gin, int l,
                                                        const double* __restrict__ Rprev, int signfix,
                                                        double* __restrict__ Minv, double* __restrict__ Rtot) {
  extern __shared__ double sm[];
  double* G = sm;              // l×l
  double* R = sm + l * l;      // l×l
  double* X = sm + 2 * l * l;  // l×l (inverse)
  __shared__ double d[kMaxL];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, q = idx - p * l;
    G[idx] = 0.5 * (Gin[idx] + Gin[q * l + p]);
    R[idx] = 0.0;
  }
  __syncthreads();
  double gmax = 0.0;
  for (int j = 0; j < l; ++j) gmax = fmax(gmax, G[j * l + j]);
  // right-looking: column j's pivot, then row j of R, then the rank-1 update
  // of the trailing block of G — every step fully parallel
  const double floor_ = 0x1p-104 * gmax;  // L (and Q1) are full rank; guard against roundoff only
  for (int j = 0; j < l; ++j) {
    const double dj = G[j * l + j];
    const double rjj = sqrt(dj > floor_ ? dj : (floor_ > 0.0 ? floor_ : 1.0));
    for (int i = j + tid; i < l; i += kThreads) R[j * l + i] = i == j ? rjj : G[j * l + i] / rjj;
    __syncthreads();
    const int w = l - j - 1;
    for (int idx = tid; idx < w * w; idx += kThreads) {
      const int a = j + 1 + idx / w, b = j + 1 + idx % w;
      G[a * l + b] -= R[j * l + a] * R[j * l + b];
    }
    __syncthreads();
  }
  // X = R⁻¹ (upper): thread j owns column j, back substitution with i
  // descending in lock-step (R reads are broadcasts)
  if (tid < l) {
    const int j = tid;
    for (int i = l - 1; i >= 0; --i) {
      double s = 0.0;
      for (int t = i + 1; t <= j; ++t) s += R[i * l + t] * X[t * l + j];
      X[i * l + j] = i <= j ? ((i == j ? 1.0 : 0.0) - s) / R[i * l + i] : 0.0;
    }
  }
  __syncthreads();
  // Rtot = R·Rprev (both upper)
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int i = idx / l, j = idx - i * l;
    double s;
    if (!Rprev) s = R[idx];
    else {
      s = 0.0;
      for (int t = i; t <= j; ++t) s += R[i * l + t] * Rprev[t * l + j];
    }
    G[idx] = s;  // reuse G for Rtot
  }
  __syncthreads();
  if (tid < l) d[tid] = (signfix && G[tid * l + tid] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int i = idx / l, j = idx - i * l;
    Minv[idx] = X[idx] * d[j];
    Rtot[idx] = G[idx] * d[i];
  }
}

void chol(Ctx& c, const double* G, int l, const double* Rprev, int signfix, double* Minv, double* Rtot) {
  ensure_smem((const void*)chol_kernel, 3 * kMaxL * kMaxL * 8);
  chol_kernel<<<1, kThreads, 3 * l * l * 8, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "cholqr_chol");
}

}  // namespace

size_t orth_ws_bytes(int64_t m, int l) {
  Sizer s;
  s.add<double>(6 * (size_t)l * l);
  const DenseA Y{nullptr, RPCA_F64, m, l, l};
  return s.total + lu_ws_bytes(m, l) + ax_ws_bytes(Y, l) + 4096;
}

size_t orth_ws_bytes(Ctx& c, int64_t m, int l) { return orth_ws_bytes(m, l) + gram_ws_bytes(c, m, l); }

void orthonormalize(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar, const double* mu) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "orthonormalize: need 1 ≤ l ≤ %d, m ≥ l", kMaxL);
  double* U = ar.get<double>((size_t)l * l);
  double* G = ar.get<double>((size_t)l * l);
  double* M1 = ar.get<double>((size_t)l * l);
  double* R1 = ar.get<double>((size_t)l * l);
  double* M2 = ar.get<double>((size_t)l * l);
  double* R2 = ar.get<double>((size_t)l * l);
  const DenseA Yd{Y, RPCA_F64, m, l, l};
  const size_t mark = ar.off;
  lu_renorm(c, Y, m, l, U, nullptr, ar, mu);  // Y ← L (of Y − 1·mu when centring is pending)
  ar.off = mark;
  TagScope ts(c, "cholqr_gram");
  gram(c, Y, Y, m, l, G, ar);              // G = LᵀL
  ar.off = mark;
  chol(c, G, l, U, 0, M1, R1);             // R1·U
  c.tag = "cholqr_trmm";
  dense_ax(c, Yd, M1, l, Y, ar);           // Q1 = L·R1⁻¹
  ar.off = mark;
  c.tag = "cholqr_gram";
  gram(c, Y, Y, m, l, G, ar);              // G = Q1ᵀQ1
  ar.off = mark;
  chol(c, G, l, R1, 1, M2, R2);            // R = D·R2·R1·U
  c.tag = "cholqr_trmm";
  dense_ax(c, Yd, M2, l, Y, ar);           // Q = Q1·R2⁻¹·D
  ar.off = mark;
  if (R_out) RPCA_CUDA(cudaMemcpyAsync(R_out, R2, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, c.stream));
}

// Row-sharded variant: the LU is the sharded tournament,
// each Gram is the all-reduced sum of the per-shard Grams (fixed rank order),
// the l×l Cholesky runs redundantly on every rank and the triangular products
// stay local.
void orthonormalize_sharded(Ctx& c, double* Y, int64_t m, int64_t row0, int l, double* R_out, Arena& ar,
                            const double* mu) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= 0, RPCA_E_SHAPE, "orthonormalize: need 1 ≤ l ≤ %d", kMaxL);
  double* U = ar.get<double>((size_t)l * l);
  double* G = ar.get<double>((size_t)l * l);
  double* M1 = ar.get<double>((size_t)l * l);
  double* R1 = ar.get<double>((size_t)l * l);
  double* M2 = ar.get<double>((size_t)l * l);
  double* R2 = ar.get<double>((size_t)l * l);
  const DenseA Yd{Y, RPCA_F64, m, l, l};
  const size_t mark = ar.off;
  lu_renorm_sharded(c, Y, m, row0, l, U, ar, mu);  // Y ← L (local rows)
  ar.off = mark;
  auto gram_all = [&] {
    c.tag = "cholqr_gram";
    gram(c, Y, Y, m, l, G, ar);  // zero when this shard has no rows
    ar.off = mark;
    allreduce_sum(c, G, (size_t)l * l);
  };
  auto trmm = [&](const double* Mx) {
    c.tag = "cholqr_trmm";
    if (m > 0) dense_ax(c, Yd, Mx, l, Y, ar);
    ar.off = mark;
  };
  TagScope ts(c, "cholqr_gram");
  gram_all();
  chol(c, G, l, U, 0, M1, R1);
  trmm(M1);
  gram_all();
  chol(c, G, l, R1, 1, M2, R2);
  trmm(M2);
  if (R_out) RPCA_CUDA(cudaMemcpyAsync(R_out, R2, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace rpca
