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
// Cost: the LU passes + one more read/write of Y per Cholesky step; the Gram
// matrices are accumulated inside the kernels that write L and Q1 (fused).
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

// One CTA: G (upper, from per-CTA partials summed in ascending CTA order) →
// R = chol(G) (upper, CᵀC = G) → Rinv; Rtot = R·Rprev (Rprev upper or NULL);
// if `signfix`, D = sign(diag(Rtot)): Minv = Rinv·D, Rtot ← D·Rtot.
constexpr int kCholThreads = 1024;

__global__ void __launch_bounds__(kCholThreads) chol_partials_kernel(const double* __restrict__ part, int nparts, int l,
                                                                 const double* __restrict__ Rprev, int signfix,
                                                                 double* __restrict__ Minv,
                                                                 double* __restrict__ Rtot) {
  extern __shared__ double sm[];
  double* G = sm;              // l×l
  double* R = sm + l * l;      // l×l
  double* X = sm + 2 * l * l;  // l×l (inverse)
  double* Red = sm + 3 * l * l; // 8 × l(l+1)/2 reduction slices
  __shared__ double d[kMaxL];
  const int tid = threadIdx.x;
  const int npairs = l * (l + 1) / 2;
  // fixed-order two-level sum of the CTA partials: kSub interleaved slices per
  // entry (8 independent loads in flight each), then the slices in order
  constexpr int kSub = 8;
  double* red = Red;
  for (int e = tid; e < npairs * kSub; e += kCholThreads) {
    const int pq = e % npairs, sub = e / npairs;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = sub;
    for (; b + 3 * kSub < nparts; b += 4 * kSub) {
      a0 += part[(int64_t)b * npairs + pq];
      a1 += part[(int64_t)(b + kSub) * npairs + pq];
      a2 += part[(int64_t)(b + 2 * kSub) * npairs + pq];
      a3 += part[(int64_t)(b + 3 * kSub) * npairs + pq];
    }
    for (; b < nparts; b += kSub) a0 += part[(int64_t)b * npairs + pq];
    red[sub * npairs + pq] = (a0 + a1) + (a2 + a3);
  }
  __syncthreads();
  for (int pq = tid; pq < npairs; pq += kCholThreads) {
    double s = 0.0;
    for (int sub = 0; sub < kSub; ++sub) s += red[sub * npairs + pq];
    int p = 0, rem = pq;
    while (rem >= l - p) { rem -= l - p; ++p; }
    G[p * l + p + rem] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kCholThreads) R[idx] = 0.0;
  __syncthreads();
  const double gmax = [&] {
    double v = 0.0;
    for (int j = 0; j < l; ++j) v = fmax(v, G[j * l + j]);
    return v;
  }();
  for (int j = 0; j < l; ++j) {
    if (tid == 0) {
      double dj = G[j * l + j];
      for (int t = 0; t < j; ++t) dj -= R[t * l + j] * R[t * l + j];
      // L (and Q1) are full rank by construction; guard against roundoff only
      const double floor_ = 0x1p-104 * gmax;
      R[j * l + j] = sqrt(dj > floor_ ? dj : (floor_ > 0.0 ? floor_ : 1.0));
    }
    __syncthreads();
    for (int i = j + 1 + tid; i < l; i += kCholThreads) {
      double s = G[j * l + i];
      for (int t = 0; t < j; ++t) s -= R[t * l + j] * R[t * l + i];
      R[j * l + i] = s / R[j * l + j];
    }
    __syncthreads();
  }
  // X = R⁻¹ (upper), thread per column
  if (tid < l) {
    const int j = tid;
    for (int i = 0; i < l; ++i) X[i * l + j] = 0.0;
    X[j * l + j] = 1.0 / R[j * l + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int t = i + 1; t <= j; ++t) s += R[i * l + t] * X[t * l + j];
      X[i * l + j] = -s / R[i * l + i];
    }
  }
  __syncthreads();
  // Rtot = R·Rprev (both upper)
  for (int idx = tid; idx < l * l; idx += kCholThreads) {
    const int i = idx / l, j = idx - i * l;
    double s;
    if (!Rprev) s = R[idx];
    else {
      s = 0.0;
      for (int t = i; t <= j; ++t) s += R[i * l + t] * Rprev[t * l + j];
      if (j < i) s = 0.0;
    }
    G[idx] = s;  // reuse G for Rtot
  }
  __syncthreads();
  if (tid < l) d[tid] = (signfix && G[tid * l + tid] < 0.0) ? -1.0 : 1.0;
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kCholThreads) {
    const int i = idx / l, j = idx - i * l;
    Minv[idx] = X[idx] * d[j];
    Rtot[idx] = G[idx] * d[i];
  }
}

// Out = In·M (M upper l×l), in place allowed (tiles staged in smem); optional
// per-CTA upper Gram partial of Out.
__global__ void __launch_bounds__(kThreads, 2) right_mult_upper_kernel(double* __restrict__ Y, int64_t m, int l,
                                                                    const double* __restrict__ M,
                                                                    double* __restrict__ gpart) {
  extern __shared__ double sm[];
  const int ldw = l | 1;
  double* Ms = sm;
  double* Ys = sm + l * l;
  for (int idx = threadIdx.x; idx < l * l; idx += kThreads) Ms[idx] = M[idx];
  const int r = threadIdx.x & 127, jph = threadIdx.x >> 7;
  constexpr int kPairs = kMaxL * (kMaxL + 1) / 2 / kThreads + 1;
  double g[kPairs];
  uint16_t gp[kPairs], gq[kPairs];
  const int npairs = l * (l + 1) / 2;
#pragma unroll
  for (int i = 0; i < kPairs; ++i) {
    g[i] = 0.0;
    const int pq = threadIdx.x + i * kThreads;
    int p = 0, rem = pq < npairs ? pq : 0;
    while (rem >= l - p) { rem -= l - p; ++p; }
    gp[i] = (uint16_t)p;
    gq[i] = (uint16_t)(p + rem);
  }
  for (int64_t r0 = (int64_t)blockIdx.x * 128; r0 < m; r0 += (int64_t)gridDim.x * 128) {
    const int rows = (int)imin64(128, m - r0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) {
      const int rr = idx / l, t = idx - rr * l;
      Ys[rr * ldw + t] = Y[r0 * l + idx];
    }
    __syncthreads();
    double out[kMaxL / 2];
    if (r < rows) {
#pragma unroll
      for (int q = 0; q < kMaxL / 2; ++q) {
        const int j = jph + 2 * q;
        if (j >= l) break;
        double s = 0.0;
        for (int t = 0; t <= j; ++t) s += Ys[r * ldw + t] * Ms[t * l + j];
        out[q] = s;
      }
    }
    __syncthreads();
    if (r < rows) {
#pragma unroll
      for (int q = 0; q < kMaxL / 2; ++q) {
        const int j = jph + 2 * q;
        if (j >= l) break;
        Ys[r * ldw + j] = out[q];
        Y[(r0 + r) * l + j] = out[q];
      }
    }
    if (gpart) {
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kPairs; ++i) {
        if (threadIdx.x + i * kThreads >= npairs) break;
        const int p = gp[i], q = gq[i];
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int rr = 0;
        for (; rr + 4 <= rows; rr += 4) {
          s0 += Ys[rr * ldw + p] * Ys[rr * ldw + q];
          s1 += Ys[(rr + 1) * ldw + p] * Ys[(rr + 1) * ldw + q];
          s2 += Ys[(rr + 2) * ldw + p] * Ys[(rr + 2) * ldw + q];
          s3 += Ys[(rr + 3) * ldw + p] * Ys[(rr + 3) * ldw + q];
        }
        for (; rr < rows; ++rr) s0 += Ys[rr * ldw + p] * Ys[rr * ldw + q];
        g[i] += (s0 + s1) + (s2 + s3);
      }
    }
  }
  if (gpart) {
#pragma unroll
    for (int i = 0; i < kPairs; ++i) {
      const int pq = threadIdx.x + i * kThreads;
      if (pq < npairs) gpart[(int64_t)blockIdx.x * npairs + pq] = g[i];
    }
  }
}

}  // namespace

size_t orth_ws_bytes(int64_t m, int l) {
  Sizer s;
  s.add<double>((size_t)296 * l * (l + 1) / 2 + 64);  // partials (≤ 2·148 CTAs)
  s.add<double>((size_t)296 * l * (l + 1) / 2 + 64);
  s.add<double>(6 * (size_t)l * l);
  return s.total + lu_ws_bytes(m, l);
}

void orthonormalize(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "orthonormalize: need 1 ≤ l ≤ %d, m ≥ l", kMaxL);
  const int P = lu_apply_grid(c, m);
  const int npairs = l * (l + 1) / 2;
  double* p1 = ar.get<double>((size_t)P * npairs);
  double* p2 = ar.get<double>((size_t)P * npairs);
  double* U = ar.get<double>((size_t)l * l);
  double* M1 = ar.get<double>((size_t)l * l);
  double* R1 = ar.get<double>((size_t)l * l);
  double* M2 = ar.get<double>((size_t)l * l);
  double* R2 = ar.get<double>((size_t)l * l);
  lu_renorm(c, Y, m, l, U, nullptr, ar, p1);
  const int smem_c = (3 * l * l + 8 * npairs) * 8;
  ensure_smem((const void*)chol_partials_kernel, (3 * kMaxL * kMaxL + 8 * kMaxL * (kMaxL + 1) / 2) * 8);
  chol_partials_kernel<<<1, kCholThreads, smem_c, c.stream>>>(p1, P, l, U, 0, M1, R1);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "cholqr_chol");
  const int smem_r = (l * l + 128 * (l | 1)) * 8;
  ensure_smem((const void*)right_mult_upper_kernel, (kMaxL * kMaxL + 128 * (kMaxL | 1)) * 8);
  right_mult_upper_kernel<<<P, kThreads, smem_r, c.stream>>>(Y, m, l, M1, p2);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "cholqr_trmm");
  chol_partials_kernel<<<1, kCholThreads, smem_c, c.stream>>>(p2, P, l, R1, 1, M2, R2);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "cholqr_chol");
  right_mult_upper_kernel<<<P, kThreads, smem_r, c.stream>>>(Y, m, l, M2, nullptr);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "cholqr_trmm");
  if (R_out) RPCA_CUDA(cudaMemcpyAsync(R_out, R2, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace rpca
