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
// A Cholesky pivot of LᵀL below 2^-40 of its largest diagonal (κ(L) ≳ 1e6,
// far from CholeskyQR2's failure at κ ≈ u^-1/2 ≈ 7e7, which LU's bounded
// multipliers make rare) flags a breakdown: the driver then re-runs the call
// with Householder TSQR for every final orthonormalisation.
constexpr double kBreakdown = 0x1p-40;

// One CTA: R = chol(G) (upper, RᵀR = G, G full l×l) → X = R⁻¹ (upper);
// Rtot = R·Rprev (Rprev upper or NULL); if `signfix`, D = sign(diag(Rtot)):
// Minv = X·D, Rtot ← D·Rtot.
__global__ void __launch_bounds__(kThreads) chol_kernel(const double* __restrict__ Gin, int l,
                                                        const double* __restrict__ Rprev, int signfix,
                                                        double* __restrict__ Minv, double* __restrict__ Rtot,
                                                        int* __restrict__ breakdown) {
  extern __shared__ double sm[];
  double* G = sm;              // l×l
  double* R = sm + l * l;      // l×l
  double* X = sm + 2 * l * l;  // l×l (inverse)
  double* P = sm + 3 * l * l;  // l×l (Rprev)
  __shared__ double d[kMaxL];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = kMaxL * kMaxL / kThreads;
  {  // every global read issued before the first use (one round trip)
    double g0[kPer], g1[kPer], pr[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + k * kThreads;
      const int p = idx / l, q = idx - p * l;
      const bool in = idx < l * l;
      g0[k] = in ? Gin[idx] : 0.0;
      g1[k] = in ? Gin[q * l + p] : 0.0;
      pr[k] = in && Rprev ? Rprev[idx] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int idx = tid + k * kThreads;
      if (idx < l * l) {
        G[idx] = 0.5 * (g0[k] + g1[k]);
        R[idx] = 0.0;
        P[idx] = pr[k];
      }
    }
  }
  __syncthreads();
  double gmax = 0.0;
  for (int j = 0; j < l; ++j) gmax = fmax(gmax, G[j * l + j]);
  // right-looking, one barrier per column: every thread forms the pivot's
  // reciprocal square root itself (same bits everywhere), then row j of R and
  // the rank-1 update of the trailing block of G, G_ab −= G_ja·G_jb / G_jj
  // (row j of G is not written in step j)
  const double floor_ = 0x1p-104 * gmax;  // L (and Q1) are full rank; guard against roundoff only
  for (int j = 0; j < l; ++j) {
    const double dj = G[j * l + j];
    if (breakdown && tid == 0 && !(dj > kBreakdown * gmax)) *breakdown = 1;
    const double dc = dj > floor_ ? dj : (floor_ > 0.0 ? floor_ : 1.0);
    const double ri = rsqrt(dc);  // 1/R_jj
    for (int i = j + tid; i < l; i += kThreads) R[j * l + i] = i == j ? dc * ri : G[j * l + i] * ri;
    if (tid == 0) d[j] = ri;
    const double ri2 = ri * ri;
    for (int a = j + 1 + warp; a < l; a += kThreads / 32) {
      const double ga = G[j * l + a] * ri2;
      for (int b = j + 1 + lane; b < l; b += 32) G[a * l + b] = fma(-ga, G[j * l + b], G[a * l + b]);
    }
    __syncthreads();
  }
  // X = R⁻¹ (upper): thread j owns column j, back substitution with i
  // descending (R reads are broadcasts), four partial sums per dot product
  if (tid < l) {
    const int j = tid;
    for (int i = l - 1; i > j; --i) X[i * l + j] = 0.0;
    for (int i = j; i >= 0; --i) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const double* ri = R + i * l;
      int t = i + 1;
      for (; t + 3 <= j; t += 4) {
        a0 = fma(ri[t], X[t * l + j], a0);
        a1 = fma(ri[t + 1], X[(t + 1) * l + j], a1);
        a2 = fma(ri[t + 2], X[(t + 2) * l + j], a2);
        a3 = fma(ri[t + 3], X[(t + 3) * l + j], a3);
      }
      for (; t <= j; ++t) a0 = fma(ri[t], X[t * l + j], a0);
      X[i * l + j] = ((i == j ? 1.0 : 0.0) - ((a0 + a1) + (a2 + a3))) * d[i];
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
      for (int t = i; t <= j; ++t) s = fma(R[i * l + t], P[t * l + j], s);
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

// The same contract for l ≤ 32 in ONE warp, no barriers: lane b holds column
// b of G, then of R (and of Rprev), in registers (LP = l rounded up to 8,
// static indices); during the Cholesky the values of other columns arrive by
// broadcast shuffles.  Order: Cholesky (right-looking), then Rtot = R·Rprev
// and its row signs, then X = R⁻¹ written with the column signs.  The two
// triangular products read the rows of R from a shared-memory copy (broadcast
// loads): with a shuffle per term they were 80% of the kernel at l = 32 (a
// shuffle in every link of the FMA chain).  Same FMA order either way.
template <int LP>
__global__ void __launch_bounds__(32) chol_warp_kernel(const double* __restrict__ Gin, int l,
                                                       const double* __restrict__ Rprev, int signfix,
                                                       double* __restrict__ Minv, double* __restrict__ Rtot,
                                                       int* __restrict__ breakdown) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x;
  const bool own = lane < l;
  double g[LP], r[LP], pc[LP], d[LP];
#pragma unroll
  for (int i = 0; i < LP; ++i) {
    const bool in = own && i < l;
    g[i] = in ? 0.5 * (Gin[i * l + lane] + Gin[lane * l + i]) : 0.0;
    pc[i] = in && Rprev ? Rprev[i * l + lane] : 0.0;
    r[i] = 0.0;
  }
  double gmax = 0.0;
#pragma unroll
  for (int j = 0; j < LP; ++j) gmax = fmax(gmax, __shfl_sync(FULL, g[j], j));  // lanes ≥ l hold 0
  const double floor_ = 0x1p-104 * gmax;
#ifndef CHOL_ROLLED
#define CHOL_ROLLED 1
#endif
  // R row-major in shared memory: Rs[i][t] = R[i][t] (lane t holds column t)
  __shared__ double Rs[LP][LP + 1];
#if CHOL_ROLLED
  // Column steps as a rolled loop over a register window (window slot t holds
  // column j + t at step j, shifted left after each step): the same FMAs in
  // the same order as the unrolled form below, at 1/LP of its code — the
  // unrolled kernel (one warp, run once per call) was bound by instruction
  // fetch.  Slots past column LP−1 hold values never read back.
  __shared__ double ds[LP];
#pragma unroll 1
  for (int j = 0; j < l; ++j) {
    const double dj = __shfl_sync(FULL, g[0], j);
    if (breakdown && lane == 0 && !(dj > kBreakdown * gmax)) *breakdown = 1;
    const double dc = dj > floor_ ? dj : (floor_ > 0.0 ? floor_ : 1.0);
    const double ri = rsqrt(dc);
    if (lane == 0) ds[j] = ri;
    const double rjb = lane == j ? dc * ri : (lane > j ? g[0] * ri : 0.0);  // R[j][lane]
    if (lane < LP) Rs[j][lane] = rjb;
#pragma unroll
    for (int t = 1; t < LP; ++t) {
      const double rja = __shfl_sync(FULL, rjb, (j + t) & 31);
      g[t] = fma(-rja, rjb, g[t]);
    }
#pragma unroll
    for (int t = 0; t < LP - 1; ++t) g[t] = g[t + 1];
    g[LP - 1] = 0.0;
  }
  for (int j = l; j < LP; ++j)
    if (lane < LP) Rs[j][lane] = 0.0;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < LP; ++i) {
    r[i] = lane < LP ? Rs[i][lane] : 0.0;
    d[i] = i < l ? ds[i] : 0.0;
  }
#else
#pragma unroll
  for (int j = 0; j < LP; ++j) {
    if (j >= l) break;
    const double dj = __shfl_sync(FULL, g[j], j);
    if (breakdown && lane == 0 && !(dj > kBreakdown * gmax)) *breakdown = 1;
    const double dc = dj > floor_ ? dj : (floor_ > 0.0 ? floor_ : 1.0);
    const double ri = rsqrt(dc);
    d[j] = ri;
    const double rjb = lane == j ? dc * ri : (lane > j ? g[j] * ri : 0.0);  // R[j][lane]
    r[j] = rjb;
#pragma unroll
    for (int a = j + 1; a < LP; ++a) {
      const double rja = __shfl_sync(FULL, rjb, a);
      g[a] = fma(-rja, rjb, g[a]);
    }
  }
#if !CHOL_ROLLED
#pragma unroll
  for (int i = 0; i < LP; ++i)
    if (lane < LP) Rs[i][lane] = r[i];
  __syncwarp();
#endif
#endif
  // Rtot = R·Rprev (column `lane`), reusing g; row signs from its diagonal
#pragma unroll
  for (int i = 0; i < LP; ++i) {
    double s = 0.0;
    if (!Rprev) {
      s = r[i];
    } else {
#pragma unroll
      for (int t = i; t < LP; ++t) s = fma(Rs[i][t], pc[t], s);
    }
    g[i] = s;
  }
  double sg[LP];
#pragma unroll
  for (int i = 0; i < LP; ++i) sg[i] = (signfix && __shfl_sync(FULL, g[i], i) < 0.0) ? -1.0 : 1.0;
  if (own)
#pragma unroll
    for (int i = 0; i < LP; ++i)
      if (i < l) Rtot[i * l + lane] = g[i] * sg[i];
  // X = R⁻¹, column `lane` (upper), back substitution; reuse pc
  double dl = 1.0;  // this column's sign
#pragma unroll
  for (int i = 0; i < LP; ++i)
    if (i == lane) dl = sg[i];
#pragma unroll
  for (int i = LP - 1; i >= 0; --i) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int t = i + 1; t < LP; ++t) {
      const double rit = Rs[i][t];
      if ((t - i) & 1) a0 = fma(rit, pc[t], a0);
      else a1 = fma(rit, pc[t], a1);
    }
    pc[i] = i < l && i <= lane ? ((i == lane ? 1.0 : 0.0) - (a0 + a1)) * d[i] : 0.0;
  }
  if (own)
#pragma unroll
    for (int i = 0; i < LP; ++i)
      if (i < l) Minv[i * l + lane] = pc[i] * dl;
}

void chol(Ctx& c, const double* G, int l, const double* Rprev, int signfix, double* Minv, double* Rtot,
          int* bd = nullptr) {
  switch ((l + 7) & ~7) {
    case 8: chol_warp_kernel<8><<<1, 32, 0, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot, bd); break;
    case 16: chol_warp_kernel<16><<<1, 32, 0, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot, bd); break;
    case 24: chol_warp_kernel<24><<<1, 32, 0, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot, bd); break;
    case 32: chol_warp_kernel<32><<<1, 32, 0, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot, bd); break;
    default:
      ensure_smem((const void*)chol_kernel, 4 * kMaxL * kMaxL * 8);
      chol_kernel<<<1, kThreads, 4 * l * l * 8, c.stream>>>(G, l, Rprev, signfix, Minv, Rtot, bd);
  }
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
  chol(c, G, l, U, 0, M1, R1, breakdown_flag(c));  // R1·U
  c.tag = "cholqr_trmm";
  dense_ax(c, Yd, M1, l, Y, ar, nullptr, true);  // Q1 = L·R1⁻¹
  ar.off = mark;
  c.tag = "cholqr_gram";
  gram(c, Y, Y, m, l, G, ar);              // G = Q1ᵀQ1
  ar.off = mark;
  chol(c, G, l, R1, 1, M2, R2);            // R = D·R2·R1·U
  c.tag = "cholqr_trmm";
  dense_ax(c, Yd, M2, l, Y, ar, nullptr, true);  // Q = Q1·R2⁻¹·D
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
    if (m > 0) dense_ax(c, Yd, Mx, l, Y, ar, nullptr, true);
    ar.off = mark;
  };
  TagScope ts(c, "cholqr_gram");
  gram_all();
  chol(c, G, l, U, 0, M1, R1, breakdown_flag(c));
  trmm(M1);
  gram_all();
  chol(c, G, l, R1, 1, M2, R2);
  trmm(M2);
  if (R_out) RPCA_CUDA(cudaMemcpyAsync(R_out, R2, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, c.stream));
}

// ---------------------------------------------------------------- fallback
// Householder TSQR (tsqr.cu) for the final orthonormalisation when the
// LU-Cholesky-QR2 above flagged a breakdown (kBreakdown): unconditionally
// backward stable, slower (≈ 4 block passes, one CTA per leaf).

namespace {
// out (l×l) = the rows × l block `in` zero-padded to l rows
__global__ void pad_rows_kernel(const double* __restrict__ in, int64_t rows, int l, double* __restrict__ out) {
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) out[idx] = idx / l < rows ? in[idx] : 0.0;
}
}  // namespace

size_t orth_house_ws_bytes(int64_t m, int l, int nranks) {
  Sizer s;
  s.add<double>((size_t)nranks * l * l * 2 + 2 * (size_t)l * l);
  s.add<double>((size_t)std::max<int64_t>(m, 1) * l);
  const int64_t stack = std::max<int64_t>((int64_t)nranks * l, l);
  return s.total + std::max(qr_ws_bytes(std::max<int64_t>(m, l), l), qr_ws_bytes(stack, l)) +
         thin_gemm_ws_bytes(std::max<int64_t>(m, 1), l, l) + 65536;
}

void orthonormalize_house(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar, const double* mu) {
  if (mu) sub_rank1(c, Y, m, l, nullptr, mu);
  qr(c, Y, m, l, R_out, ar);
}

// Rows [row0, row0+m) of a row-sharded block: local QR (Y_p = Q_p·R_p; a shard
// of fewer than l rows is its own R, zero-padded, with Q_p = I), the l×l R_p
// all-gathered in rank order, QR of the stack (the same bytes on every rank ⇒
// the same Q_s, R), Y_p ← Q_p·Q_s[rank].  diag(R) ≥ 0 from the stack's QR.
void orthonormalize_house_sharded(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar,
                                  const double* mu) {
  const int P = comm_size(c), rank = c.comm ? c.comm->rank : 0;
  const size_t ll = (size_t)l * l;
  double* Rp = ar.get<double>(ll);
  double* stack = ar.get<double>((size_t)P * ll);
  double* Rs = ar.get<double>(ll);
  double* tmp = ar.get<double>((size_t)std::max<int64_t>(m, 1) * l);
  const size_t mark = ar.off;
  if (mu && m > 0) sub_rank1(c, Y, m, l, nullptr, mu);
  const bool local_qr = m >= l;
  if (local_qr) {
    qr(c, Y, m, l, Rp, ar);  // Y ← Q_p
    ar.off = mark;
  } else {
    pad_rows_kernel<<<1, 256, 0, c.stream>>>(Y, m, l, Rp);
    RPCA_CHECK_LAUNCH();
    count_launch(c);
  }
  allgather_bytes(c, Rp, stack, ll * sizeof(double));
  qr(c, stack, (int64_t)P * l, l, Rs, ar);  // stack ← Q_s (P·l × l)
  ar.off = mark;
  const double* slice = stack + (size_t)rank * ll;
  if (local_qr) {
    thin_gemm(c, Y, m, l, slice, l, nullptr, tmp, l, RPCA_F64, ar);
    RPCA_CUDA(cudaMemcpyAsync(Y, tmp, (size_t)m * l * 8, cudaMemcpyDeviceToDevice, c.stream));
  } else if (m > 0) {
    RPCA_CUDA(cudaMemcpyAsync(Y, slice, (size_t)m * l * 8, cudaMemcpyDeviceToDevice, c.stream));
  }
  ar.off = mark;
  if (R_out) RPCA_CUDA(cudaMemcpyAsync(R_out, Rs, ll * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace rpca
