// small.cu — the l×l work of §8(a) step a7 and of the Nyström path, in one
// CTA each (l ≤ 64: a 32 KB fp64 matrix in shared memory).
//
// jacobi_svd_small: the SVD of eq. (i3), PAPER.md:133-139 ("W Σ V* = B"),
// applied to the l×l triangular factor R of Bᵀ = Q_B·R (so B = Rᵀ Q_Bᵀ).
// One-sided Hestenes Jacobi on the columns of R (readings Q9/Q18):
// rotate a pair iff |γ| > l·2^-52·sqrt(αβ) — the rounding level of an l-term
// dot product (the oracle's 2^-52 is below it, so its cyclic sweeps keep
// rotating on rounding noise until the 30-sweep cap) — stop after a sweep
// without a rotation or after 30 sweeps.  Pairs are scheduled in parallel rounds
// (round-robin tournament: l/2 disjoint pairs per round, one warp per pair);
// the oracle sweeps cyclically — same fixed point up to rounding.
// Result: R·W = Vr·diag(σ), σ sorted non-increasing (stable), zero-σ
// columns of Vr completed by Gram–Schmidt of e_1, e_2, ….
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

// Zero-σ completion (rare): column col of Vout (l×l row-major) with σ = 0 is
// replaced by the Gram–Schmidt residual of the first e_t that keeps a norm
// ≥ 1/2 against the other columns (the largest residual if none does).
__device__ void complete_zero_sigma(const double* sigma, double* Vout, int l) {
  for (int col = 0; col < l; ++col) {
    if (sigma[col] > 0.0) continue;
    double best = -1.0;
    double v[kMaxL], bv[kMaxL];
    for (int t = 0; t < l; ++t) {
      for (int i = 0; i < l; ++i) v[i] = (i == t) ? 1.0 : 0.0;
      for (int pass = 0; pass < 2; ++pass)
        for (int s = 0; s < l; ++s) {
          if (s == col || (sigma[s] == 0.0 && s > col)) continue;
          double d = 0.0;
          for (int i = 0; i < l; ++i) d += Vout[i * l + s] * v[i];
          for (int i = 0; i < l; ++i) v[i] -= d * Vout[i * l + s];
        }
      double nv = 0.0;
      for (int i = 0; i < l; ++i) nv += v[i] * v[i];
      nv = sqrt(nv);
      if (nv > best) {
        best = nv;
        for (int i = 0; i < l; ++i) bv[i] = v[i];
      }
      if (nv >= 0.5) break;
    }
    for (int i = 0; i < l; ++i) Vout[i * l + col] = bv[i] / best;
  }
}

// Jacobi rotation zeroing γ between columns of squared norms α (lower index)
// and β: t = tan θ = sign(β−α)·2γ / (|β−α| + h), h = √((β−α)² + 4γ²), and
// since 1 + t² = 2h·d / d² with d = |β−α| + h:  cs = d/√(2hd), sn = ±2γ/√(2hd).
// One square root and one reciprocal square root on the dependent chain (the
// reciprocal of d, for tγ = the norm update, runs beside the latter).  The
// operands are O(l) after the 2^-E prescale of R, so no hypot scaling.
__device__ __forceinline__ void jacobi_rotation(double al, double be, double g, double& cs, double& sn,
                                                double& tg) {
  const double tau = be - al, sig = tau >= 0.0 ? 2.0 * g : -2.0 * g;
  const double h = sqrt(fma(tau, tau, sig * sig));
  const double d = fabs(tau) + h;
  const double r = rsqrt(2.0 * h * d);
  cs = d * r;
  sn = sig * r;
  tg = sig * g * rcp_nr(d);
}

// 2^-E with 2^E ≥ max |x| (the exponent field of the max |x|, clamped so both
// 2^±E are normal): applied to R it is exact and bounds every norm by O(l)
__device__ __forceinline__ int scale_exp_of(unsigned hi_max) {
  const int f = (int)(hi_max >> 20);  // biased exponent of the largest |R_ij|
  return f == 0 ? 0 : max(-1000, min(1000, f - 1022));
}
__device__ __forceinline__ double pow2(int e) { return __hiloint2double((1023 + e) << 20, 0); }

constexpr int kJThreads = 1024;  // one warp per column pair: l/2 ≤ 32 pairs in flight

__global__ void __launch_bounds__(kJThreads) jacobi_kernel(const double* __restrict__ R, int l,
                                                           double* __restrict__ sigma, double* __restrict__ Wout,
                                                           double* __restrict__ Vout) {
  // column-major: Mc[p*l + i] = M[i][p]; Wc likewise
  extern __shared__ double sm[];
  double* Mc = sm;
  double* Wc = sm + l * l;
  __shared__ double nrm[kMaxL];
  __shared__ double nrm2[kMaxL];  // ‖M[:, p]‖², refreshed every sweep, updated by each rotation
  __shared__ int rank_[kMaxL];
  __shared__ int rotated[2];
  __shared__ unsigned hmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nwarp = nthr >> 5;  // one warp per pair of a round
  if (tid == 0) hmax = 0u;
  __syncthreads();
  unsigned hm = 0u;
  for (int idx = tid; idx < l * l; idx += nthr) hm = max(hm, (unsigned)__double2hiint(R[idx]) & 0x7FFFFFFFu);
  hm = __reduce_max_sync(0xffffffffu, hm);
  if (lane == 0) atomicMax(&hmax, hm);
  __syncthreads();
  const int E = scale_exp_of(hmax);
  const double down = pow2(-E);
  for (int idx = tid; idx < l * l; idx += nthr) {
    const int i = idx / l, p = idx % l;
    Mc[p * l + i] = R[idx] * down;
    Wc[p * l + i] = (i == p) ? 1.0 : 0.0;
  }
  if (tid < 2) rotated[tid] = 0;
  __syncthreads();
  const int lp = (l + 1) & ~1;  // players (one dummy if l is odd)
  const double eps = 0x1p-52 * (double)l, eps2 = eps * eps;
  for (int sweep = 0; sweep < 30 && l > 1; ++sweep) {
    for (int p = warp; p < l; p += nwarp) {
      double s = 0.0;
      for (int i = lane; i < l; i += 32) s = fma(Mc[p * l + i], Mc[p * l + i], s);
      s = warp_sum(s);
      if (lane == 0) nrm2[p] = s;
    }
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      const int k = warp;
      if (k < lp / 2) {
        auto player = [&](int i) {  // 1 + (i − 1 + round) mod (lp − 1), both terms < lp − 1
          const int v = i - 1 + round;
          return i == 0 ? 0 : 1 + (v >= lp - 1 ? v - (lp - 1) : v);
        };
        int p = player(k), q = player(lp - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        if (q < l) {
          // lanes own rows i = lane, lane + 32 (l ≤ 64)
          const double x0 = lane < l ? Mc[p * l + lane] : 0.0, y0 = lane < l ? Mc[q * l + lane] : 0.0;
          const double x1 = lane + 32 < l ? Mc[p * l + lane + 32] : 0.0;
          const double y1 = lane + 32 < l ? Mc[q * l + lane + 32] : 0.0;
          // only γ is reduced; α, β follow the rotations exactly in exact
          // arithmetic (α' = α − tγ, β' = β + tγ) and are recomputed per sweep
          const double g = warp_sum(fma(x0, y0, x1 * y1));
          const double a = nrm2[p], b = nrm2[q];
          if (g * g > eps2 * (a * b)) {
            double cs, sn, tg;
            jacobi_rotation(a, b, g, cs, sn, tg);
            if (lane == 0) {
              rotated[sweep & 1] = 1;
              nrm2[p] = a - tg;
              nrm2[q] = b + tg;
            }
            if (lane < l) {
              Mc[p * l + lane] = cs * x0 - sn * y0;
              Mc[q * l + lane] = sn * x0 + cs * y0;
              const double u = Wc[p * l + lane], v = Wc[q * l + lane];
              Wc[p * l + lane] = cs * u - sn * v;
              Wc[q * l + lane] = sn * u + cs * v;
            }
            if (lane + 32 < l) {
              Mc[p * l + lane + 32] = cs * x1 - sn * y1;
              Mc[q * l + lane + 32] = sn * x1 + cs * y1;
              const double u = Wc[p * l + lane + 32], v = Wc[q * l + lane + 32];
              Wc[p * l + lane + 32] = cs * u - sn * v;
              Wc[q * l + lane + 32] = sn * u + cs * v;
            }
          }
        }
      }
      __syncthreads();
    }
    const int any = rotated[sweep & 1];
    __syncthreads();
    if (tid == 0) rotated[sweep & 1] = 0;
    if (!any) break;
  }
  // σ_p = ‖M[:, p]‖
  for (int p = warp; p < l; p += nwarp) {
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s += Mc[p * l + i] * Mc[p * l + i];
    s = warp_sum(s);
    if (lane == 0) nrm[p] = sqrt(s);
  }
  __syncthreads();
  if (tid < l) {  // stable descending rank
    int r = 0;
    for (int i = 0; i < l; ++i) r += (nrm[i] > nrm[tid]) || (nrm[i] == nrm[tid] && i < tid);
    rank_[tid] = r;
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nthr) {
    const int p = idx / l, i = idx % l;
    const int rp = rank_[p];
    Wout[i * l + rp] = Wc[p * l + i];
    Vout[i * l + rp] = nrm[p] > 0.0 ? Mc[p * l + i] / nrm[p] : 0.0;
  }
  if (tid < l) sigma[rank_[tid]] = nrm[tid] * pow2(E);
  __syncthreads();
  __threadfence_block();
  if (tid == 0) complete_zero_sigma(sigma, Vout, l);
}

// The same sweeps for l ≤ 32 in one warp, lane p owning column p of M and of
// W in registers: a round exchanges the partner's column by shuffles, both
// lanes of a pair compute the identical γ (same products, same order) and
// hence the identical rotation, and no barrier separates the rounds.
template <int LP>
__global__ void __launch_bounds__(32) jacobi_warp_kernel(const double* __restrict__ R, int l,
                                                         double* __restrict__ sigma, double* __restrict__ Wout,
                                                         double* __restrict__ Vout) {
  const unsigned full = 0xffffffffu;
  const int p = threadIdx.x;
  double m[LP], w[LP], y[LP];
  unsigned hm = 0u;
#pragma unroll
  for (int i = 0; i < LP; ++i) {
    m[i] = (i < l && p < l) ? R[i * l + p] : 0.0;
    w[i] = (i == p) ? 1.0 : 0.0;
    hm = max(hm, (unsigned)__double2hiint(m[i]) & 0x7FFFFFFFu);
  }
  const int E = scale_exp_of(__reduce_max_sync(full, hm));
  const double down = pow2(-E);
#pragma unroll
  for (int i = 0; i < LP; ++i) m[i] *= down;
  const int lp = (l + 1) & ~1;
  const double eps = 0x1p-52 * (double)l, eps2 = eps * eps;
  for (int sweep = 0; sweep < 30 && l > 1; ++sweep) {
    double a = 0.0;
#pragma unroll
    for (int i = 0; i < LP; ++i) a = fma(m[i], m[i], a);
    bool any = false;
    for (int round = 0; round < lp - 1; ++round) {
      // position of player p (inverse of player() in jacobi_kernel), its partner
      int q;
      if (p >= lp) q = p;
      else {
        int pos = 0;
        if (p > 0) { const int v = p - 1 - round; pos = 1 + (v < 0 ? v + (lp - 1) : v); }
        const int k = lp - 1 - pos;
        const int v = k - 1 + round;
        q = k == 0 ? 0 : 1 + (v >= lp - 1 ? v - (lp - 1) : v);
      }
      const bool pair = p < l && q < l;
      const int src = pair ? q : p;
      double g0 = 0.0, g1 = 0.0;
#pragma unroll
      for (int i = 0; i < LP; ++i) {
        y[i] = __shfl_sync(full, m[i], src);
        if (i & 1) g1 = fma(m[i], y[i], g1); else g0 = fma(m[i], y[i], g0);
      }
      const double g = g0 + g1;
      const double b = __shfl_sync(full, a, src);
      const bool lo = p < q;
      const double al = lo ? a : b, be = lo ? b : a;
      const bool act = pair && g * g > eps2 * (al * be);
      if (!__any_sync(full, act)) continue;
      any |= act;
      double cs = 1.0, sn = 0.0;
      if (act) {
        double tg;
        jacobi_rotation(al, be, g, cs, sn, tg);
        a = lo ? al - tg : be + tg;
        if (!lo) sn = -sn;  // hi column: sn·x + cs·y = cs·own − (−sn)·partner
      }
#pragma unroll
      for (int i = 0; i < LP; ++i) {
        const double wq = __shfl_sync(full, w[i], src);
        m[i] = cs * m[i] - sn * y[i];
        w[i] = cs * w[i] - sn * wq;
      }
    }
    if (!__any_sync(full, any)) break;
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < LP; ++i) s += m[i] * m[i];
  const double nrm = sqrt(s);
  int r = 0;
  for (int i = 0; i < l; ++i) {
    const double ni = __shfl_sync(full, nrm, i);
    r += (ni > nrm) || (ni == nrm && i < p);
  }
  if (p < l) {
#pragma unroll
    for (int i = 0; i < LP; ++i)
      if (i < l) {
        Wout[i * l + r] = w[i];
        Vout[i * l + r] = nrm > 0.0 ? m[i] / nrm : 0.0;
      }
    sigma[r] = nrm * pow2(E);
  }
  __syncwarp();
  __threadfence_block();
  if (p == 0) complete_zero_sigma(sigma, Vout, l);
}


// ---------------------------------------------------------------- Nyström
// Upper inverse X = C⁻¹ of an upper-triangular l×l C (thread per column).
__device__ void upper_inverse(const double* C, int l, double* X) {
  const int j = threadIdx.x;
  if (j < l) {
    for (int i = 0; i < l; ++i) X[i * l + j] = 0.0;
    X[j * l + j] = 1.0 / C[j * l + j];
    for (int i = j - 1; i >= 0; --i) {
      double s = 0.0;
      for (int t = i + 1; t <= j; ++t) s += C[i * l + t] * X[t * l + j];
      X[i * l + j] = -s / C[i * l + i];
    }
  }
}

__global__ void __launch_bounds__(kThreads) shift_chol_kernel(const double* __restrict__ G,
                                                              const double* __restrict__ fro2, int l, double sqrt_n,
                                                              double u, double* __restrict__ Minv,
                                                              double* __restrict__ nu_out, int* __restrict__ status) {
  extern __shared__ double sm[];
  double* B = sm;          // l×l, B2 = sym(G)
  double* C = sm + l * l;  // upper Cholesky factor
  __shared__ int fail;
  __shared__ double nu_s;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, q = idx % l;
    B[idx] = 0.5 * (G[p * l + q] + G[q * l + p]);
  }
  const double fro = sqrt(*fro2);
  if (tid == 0) nu_s = u * sqrt_n * fro;
  __syncthreads();
  if (fro == 0.0) {  // A·Q = 0: nothing to approximate (DESIGN.md reading)
    for (int idx = tid; idx < l * l; idx += kThreads) Minv[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
    if (tid == 0) { *nu_out = 0.0; *status = 2; }
    return;
  }
  int ok = 0;
  for (int attempt = 0; attempt <= 5 && !ok; ++attempt) {
    if (tid == 0) fail = 0;
    for (int idx = tid; idx < l * l; idx += kThreads) C[idx] = 0.0;
    __syncthreads();
    const double nu = nu_s;
    for (int j = 0; j < l; ++j) {
      if (tid == 0) {
        double d = B[j * l + j] + nu;
        for (int t = 0; t < j; ++t) d -= C[t * l + j] * C[t * l + j];
        if (!(d > 0.0)) fail = 1;
        else C[j * l + j] = sqrt(d);
      }
      __syncthreads();
      if (fail) break;
      for (int i = j + 1 + tid; i < l; i += kThreads) {
        double s = B[j * l + i];
        for (int t = 0; t < j; ++t) s -= C[t * l + j] * C[t * l + i];
        C[j * l + i] = s / C[j * l + j];
      }
      __syncthreads();
    }
    if (!fail) ok = 1;
    else {
      __syncthreads();
      if (tid == 0) nu_s *= 10.0;
      __syncthreads();
    }
  }
  if (!ok) {
    if (tid == 0) { *nu_out = nu_s; *status = 1; }
    return;
  }
  upper_inverse(C, l, B);  // reuse B as X
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kThreads) Minv[idx] = B[idx];
  if (tid == 0) { *nu_out = nu_s; *status = 0; }
}

// Parallel (Brent–Luk) two-sided Jacobi on a symmetric l×l matrix in shared
// memory: on return A is diagonal (its eigenvalues) and E (initialised here)
// holds the eigenvectors as columns.  Rotate iff |a_pq| > 2^-52·√|a_pp|·√|a_qq|,
// ≤ 30 sweeps (the oracle's rule, reading Q18).
__device__ void sym_jacobi(double* A, double* E, int l) {
  __shared__ double cs_[kMaxL / 2], sn_[kMaxL / 2];
  __shared__ int pp_[kMaxL / 2], qq_[kMaxL / 2];
  __shared__ int rotated;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < l * l; idx += blockDim.x) E[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
  __syncthreads();
  const int lp = (l + 1) & ~1;
  const double eps = 0x1p-52;
  for (int sweep = 0; sweep < 30 && l > 1; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < lp - 1; ++round) {
      for (int k = tid; k < lp / 2; k += blockDim.x) {
        auto player = [&](int i) {  // 1 + (i − 1 + round) mod (lp − 1), both terms < lp − 1
          const int v = i - 1 + round;
          return i == 0 ? 0 : 1 + (v >= lp - 1 ? v - (lp - 1) : v);
        };
        int p = player(k), q = player(lp - 1 - k);
        if (p > q) { const int t = p; p = q; q = t; }
        double c = 1.0, s = 0.0;
        if (q < l) {
          const double apq = A[p * l + q], app = A[p * l + p], aqq = A[q * l + q];
          if (fabs(apq) > eps * sqrt(fabs(app)) * sqrt(fabs(aqq))) {  // no overflow of app·aqq
            const double zeta = (aqq - app) / (2.0 * apq);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
            c = 1.0 / sqrt(1.0 + t * t);
            s = c * t;
            rotated = 1;
          }
        }
        pp_[k] = p; qq_[k] = q; cs_[k] = c; sn_[k] = s;
      }
      __syncthreads();
      // columns: A ← A·J, E ← E·J
      for (int idx = tid; idx < (lp / 2) * l; idx += blockDim.x) {
        const int k = idx / l, r = idx % l;
        const int p = pp_[k], q = qq_[k];
        if (q >= l || sn_[k] == 0.0) continue;
        const double c = cs_[k], s = sn_[k];
        const double x = A[r * l + p], y = A[r * l + q];
        A[r * l + p] = c * x - s * y;
        A[r * l + q] = s * x + c * y;
        const double u = E[r * l + p], v = E[r * l + q];
        E[r * l + p] = c * u - s * v;
        E[r * l + q] = s * u + c * v;
      }
      __syncthreads();
      // rows: A ← Jᵀ·A
      for (int idx = tid; idx < (lp / 2) * l; idx += blockDim.x) {
        const int k = idx / l, r = idx % l;
        const int p = pp_[k], q = qq_[k];
        if (q >= l || sn_[k] == 0.0) continue;
        const double c = cs_[k], s = sn_[k];
        const double x = A[p * l + r], y = A[q * l + r];
        A[p * l + r] = c * x - s * y;
        A[q * l + r] = s * x + c * y;
      }
      __syncthreads();
      for (int k = tid; k < lp / 2; k += blockDim.x)
        if (qq_[k] < l && sn_[k] != 0.0) A[pp_[k] * l + qq_[k]] = A[qq_[k] * l + pp_[k]] = 0.0;
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
}

// Regularised inverse square root of the symmetric B2: Minv = E·diag(d)·Eᵀ.
__global__ void __launch_bounds__(kThreads) sqrt_inv_kernel(const double* __restrict__ G, int l,
                                                            double* __restrict__ Minv, double* __restrict__ nu_out,
                                                            int* __restrict__ status) {
  extern __shared__ double sm[];
  double* A = sm;          // l×l row-major
  double* E = sm + l * l;  // eigenvectors (columns)
  __shared__ double mu[kMaxL], dd[kMaxL];
  __shared__ int rk[kMaxL];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, q = idx % l;
    A[idx] = 0.5 * (G[p * l + q] + G[q * l + p]);
  }
  __syncthreads();
  sym_jacobi(A, E, l);
  if (tid < l) {
    int r = 0;
    const double v = A[tid * l + tid];
    for (int i = 0; i < l; ++i) {
      const double w = A[i * l + i];
      r += (w > v) || (w == v && i < tid);
    }
    rk[tid] = r;
  }
  __syncthreads();
  if (tid < l) mu[rk[tid]] = A[tid * l + tid];
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int j = 0; j < l; ++j) mx = fmax(mx, fabs(mu[j]));
    const int bad = mu[l - 1] < -1e-6 * mx;
    const double smax = sqrt(fmax(mu[0], 0.0));
    for (int j = 0; j < l; ++j) {
      const double sj = sqrt(fmax(mu[j], 0.0));
      dd[j] = (sj > 1e-12 * smax && sj > 0.0) ? 1.0 / sj : 0.0;
    }
    *status = bad ? 1 : 0;
    *nu_out = 0.0;
  }
  __syncthreads();
  // Minv[p][q] = Σ_t E[p][t'] d_t E[q][t'] where t' is the column of rank t
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, q = idx % l;
    double s = 0.0;
    for (int t = 0; t < l; ++t) s += E[p * l + t] * dd[rk[t]] * E[q * l + t];
    Minv[idx] = s;
  }
}

// reig: T = sym(G) = E·diag(λ)·Eᵀ; the
// eigenvalues ordered by |λ| descending (ties: the larger λ, then the lower
// index — the oracle's order), lam[j] = λ of rank j (signed), Eo[:, j] its
// eigenvector.
__global__ void __launch_bounds__(kThreads) sym_eig_abs_kernel(const double* __restrict__ G, int l,
                                                               double* __restrict__ lam, double* __restrict__ Eo) {
  extern __shared__ double sm[];
  double* A = sm;
  double* E = sm + l * l;
  __shared__ int col_of[kMaxL];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, q = idx % l;
    A[idx] = 0.5 * (G[p * l + q] + G[q * l + p]);
  }
  __syncthreads();
  sym_jacobi(A, E, l);
  // rank among the eigenvalues in the oracle's order: oracle_jacobi_eig sorts
  // λ non-increasing (stable in index), then reig stable-sorts by |λ| with the
  // larger λ first on |λ| ties — both tie-breaks reduce to the lower index
  if (tid < l) {
    const double v = A[tid * l + tid];
    int r = 0;
    for (int i = 0; i < l; ++i) {
      const double w = A[i * l + i];
      const bool before = fabs(w) > fabs(v) || (fabs(w) == fabs(v) && (w > v || (w == v && i < tid)));
      r += before;
    }
    col_of[r] = tid;
  }
  __syncthreads();
  for (int j = tid; j < l; j += kThreads) lam[j] = A[col_of[j] * l + col_of[j]];
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int p = idx / l, j = idx % l;
    Eo[idx] = E[p * l + col_of[j]];
  }
}

template <class T>
__global__ void lambda_kernel(const double* __restrict__ sigma, const double* __restrict__ nu, int k,
                              T* __restrict__ lam) {
  const int j = threadIdx.x;
  if (j < k) {
    const double v = sigma[j] * sigma[j] - *nu;
    lam[j] = static_cast<T>(v > 0.0 ? v : 0.0);
  }
}

__global__ void power_step_kernel(const double* __restrict__ nz2, double* __restrict__ z, double* __restrict__ x,
                                  int64_t n, double* __restrict__ est, int* __restrict__ done) {
  const double nz = sqrt(*nz2);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!*done) {
      if (nz == 0.0) { *est = 0.0; *done = 1; }
      else *est = sqrt(nz);
    }
  }
  const double inv = nz > 0.0 ? 1.0 / nz : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = z[i] * inv;
}

}  // namespace

void jacobi_svd_small(Ctx& c, const double* R, int l, double* sigma, double* W, double* Vr) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "jacobi: l=%d", l);
#ifndef JACOBI_NO_WARP  // ablation: the shared-memory kernel for every l
  if (l <= 32) {
    auto k = l <= 8 ? jacobi_warp_kernel<8> : l <= 16 ? jacobi_warp_kernel<16>
           : l <= 24 ? jacobi_warp_kernel<24> : jacobi_warp_kernel<32>;
    k<<<1, 32, 0, c.stream>>>(R, l, sigma, W, Vr);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "jacobi");
    return;
  }
#endif
  const int smem = 2 * l * l * 8;
  ensure_smem((const void*)jacobi_kernel, 2 * kMaxL * kMaxL * 8);
  const int threads = 32 * std::max(1, ((l + 1) & ~1) / 2);  // one warp per pair of a round
  jacobi_kernel<<<1, threads, smem, c.stream>>>(R, l, sigma, W, Vr);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "jacobi");
}


void nystrom_shift_chol(Ctx& c, const double* G, const double* fro2, int l, int64_t n, double unit_roundoff,
                        double* Minv, double* nu, int* status) {
  ensure_smem((const void*)shift_chol_kernel, 2 * kMaxL * kMaxL * 8);
  shift_chol_kernel<<<1, kThreads, 2 * l * l * 8, c.stream>>>(G, fro2, l, sqrt((double)n), unit_roundoff, Minv, nu,
                                                              status);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void nystrom_sqrt(Ctx& c, const double* G, int l, double* Minv, double* nu, int* status) {
  ensure_smem((const void*)sqrt_inv_kernel, 2 * kMaxL * kMaxL * 8);
  sqrt_inv_kernel<<<1, kThreads, 2 * l * l * 8, c.stream>>>(G, l, Minv, nu, status);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void sym_eig_abs(Ctx& c, const double* G, int l, double* lam, double* E) {
  const int smem = 2 * l * l * 8;
  ensure_smem((const void*)sym_eig_abs_kernel, 2 * kMaxL * kMaxL * 8);
  sym_eig_abs_kernel<<<1, kThreads, smem, c.stream>>>(G, l, lam, E);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "jacobi");
}

void nystrom_lambda(Ctx& c, const double* sigma, const double* nu, int k, void* lam, int dtype) {
  if (dtype == RPCA_F64) lambda_kernel<double><<<1, 64, 0, c.stream>>>(sigma, nu, k, (double*)lam);
  else lambda_kernel<float><<<1, 64, 0, c.stream>>>(sigma, nu, k, (float*)lam);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void power_step(Ctx& c, const double* nz2, double* z, double* x, int64_t n, double* est, int* done) {
  const unsigned grid = (unsigned)std::min<int64_t>(std::max<int64_t>(1, cdiv(n, 256)), (int64_t)c.num_sms * 8);
  power_step_kernel<<<grid, 256, 0, c.stream>>>(nz2, z, x, n, est, done);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

}  // namespace rpca
