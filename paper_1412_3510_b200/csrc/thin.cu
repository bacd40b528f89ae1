// thin.cu — kernels on the thin blocks (m×l, n×l, l×l) of the randomized PCA
// path: operand packing for the DMMA kernels, the rank-1 centring corrections
// of PAPER.md:427-435 ("Q = A*Q - ones(m,1)*(c*Q)"), column means
// (PAPER.md:428-429), the lift U = Q·W of eq. (i4) and
// the sign convention of DESIGN.md reading Q10.  All HBM-bound; every
// reduction runs in a fixed order (fixed row chunks, ascending).
#include "comm.cuh"

namespace rpca {
namespace {

constexpr int kChunk = 8192;  // rows per partial in the two-stage reductions

// Packed X for dense_ax (fragment-major, see dense_ax.cu):
// Xp[kb][s][nt][lane] = X[kb*32 + 16*(s>>2) + 4*(lane&3) + 2*((s>>1)&1) + (s&1)][nt*8 + (lane>>2)]
template <int NT>  // as pack_y_kernel: no runtime 64-bit division per element
__global__ void pack_x_kernel(const double* __restrict__ X, int64_t n, int l, int64_t total,
                              double* __restrict__ Xp) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    int64_t t = idx >> 5;
    const int nt = (int)(t % NT);
    t /= NT;
    const int s = (int)(t & 7);
    const int64_t kb = t >> 3;
    const int64_t k = kb * 32 + 16 * (s >> 2) + 4 * (lane & 3) + 2 * ((s >> 1) & 1) + (s & 1);
    const int j = nt * 8 + (lane >> 2);
    Xp[idx] = (k < n && j < l) ? X[k * l + j] : 0.0;
  }
}

// Packed Y for dense_aty: Yp[g][s][nt][lane] = Y[8g + 2*(lane&3) + s][nt*8 + (lane>>2)]
// NT = ⌈l/8⌉ is a template constant: a runtime 64-bit division per element
// had made this copy instruction-bound (C2: 12 µs for 35 MB)
template <int NT>
__global__ void pack_y_kernel(const double* __restrict__ Y, int64_t m, int l, int64_t total,
                              const double* __restrict__ ymean, double* __restrict__ Yp) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int lane = (int)(idx & 31);
    int64_t t = idx >> 5;
    const int nt = (int)(t % NT);
    t /= NT;
    const int s = (int)(t & 1);
    const int64_t g = t >> 1;
    const int64_t i = 8 * g + 2 * (lane & 3) + s;
    const int j = nt * 8 + (lane >> 2);
    Yp[idx] = (i < m && j < l) ? Y[i * l + j] - (ymean ? ymean[j] : 0.0) : 0.0;
  }
}

// partial[b][j] = Σ_{i in chunk b} a[i]·X[i][j]  (a == NULL ⇒ 1); chunks of
// kColChunk rows, threads (phase, column) read whole rows (coalesced), eight
// independent accumulators per thread, fixed order
constexpr int kColChunk = 2048;
__global__ void __launch_bounds__(256) wcolsum_partial(const double* __restrict__ a, const double* __restrict__ X,
                                                      int64_t rows, int l, int64_t ldx, double* __restrict__ part) {
  __shared__ double red[256];
  const int64_t r0 = (int64_t)blockIdx.x * kColChunk;
  const int64_t r1 = min(rows, r0 + kColChunk);
  const int phases = 256 / l;  // l ≤ 64 ⇒ ≥ 4 phases
  const int ph = threadIdx.x / l, j = threadIdx.x % l;
  double s[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) s[u] = 0.0;
  if (ph < phases) {
    int64_t i = r0 + ph;
    for (; i + 7 * phases < r1; i += 8 * phases) {  // eight loads in flight per thread
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = X[(i + u * phases) * ldx + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s[u] += (a ? a[i + u * phases] : 1.0) * x[u];
    }
    for (; i < r1; i += phases) s[0] += (a ? a[i] : 1.0) * X[i * ldx + j];
  }
  red[threadIdx.x] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  __syncthreads();
  if (threadIdx.x < l) {
    double t = 0.0;
    for (int p = 0; p < phases; ++p) t += red[p * l + threadIdx.x];
    part[(int64_t)blockIdx.x * l + threadIdx.x] = t;
  }
}

// v[j] = scale·Σ_b part[b][j]: warp w of the 32 sums the partials
// b ≡ w (mod 32) in ascending order (eight loads in flight), then the 32
// warp sums are added in order — fixed order, one CTA
constexpr int kSumWarps = 32;
__global__ void __launch_bounds__(32 * kSumWarps) sum_partials_8w(const double* __restrict__ part, int64_t nparts,
                                                                 int l, double scale, double* __restrict__ v) {
  __shared__ double red[kSumWarps][kMaxL];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int W = kSumWarps;
  for (int j = lane; j < l; j += 32) {
    double s = 0.0;
    int64_t b = warp;
    for (; b + 7 * W < nparts; b += 8 * W) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = part[(b + W * u) * l + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += x[u];
    }
    for (; b < nparts; b += W) s += part[b * l + j];
    red[warp][j] = s;
  }
  __syncthreads();
  if (threadIdx.x < l) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < W; ++w) t += red[w][threadIdx.x];
    v[threadIdx.x] = t * scale;
  }
}


__global__ void sub_rank1_kernel(double* __restrict__ Y, int64_t rows, int l, const double* __restrict__ u,
                                 const double* __restrict__ v, double alpha) {
  const int64_t total = rows * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / l;
    const int j = (int)(idx - i * l);
    Y[idx] -= (u ? u[i] : 1.0) * (alpha * v[j]);
  }
}

template <class T>
__global__ void colsum_dense_partial(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                     double* __restrict__ part) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t r0 = (int64_t)blockIdx.y * kChunk, r1 = min(m, r0 + kChunk);
  double s = 0.0;
  for (int64_t i = r0; i < r1; ++i) s += static_cast<double>(A[i * lda + j]);
  part[(int64_t)blockIdx.y * n + j] = s;
}

__global__ void colsum_dense_final(const double* __restrict__ part, int64_t nparts, int64_t n, double inv_m,
                                   double* __restrict__ c) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int64_t b = 0; b < nparts; ++b) s += part[b * n + j];
  c[j] = s * inv_m;
}

template <class T>
__device__ __forceinline__ T cast_out(double v) { return static_cast<T>(v); }

// Wk (l×k) = W[:, :k]·diag(sign)   (W l×l, sign may be NULL)
__global__ void scale_cols_kernel(const double* __restrict__ W, int l, int k, const double* __restrict__ sign,
                                  double* __restrict__ Wk) {
  for (int idx = threadIdx.x; idx < l * k; idx += blockDim.x) {
    const int t = idx / k, j = idx - t * k;
    Wk[idx] = W[t * l + j] * (sign ? sign[j] : 1.0);
  }
}

struct ArgBest {
  double v;
  int64_t i;
};
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

// per (chunk, column) largest |V[i][j]| with the lowest i on ties
__global__ void argmax_partial(const double* __restrict__ V, int64_t rows, int k, int64_t ldv,
                               double* __restrict__ pv, int64_t* __restrict__ pi) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  const int j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * kChunk, r1 = min(rows, r0 + kChunk);
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double v = fabs(V[i * ldv + j]);
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o && better(sv[threadIdx.x + o], si[threadIdx.x + o], sv[threadIdx.x], si[threadIdx.x])) {
      sv[threadIdx.x] = sv[threadIdx.x + o];
      si[threadIdx.x] = si[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[(int64_t)blockIdx.x * k + j] = sv[0];
    pi[(int64_t)blockIdx.x * k + j] = si[0];
  }
}

__global__ void argmax_final(const double* __restrict__ V, int64_t ldv, const double* __restrict__ pv,
                             const int64_t* __restrict__ pi, int64_t nparts, int k, double* __restrict__ sign) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t b = 0; b < nparts; ++b) {
    if (better(pv[b * k + j], pi[b * k + j], bv, bi)) { bv = pv[b * k + j]; bi = pi[b * k + j]; }
  }
  sign[j] = (bi != INT64_MAX && V[bi * ldv + j] < 0.0) ? -1.0 : 1.0;
}

// Row-sharded variant, stage 1: this shard's winner of column j as the triple
// (|v|, global row, sign) — the row index is exact as a double below 2^53
__global__ void argmax_local_triple(const double* __restrict__ V, int64_t ldv, const double* __restrict__ pv,
                                    const int64_t* __restrict__ pi, int64_t nparts, int k, int64_t row0,
                                    double* __restrict__ trip) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double bv = -1.0;
  int64_t bi = INT64_MAX;
  for (int64_t b = 0; b < nparts; ++b) {
    if (better(pv[b * k + j], pi[b * k + j], bv, bi)) { bv = pv[b * k + j]; bi = pi[b * k + j]; }
  }
  trip[3 * j] = bv;
  trip[3 * j + 1] = bi == INT64_MAX ? 9.0e15 : (double)(row0 + bi);
  trip[3 * j + 2] = (bi != INT64_MAX && V[bi * ldv + j] < 0.0) ? -1.0 : 1.0;
}

// stage 2 (after the all-gather): the best triple over the ranks, same rule
__global__ void argmax_ranks(const double* __restrict__ trip, int P, int k, double* __restrict__ sign) {
  const int j = threadIdx.x;
  if (j >= k) return;
  double bv = -1.0, bs = 1.0;
  int64_t bi = INT64_MAX;
  for (int r = 0; r < P; ++r) {
    const double* t = trip + ((size_t)r * k + j) * 3;
    if (better(t[0], (int64_t)t[1], bv, bi)) { bv = t[0]; bi = (int64_t)t[1]; bs = t[2]; }
  }
  sign[j] = bs;
}

template <class T>
__global__ void copy_cast_kernel(const double* __restrict__ s, T* __restrict__ d, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = static_cast<T>(s[i]);
}


template <class T>
__global__ void scale_cast_kernel(const double* __restrict__ src, int64_t rows, int k, const double* __restrict__ sign,
                                  T* __restrict__ dst, int64_t ldd) {
  const int64_t total = rows * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / k;
    const int j = (int)(idx - i * k);
    dst[i * ldd + j] = static_cast<T>(src[idx] * (sign ? sign[j] : 1.0));
  }
}

// Out[i][j] = Σ_{t} (In[i][t] + nu·Q[i][t])·M[t][j]   (M l×l; nu from device; Q may be NULL)
__global__ void right_mult_kernel(const double* __restrict__ In, const double* __restrict__ Q,
                                  const double* __restrict__ nu_p, const double* __restrict__ M, int64_t rows, int l,
                                  double* __restrict__ Out) {
  extern __shared__ double sm[];
  double* Ms = sm;
  double* Is = sm + l * l;
  const double nu = (Q && nu_p) ? *nu_p : 0.0;
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) Ms[idx] = M[idx];
  for (int64_t r0 = (int64_t)blockIdx.x * 64; r0 < rows; r0 += (int64_t)gridDim.x * 64) {
    const int nr = (int)imin64(64, rows - r0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nr * l; idx += blockDim.x)
      Is[idx] = In[r0 * l + idx] + (Q ? nu * Q[r0 * l + idx] : 0.0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nr * l; idx += blockDim.x) {
      const int r = idx / l, j = idx % l;
      double s = 0.0;
      for (int t = 0; t < l; ++t) s += Is[r * l + t] * Ms[t * l + j];
      Out[(r0 + r) * l + j] = s;
    }
  }
}

// y[i] -= Σ_j U[i][j]·t[j]   (U rows×k, ld ldu)
__global__ void rank_k_sub_kernel(double* __restrict__ y, const double* __restrict__ U, int64_t ldu,
                                  const double* __restrict__ t, int64_t rows, int k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += U[i * ldu + j] * t[j];
    y[i] -= s;
  }
}

__global__ void hadamard_kernel(double* __restrict__ t, const double* __restrict__ S, int k) {
  const int j = threadIdx.x;
  if (j < k) t[j] *= S[j];
}

__global__ void finite_check_kernel(const double* __restrict__ x, int64_t count, int* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

unsigned grid_for(Ctx& c, int64_t work, int per = 256) {
  int64_t b = cdiv(work, per);
  const int64_t cap = (int64_t)c.num_sms * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}


}  // namespace

int64_t packx_elems(int64_t n, int l) { return cdiv(n, 32) * 256 * cdiv(l, 8); }
int64_t packy_elems(int64_t m, int l) { return cdiv(m, 32) * 4 * 64 * cdiv(l, 8); }

void pack_x(Ctx& c, const double* X, int64_t n, int l, double* Xp) {
  const int NT = (int)cdiv(l, 8);
  const int64_t total = packx_elems(n, l);
  const unsigned g = grid_for(c, total);
  switch (NT) {
#define RPCA_PACK_X(N) \
  case N: pack_x_kernel<N><<<g, 256, 0, c.stream>>>(X, n, l, total, Xp); break;
    RPCA_PACK_X(1) RPCA_PACK_X(2) RPCA_PACK_X(3) RPCA_PACK_X(4)
    RPCA_PACK_X(5) RPCA_PACK_X(6) RPCA_PACK_X(7) RPCA_PACK_X(8)
#undef RPCA_PACK_X
    default: RPCA_REQUIRE(false, RPCA_E_SHAPE, "pack_x: l=%d > 64", l);
  }
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "pack_x");
}

void pack_y(Ctx& c, const double* Y, int64_t m, int l, double* Yp, const double* ymean) {
  const int NT = (int)cdiv(l, 8);
  const int64_t total = packy_elems(m, l);
  const unsigned g = grid_for(c, total);
  switch (NT) {
#define RPCA_PACK_Y(N) \
  case N: pack_y_kernel<N><<<g, 256, 0, c.stream>>>(Y, m, l, total, ymean, Yp); break;
    RPCA_PACK_Y(1) RPCA_PACK_Y(2) RPCA_PACK_Y(3) RPCA_PACK_Y(4)
    RPCA_PACK_Y(5) RPCA_PACK_Y(6) RPCA_PACK_Y(7) RPCA_PACK_Y(8)
#undef RPCA_PACK_Y
    default: RPCA_REQUIRE(false, RPCA_E_SHAPE, "pack_y: l=%d > 64", l);
  }
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "pack_y");
}

void weighted_colsum(Ctx& c, const double* a, const double* X, int64_t rows, int l, double* v, Arena& ar,
                     int64_t ldx, double scale) {
  if (ldx <= 0) ldx = l;
  const int64_t nparts = std::max<int64_t>(1, cdiv(rows, kColChunk));
  double* part = ar.get<double>(nparts * l);
  wcolsum_partial<<<(unsigned)nparts, 256, 0, c.stream>>>(a, X, rows, l, ldx, part);
  RPCA_CHECK_LAUNCH();
  sum_partials_8w<<<1, 32 * kSumWarps, 0, c.stream>>>(part, nparts, l, scale, v);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 2);
}

// dst rows (ld ldd elements) ← src rows (ld lds): a warp per row, 4-byte
// words, coalesced (the source rows are only 4- or 8-byte aligned)
__global__ void copy_rows_kernel(const uint32_t* __restrict__ src, int64_t lds, uint32_t* __restrict__ dst,
                                 int64_t ldd, int64_t rows, int64_t wpr) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    const uint32_t* s = src + r * lds;
    uint32_t* d = dst + r * ldd;
    int64_t t = lane;
    for (; t + 96 < wpr; t += 128) {  // four loads in flight
      const uint32_t a = s[t], b = s[t + 32], c = s[t + 64], e = s[t + 96];
      d[t] = a;
      d[t + 32] = b;
      d[t + 64] = c;
      d[t + 96] = e;
    }
    for (; t < wpr; t += 32) d[t] = s[t];
  }
}

void copy_rows(Ctx& c, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols, int es) {
  if (rows == 0) return;
  const int64_t w = es / 4;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(rows, 8), (int64_t)c.num_sms * 16);
  copy_rows_kernel<<<grid, 256, 0, c.stream>>>(static_cast<const uint32_t*>(src), lds * w, static_cast<uint32_t*>(dst),
                                               ldd * w, rows, cols * w);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "pad_copy");
}

__global__ void add_into_kernel(double* __restrict__ Z, const double* __restrict__ W, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    Z[i] += W[i];
}

void add_into(Ctx& c, double* Z, const double* W, int64_t count) {
  if (count == 0) return;
  add_into_kernel<<<grid_for(c, count), 256, 0, c.stream>>>(Z, W, count);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "stream_accumulate");
}

void sub_rank1(Ctx& c, double* Y, int64_t rows, int l, const double* u, const double* v, double alpha) {
  sub_rank1_kernel<<<grid_for(c, rows * l), 256, 0, c.stream>>>(Y, rows, l, u, v, alpha);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void colmeans_dense(Ctx& c, const void* A, int dtype, int64_t m, int64_t n, int64_t lda, int64_t m_total,
                    double* cmean, Arena& ar) {
  const int64_t nparts = std::max<int64_t>(1, cdiv(m, kChunk));
  double* part = ar.get<double>(nparts * n);
  dim3 grid((unsigned)cdiv(n, 256), (unsigned)nparts);
  if (dtype == RPCA_F64)
    colsum_dense_partial<double><<<grid, 256, 0, c.stream>>>((const double*)A, m, n, lda, part);
  else
    colsum_dense_partial<float><<<grid, 256, 0, c.stream>>>((const float*)A, m, n, lda, part);
  RPCA_CHECK_LAUNCH();
  colsum_dense_final<<<(unsigned)cdiv(n, 256), 256, 0, c.stream>>>(part, nparts, n, 1.0 / (double)m_total, cmean);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 2, "colmeans");
}

size_t thin_gemm_ws_bytes(int64_t rows, int l, int k) {
  Sizer s;
  s.add<double>((size_t)l * k);
  s.add<double>((size_t)rows * k);
  s.add<char>(ax_ws_bytes(DenseA{nullptr, RPCA_F64, rows, l, l}, k));
  return s.total + 4096;
}

// Out = In·W[:, :k]·diag(sign) on the fp64 tensor-core pass kernel (dense_ax
// with the thin block as "A"): W' = W[:, :k]·diag(sign) is formed first; an fp64
// output with ldo = k is written directly, otherwise through an fp64 temporary
// and a casting copy
void thin_gemm(Ctx& c, const double* In, int64_t rows, int l, const double* W, int k, const double* sign, void* Out,
               int64_t ldo, int out_dtype, Arena& ar) {
  if (rows == 0) return;
  const size_t mark = ar.off;
  double* Wk = ar.get<double>((size_t)l * k);
  scale_cols_kernel<<<1, 256, 0, c.stream>>>(W, l, k, sign, Wk);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
  TagScope ts(c, "thin_gemm");
  const DenseA A{In, RPCA_F64, rows, l, l};
  if (out_dtype == RPCA_F64 && ldo == k) {
    dense_ax(c, A, Wk, k, (double*)Out, ar);
  } else {
    double* tmp = ar.get<double>((size_t)rows * k);
    dense_ax(c, A, Wk, k, tmp, ar);
    scale_cast(c, tmp, rows, k, nullptr, Out, ldo, out_dtype);
  }
  ar.off = mark;
}

void column_signs(Ctx& c, const double* V, int64_t rows, int k, int64_t ldv, double* sign, Arena& ar) {
  const int64_t nparts = std::max<int64_t>(1, cdiv(rows, kChunk));
  double* pv = ar.get<double>(nparts * k);
  int64_t* pi = ar.get<int64_t>(nparts * k);
  argmax_partial<<<dim3((unsigned)nparts, (unsigned)k), 256, 0, c.stream>>>(V, rows, k, ldv, pv, pi);
  RPCA_CHECK_LAUNCH();
  argmax_final<<<1, 64, 0, c.stream>>>(V, ldv, pv, pi, nparts, k, sign);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 2);
}

void column_signs_sharded(Ctx& c, const double* V, int64_t rows, int64_t row0, int k, int64_t ldv, double* sign,
                          Arena& ar) {
  const int P = comm_size(c);
  const int64_t nparts = std::max<int64_t>(1, cdiv(rows, kChunk));
  double* pv = ar.get<double>(nparts * k);
  int64_t* pi = ar.get<int64_t>(nparts * k);
  double* trip = ar.get<double>(3 * (size_t)k);
  double* all = ar.get<double>(3 * (size_t)k * P);
  argmax_partial<<<dim3((unsigned)nparts, (unsigned)k), 256, 0, c.stream>>>(V, rows, k, ldv, pv, pi);
  RPCA_CHECK_LAUNCH();
  argmax_local_triple<<<1, 64, 0, c.stream>>>(V, ldv, pv, pi, nparts, k, row0, trip);
  RPCA_CHECK_LAUNCH();
  allgather_bytes(c, trip, all, 3 * sizeof(double) * k);
  argmax_ranks<<<1, 64, 0, c.stream>>>(all, P, k, sign);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 3);
}


void scale_cast(Ctx& c, const double* src, int64_t rows, int k, const double* sign, void* dst, int64_t ldd,
                int dtype) {
  if (dtype == RPCA_F64)
    scale_cast_kernel<double><<<grid_for(c, rows * k), 256, 0, c.stream>>>(src, rows, k, sign, (double*)dst, ldd);
  else
    scale_cast_kernel<float><<<grid_for(c, rows * k), 256, 0, c.stream>>>(src, rows, k, sign, (float*)dst, ldd);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void right_mult(Ctx& c, const double* In, const double* Q, const double* nu, const double* M, int64_t rows, int l,
                double* Out) {
  const size_t smem = (size_t)(l * l + 64 * l) * 8;
  ensure_smem((const void*)right_mult_kernel, (int)((kMaxL * kMaxL + 64 * kMaxL) * 8));
  right_mult_kernel<<<grid_for(c, rows, 64), 256, smem, c.stream>>>(In, Q, nu, M, rows, l, Out);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void rank_k_sub(Ctx& c, double* y, const double* U, int64_t ldu, const double* t, int64_t rows, int k) {
  if (k == 0) return;
  rank_k_sub_kernel<<<grid_for(c, rows), 256, 0, c.stream>>>(y, U, ldu, t, rows, k);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void finite_check(Ctx& c, const double* x, int64_t count, int* flag) {
  if (count == 0) return;
  finite_check_kernel<<<grid_for(c, count, 1024), 256, 0, c.stream>>>(x, count, flag);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "finite_check");
}

void hadamard(Ctx& c, double* t, const double* S, int k) {
  if (k == 0) return;
  hadamard_kernel<<<1, 256, 0, c.stream>>>(t, S, k);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

void copy_cast(Ctx& c, const double* src, void* dst, int64_t count, int dtype) {
  if (dtype == RPCA_F64)
    copy_cast_kernel<double><<<grid_for(c, count), 256, 0, c.stream>>>(src, (double*)dst, count);
  else
    copy_cast_kernel<float><<<grid_for(c, count), 256, 0, c.stream>>>(src, (float*)dst, count);
  RPCA_CHECK_LAUNCH();
  count_launch(c);
}

}  // namespace rpca
