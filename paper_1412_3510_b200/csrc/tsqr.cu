// tsqr.cu — §8(a) steps a5/a7: Householder QR of a tall-skinny block.
//
// PAPER.md:169-172 ("applying the Gram-Schmidt process (or other methods for
// constructing QR decompositions) ... yields an orthonormal basis"),
// PAPER.md:406-425 (§5: the last renormalisation is a QR, "[Q,R,E] =
// qr(Q,0)"; pivoting "is not necessary", reading Q4).  Householder keeps Q
// orthonormal to working precision even for rank-deficient blocks (the
// PROPACK matrices of §6), which CholeskyQR cannot.
//
// B200 design — TSQR tree with an implicit Q:
//   factor: leaves of 256 (l ≤ 32) / 128 rows, one CTA each, Householder in
//   shared memory (reflectors v, β = 2/vᵀv stored per block, R written out);
//   groups of G stacked R's are factored the same way until one R is left.
//   expand: from the root down, each group applies its reflectors (in reverse)
//   to [C; 0], C = its slice of the parent's Q; the root starts from I and
//   fixes signs so that diag(R) ≥ 0 (as the oracle).  Leaves write Q in place.
// Traffic: Y read once, V written and read once, Q written once (4·m·l·8 B).
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kThreads / 32; ++w) s += red[w];
  return s;
}

// Householder QR of W (rows × l, shared, row-major).  V (rows × l, shared)
// receives the reflectors (zero above the diagonal), beta[j] = 2/vᵀv (0 ⇒ H = I).
// After return the upper triangle of W's first min(rows,l) rows is R.
__device__ void householder(double* W, double* V, double* beta, double* wvec, int rows, int l, double* red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int steps = min(rows, l);
  for (int idx = tid; idx < rows * l; idx += kThreads) V[idx] = 0.0;
  __syncthreads();
  for (int j = 0; j < steps; ++j) {
    double part = 0.0;
    for (int r = j + tid; r < rows; r += kThreads) part += W[r * l + j] * W[r * l + j];
    const double nx2 = block_sum(part, red);
    const double nx = sqrt(nx2);
    const double x0 = W[j * l + j];
    const double sg = x0 >= 0.0 ? 1.0 : -1.0;
    const double b = nx > 0.0 ? 1.0 / (nx * (nx + fabs(x0))) : 0.0;  // 2/vᵀv, vᵀv = 2·nx·(nx+|x0|)
    if (tid == 0) beta[j] = b;
    for (int r = j + tid; r < rows; r += kThreads) V[r * l + j] = (r == j) ? x0 + sg * nx : W[r * l + j];
    __syncthreads();
    if (b != 0.0) {
      // w_t = vᵀ W[:, t] for t ≥ j (warp per column)
      for (int t = j + warp; t < l; t += kThreads / 32) {
        double s = 0.0;
        for (int r = j + lane; r < rows; r += 32) s += V[r * l + j] * W[r * l + t];
        s = warp_sum(s);
        if (lane == 0) wvec[t] = s;
      }
      __syncthreads();
      const int nt = l - j;
      for (int idx = tid; idx < (rows - j) * nt; idx += kThreads) {
        const int r = j + idx / nt, t = j + idx % nt;
        W[r * l + t] -= b * V[r * l + j] * wvec[t];
      }
    }
    __syncthreads();
  }
}

// Apply H_0 ⋯ H_{steps-1} (reflectors in V) to C (rows × l, shared): C ← Q·C.
__device__ void apply_q(const double* V, const double* beta, double* C, double* wvec, int rows, int l) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int steps = min(rows, l);
  for (int j = steps - 1; j >= 0; --j) {
    const double b = beta[j];
    if (b == 0.0) continue;  // uniform across the CTA
    for (int t = warp; t < l; t += kThreads / 32) {
      double s = 0.0;
      for (int r = j + lane; r < rows; r += 32) s += V[r * l + j] * C[r * l + t];
      s = warp_sum(s);
      if (lane == 0) wvec[t] = s;
    }
    __syncthreads();
    for (int idx = tid; idx < (rows - j) * l; idx += kThreads) {
      const int r = j + idx / l, t = idx % l;
      C[r * l + t] -= b * V[r * l + j] * wvec[t];
    }
    __syncthreads();
  }
}

// factor: leaf (rows of Y) or tree (stack of up to G R's of the level below).
// Outputs per group g: Vout[g] (cap × l), bout[g] (l), Rout[g] (l×l).
__global__ void __launch_bounds__(kThreads) qr_factor_kernel(const double* __restrict__ src, int64_t src_rows, int l,
                                                             int leaf, int cap, int64_t n_in,
                                                             double* __restrict__ Vout, double* __restrict__ bout,
                                                             double* __restrict__ Rout) {
  extern __shared__ double sm[];
  __shared__ double red[kThreads / 32];
  __shared__ double wvec[kMaxL];
  __shared__ double beta[kMaxL];
  double* W = sm;
  double* V = sm + (size_t)cap * l;
  const int64_t g = blockIdx.x;
  int rows;
  if (leaf) {
    const int64_t r0 = g * cap;
    rows = (int)imin64(cap, src_rows - r0);
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) W[idx] = src[r0 * l + idx];
  } else {
    const int G = cap / l;
    const int64_t i0 = g * G;
    const int nr = (int)imin64(G, n_in - i0);
    rows = nr * l;
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) W[idx] = src[i0 * l * l + idx];
  }
  __syncthreads();
  householder(W, V, beta, wvec, rows, l, red);
  for (int idx = threadIdx.x; idx < cap * l; idx += kThreads) Vout[g * cap * l + idx] = idx < rows * l ? V[idx] : 0.0;
  for (int j = threadIdx.x; j < l; j += kThreads) bout[g * l + j] = j < min(rows, l) ? beta[j] : 0.0;
  for (int idx = threadIdx.x; idx < l * l; idx += kThreads) {
    const int j = idx / l, t = idx % l;
    Rout[g * l * l + idx] = (j < rows && t >= j) ? W[idx] : 0.0;
  }
}

// expand: C = parent slice (or I at the root), apply this group's reflectors,
// write Q (leaf: rows of Y; inner: Qout[g] cap × l).  At the root, signs are
// fixed so diag(R) ≥ 0 and R is written to Rfinal (may be NULL).
__global__ void __launch_bounds__(kThreads) qr_expand_kernel(const double* __restrict__ V, const double* __restrict__ bv,
                                                             int l, int cap, int leaf, int64_t total_rows,
                                                             int64_t n_groups, const double* __restrict__ Cparent,
                                                             int root, const double* __restrict__ Rroot,
                                                             double* __restrict__ Rfinal, double* __restrict__ Qout) {
  extern __shared__ double sm[];
  __shared__ double wvec[kMaxL];
  __shared__ double beta[kMaxL];
  __shared__ double dsign[kMaxL];
  double* C = sm;
  double* Vs = sm + (size_t)cap * l;
  const int64_t g = blockIdx.x;
  int rows;
  if (leaf) rows = (int)imin64(cap, total_rows - g * cap);
  else rows = (int)imin64(cap / l, n_groups - g * (cap / l)) * l;
  (void)n_groups;
  for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) {
    const int r = idx / l, t = idx % l;
    double cv;
    if (root) cv = (r == t) ? 1.0 : 0.0;
    else cv = r < l ? Cparent[g * l * l + idx] : 0.0;  // parent's slice for group g is rows [g·l, g·l+l)
    C[idx] = cv;
    Vs[idx] = V[g * (int64_t)cap * l + idx];
  }
  for (int j = threadIdx.x; j < l; j += kThreads) beta[j] = bv[g * l + j];
  __syncthreads();
  apply_q(Vs, beta, C, wvec, rows, l);
  if (root) {
    for (int j = threadIdx.x; j < l; j += kThreads) dsign[j] = Rroot[j * l + j] < 0.0 ? -1.0 : 1.0;
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) C[idx] *= dsign[idx % l];
    if (Rfinal)
      for (int idx = threadIdx.x; idx < l * l; idx += kThreads) Rfinal[idx] = Rroot[idx] * dsign[idx / l];
    __syncthreads();
  }
  if (leaf) {
    const int64_t r0 = g * cap;
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) Qout[r0 * l + idx] = C[idx];
  } else {
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) Qout[g * (int64_t)cap * l + idx] = C[idx];
  }
}

int leaf_rows_for(int l) { return l <= 32 ? 256 : 128; }
int group_for(int l) { return std::max(2, std::min(16, 10240 / (l * l))); }

struct Level {
  int64_t ngroups;
  int cap;  // rows per group
  double *V, *b, *R, *Q;
};

std::vector<Level> plan(int64_t m, int l) {
  std::vector<Level> lv;
  const int lr = leaf_rows_for(l), G = group_for(l);
  int64_t n = cdiv(m, lr);
  lv.push_back({n, lr, nullptr, nullptr, nullptr, nullptr});
  while (n > 1) {
    n = cdiv(n, G);
    lv.push_back({n, G * l, nullptr, nullptr, nullptr, nullptr});
  }
  return lv;
}

}  // namespace

size_t qr_ws_bytes(int64_t m, int l) {
  Sizer s;
  auto lv = plan(m, l);
  for (size_t i = 0; i < lv.size(); ++i) {
    s.add<double>(lv[i].ngroups * lv[i].cap * (int64_t)l);
    s.add<double>(lv[i].ngroups * (int64_t)l);
    s.add<double>(lv[i].ngroups * (int64_t)l * l);
    if (i > 0) s.add<double>(lv[i].ngroups * lv[i].cap * (int64_t)l);
  }
  return s.total;
}

void qr(Ctx& c, double* Y, int64_t m, int l, double* R_out, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "qr: need 1 ≤ l ≤ %d and m ≥ l", kMaxL);
  auto lv = plan(m, l);
  for (size_t i = 0; i < lv.size(); ++i) {
    lv[i].V = ar.get<double>(lv[i].ngroups * lv[i].cap * (int64_t)l);
    lv[i].b = ar.get<double>(lv[i].ngroups * (int64_t)l);
    lv[i].R = ar.get<double>(lv[i].ngroups * (int64_t)l * l);
    lv[i].Q = i > 0 ? ar.get<double>(lv[i].ngroups * lv[i].cap * (int64_t)l) : nullptr;
  }
  int maxcap = 0;
  for (auto& x : lv) maxcap = std::max(maxcap, x.cap);
  const size_t smem_max = (size_t)2 * maxcap * l * 8;
  ensure_smem((const void*)qr_factor_kernel, (int)smem_max);
  ensure_smem((const void*)qr_expand_kernel, (int)smem_max);
  // factor, bottom-up
  for (size_t i = 0; i < lv.size(); ++i) {
    const size_t smem = (size_t)2 * lv[i].cap * l * 8;
    const double* src = i == 0 ? Y : lv[i - 1].R;
    const int64_t n_in = i == 0 ? m : lv[i - 1].ngroups;
    qr_factor_kernel<<<(unsigned)lv[i].ngroups, kThreads, smem, c.stream>>>(src, m, l, i == 0, lv[i].cap, n_in,
                                                                           lv[i].V, lv[i].b, lv[i].R);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, i == 0 ? "qr_leaf" : "qr_tree");
  }
  // expand, top-down
  const double* Rroot = lv.back().R;
  for (int i = (int)lv.size() - 1; i >= 0; --i) {
    const size_t smem = (size_t)2 * lv[i].cap * l * 8;
    const bool root = i == (int)lv.size() - 1;
    const double* Cp = root ? nullptr : lv[i + 1].Q;
    double* out = i == 0 ? Y : lv[i].Q;
    const int64_t n_groups_below = i == 0 ? 0 : lv[i - 1].ngroups;
    qr_expand_kernel<<<(unsigned)lv[i].ngroups, kThreads, smem, c.stream>>>(
        lv[i].V, lv[i].b, l, lv[i].cap, i == 0, m, n_groups_below, Cp, root, Rroot, root ? R_out : nullptr, out);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, i == 0 ? "qr_expand_leaf" : "qr_expand_tree");
  }
}

}  // namespace rpca
