// tslu.cu — §8(a) step a3: LU renormalisation of a tall-skinny block.
//
// PAPER.md:382-404 (§5): "computing the LU decomposition is typically more
// efficient than computing the QR decomposition, and both are sufficient for
// most stages" — "[Q,R] = lu(Q)", i.e. Q ← the row-permuted unit lower factor
// L with Y = L·U (MATLAB's two-output lu; reading Q3).
//
// B200 design — tournament pivoting (CALU):
//   1. leaf kernel: one CTA per block of 256 (l ≤ 32) or 128 rows runs GEPP in
//      shared memory and nominates l candidate pivot rows (original rows);
//   2. tree kernel: groups of G candidate sets are stacked (original values
//      gathered from Y) and reduced by GEPP again, until one set is left; the
//      last GEPP gives the pivot order, U (l×l) and the multipliers of the pivot
//      rows (Lp), and the substitution matrix M with x = y·M ⇔ x·U = y
//      (x_j = 0 where U_jj = 0 — the exact-zero-pivot rule of reading Q3);
//   3. apply kernel: L = Y·M for every row (HBM-bound), pivot rows overwritten
//      with their exact unit-lower rows from Lp.
// Pivot choice: largest |·| among active rows, lowest original row on ties.
// Tournament pivots differ from plain GEPP, so L differs from the oracle's L
// but span(L) = span(Y) whenever U is nonsingular (compare spans, Q3).
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

struct Best {
  double v;
  int64_t id;
  int r;
};

__device__ __forceinline__ bool better(double v, int64_t id, double bv, int64_t bid) {
  return v > bv || (v == bv && id < bid);
}

// GEPP on W (rows × ldw, shared), ids = original row numbers.  After return,
// piv[j] = local row of pivot j (j < steps), active[] = 0 for pivot rows, and
// W holds multipliers left of each row's pivot column (for pivot rows) / of
// every column (others) and the eliminated values right of it.
__device__ void gepp(double* W, int ldw, const int64_t* ids, int rows, int l, int steps, int* piv, uint8_t* active,
                     double* rv, int64_t* ri, int* rr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < steps; ++j) {
    double bv = -1.0;
    int64_t bid = INT64_MAX;
    int br = -1;
    for (int r = tid; r < rows; r += kThreads) {
      if (!active[r]) continue;
      const double v = fabs(W[r * ldw + j]);
      if (better(v, ids[r], bv, bid)) { bv = v; bid = ids[r]; br = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oid = __shfl_xor_sync(0xffffffffu, bid, o);
      const int orr = __shfl_xor_sync(0xffffffffu, br, o);
      if (better(ov, oid, bv, bid)) { bv = ov; bid = oid; br = orr; }
    }
    if (lane == 0) { rv[warp] = bv; ri[warp] = bid; rr[warp] = br; }
    __syncthreads();
    if (tid == 0) {
      double b = rv[0];
      int64_t bi = ri[0];
      int r = rr[0];
      for (int w = 1; w < kThreads / 32; ++w)
        if (better(rv[w], ri[w], b, bi)) { b = rv[w]; bi = ri[w]; r = rr[w]; }
      piv[j] = r;
      active[r] = 0;
    }
    __syncthreads();
    const int pr = piv[j];
    const double u = W[pr * ldw + j];
    for (int r = tid; r < rows; r += kThreads)
      if (active[r]) W[r * ldw + j] = (u != 0.0) ? W[r * ldw + j] / u : 0.0;
    __syncthreads();
    const int nt = l - j - 1;
    if (nt > 0 && u != 0.0) {
      for (int idx = tid; idx < rows * nt; idx += kThreads) {
        const int r = idx / nt, t = j + 1 + idx % nt;
        if (active[r]) W[r * ldw + t] -= W[r * ldw + j] * W[pr * ldw + t];
      }
    }
    __syncthreads();
  }
}

// One CTA: rows from Y (leaf: contiguous block; tree: a group of candidate
// sets), GEPP, l nominated original rows → cand_out[blockIdx.x*l ...] (-1 pad).
// If final, also U, Lp, piv and the substitution matrix M.
__global__ void __launch_bounds__(kThreads) lu_select_kernel(const double* __restrict__ Y, int64_t m, int l,
                                                             int leaf, int64_t leaf_rows,
                                                             const int64_t* __restrict__ cand_in, int64_t n_in,
                                                             int G, int64_t* __restrict__ cand_out, int final_,
                                                             double* __restrict__ U, double* __restrict__ Lp,
                                                             double* __restrict__ M, int64_t* __restrict__ piv_out) {
  extern __shared__ double sm[];
  __shared__ double rv[kThreads / 32];
  __shared__ int64_t ri[kThreads / 32];
  __shared__ int rr[kThreads / 32];
  __shared__ int piv[kMaxL];
  __shared__ int nrows_s;
  const int cap = leaf ? (int)leaf_rows : G * l;
  const int ldw = l;
  double* W = sm;
  int64_t* ids = reinterpret_cast<int64_t*>(W + (size_t)cap * ldw);
  uint8_t* active = reinterpret_cast<uint8_t*>(ids + cap);
  const int tid = threadIdx.x;

  if (leaf) {
    const int64_t r0 = (int64_t)blockIdx.x * leaf_rows;
    const int rows = (int)imin64(leaf_rows, m - r0);
    if (tid == 0) nrows_s = rows;
    for (int r = tid; r < rows; r += kThreads) { ids[r] = r0 + r; active[r] = 1; }
    for (int idx = tid; idx < rows * l; idx += kThreads) W[idx] = Y[r0 * l + idx];
  } else {
    // compact the valid candidates of this group (ascending slot order)
    if (tid == 0) {
      int cnt = 0;
      const int64_t s0 = (int64_t)blockIdx.x * G * l, s1 = imin64(n_in * l, s0 + (int64_t)G * l);
      for (int64_t s = s0; s < s1; ++s)
        if (cand_in[s] >= 0) { ids[cnt] = cand_in[s]; active[cnt] = 1; ++cnt; }
      nrows_s = cnt;
    }
    __syncthreads();
    const int rows = nrows_s;
    for (int idx = tid; idx < rows * l; idx += kThreads) {
      const int r = idx / l, t = idx % l;
      W[idx] = Y[ids[r] * l + t];
    }
  }
  __syncthreads();
  const int rows = nrows_s;
  const int steps = min(rows, l);
  gepp(W, ldw, ids, rows, l, steps, piv, active, rv, ri, rr);
  for (int j = tid; j < l; j += kThreads)
    cand_out[(int64_t)blockIdx.x * l + j] = j < steps ? ids[piv[j]] : -1;
  if (!final_) return;
  // final set: U (upper), Lp (unit lower of the pivot rows), piv, M
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int j = idx / l, t = idx % l;
    const double w = W[piv[j] * ldw + t];
    U[idx] = t >= j ? w : 0.0;
    Lp[idx] = t < j ? w : (t == j ? 1.0 : 0.0);
  }
  for (int j = tid; j < l; j += kThreads) piv_out[j] = ids[piv[j]];
  __syncthreads();
  // M row t = solution x of x·U = e_t with the zero-pivot rule
  if (tid < l) {
    const int t = tid;
    for (int j = 0; j < l; ++j) {
      double s = (j == t) ? 1.0 : 0.0;
      for (int q = 0; q < j; ++q) s -= M[t * l + q] * U[q * l + j];
      const double ujj = U[j * l + j];
      M[t * l + j] = (ujj != 0.0) ? s / ujj : 0.0;
    }
  }
}

// L = Y·M (in place), pivot rows ← Lp rows.  One CTA per 128 rows.
__global__ void __launch_bounds__(kThreads) lu_apply_kernel(double* __restrict__ Y, int64_t m, int l,
                                                            const double* __restrict__ M,
                                                            const double* __restrict__ Lp,
                                                            const int64_t* __restrict__ piv) {
  extern __shared__ double sm[];
  double* Ms = sm;               // l×l
  double* Ys = sm + l * l;       // 128×l
  __shared__ int64_t ps[kMaxL];
  for (int idx = threadIdx.x; idx < l * l; idx += kThreads) Ms[idx] = M[idx];
  for (int j = threadIdx.x; j < l; j += kThreads) ps[j] = piv[j];
  for (int64_t r0 = (int64_t)blockIdx.x * 128; r0 < m; r0 += (int64_t)gridDim.x * 128) {
    const int rows = (int)imin64(128, m - r0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) Ys[idx] = Y[r0 * l + idx];
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) {
      const int r = idx / l, j = idx % l;
      const int64_t gi = r0 + r;
      int pj = -1;
      for (int q = 0; q < l; ++q)
        if (ps[q] == gi) pj = q;
      double s;
      if (pj >= 0) {
        s = Lp[pj * l + j];
      } else {
        s = 0.0;
        for (int t = 0; t <= j; ++t) s += Ys[r * l + t] * Ms[t * l + j];
      }
      Y[gi * l + j] = s;
    }
  }
}

int leaf_rows_for(int l) { return l <= 32 ? 256 : 128; }
int group_for(int l) { return std::max(2, std::min(32, 20480 / (l * l))); }

size_t select_smem(int cap, int l) { return (size_t)cap * l * 8 + (size_t)cap * 8 + (size_t)cap + 16; }

}  // namespace

size_t lu_ws_bytes(int64_t m, int l) {
  Sizer s;
  const int64_t nblk = cdiv(m, leaf_rows_for(l));
  s.add<int64_t>(nblk * l);
  s.add<int64_t>(nblk * l);
  s.add<double>(3 * (size_t)l * l);
  s.add<int64_t>(l);
  return s.total;
}

void lu_renorm(Ctx& c, double* Y, int64_t m, int l, double* U_out, int64_t* piv_out, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "lu_renorm: need 1 ≤ l ≤ %d and m ≥ l", kMaxL);
  const int lr = leaf_rows_for(l);
  const int G = group_for(l);
  const int64_t nblk = cdiv(m, lr);
  int64_t* ca = ar.get<int64_t>(nblk * l);
  int64_t* cb = ar.get<int64_t>(nblk * l);
  double* U = ar.get<double>((size_t)l * l);
  double* Lp = ar.get<double>((size_t)l * l);
  double* M = ar.get<double>((size_t)l * l);
  int64_t* piv = ar.get<int64_t>(l);
  const size_t smem_leaf = select_smem(lr, l), smem_tree = select_smem(G * l, l);
  RPCA_CUDA(cudaFuncSetAttribute(lu_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)std::max(smem_leaf, smem_tree)));
  lu_select_kernel<<<(unsigned)nblk, kThreads, smem_leaf, c.stream>>>(Y, m, l, 1, lr, nullptr, 0, G, ca,
                                                                      nblk == 1, U, Lp, M, piv);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_leaf");
  int64_t n = nblk;
  while (n > 1) {
    const int64_t ng = cdiv(n, G);
    lu_select_kernel<<<(unsigned)ng, kThreads, smem_tree, c.stream>>>(Y, m, l, 0, lr, ca, n, G, cb, ng == 1, U, Lp,
                                                                      M, piv);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "lu_tree");
    std::swap(ca, cb);
    n = ng;
  }
  const size_t smem_apply = (size_t)(l * l + 128 * l) * 8;
  RPCA_CUDA(cudaFuncSetAttribute(lu_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_apply));
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(m, 128), (int64_t)c.num_sms * 4);
  lu_apply_kernel<<<grid, kThreads, smem_apply, c.stream>>>(Y, m, l, M, Lp, piv);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_apply");
  if (U_out) RPCA_CUDA(cudaMemcpyAsync(U_out, U, sizeof(double) * l * l, cudaMemcpyDeviceToDevice, c.stream));
  if (piv_out) RPCA_CUDA(cudaMemcpyAsync(piv_out, piv, sizeof(int64_t) * l, cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace rpca
