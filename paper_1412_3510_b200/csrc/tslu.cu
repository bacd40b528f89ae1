// tslu.cu — §8(a) step a3: LU renormalisation of a tall-skinny block.
//
// PAPER.md:382-404 (§5): "computing the LU decomposition is typically more
// efficient than computing the QR decomposition, and both are sufficient for
// most stages" — "[Q,R] = lu(Q)", i.e. Q ← the row-permuted unit lower factor
// L with Y = L·U (MATLAB's two-output lu; reading Q3).
//
// B200 design — tournament pivoting (CALU):
//   1. leaf kernel: one CTA per block of 256 rows runs GEPP and nominates l
//      candidate pivot rows (original rows);
//   2. tree kernel: groups of G candidate sets are stacked (original values
//      gathered from Y) and reduced by GEPP again, until one set is left; the
//      last GEPP gives the pivot order, U (l×l) and the multipliers of the pivot
//      rows (Lp);
//   3. apply kernel: every CTA first forms the substitution matrix M with
//      x = y·M ⇔ x·U = y (x_j = 0 where U_jj = 0 — the exact-zero-pivot rule of
//      reading Q3), then L = Y·M for its rows (HBM-bound); pivot rows are
//      overwritten with their exact unit-lower rows from Lp.  Optionally the
//      CTA also accumulates LᵀL for the Cholesky-QR that follows (cholqr.cu).
// GEPP inside a CTA: thread t owns rows t, t+256, … held in REGISTERS (the
// kernel is templated on l rounded up to 8); the pivot row is read from a
// shared-memory mirror that every thread refreshes after its update; the
// argmax of column j+1 is reduced while column j is eliminated, so each column
// costs one __syncthreads.  Pivot: largest |·| among active rows, lowest
// original row on ties.  Tournament pivots differ from plain GEPP, so L differs
// from the oracle's L but span(L) = span(Y) whenever U is nonsingular.
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

struct Cand {
  double v;
  int r;  // local row (ties are broken by ids[r])
};

__device__ __forceinline__ bool better(double v, int r, double bv, int br, const int64_t* ids) {
  if (v != bv) return v > bv;
  if (br < 0) return r >= 0;
  if (r < 0) return false;
  return ids[r] < ids[br];
}

__device__ __forceinline__ Cand warp_best(Cand c, const int64_t* ids) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, c.v, o);
    const int orr = __shfl_xor_sync(0xffffffffu, c.r, o);
    if (better(ov, orr, c.v, c.r, ids)) { c.v = ov; c.r = orr; }
  }
  return c;
}

// GEPP on W (rows × ldw, shared; ldw odd ⇒ conflict-free row-per-thread
// access).  Thread t owns rows t, t+256, … (active flags in registers).  One
// __syncthreads per column: the argmax of column j+1 is reduced while column j
// is eliminated and every thread redundantly combines the eight warp winners.
// piv[j] = local pivot row of column j; W ends with the multipliers left of
// each row's pivot column and its eliminated values right of it.
__device__ void gepp(double* W, int ldw, const int64_t* ids, int rows, int l, int steps, int* piv,
                     Cand (*slot)[kWarps]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kMaxR = 3;
  bool act[kMaxR];
  Cand c{-1.0, -1};
#pragma unroll
  for (int q = 0; q < kMaxR; ++q) {
    const int r = tid + q * kThreads;
    act[q] = r < rows;
    if (act[q]) {
      const double v = fabs(W[r * ldw]);
      if (better(v, r, c.v, c.r, ids)) c = Cand{v, r};
    }
  }
  c = warp_best(c, ids);
  if (lane == 0) slot[0][warp] = c;
  __syncthreads();
  for (int j = 0; j < steps; ++j) {
    Cand b = slot[j & 1][0];
#pragma unroll
    for (int wi = 1; wi < kWarps; ++wi) {
      const Cand o = slot[j & 1][wi];
      if (better(o.v, o.r, b.v, b.r, ids)) b = o;
    }
    const int p = b.r;
    if (tid == 0) piv[j] = p;
    const double* prow = W + p * ldw;
    const double u = prow[j];
    const double uinv = (u != 0.0) ? __drcp_rn(u) : 0.0;
    Cand nc{-1.0, -1};
#pragma unroll
    for (int q = 0; q < kMaxR; ++q) {
      const int r = tid + q * kThreads;
      if (!act[q]) continue;
      if (r == p) { act[q] = false; continue; }
      double* wr = W + r * ldw;
      const double mult = wr[j] * uinv;
      wr[j] = mult;
      if (mult != 0.0) {
        // chunks of 8: all loads issued before the stores (a row never aliases the pivot row)
        int t = j + 1;
        for (; t + 8 <= l; t += 8) {
          double pv[8], wv[8];
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8) { pv[u8] = prow[t + u8]; wv[u8] = wr[t + u8]; }
#pragma unroll
          for (int u8 = 0; u8 < 8; ++u8) wr[t + u8] = wv[u8] - mult * pv[u8];
        }
        for (; t < l; ++t) wr[t] -= mult * prow[t];
      }
      if (j + 1 < steps) {
        const double v = fabs(wr[j + 1]);
        if (better(v, r, nc.v, nc.r, ids)) nc = Cand{v, r};
      }
    }
    nc = warp_best(nc, ids);
    if (lane == 0) slot[(j + 1) & 1][warp] = nc;
    __syncthreads();
  }
}

// One CTA: rows from Y (leaf: contiguous block; tree: a group of candidate
// sets), GEPP, l nominated original rows → cand_out[blockIdx.x*l ...] (-1 pad).
// If final, also U, Lp and the original pivot rows piv_out.
__global__ void __launch_bounds__(kThreads) lu_select_kernel(const double* __restrict__ Y, int64_t m, int l, int leaf,
                                                             int64_t leaf_rows, const int64_t* __restrict__ cand_in,
                                                             int64_t n_in, int G, int64_t* __restrict__ cand_out,
                                                             int final_, double* __restrict__ U,
                                                             double* __restrict__ Lp, int64_t* __restrict__ piv_out,
                                                             double* __restrict__ M) {
  extern __shared__ double sm[];
  __shared__ Cand slot[2][kWarps];
  __shared__ int piv[kMaxL];
  __shared__ int nrows_s;
  const int cap = leaf ? (int)leaf_rows : G * l;
  const int ldw = l | 1;
  double* W = sm;
  int64_t* ids = reinterpret_cast<int64_t*>(W + (size_t)cap * ldw);
  const int tid = threadIdx.x;

  if (leaf) {
    const int64_t r0 = (int64_t)blockIdx.x * leaf_rows;
    if (tid == 0) nrows_s = (int)imin64(leaf_rows, m - r0);
    for (int r = tid; r < cap; r += kThreads) ids[r] = r0 + r;
  } else {
    // compact the valid candidates of this group (ascending slot order)
    if (tid < 32) {
      const int64_t s0 = (int64_t)blockIdx.x * G * l, s1 = imin64(n_in * l, s0 + (int64_t)G * l);
      int base = 0;
      for (int64_t s = s0; s < s1; s += 32) {
        const int64_t id = (s + tid < s1) ? cand_in[s + tid] : -1;
        const unsigned mask = __ballot_sync(0xffffffffu, id >= 0);
        if (id >= 0) ids[base + __popc(mask & ((1u << tid) - 1u))] = id;
        base += __popc(mask);
      }
      if (tid == 0) nrows_s = base;
    }
  }
  __syncthreads();
  const int rows = nrows_s;
  for (int idx = tid; idx < rows * l; idx += kThreads) {
    const int r = idx / l, t = idx - r * l;
    W[r * ldw + t] = Y[ids[r] * l + t];
  }
  __syncthreads();
  const int steps = min(rows, l);
  gepp(W, ldw, ids, rows, l, steps, piv, slot);
  for (int j = tid; j < l; j += kThreads) cand_out[(int64_t)blockIdx.x * l + j] = j < steps ? ids[piv[j]] : -1;
  if (!final_) return;
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int j = idx / l, t = idx - j * l;
    const double v = W[piv[j] * ldw + t];
    U[idx] = t >= j ? v : 0.0;
    Lp[idx] = t < j ? v : (t == j ? 1.0 : 0.0);
  }
  for (int j = tid; j < l; j += kThreads) piv_out[j] = ids[piv[j]];
  __syncthreads();
  // M = U⁻¹ with the zero-pivot rule (a zero U_ii zeroes row i of M: x_i = 0
  // for every input of the row substitution x·U = y, reading Q3): column j by
  // one warp, M[j][j] = 1/U_jj, M[i][j] = −(Σ_{t=i+1..j} U_it M_tj)/U_ii.
  double* Ms = reinterpret_cast<double*>(ids + cap);  // l×l after the row ids
  const int lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < l; j += kWarps) {
    for (int i = lane; i < l; i += 32) Ms[i * l + j] = 0.0;
    __syncwarp();
    for (int i = j; i >= 0; --i) {
      double acc = 0.0;
      for (int t = i + 1 + lane; t <= j; t += 32) acc += W[piv[i] * ldw + t] * Ms[t * l + j];
      acc = warp_sum(acc);
      const double uii = W[piv[i] * ldw + i];
      if (lane == 0) Ms[i * l + j] = (uii != 0.0) ? ((i == j ? 1.0 : 0.0) - acc) / uii : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += kThreads) M[idx] = Ms[idx];
}

// L = Y·M (in place) with M = U⁻¹ formed per CTA (zero-pivot rule: a zero
// U_ii zeroes row i of M, i.e. x_i = 0 for every input, as the row
// substitution x·U = y of reading Q3 prescribes), pivot rows ← Lp rows.  CTAs
// walk 128-row tiles; if `gpart` is given each CTA also writes its partial
// Gram Σ L_rᵀ L_r (upper triangle) for the Cholesky-QR that follows.
__global__ void __launch_bounds__(kThreads, 2) lu_apply_kernel(double* __restrict__ Y, int64_t m, int l,
                                                            const double* __restrict__ M,
                                                            const double* __restrict__ Lp,
                                                            const int64_t* __restrict__ piv,
                                                            double* __restrict__ gpart) {
  extern __shared__ double sm[];
  const int ldw = l | 1;
  double* Ms = sm;                 // l×l
  double* Ys = sm + l * l;         // 128×ldw
  __shared__ int pivpos[128];
  for (int idx = threadIdx.x; idx < l * l; idx += kThreads) Ms[idx] = M[idx];
  const int r = threadIdx.x & 127, jph = threadIdx.x >> 7;  // 2 column phases
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
    for (int idx = threadIdx.x; idx < 128; idx += kThreads) pivpos[idx] = -1;
    for (int idx = threadIdx.x; idx < rows * l; idx += kThreads) {
      const int rr = idx / l, t = idx - rr * l;
      Ys[rr * ldw + t] = Y[r0 * l + idx];
    }
    __syncthreads();
    if (threadIdx.x < l) {
      const int64_t pr = piv[threadIdx.x] - r0;
      if (pr >= 0 && pr < rows) pivpos[pr] = threadIdx.x;
    }
    __syncthreads();
    double out[kMaxL / 2];
    if (r < rows) {
      const int pj = pivpos[r];
#pragma unroll
      for (int q = 0; q < kMaxL / 2; ++q) {
        const int j = jph + 2 * q;
        if (j >= l) break;
        double s;
        if (pj >= 0) {
          s = Lp[pj * l + j];
        } else {
          double s0 = 0.0, s1 = 0.0;
          int t = 0;
          for (; t + 1 <= j; t += 2) {
            s0 += Ys[r * ldw + t] * Ms[t * l + j];
            s1 += Ys[r * ldw + t + 1] * Ms[(t + 1) * l + j];
          }
          if (t <= j) s0 += Ys[r * ldw + t] * Ms[t * l + j];
          s = s0 + s1;
        }
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

constexpr int kLeafRows = 256;

// a tree group holds ≤ 3·256 rows (3 rows per thread in gepp) and ≤ ~200 KB
int group_for(int l) {
  const int max_rows = std::min(kThreads * 3, 21000 / (l | 1));
  return std::max(2, std::min(32, max_rows / l));
}

size_t select_smem(int cap, int l) { return (size_t)cap * (l | 1) * 8 + (size_t)cap * 8 + (size_t)l * l * 8 + 16; }

void select(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
            int G, int64_t* cout, int final_, double* U, double* Lp, int64_t* piv, double* M) {
  const int cap = leaf ? kLeafRows : G * l;
  ensure_smem((const void*)lu_select_kernel, 220 * 1024);
  lu_select_kernel<<<grid, kThreads, select_smem(cap, l), c.stream>>>(Y, m, l, leaf, kLeafRows, cin, n_in, G, cout,
                                                                     final_, U, Lp, piv, M);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, leaf ? "lu_leaf" : "lu_tree");
}

}  // namespace

size_t lu_ws_bytes(int64_t m, int l) {
  Sizer s;
  const int64_t nblk = cdiv(m, kLeafRows);
  s.add<int64_t>(nblk * l);
  s.add<int64_t>(nblk * l);
  s.add<double>(4 * (size_t)l * l);
  s.add<int64_t>(l);
  return s.total;
}

int lu_apply_grid(Ctx& c, int64_t m) { return (int)std::min<int64_t>(cdiv(m, 128), (int64_t)c.num_sms * 2); }

void lu_renorm(Ctx& c, double* Y, int64_t m, int l, double* U_out, int64_t* piv_out, Arena& ar, double* gpart) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "lu_renorm: need 1 ≤ l ≤ %d and m ≥ l", kMaxL);
  const int G = group_for(l);
  const int64_t nblk = cdiv(m, kLeafRows);
  int64_t* ca = ar.get<int64_t>(nblk * l);
  int64_t* cb = ar.get<int64_t>(nblk * l);
  double* U = U_out ? U_out : ar.get<double>((size_t)l * l);
  double* Lp = ar.get<double>((size_t)l * l);
  int64_t* piv = ar.get<int64_t>(l);
  double* M = ar.get<double>((size_t)l * l);
  select(c, (unsigned)nblk, Y, m, l, 1, nullptr, 0, G, ca, nblk == 1, U, Lp, piv, M);
  int64_t n = nblk;
  while (n > 1) {
    const int64_t ng = cdiv(n, G);
    select(c, (unsigned)ng, Y, m, l, 0, ca, n, G, cb, ng == 1, U, Lp, piv, M);
    std::swap(ca, cb);
    n = ng;
  }
  const size_t smem_apply = (size_t)(l * l + 128 * (l | 1)) * 8;
  ensure_smem((const void*)lu_apply_kernel, (int)((kMaxL * kMaxL + 128 * (kMaxL | 1)) * 8));
  const unsigned grid = (unsigned)lu_apply_grid(c, m);
  lu_apply_kernel<<<grid, kThreads, smem_apply, c.stream>>>(Y, m, l, M, Lp, piv, gpart);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_apply");
  if (piv_out) RPCA_CUDA(cudaMemcpyAsync(piv_out, piv, sizeof(int64_t) * l, cudaMemcpyDeviceToDevice, c.stream));
}

}  // namespace rpca
