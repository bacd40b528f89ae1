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
#include "comm.cuh"

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
                                                             double* __restrict__ M,
                                                             const double* __restrict__ rows_in,
                                                             double* __restrict__ rows_out) {
  // leaf: 1 = contiguous rows of Y; 0 = candidate ids into Y; 2 = candidate
  // rows given directly (rows_in, one l-vector per slot; ids are global rows
  // — the all-gathered local winners of a row-sharded LU)
  extern __shared__ double sm[];
  __shared__ Cand slot[2][kWarps];
  __shared__ int piv[kMaxL];
  __shared__ int nrows_s;
  const int cap = leaf == 1 ? (int)leaf_rows : G * l;
  const int ldw = l | 1;
  double* W = sm;
  int64_t* ids = reinterpret_cast<int64_t*>(W + (size_t)cap * ldw);
  int* slot_of = reinterpret_cast<int*>(ids + cap);
  const int tid = threadIdx.x;

  if (leaf == 1) {
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
        if (id >= 0) {
          const int pos = base + __popc(mask & ((1u << tid) - 1u));
          ids[pos] = id;
          slot_of[pos] = (int)(s + tid - s0);
        }
        base += __popc(mask);
      }
      if (tid == 0) nrows_s = base;
    }
  }
  __syncthreads();
  const int rows = nrows_s;
  for (int idx = tid; idx < rows * l; idx += kThreads) {
    const int r = idx / l, t = idx - r * l;
    W[r * ldw + t] = leaf == 2 ? rows_in[((int64_t)blockIdx.x * G * l + slot_of[r]) * l + t] : Y[ids[r] * l + t];
  }
  __syncthreads();
  const int steps = min(rows, l);
  gepp(W, ldw, ids, rows, l, steps, piv, slot);
  for (int j = tid; j < l; j += kThreads) cand_out[(int64_t)blockIdx.x * l + j] = j < steps ? ids[piv[j]] : -1;
  if (rows_out) {  // direct mode: forward the winners' original rows to the next level
    for (int idx = tid; idx < l * l; idx += kThreads) {
      const int j = idx / l, t = idx - j * l;
      rows_out[(int64_t)blockIdx.x * l * l + idx] =
          j < steps ? rows_in[((int64_t)blockIdx.x * G * l + slot_of[piv[j]]) * l + t] : 0.0;
    }
  }
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
  double* Ms = reinterpret_cast<double*>(ids + cap) + (cap + 1) / 2;  // l×l after ids and slot_of
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

// Y[piv[j] − row0] ← Lp[j] for the pivot rows this shard holds (their exact
// unit-lower rows)
__global__ void pivot_rows_kernel(double* __restrict__ Y, int64_t m, int64_t row0, int l,
                                  const double* __restrict__ Lp, const int64_t* __restrict__ piv) {
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int j = idx / l, t = idx - j * l;
    const int64_t r = piv[j] - row0;
    if (r >= 0 && r < m) Y[r * l + t] = Lp[idx];
  }
}

// rows_out[j] = Y[cand[j]] (l-vectors), gid[j] = row0 + cand[j] (−1 kept) — the
// local tournament winners packaged for the all-gather of a sharded LU
__global__ void pack_candidates_kernel(const double* __restrict__ Y, int l, int64_t row0,
                                       const int64_t* __restrict__ cand, double* __restrict__ rows_out,
                                       int64_t* __restrict__ gid) {
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int j = idx / l, t = idx - j * l;
    const int64_t r = cand[j];
    rows_out[idx] = r >= 0 ? Y[r * l + t] : 0.0;
    if (t == 0) gid[j] = r >= 0 ? row0 + r : -1;
  }
}

constexpr int kLeafRows = 256;

// a tree group holds ≤ 3·256 rows (3 rows per thread in gepp) and ≤ ~200 KB
int group_for(int l) {
  const int max_rows = std::min(kThreads * 3, 21000 / (l | 1));
  return std::max(2, std::min(32, max_rows / l));
}

size_t select_smem(int cap, int l) {
  return (size_t)cap * (l | 1) * 8 + (size_t)cap * 8 + (size_t)(cap + 1) / 2 * 8 + (size_t)l * l * 8 + 16;
}

void select(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
            int G, int64_t* cout, int final_, double* U, double* Lp, int64_t* piv, double* M,
            const double* rows_in = nullptr, double* rows_out = nullptr) {
  const int cap = leaf == 1 ? kLeafRows : G * l;
  ensure_smem((const void*)lu_select_kernel, 220 * 1024);
  const size_t smem = select_smem(cap, l) - (final_ ? 0 : (size_t)l * l * 8);
  lu_select_kernel<<<grid, kThreads, smem, c.stream>>>(Y, m, l, leaf, kLeafRows, cin, n_in, G, cout, final_, U, Lp,
                                                       piv, M, rows_in, rows_out);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, leaf == 1 ? "lu_leaf" : "lu_tree");
}

// Tournament over rows [0, m) of Y down to one candidate set; returns the set
// (l entries, local row indices, −1 padded).  If `finalize`, the last level
// also writes U, Lp, piv and M.
int64_t* tournament(Ctx& c, const double* Y, int64_t m, int l, bool finalize, double* U, double* Lp, int64_t* piv,
                    double* M, Arena& ar) {
  const int G = group_for(l);
  const int64_t nblk = std::max<int64_t>(1, cdiv(m, kLeafRows));
  int64_t* ca = ar.get<int64_t>(nblk * l);
  int64_t* cb = ar.get<int64_t>(nblk * l);
  if (m == 0) {
    RPCA_CUDA(cudaMemsetAsync(ca, 0xFF, sizeof(int64_t) * l, c.stream));  // no local rows: all −1
    return ca;
  }
  select(c, (unsigned)nblk, Y, m, l, 1, nullptr, 0, G, ca, finalize && nblk == 1, U, Lp, piv, M);
  int64_t n = nblk;
  while (n > 1) {
    const int64_t ng = cdiv(n, G);
    select(c, (unsigned)ng, Y, m, l, 0, ca, n, G, cb, finalize && ng == 1, U, Lp, piv, M);
    std::swap(ca, cb);
    n = ng;
  }
  return ca;
}

// L = Y·M on the fp64 tensor-core pass kernel (in place: every output row is
// written only after all of its own K-chunks were read), then the pivot rows
// this shard holds get their exact unit-lower rows
void apply_l(Ctx& c, double* Y, int64_t m, int64_t row0, int l, const double* M, const double* Lp,
             const int64_t* piv, Arena& ar) {
  if (m > 0) {
    TagScope ts(c, "lu_apply");
    dense_ax(c, DenseA{Y, RPCA_F64, m, l, l}, M, l, Y, ar);
  }
  pivot_rows_kernel<<<1, 256, 0, c.stream>>>(Y, m, row0, l, Lp, piv);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_pivot_rows");
}

}  // namespace

size_t lu_ws_bytes(int64_t m, int l) {
  Sizer s;
  s.add<char>(ax_ws_bytes(DenseA{nullptr, RPCA_F64, m, l, l}, l) + 4096);
  const int64_t nblk = std::max<int64_t>(1, cdiv(m, kLeafRows));
  s.add<int64_t>(nblk * l);
  s.add<int64_t>(nblk * l);
  s.add<double>(4 * (size_t)l * l);
  s.add<int64_t>(l);
  s.add<double>((size_t)2 * kMaxL * (size_t)(kMaxL + 1) * 64 + 2 * kMaxL * kMaxL);  // sharded: gathered rows + ids
  return s.total;
}

void lu_renorm(Ctx& c, double* Y, int64_t m, int l, double* U_out, int64_t* piv_out, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "lu_renorm: need 1 ≤ l ≤ %d and m ≥ l", kMaxL);
  double* U = U_out ? U_out : ar.get<double>((size_t)l * l);
  double* Lp = ar.get<double>((size_t)l * l);
  int64_t* piv = ar.get<int64_t>(l);
  double* M = ar.get<double>((size_t)l * l);
  const size_t mark = ar.off;
  tournament(c, Y, m, l, true, U, Lp, piv, M, ar);
  ar.off = mark;
  apply_l(c, Y, m, 0, l, M, Lp, piv, ar);
  if (piv_out) RPCA_CUDA(cudaMemcpyAsync(piv_out, piv, sizeof(int64_t) * l, cudaMemcpyDeviceToDevice, c.stream));
}

// Row-sharded LU: every rank runs the tournament on its rows
// [row0, row0+m); the winners (l rows + their global ids) are all-gathered and
// every rank runs the final GEPP on the same P·l rows — identical U, pivots and
// M everywhere — then applies L = Y·M to its own rows.
void lu_renorm_sharded(Ctx& c, double* Y, int64_t m, int64_t row0, int l, double* U_out, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= 0, RPCA_E_SHAPE, "lu_renorm: need 1 ≤ l ≤ %d", kMaxL);
  const int P = comm_size(c);
  RPCA_REQUIRE(P <= 64, RPCA_E_ARG, "at most 64 ranks");
  double* U = U_out ? U_out : ar.get<double>((size_t)l * l);
  double* Lp = ar.get<double>((size_t)l * l);
  int64_t* piv = ar.get<int64_t>(l);
  double* M = ar.get<double>((size_t)l * l);
  double* rows_send = ar.get<double>((size_t)l * l);
  int64_t* ids_send = ar.get<int64_t>(l);
  double* rows_a = ar.get<double>((size_t)l * l * P);
  double* rows_b = ar.get<double>((size_t)l * l * P);
  int64_t* ids_a = ar.get<int64_t>((size_t)l * P);
  int64_t* ids_b = ar.get<int64_t>((size_t)l * P);
  const size_t mark = ar.off;
  const int64_t* cand = tournament(c, Y, m, l, false, nullptr, nullptr, nullptr, nullptr, ar);
  pack_candidates_kernel<<<1, 256, 0, c.stream>>>(Y, l, row0, cand, rows_send, ids_send);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_pack");
  ar.off = mark;
  allgather_bytes(c, rows_send, rows_a, sizeof(double) * l * l);
  allgather_bytes(c, ids_send, ids_a, sizeof(int64_t) * l);
  // tournament over the P gathered sets with rows given directly; every rank
  // runs the same launches on the same bytes, so U, piv and M agree bitwise
  const int G = group_for(l);
  int64_t n = P;
  for (;;) {
    const int64_t ng = cdiv(n, G);
    select(c, (unsigned)ng, nullptr, 0, l, 2, ids_a, n, G, ids_b, ng == 1, U, Lp, piv, M, rows_a,
           ng == 1 ? nullptr : rows_b);
    if (ng == 1) break;
    std::swap(rows_a, rows_b);
    std::swap(ids_a, ids_b);
    n = ng;
  }
  apply_l(c, Y, m, row0, l, M, Lp, piv, ar);
}

}  // namespace rpca
