// tslu.cu — §8(a) step a3: LU renormalisation of a tall-skinny block.
//
// PAPER.md:382-404 (§5): "computing the LU decomposition is typically more
// efficient than computing the QR decomposition, and both are sufficient for
// most stages" — "[Q,R] = lu(Q)", i.e. Q ← the row-permuted unit lower factor
// L with Y = L·U (MATLAB's two-output lu; reading Q3).
//
// B200 design — tournament pivoting (CALU):
//   1. leaf kernel: a persistent CTA walks blocks of R·256 rows (the next
//      block bulk-copied into shared memory meanwhile), runs GEPP on each and
//      nominates l candidate pivot rows (original rows);
//   2. tree kernel: groups of G candidate sets are stacked (original values
//      gathered from Y) and reduced by GEPP again, until one set is left; the
//      last GEPP gives the pivot order, U (l×l) and the multipliers of the pivot
//      rows (Lp);
//   3. apply kernel: every CTA first forms the substitution matrix M with
//      x = y·M ⇔ x·U = y (x_j = 0 where U_jj = 0 — the exact-zero-pivot rule of
//      reading Q3), then L = Y·M for its rows (HBM-bound); pivot rows are
//      overwritten with their exact unit-lower rows from Lp.
// GEPP inside a CTA: thread t owns rows t·R … t·R+R−1 held in REGISTERS (the
// kernel is templated on l rounded up to 8, every column step is unrolled so
// all register indices are static).  Per column: the argmax over the warp is
// two redux.sync.max on the bits of |v| (a non-negative double orders like its
// bit pattern) plus a ballot for the lowest lane on ties; each warp's winner
// lane publishes its (key, row), its reciprocal and the panel part of its row
// to shared memory; ONE __syncthreads; every warp then reduces the 8 warp winners the
// same way (lanes 0-7 hold the keys) and reads the pivot row with broadcast
// loads.  Local row order = original row
// order (leaves are contiguous; tree candidates are sorted by id within each
// set and sets cover ascending row ranges), so "lowest local row" is the
// lowest-original-row tie rule.  Tournament pivots differ from plain GEPP, so
// L differs from the oracle's L but span(L) = span(Y) whenever U is
// nonsingular.
#include <type_traits>
#include <utility>

#include "comm.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// rows per thread: leaves favour occupancy, tree levels (few CTAs, latency-
// bound) favour bigger groups so the tournament has fewer levels
#ifndef LU_NOM_U32
#define LU_NOM_U32 32  // rows in flight per warp in the nomination loads, l ≤ 32
#endif
#ifndef LU_NOM_U64
#define LU_NOM_U64 16  // … l > 32
#endif
#ifndef LU_LEAF_R24
#define LU_LEAF_R24 1  // rows per thread of the leaves for 16 < LP ≤ 24
#endif
#ifndef LU_LEAF_R32
#define LU_LEAF_R32 2  // … for 24 < LP ≤ 32 (C5: leaves +0.8 ms, tree −1.0 ms)
#endif
constexpr int leaf_rows_per_thread(int LP) {
  return LP <= 8 ? 4 : (LP <= 16 ? 2 : (LP <= 24 ? LU_LEAF_R24 : (LP <= 32 ? LU_LEAF_R32 : 1)));
}
#ifndef LU_TREE_R32
#define LU_TREE_R32 1  // rows per thread of the fp64 last level for 8 < LP ≤ 32 (1: −21% vs 2)
#endif
constexpr int tree_rows_per_thread(int LP) { return LP <= 8 ? 4 : (LP <= 32 ? LU_TREE_R32 : 1); }

// two CTAs per SM (registers capped at 128) while a thread's rows fit
#ifndef LU_TWO_BLOCK_MAX
#define LU_TWO_BLOCK_MAX 32
#endif

template <int LP, int RR>
struct SelCfg {
  static constexpr int R = RR;
  static constexpr int kCap = kThreads * R;  // rows per CTA
  static constexpr int kMinBlocks = R * LP <= LU_TWO_BLOCK_MAX ? 2 : 1;
};

// Pivot key of a value: the high word of |v| (11 exponent + 20 mantissa bits)
// + 1, so 0 means "no candidate".  The pivot of a column is therefore a row
// whose |value| is within 2^-20 (relative) of the column maximum — the lowest
// such row (tournament LU): multipliers stay ≤ 1 + 2^-20.
__device__ __forceinline__ uint32_t piv_key(double v) {
  return ((uint32_t)__double2hiint(v) & 0x7FFFFFFFu) + 1u;
}

// w[t−1] ← w[t] − mult·prow[t] for t < W (the live width), w[W−1.. ] ← 0
template <int LP, int W>
__device__ __forceinline__ void eliminate(double (&w)[LP], const double* prow, double mult) {
#pragma unroll
  for (int t = 1; t < W; ++t) w[t - 1] = fma(-mult, prow[t], w[t]);
#pragma unroll
  for (int t = W - 1; t < LP; ++t) w[t] = 0.0;
}

// rank-ns update of the trailing columns then the shift to the next panel:
// w[t] −= Σ_{s<ns} w[s]·U12[s][t−8] for 8 ≤ t < W, then w[t] ← w[t+8]
template <int LP, int W>
__device__ __forceinline__ void trail_update(double (&w)[LP], const double (*u12)[LP], int ns) {
  double m[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) m[s] = s < ns ? w[s] : 0.0;
#pragma unroll
  for (int t = 8; t < W; ++t) {
    double v = w[t];
#pragma unroll
    for (int s = 0; s < 8; ++s) v = fma(-m[s], u12[s][t - 8], v);
    w[t] = v;
  }
#pragma unroll
  for (int t = 0; t + 8 < LP; ++t) w[t] = w[t + 8];
#pragma unroll
  for (int t = LP - 8; t < LP; ++t) w[t] = 0.0;
}

// One CTA: rows from Y (leaf: contiguous block; tree: a group of candidate
// sets), GEPP, l nominated original rows → cand_out[blockIdx.x*l ...] (-1 pad).
// If final, also U, Lp and the original pivot rows piv_out (M = U⁻¹ follows in
// u_inverse_warp_kernel).
//   leaf: 1 = contiguous rows of Y; 0 = candidate ids into Y; 2 = candidate
//   rows given directly (rows_in, one l-vector per slot; ids are global rows
//   — the all-gathered local winners of a row-sharded LU)
template <int LP, int RR, bool BULK>
__global__ void __launch_bounds__(kThreads, SelCfg<LP, RR>::kMinBlocks)
    lu_select_kernel(const double* __restrict__ Y, int64_t m, int l, int leaf, const int64_t* __restrict__ cand_in,
                     int64_t n_in, int G, int64_t* __restrict__ cand_out, int final_, double* __restrict__ U,
                     double* __restrict__ Lp, int64_t* __restrict__ piv_out, double* __restrict__ M,
                     const double* __restrict__ rows_in, double* __restrict__ rows_out,
                     const double* __restrict__ mu, int bulk) {
  using Cfg = SelCfg<LP, RR>;
  constexpr int R = Cfg::R, CAP = Cfg::kCap;
  __shared__ int64_t ids[CAP];
  __shared__ int slot_of[CAP];
  __shared__ uint2 slot[2][kWarps];  // {pivot key, local row} of each warp's winner
  __shared__ double suinv[2][kWarps];
  __shared__ __align__(16) double pbuf[2][kWarps][8];  // panel part of each warp winner's row
  __shared__ double traw[8][LP];                         // raw trailing parts of the panel's pivot rows
  __shared__ double l11[8][8];                           // the panel's unit-lower multipliers
  __shared__ double u12[8][LP];                          // trailing rows of U
  __shared__ int piv[LP];
  __shared__ int nrows_s;
  __shared__ int setcnt[CAP + 1];
  __shared__ uint64_t full_bar;
  // final: LP × LP published pivot rows and the multipliers; bulk: the staged
  // rows of the next leaf (CAP × l, row-major as in Y)
  extern __shared__ double keep[];
  double* msm = keep + LP * LP;  // final only: multiplier of (step j, row r) at j·CAP + r
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // bulk (leaves only, never final): a persistent CTA walks leaves b, b+grid, …
  // and a 1-D bulk copy stages the next leaf's rows (contiguous in Y) in
  // shared memory while the current leaf runs its GEPP on registers
  bulk = BULK && bulk;  // the staging code exists in the BULK instantiation only
  const int64_t nleaf = (leaf == 1 && bulk) ? (m + CAP - 1) / CAP : (int64_t)blockIdx.x + 1;
  auto leaf_bytes = [&](int64_t b) -> uint32_t {
    return (uint32_t)(imin64(CAP, m - b * CAP) * l * 8) & ~15u;  // an odd last double is read from Y
  };
  if (leaf == 1 && bulk) {
    if (tid == 0) {
      mbar_init(&full_bar, 1);
      fence_barrier_init();
      const int64_t b = blockIdx.x;
      mbar_arrive_expect_tx(&full_bar, leaf_bytes(b));
      if (leaf_bytes(b)) bulk_load(keep, Y + b * CAP * l, leaf_bytes(b), &full_bar);
    }
    __syncthreads();
  }
  uint32_t it = 0;
  for (int64_t blk = blockIdx.x; blk < nleaf; blk += gridDim.x, ++it) {
  if (leaf == 1) {
    const int64_t r0 = blk * CAP;
    if (tid == 0) nrows_s = (int)imin64(CAP, m - r0);
    for (int r = tid; r < CAP; r += kThreads) ids[r] = r0 + r;
  } else {
    // compact the valid candidates of this group: sets in ascending order,
    // each set's ids sorted ascending (rank = #smaller valid ids in the set)
    const int64_t s0 = blk * G * l, s1 = imin64(n_in * l, s0 + (int64_t)G * l);
    const int nslots = (int)(s1 - s0), nsets = (nslots + l - 1) / l;
    for (int s = tid; s < nslots; s += kThreads) ids[s] = cand_in[s0 + s];
    __syncthreads();
    for (int st = tid; st < nsets; st += kThreads) {
      int cnt = 0;
      for (int t = st * l; t < min(nslots, st * l + l); ++t) cnt += ids[t] >= 0;
      setcnt[st + 1] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
      setcnt[0] = 0;
      for (int st = 0; st < nsets; ++st) setcnt[st + 1] += setcnt[st];
      nrows_s = setcnt[nsets];
    }
    __syncthreads();
    int64_t myid[(CAP + kThreads - 1) / kThreads];
    int mypos[(CAP + kThreads - 1) / kThreads];
#pragma unroll
    for (int q = 0; q < (CAP + kThreads - 1) / kThreads; ++q) {
      const int s = tid + q * kThreads;
      mypos[q] = -1;
      myid[q] = -1;
      if (s < nslots && ids[s] >= 0) {
        const int st = s / l;
        const int64_t id = ids[s];
        int rank = 0;
        for (int t = st * l; t < min(nslots, st * l + l); ++t) rank += (ids[t] >= 0 && ids[t] < id);
        mypos[q] = setcnt[st] + rank;
        myid[q] = id;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < (CAP + kThreads - 1) / kThreads; ++q)
      if (mypos[q] >= 0) {
        ids[mypos[q]] = myid[q];
        slot_of[mypos[q]] = tid + q * kThreads;
      }
  }
  __syncthreads();
  const int rows = nrows_s;
  const int steps = min(rows, l);

  // this thread's rows → registers (zero beyond l / beyond rows)
  double w[R][LP];
  bool act[R];
  int pstep[R];  // ≥ 0: pivot step within the current panel (−1: not a pivot)
  const bool staged = leaf == 1 && bulk;
  if (staged) mbar_wait(&full_bar, it & 1u);
  const uint32_t nstaged = staged ? leaf_bytes(blk) / 8 : 0u;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const int r = tid * R + q;
    act[q] = r < rows;
    pstep[q] = -1;
    const double* src = nullptr;
    if (act[q])
      src = leaf == 2                             ? rows_in + (blk * G * l + slot_of[r]) * l
            : (uint32_t)((r + 1) * l) <= nstaged ? keep + r * l
                                                  : Y + ids[r] * l;
    // a pending centring of Y (the projector P of DESIGN.md reading Q8) is
    // applied on load; direct rows (leaf 2) arrive centred
    const bool sub = mu != nullptr && leaf != 2;
#pragma unroll
    for (int t = 0; t < LP; ++t) w[q][t] = (act[q] && t < l) ? src[t] - (sub ? mu[t] : 0.0) : 0.0;
  }
  if (staged) {
    __syncthreads();  // every row is in registers: the buffer takes the next leaf
    const int64_t nb = blk + gridDim.x;
    if (tid == 0 && nb < nleaf) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&full_bar, leaf_bytes(nb));
      if (leaf_bytes(nb)) bulk_load(keep, Y + nb * CAP * l, leaf_bytes(nb), &full_bar);
    }
  }

  // Blocked GEPP, panels of 8 columns.  Registers hold each row SHIFTED so
  // the current panel is w[q][0..7] (static indices; the loop over panels is
  // rolled — a straight-line unroll over all columns overflows the
  // instruction cache).  Panel step s: argmax of column s, the warp winner
  // publishes only the panel part of its row (≤ 8 values), one barrier, then
  // each row eliminates the panel columns and keeps its multiplier in w[q][s].
  // Panel end: the panel's pivot rows publish their raw trailing parts, the
  // trailing rows of U are formed by forward substitution with the panel's
  // unit-lower L11 (one thread per column), and every other row applies the
  // rank-8 update w_trail −= Σ_s mult_s·U12[s] and shifts left by 8.  Same
  // pivots as column-by-column GEPP; only the order of the trailing updates
  // differs.  Final level: U rows go to `keep`, multipliers to `msm`.
  for (int pb = 0; pb < steps; pb += 8) {
    const int ns = min(8, steps - pb);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s >= ns) break;
      const int j = pb + s;
      uint32_t best = 0;
      int bq = 0;
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (act[q]) {
          const uint32_t k = piv_key(w[q][s]);
          if (k > best) { best = k; bq = q; }
        }
      const uint32_t mk = __reduce_max_sync(0xffffffffu, best);
      const int wl = __ffs(__ballot_sync(0xffffffffu, best == mk)) - 1;  // lowest lane = lowest row
      if (lane == wl) {
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (q == bq) {
            slot[j & 1][warp] = make_uint2(mk, (uint32_t)(tid * R + q));
            suinv[j & 1][warp] = rcp_nr(w[q][s]);
#pragma unroll
            for (int t = s; t < 8; ++t) pbuf[j & 1][warp][t] = w[q][t];
          }
      }
      __syncthreads();
      // max over the 8 warp winners: lanes 0-7 hold their keys, one redux and
      // a ballot (lowest warp = lowest rows on ties)
      const uint32_t kv = lane < kWarps ? slot[j & 1][lane].x : 0u;
      const uint32_t gk = __reduce_max_sync(0xffffffffu, kv);
      const int ww = __ffs(__ballot_sync(0xffffffffu, kv == gk)) - 1;
      const int p = (int)slot[j & 1][ww].y;
      const double uinv = suinv[j & 1][ww];
      const double* prow = pbuf[j & 1][ww];
      if (tid == 0) piv[j] = p;
      if (final_ && tid < 8 - s) keep[j * LP + tid] = prow[s + tid];  // U[j][j .. pb+7]
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (!act[q]) continue;
        if (tid * R + q == p) {
          act[q] = false;
          pstep[q] = s;  // this row is the panel's s-th pivot
          continue;
        }
        const double mult = w[q][s] * uinv;
        w[q][s] = mult;
        if (final_) msm[j * CAP + tid * R + q] = mult;
#pragma unroll
        for (int t = s + 1; t < 8; ++t) w[q][t] = fma(-mult, prow[t], w[q][t]);
      }
    }
    if (pb + 8 >= LP) break;  // no trailing columns
    // ---- panel end: U12 (rows of U right of the panel) by forward substitution
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (pstep[q] >= 0) {
        const int sp = pstep[q];
#pragma unroll
        for (int t = 8; t < LP; ++t) traw[sp][t - 8] = w[q][t];
#pragma unroll
        for (int t = 0; t < 8; ++t) l11[sp][t] = t < sp ? w[q][t] : 0.0;
        pstep[q] = -2;  // published; the row is done
      }
    __syncthreads();
    if (tid < LP - 8) {
      double u[8];
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        double v = sp < ns ? traw[sp][tid] : 0.0;
#pragma unroll
        for (int s2 = 0; s2 < sp; ++s2) v = fma(-l11[sp][s2], u[s2], v);
        u[sp] = v;
        u12[sp][tid] = v;
        if (final_ && sp < ns) keep[(pb + sp) * LP + (8 - sp) + tid] = v;  // U[j][pb+8+tid]
      }
    }
    __syncthreads();
    const int live = LP - pb;  // columns beyond are zero in every row
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if (!act[q]) continue;
      if (live > LP / 2) trail_update<LP, LP>(w[q], u12, ns);
      else trail_update<LP, LP / 2>(w[q], u12, ns);
    }
  }
  __syncthreads();
  for (int j = tid; j < l; j += kThreads) cand_out[blk * l + j] = j < steps ? ids[piv[j]] : -1;
  if (rows_out) {  // direct mode: forward the winners' original rows to the next level
    for (int idx = tid; idx < l * l; idx += kThreads) {
      const int j = idx / l, t = idx - j * l;
      rows_out[blk * l * l + idx] = j < steps ? rows_in[(blk * G * l + slot_of[piv[j]]) * l + t] : 0.0;
    }
  }
  if (!final_) {
    __syncthreads();  // ids / piv are rewritten by the next leaf
    continue;
  }
  // keep[j] = pivot row j as published (columns j.. at 0..LP−j−1); its
  // multiplier of step s < j is msm[s·CAP + piv[j]]
  for (int idx = tid; idx < l * l; idx += kThreads) {
    const int j = idx / l, c = idx - j * l;
    const double u = c >= j ? keep[j * LP + c - j] : 0.0;
    U[idx] = u;
    Lp[idx] = c < j ? msm[c * CAP + piv[j]] : (c == j ? 1.0 : 0.0);
  }
  for (int j = tid; j < l; j += kThreads) piv_out[j] = ids[piv[j]];
  // M = U⁻¹ follows in u_inverse_warp_kernel (one thread per column in
  // registers; here, one column per thread re-read every term from shared
  // memory — 20-66k cycles, up to half of this kernel)
  }  // leaves
}

// ---------------------------------------------------------------------------
// Nomination levels in fp32 (every tournament level but the last).  A level
// only NOMINATES l candidate rows of its block — the last level re-reads the
// candidates' original fp64 rows and runs the exact fp64 GEPP that fixes the
// pivots, U and M, so L = Y·U⁻¹ stays an exact factorisation whatever was
// nominated (reading Q3).  fp32 halves the registers a row
// takes (two CTAs per SM instead of one) and the FFMA / MUFU latencies of the
// step chain.  Each column is scaled by an exact power of two so that its
// largest |value| in the block is in [1, 2) — column scaling leaves GEPP's
// pivot choices unchanged, and the fp32 range then covers every column
// whatever the fp64 magnitudes.  A column whose remaining values are all
// below 2^-100 of its block maximum counts as zero (no elimination).


// a·b + c on both halves of a float pair: one FFMA2
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// MINB: CTAs per SM the registers are capped for — 3 for the wide leaves and
// big tree levels of 32 < l < 64 (80 registers, a few spilled: the third
// CTA's step chain hides more of the other two's), else 2
template <int LP, int R, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    lu_nominate_kernel(const double* __restrict__ Y, int64_t m, int l, int leaf, const int64_t* __restrict__ cand_in,
                       int64_t n_in, int G, int64_t* __restrict__ cand_out, const double* __restrict__ mu) {
  constexpr int CAP = kThreads * R;
  __shared__ int64_t ids[CAP];
  __shared__ int setcnt[CAP + 1];
  __shared__ uint32_t slot[2][kWarps];  // each warp's winning packed key
  __shared__ __align__(16) float pbuf[2][kWarps][8];
  __shared__ float traw[8][LP];
  __shared__ float l11[8][8];
  __shared__ __align__(16) float u12[8][LP];
  __shared__ int piv[LP];
  __shared__ int colexp[LP];
  __shared__ int nrows_s;
  extern __shared__ float stage[];  // CAP × (l+1) scaled fp32 rows
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t blk = blockIdx.x;
  for (int t = tid; t < LP; t += kThreads) colexp[t] = 0;
  if (leaf == 1) {
    const int64_t r0 = blk * CAP;
    if (tid == 0) nrows_s = (int)imin64(CAP, m - r0);
    for (int r = tid; r < CAP; r += kThreads) ids[r] = r0 + r;
  } else {
    // valid candidates of this group in ascending id order within each set
    // (sets cover ascending row ranges, so ascending overall)
    const int64_t s0 = blk * G * l, s1 = imin64(n_in * l, s0 + (int64_t)G * l);
    const int nslots = (int)(s1 - s0), nsets = (nslots + l - 1) / l;
    for (int st = tid; st < nsets; st += kThreads) {
      int cnt = 0;
      for (int t = st * l; t < min(nslots, st * l + l); ++t) cnt += cand_in[s0 + t] >= 0;
      setcnt[st + 1] = cnt;
    }
    __syncthreads();
    if (tid == 0) {
      setcnt[0] = 0;
      for (int st = 0; st < nsets; ++st) setcnt[st + 1] += setcnt[st];
      nrows_s = setcnt[nsets];
    }
    __syncthreads();
    for (int s = tid; s < nslots; s += kThreads) {
      const int64_t id = cand_in[s0 + s];
      if (id < 0) continue;
      const int st = s / l;
      int rank = 0;
      for (int t = st * l; t < min(nslots, st * l + l); ++t) {
        const int64_t o = cand_in[s0 + t];
        rank += (o >= 0 && o < id);
      }
      ids[setcnt[st] + rank] = id;
    }
  }
  __syncthreads();
  const int rows = nrows_s;
  const int steps = min(rows, l);
  bool act[R];
  int pstep[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    act[q] = tid * R + q < rows;
    pstep[q] = -1;
  }
  // Rows are read coalesced — warp w takes rows w, w+8, …, lane j columns j
  // and j+32 (a thread-per-row read touched one 32-byte sector per lane and
  // saturated L1: ncu, profiles/r02_lu_nominate.md) — twice: pass 1 takes the
  // per-column exponent maxima (pending centring applied on load), pass 2
  // (L1/L2-hot) writes the scaled fp32 rows to shared memory at a stride of
  // l+1 floats, from where each thread loads its own rows bank-conflict free.
  const int sl = l + 1;
  {
    const double m0 = (mu && lane < l) ? mu[lane] : 0.0, m1 = (mu && lane + 32 < l) ? mu[lane + 32] : 0.0;
    // U rows' loads in flight per warp (the loads are latency-bound: a
    // leaf's rows arrive in ⌈rows / (8·U)⌉ round trips per pass); rows of
    // l ≤ 32 take one double per lane
    constexpr bool kTwo = LP > 32;
    constexpr int U8 = kTwo ? (MINB >= 3 ? 8 : LU_NOM_U64) : (MINB >= 3 ? 16 : LU_NOM_U32);
    // CONTIG: a full leaf (rows = CAP consecutive rows of Y) — plain strided
    // addresses, no per-row bounds or id lookups (the address arithmetic and
    // predicates were most of the leaf's instructions: ncu, C5 leaf)
    const double* yb = Y + (leaf == 1 ? blk * (int64_t)CAP * l : 0) + lane;
    // EXACT: l == LP (C5's l = 32) — row stride, bounds and the stage stride
    // become compile-time constants (immediate address offsets)
    auto passes = [&](auto CONTIG, auto EXACT) {
      constexpr bool kContig = decltype(CONTIG)::value;
      const int ll = decltype(EXACT)::value ? LP : l, sll = ll + 1;
      auto load8 = [&](int r0, double (&v0)[U8], double (&v1)[U8]) {
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int r = r0 + u * kWarps;
          if constexpr (kContig) {
            const int o = r * ll;
            v0[u] = lane < ll ? yb[o] : 0.0;
            if constexpr (kTwo) v1[u] = lane + 32 < ll ? yb[o + 32] : 0.0;
          } else {
            const double* y = Y + (r < rows ? ids[r] : 0) * l;
            v0[u] = (r < rows && lane < l) ? y[lane] : 0.0;
            if constexpr (kTwo) v1[u] = (r < rows && lane + 32 < l) ? y[lane + 32] : 0.0;
          }
        }
      };
      const int nr = kContig ? CAP : rows;
      unsigned f0 = 0, f1 = 0;
      for (int r0 = warp; r0 < nr; r0 += kWarps * U8) {
        double v0[U8], v1[U8];
        load8(r0, v0, v1);
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          if (!kContig && r0 + u * kWarps >= rows) break;
          f0 = max(f0, (unsigned)(__double_as_longlong(v0[u] - m0) >> 52) & 0x7FFu);
          if constexpr (kTwo) f1 = max(f1, (unsigned)(__double_as_longlong(v1[u] - m1) >> 52) & 0x7FFu);
        }
      }
      if (lane < ll && f0) atomicMax(&colexp[lane], (int)f0);
      if (kTwo && lane + 32 < ll && f1) atomicMax(&colexp[lane + 32], (int)f1);
      __syncthreads();
      // 2^(1023 − f) (field f ≥ 1): the column maximum lands in [1, 2) ([2, 4)
      // for the top binade, whose 2^-1023 would be subnormal)
      auto scale = [](int f) { return f ? __longlong_as_double((long long)(2046 - min(f, 2045)) << 52) : 0.0; };
      const double s0 = lane < ll ? scale(colexp[lane]) : 0.0, s1 = lane + 32 < ll ? scale(colexp[lane + 32]) : 0.0;
      for (int r0 = warp; r0 < nr; r0 += kWarps * U8) {
        double v0[U8], v1[U8];
        load8(r0, v0, v1);
#pragma unroll
        for (int u = 0; u < U8; ++u) {
          const int r = r0 + u * kWarps;
          if (!kContig && r >= rows) break;
          if (lane < ll) stage[r * sll + lane] = (float)((v0[u] - m0) * s0);
          if (kTwo && lane + 32 < ll) stage[r * sll + lane + 32] = (float)((v1[u] - m1) * s1);
        }
      }
    };
    static_assert(CAP % (kWarps * U8) == 0, "a full leaf is a whole number of load batches");
    if (leaf == 1 && rows == CAP && l == LP) passes(std::true_type{}, std::true_type{});
    else if (leaf == 1 && rows == CAP) passes(std::true_type{}, std::false_type{});
    else passes(std::false_type{}, std::false_type{});
  }
  __syncthreads();
  float w[R][LP];
  uint32_t amask[R];  // all ones while the row may still be chosen
#pragma unroll
  for (int q = 0; q < R; ++q) {
#pragma unroll
    for (int t = 0; t < LP; ++t) w[q][t] = (act[q] && t < l) ? stage[(tid * R + q) * sl + t] : 0.f;
    amask[q] = act[q] ? 0xFFFFFFFFu : 0u;
  }
  // Blocked GEPP in 8-column panels (the fp64 kernel's scheme, lu_select_kernel),
  // every panel and step unrolled so each register index is static.
  // The pivot key packs the value and the row: bits [RB, 32) hold
  // (|v|'s bits ≫ RB) + 1 (a 2^-(23-RB)-relative comparison, RB = log2 CAP),
  // bits [0, RB) hold CAP−1−row, so ONE unsigned max gives the largest |v|
  // and, among equal keys, the lowest row.  A row leaves the competition by
  // its key mask only: chosen rows keep being updated like the others (their
  // values are never read again — the panel end takes their multipliers and
  // trailing part before any later update reaches them), so a step is
  // straight-line code.  Every warp publishes its winner's whole panel (two
  // 16-byte stores).
  constexpr int RB = CAP <= 256 ? 8 : (CAP <= 512 ? 9 : 10);
#ifdef LU_NOM_LOAD_ONLY  // timing ablation: the loads without the elimination
  for (int j = tid; j < steps; j += kThreads) piv[j] = j;
  if (w[0][0] == 1.2345f && w[R - 1][LP - 1] == 2.5f) piv[0] = 1;
  if (false)
#endif
#ifndef LU_NOM_ROLLED
#define LU_NOM_ROLLED 1
#endif
#if LU_NOM_ROLLED
  // Panels as a rolled loop over a register window: the panel is always
  // w[·][0, 8) and its trailing columns w[·][8, LP); after each panel the
  // window shifts left by 8 columns.  Same operations in the same order as
  // the unrolled form below (the shifted-in tail holds zeros and gets zero
  // U12 columns), at 1/(LP/8) of its code: the unrolled kernel (~6k
  // instructions for LP = 24) stalled on instruction fetch ("no_instructions"
  // 44% of the leaf's samples, most of a 9-CTA tree level's).
#pragma unroll 1
  for (int pb = 0; pb < steps; pb += 8) {
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int j = pb + s;
      if (j >= steps) break;
      uint32_t key[R], best = 0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        key[q] = (((((__float_as_uint(w[q][s]) & 0x7FFFFFFFu) >> RB) + 1u) << RB) |
                  (uint32_t)(CAP - 1 - (tid * R + q))) & amask[q];
        best = max(best, key[q]);
      }
      const uint32_t mk = __reduce_max_sync(0xffffffffu, best);
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (key[q] == mk && mk != 0u) {  // the (unique) winning row of this warp
          float4* d = reinterpret_cast<float4*>(pbuf[j & 1][warp]);
          d[0] = make_float4(w[q][0], w[q][1], w[q][2], w[q][3]);
          d[1] = make_float4(w[q][4], w[q][5], w[q][6], w[q][7]);
        }
      if (lane == 0) slot[j & 1][warp] = mk;
      __syncthreads();
      const uint32_t kv = lane < kWarps ? slot[j & 1][lane] : 0u;
      const uint32_t gk = __reduce_max_sync(0xffffffffu, kv);
      const int p = (int)(CAP - 1 - (gk & (CAP - 1)));
      const float4* pr4 = reinterpret_cast<const float4*>(pbuf[j & 1][p / (32 * R)]);
      const float4 pa = pr4[0], pc = pr4[1];
      const float pr[8] = {pa.x, pa.y, pa.z, pa.w, pc.x, pc.y, pc.z, pc.w};
      float rc;  // MUFU reciprocal (nomination only needs ~1 ulp); tiny pivot ⇒ a zero column
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(pr[s]));
      const float uinv = fabsf(pr[s]) >= 0x1p-100f ? rc : 0.f;
      if (tid == 0) piv[j] = p;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (tid * R + q == p) {
          pstep[q] = s;
          amask[q] = 0u;
        }
        const float mult = w[q][s] * uinv;
        w[q][s] = mult;
#pragma unroll
        for (int t = s + 1; t < 8; ++t) w[q][t] = fmaf(-mult, pr[t], w[q][t]);
      }
    }
    if (pb + 8 >= steps || LP == 8) break;  // no later step reads the trailing columns
    const int nt = LP - pb - 8;             // real trailing columns
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (pstep[q] >= 0) {  // this panel's pivot rows: multipliers and trailing part
        const int sp = pstep[q];
#pragma unroll
        for (int t = 8; t < LP; ++t) traw[sp][t - 8] = w[q][t];
#pragma unroll
        for (int t = 0; t < 8; ++t) l11[sp][t] = t < sp ? w[q][t] : 0.f;
        pstep[q] = -1;
      }
    __syncthreads();
    if (tid < LP - 8) {  // U12 = L11⁻¹·(pivot rows' trailing part), one column per thread
      float u[8];
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        float v = traw[sp][tid];
#pragma unroll
        for (int s2 = 0; s2 < sp; ++s2) v = fmaf(-l11[sp][s2], u[s2], v);
        u[sp] = v;
        u12[sp][tid] = tid < nt ? v : 0.f;
      }
    }
    __syncthreads();
    // trailing update w[t] −= Σ_s w[s]·U12[s][t] (s ascending), two columns
    // per FFMA2, then the window moves to the next panel
#pragma unroll
    for (int q = 0; q < R; ++q) {
      float2 nm[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) nm[s] = make_float2(-w[q][s], -w[q][s]);
#pragma unroll
      for (int t = 8; t < LP; t += 4) {
        float2 v0 = make_float2(w[q][t], w[q][t + 1]), v1 = make_float2(w[q][t + 2], w[q][t + 3]);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const float4 u = *reinterpret_cast<const float4*>(&u12[s][t - 8]);
          v0 = ffma2(nm[s], make_float2(u.x, u.y), v0);
          v1 = ffma2(nm[s], make_float2(u.z, u.w), v1);
        }
        w[q][t - 8] = v0.x;
        w[q][t - 7] = v0.y;
        w[q][t - 6] = v1.x;
        w[q][t - 5] = v1.y;
      }
#pragma unroll
      for (int t = LP - 8; t < LP; ++t) w[q][t] = 0.f;
    }
  }
#else
#pragma unroll
  for (int P = 0; P < LP / 8; ++P) {
    const int pb = 8 * P;
    if (pb >= steps) break;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int j = pb + s;
      if (j >= steps) break;
      uint32_t key[R], best = 0;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        key[q] = (((((__float_as_uint(w[q][j]) & 0x7FFFFFFFu) >> RB) + 1u) << RB) |
                  (uint32_t)(CAP - 1 - (tid * R + q))) & amask[q];
        best = max(best, key[q]);
      }
      const uint32_t mk = __reduce_max_sync(0xffffffffu, best);
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (key[q] == mk && mk != 0u) {  // the (unique) winning row of this warp
          float4* d = reinterpret_cast<float4*>(pbuf[j & 1][warp]);
          d[0] = make_float4(w[q][pb], w[q][pb + 1], w[q][pb + 2], w[q][pb + 3]);
          d[1] = make_float4(w[q][pb + 4], w[q][pb + 5], w[q][pb + 6], w[q][pb + 7]);
        }
      if (lane == 0) slot[j & 1][warp] = mk;
      __syncthreads();
      const uint32_t kv = lane < kWarps ? slot[j & 1][lane] : 0u;
      const uint32_t gk = __reduce_max_sync(0xffffffffu, kv);
      const int p = (int)(CAP - 1 - (gk & (CAP - 1)));
      const float4* pr4 = reinterpret_cast<const float4*>(pbuf[j & 1][p / (32 * R)]);
      const float4 pa = pr4[0], pc = pr4[1];
      const float pr[8] = {pa.x, pa.y, pa.z, pa.w, pc.x, pc.y, pc.z, pc.w};
      float rc;  // MUFU reciprocal (nomination only needs ~1 ulp); tiny pivot ⇒ a zero column
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(pr[s]));
      const float uinv = fabsf(pr[s]) >= 0x1p-100f ? rc : 0.f;
      if (tid == 0) piv[j] = p;
#pragma unroll
      for (int q = 0; q < R; ++q) {
        if (tid * R + q == p) {
          pstep[q] = s;
          amask[q] = 0u;
        }
        const float mult = w[q][j] * uinv;
        w[q][j] = mult;
#pragma unroll
        for (int t = s + 1; t < 8; ++t) w[q][pb + t] = fmaf(-mult, pr[t], w[q][pb + t]);
      }
    }
    if (pb + 8 >= steps) break;  // no later step reads the trailing columns
    const int nt = LP - pb - 8;  // trailing columns (a constant after unrolling)
#pragma unroll
    for (int q = 0; q < R; ++q)
      if (pstep[q] >= 0) {  // this panel's pivot rows: multipliers and trailing part
        const int sp = pstep[q];
#pragma unroll
        for (int t = pb + 8; t < LP; ++t) traw[sp][t - pb - 8] = w[q][t];
#pragma unroll
        for (int t = 0; t < 8; ++t) l11[sp][t] = t < sp ? w[q][pb + t] : 0.f;
        pstep[q] = -1;
      }
    __syncthreads();
    if (tid < nt) {  // U12 = L11⁻¹·(pivot rows' trailing part), one column per thread
      float u[8];
#pragma unroll
      for (int sp = 0; sp < 8; ++sp) {
        float v = traw[sp][tid];
#pragma unroll
        for (int s2 = 0; s2 < sp; ++s2) v = fmaf(-l11[sp][s2], u[s2], v);
        u[sp] = v;
        u12[sp][tid] = v;
      }
    }
    __syncthreads();
    // trailing update w[t] −= Σ_s w[pb+s]·U12[s][t] (s ascending), two columns
    // per FFMA2
#pragma unroll
    for (int q = 0; q < R; ++q) {
      float2 nm[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) nm[s] = make_float2(-w[q][pb + s], -w[q][pb + s]);
#pragma unroll
      for (int t = pb + 8; t < LP; t += 4) {
        float2 v0 = make_float2(w[q][t], w[q][t + 1]), v1 = make_float2(w[q][t + 2], w[q][t + 3]);
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const float4 u = *reinterpret_cast<const float4*>(&u12[s][t - pb - 8]);
          v0 = ffma2(nm[s], make_float2(u.x, u.y), v0);
          v1 = ffma2(nm[s], make_float2(u.z, u.w), v1);
        }
        w[q][t] = v0.x;
        w[q][t + 1] = v0.y;
        w[q][t + 2] = v1.x;
        w[q][t + 3] = v1.y;
      }
    }
  }
#endif
  __syncthreads();
  for (int j = tid; j < l; j += kThreads) cand_out[blk * l + j] = j < steps ? ids[piv[j]] : -1;
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
                                       const int64_t* __restrict__ cand, const double* __restrict__ mu,
                                       double* __restrict__ rows_out, int64_t* __restrict__ gid) {
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int j = idx / l, t = idx - j * l;
    const int64_t r = cand[j];
    rows_out[idx] = r >= 0 ? Y[r * l + t] - (mu ? mu[t] : 0.0) : 0.0;
    if (t == 0) gid[j] = r >= 0 ? row0 + r : -1;
  }
}

int lp_of(int l) { return (l + 7) & ~7; }
int leaf_cap(int l) { return kThreads * leaf_rows_per_thread(lp_of(l)); }
int tree_cap(int l) { return kThreads * tree_rows_per_thread(lp_of(l)); }
// a tree group stacks G candidate sets of l rows into one CTA's rows
int group_for(int l) { return std::max(2, tree_cap(l) / l); }

template <int LP, int R>
void select_lpr(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
                int G, int64_t* cout, int final_, double* U, double* Lp, int64_t* piv, double* M,
                const double* rows_in, double* rows_out, const double* mu) {
  constexpr int CAP = SelCfg<LP, R>::kCap;
  // leaves that are not the last level run persistent with bulk-staged rows —
  // in the one-CTA-per-SM configurations (with two CTAs per SM the second one
  // already hides the row loads, and the 128-register cap has no room for
  // the staging state)
  constexpr bool kBulkOK = SelCfg<LP, R>::kMinBlocks == 1;
  const int bulk = kBulkOK && leaf == 1 && !final_ && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  const size_t smem = final_ ? (size_t)(LP * LP + (size_t)CAP * l) * 8 : bulk ? (size_t)CAP * l * 8 : 0;
  const void* fn = bulk ? (const void*)lu_select_kernel<LP, R, kBulkOK> : (const void*)lu_select_kernel<LP, R, false>;
  if (smem) ensure_smem(fn, (int)smem);
  if (bulk) {
    int occ = 0;
    RPCA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem));
    grid = (unsigned)std::min<int64_t>(grid, (int64_t)c.num_sms * std::max(1, occ));
  }
  if (bulk)
    lu_select_kernel<LP, R, kBulkOK><<<grid, kThreads, smem, c.stream>>>(Y, m, l, leaf, cin, n_in, G, cout, final_, U,
                                                                         Lp, piv, M, rows_in, rows_out, mu, bulk);
  else
    lu_select_kernel<LP, R, false><<<grid, kThreads, smem, c.stream>>>(Y, m, l, leaf, cin, n_in, G, cout, final_, U,
                                                                       Lp, piv, M, rows_in, rows_out, mu, 0);
}

template <int LP>
void select_lp(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
               int G, int64_t* cout, int final_, double* U, double* Lp, int64_t* piv, double* M,
               const double* rows_in, double* rows_out, const double* mu) {
  if (leaf == 1)
    select_lpr<LP, leaf_rows_per_thread(LP)>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, final_, U, Lp, piv, M,
                                             rows_in, rows_out, mu);
  else
    select_lpr<LP, tree_rows_per_thread(LP)>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, final_, U, Lp, piv, M,
                                             rows_in, rows_out, mu);
}

// M = U⁻¹ for l ≤ 32 in one warp (the last tournament level's U), lane j =
// column j of M in registers, U's rows broadcast from shared memory: the
// same sums in the same order as the column-serial loop of lu_select_kernel
// — a term goes to accumulator (t−i−1) mod 4 while it belongs to that loop's
// unrolled-by-4 part, else to a0 — so M is bitwise the same; there every
// term re-read its M[t][j] from shared memory (≈ 20k cycles at l = 22).
// Terms beyond j multiply M[t][j] = 0 and leave the sums unchanged.
template <int LP>
__global__ void __launch_bounds__(32) u_inverse_warp_kernel(const double* __restrict__ U, int l,
                                                            double* __restrict__ M) {
  __shared__ double Us[LP][LP + 1];
  __shared__ double udr[LP];
  const int j = threadIdx.x;  // one thread per column
#pragma unroll
  for (int i = 0; i < LP; ++i)
    if (j < LP) Us[i][j] = (i < l && j < l) ? U[i * l + j] : 0.0;
  if (j < LP) {
    const double uii = j < l ? U[j * l + j] : 0.0;
    udr[j] = uii != 0.0 ? 1.0 / uii : 0.0;
  }
  __syncwarp();
  double mc[LP];
#pragma unroll
  for (int i = LP - 1; i >= 0; --i) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int mainend = i + 4 * ((j - i) >> 2);  // last term of the unrolled part (j ≥ i)
#pragma unroll
    for (int t = i + 1; t < LP; ++t) {
      const double u = Us[i][t];
      const int k = (t - i - 1) & 3;
      if (k == 0) {
        a0 = fma(u, mc[t], a0);
      } else {  // branch-free: the choice differs across lanes
        const bool main_ = t <= mainend;
        const double x0 = fma(u, mc[t], a0);
        if (k == 1) {
          const double xk = fma(u, mc[t], a1);
          a1 = main_ ? xk : a1;
        } else if (k == 2) {
          const double xk = fma(u, mc[t], a2);
          a2 = main_ ? xk : a2;
        } else {
          const double xk = fma(u, mc[t], a3);
          a3 = main_ ? xk : a3;
        }
        a0 = main_ ? a0 : x0;
      }
    }
    mc[i] = (i < l && j < l && j >= i) ? ((i == j ? 1.0 : 0.0) - ((a0 + a1) + (a2 + a3))) * udr[i] : 0.0;
  }
  if (j < l)
#pragma unroll
    for (int i = 0; i < LP; ++i)
      if (i < l) M[i * l + j] = mc[i];
}

// M = U⁻¹ for 32 < l ≤ 64: two warps, thread j = column j, right-looking —
// as soon as M[t][j] is known it updates every row above it, acc_i +=
// U_it·M_tj (independent across i; U's column t broadcast from shared
// memory), so the dependence chain per row is one FMA and the scaling.  The
// column-serial order of u_inverse_warp_kernel would chain every term through
// one accumulator (68 µs at l = 52); here the sum for M[i][j] runs over t
// descending (deterministic; ≈ 1 ulp from the column-serial sums).
template <int LP>
__global__ void __launch_bounds__(64) u_inverse_rl_kernel(const double* __restrict__ U, int l,
                                                          double* __restrict__ M) {
  __shared__ double Us[LP][LP + 1];
  __shared__ double udr[LP];
  const int j = threadIdx.x;
#pragma unroll
  for (int i = 0; i < LP; ++i)
    if (j < LP) Us[i][j] = (i < l && j < l) ? U[i * l + j] : 0.0;
  if (j < LP) {
    const double uii = j < l ? U[j * l + j] : 0.0;
    udr[j] = uii != 0.0 ? 1.0 / uii : 0.0;
  }
  __syncthreads();
  double acc[LP];
#pragma unroll
  for (int i = 0; i < LP; ++i) acc[i] = 0.0;
#pragma unroll
  for (int t = LP - 1; t >= 0; --t) {
    const double mt = (t < l && j < l && j >= t) ? ((t == j ? 1.0 : 0.0) - acc[t]) * udr[t] : 0.0;
    if (t < l && j < l) M[t * l + j] = mt;
#pragma unroll
    for (int i = 0; i < t; ++i) acc[i] = fma(Us[i][t], mt, acc[i]);
  }
}

void select(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
            int G, int64_t* cout, int final_, double* U, double* Lp, int64_t* piv, double* M,
            const double* rows_in = nullptr, double* rows_out = nullptr, const double* mu = nullptr) {
#define RPCA_SEL(LPV)                                                                                      \
  case LPV:                                                                                                \
    select_lp<LPV>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, final_, U, Lp, piv, M, rows_in, rows_out, mu); \
    break;
  switch (lp_of(l)) {
    RPCA_SEL(8)
    RPCA_SEL(16)
    RPCA_SEL(24)
    RPCA_SEL(32)
    RPCA_SEL(40)
    RPCA_SEL(48)
    RPCA_SEL(56)
    RPCA_SEL(64)
    default: RPCA_REQUIRE(false, RPCA_E_SHAPE, "lu: l=%d > %d", l, kMaxL);
  }
#undef RPCA_SEL
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, leaf == 1 ? "lu_leaf" : "lu_tree");
  if (final_) {
    switch (lp_of(l)) {
      case 8: u_inverse_warp_kernel<8><<<1, 32, 0, c.stream>>>(U, l, M); break;
      case 16: u_inverse_warp_kernel<16><<<1, 32, 0, c.stream>>>(U, l, M); break;
      case 24: u_inverse_warp_kernel<24><<<1, 32, 0, c.stream>>>(U, l, M); break;
      case 32: u_inverse_warp_kernel<32><<<1, 32, 0, c.stream>>>(U, l, M); break;
      case 40: u_inverse_rl_kernel<40><<<1, 64, 0, c.stream>>>(U, l, M); break;
      case 48: u_inverse_rl_kernel<48><<<1, 64, 0, c.stream>>>(U, l, M); break;
      case 56: u_inverse_rl_kernel<56><<<1, 64, 0, c.stream>>>(U, l, M); break;
      default: u_inverse_rl_kernel<64><<<1, 64, 0, c.stream>>>(U, l, M); break;
    }
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "lu_tree");
  }
}

#ifndef LU_NOM_R32
#define LU_NOM_R32 2
#endif
constexpr int nominate_rows_per_thread(int LP) { return LP <= 16 ? 4 : (LP <= 32 ? LU_NOM_R32 : 1); }
int nominate_cap(int l) { return kThreads * nominate_rows_per_thread(lp_of(l)); }

template <int LP>
void nominate_lp(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin,
                 int64_t n_in, int G, int64_t* cout, const double* mu) {
  constexpr int R = nominate_rows_per_thread(LP);
  const int smem = kThreads * R * (l + 1) * 4;
  if constexpr (LP > 32 && LP < 64) {
    if (grid >= 2u * (unsigned)c.num_sms) {  // enough CTAs to fill three per SM
      ensure_smem((const void*)lu_nominate_kernel<LP, R, 3>, kThreads * R * (LP + 1) * 4);
      lu_nominate_kernel<LP, R, 3><<<grid, kThreads, smem, c.stream>>>(Y, m, l, leaf, cin, n_in, G, cout, mu);
      return;
    }
  }
  ensure_smem((const void*)lu_nominate_kernel<LP, R, 2>, kThreads * R * (LP + 1) * 4);
  lu_nominate_kernel<LP, R, 2><<<grid, kThreads, smem, c.stream>>>(Y, m, l, leaf, cin, n_in, G, cout, mu);
}

void nominate(Ctx& c, unsigned grid, const double* Y, int64_t m, int l, int leaf, const int64_t* cin, int64_t n_in,
              int G, int64_t* cout, const double* mu) {
  switch (lp_of(l)) {
    case 8: nominate_lp<8>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 16: nominate_lp<16>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 24: nominate_lp<24>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 32: nominate_lp<32>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 40: nominate_lp<40>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 48: nominate_lp<48>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 56: nominate_lp<56>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    case 64: nominate_lp<64>(c, grid, Y, m, l, leaf, cin, n_in, G, cout, mu); break;
    default: RPCA_REQUIRE(false, RPCA_E_SHAPE, "lu: l=%d > %d", l, kMaxL);
  }
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, leaf == 1 ? "lu_leaf" : "lu_tree");
}

bool lu_f64_nomination() {
  static const bool v = getenv("RPCA_LU_F64_LEAF") != nullptr;  // ablation: the round-1 fp64 nomination
  return v;
}

// Tournament over rows [0, m) of Y down to one candidate set; returns the set
// (l entries, local row indices, −1 padded).  If `finalize`, the last level
// (fp64 GEPP on the candidates' original rows) also writes U, Lp, piv and M;
// every other level nominates in fp32 (lu_nominate_kernel).
int64_t* tournament(Ctx& c, const double* Y, int64_t m, int l, bool finalize, double* U, double* Lp, int64_t* piv,
                    double* M, Arena& ar, const double* mu) {
  const bool f64 = lu_f64_nomination();
  const int G64 = group_for(l);
  const int Gn = f64 ? G64 : std::max(2, nominate_cap(l) / l);
  const int64_t leafcap = f64 ? leaf_cap(l) : nominate_cap(l);
  const int64_t nblk = std::max<int64_t>(1, cdiv(m, leafcap));
  int64_t* ca = ar.get<int64_t>(nblk * l);
  int64_t* cb = ar.get<int64_t>(nblk * l);
  if (m == 0) {
    RPCA_CUDA(cudaMemsetAsync(ca, 0xFF, sizeof(int64_t) * l, c.stream));  // no local rows: all −1
    return ca;
  }
  if (finalize && m <= leaf_cap(l)) {  // one block: the exact GEPP directly
    select(c, 1u, Y, m, l, 1, nullptr, 0, G64, ca, 1, U, Lp, piv, M, nullptr, nullptr, mu);
    return ca;
  }
  if (f64) select(c, (unsigned)nblk, Y, m, l, 1, nullptr, 0, G64, ca, 0, U, Lp, piv, M, nullptr, nullptr, mu);
  else nominate(c, (unsigned)nblk, Y, m, l, 1, nullptr, 0, Gn, ca, mu);
  int64_t n = nblk;
  for (;;) {
    const bool last = finalize && n <= G64;
    if (!last && n <= 1) break;
    const int G = last ? G64 : Gn;
    const int64_t ng = cdiv(n, G);
    if (last || f64) select(c, (unsigned)ng, Y, m, l, 0, ca, n, G, cb, last ? 1 : 0, U, Lp, piv, M, nullptr, nullptr, mu);
    else nominate(c, (unsigned)ng, Y, m, l, 0, ca, n, G, cb, mu);
    std::swap(ca, cb);
    n = ng;
    if (last) break;
  }
  return ca;
}

// L = Y·M on the fp64 tensor-core pass kernel (in place: every output row is
// written only after all of its own K-chunks were read), then the pivot rows
// this shard holds get their exact unit-lower rows
// cx_j = Σ_t mu_t·M_tj: (Y − 1·mu)·M = Y·M − 1·cx
__global__ void mu_times_m_kernel(const double* __restrict__ mu, const double* __restrict__ M, int l,
                                  double* __restrict__ cx) {
  const int j = threadIdx.x;
  if (j >= l) return;
  double s = 0.0;
  for (int t = 0; t < l; ++t) s += mu[t] * M[t * l + j];
  cx[j] = s;
}

void apply_l(Ctx& c, double* Y, int64_t m, int64_t row0, int l, const double* M, const double* Lp,
             const int64_t* piv, Arena& ar, const double* mu) {
  if (m > 0) {
    const size_t mark = ar.off;
    double* cx = nullptr;
    if (mu) {  // L = (Y − 1·mu)·M: the pending centring enters the epilogue
      cx = ar.get<double>(kMaxL);
      mu_times_m_kernel<<<1, 64, 0, c.stream>>>(mu, M, l, cx);
      RPCA_CHECK_LAUNCH();
      count_launch(c, 1, "misc");
    }
    TagScope ts(c, "lu_apply");
    dense_ax(c, DenseA{Y, RPCA_F64, m, l, l}, M, l, Y, ar, cx, true);  // M = U⁻¹ is upper triangular
    ar.off = mark;
  }
  pivot_rows_kernel<<<1, 256, 0, c.stream>>>(Y, m, row0, l, Lp, piv);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "lu_pivot_rows");
}

}  // namespace

size_t lu_ws_bytes(int64_t m, int l) {
  Sizer s;
  s.add<char>(ax_ws_bytes(DenseA{nullptr, RPCA_F64, m, l, l}, l) + 4096);
  const int64_t nblk = std::max<int64_t>(1, cdiv(m, 256));
  s.add<int64_t>(nblk * l);
  s.add<int64_t>(nblk * l);
  s.add<double>(4 * (size_t)l * l);
  s.add<int64_t>(l);
  s.add<double>((size_t)2 * kMaxL * (size_t)(kMaxL + 1) * 64 + 2 * kMaxL * kMaxL);  // sharded: gathered rows + ids
  s.add<double>(kMaxL);                                                                 // mu·M
  return s.total;
}

void lu_renorm(Ctx& c, double* Y, int64_t m, int l, double* U_out, int64_t* piv_out, Arena& ar, const double* mu) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL && m >= l, RPCA_E_SHAPE, "lu_renorm: need 1 ≤ l ≤ %d and m ≥ l", kMaxL);
  double* U = U_out ? U_out : ar.get<double>((size_t)l * l);
  double* Lp = ar.get<double>((size_t)l * l);
  int64_t* piv = ar.get<int64_t>(l);
  double* M = ar.get<double>((size_t)l * l);
  const size_t mark = ar.off;
  tournament(c, Y, m, l, true, U, Lp, piv, M, ar, mu);
  ar.off = mark;
  apply_l(c, Y, m, 0, l, M, Lp, piv, ar, mu);
  if (piv_out) RPCA_CUDA(cudaMemcpyAsync(piv_out, piv, sizeof(int64_t) * l, cudaMemcpyDeviceToDevice, c.stream));
}

// Row-sharded LU: every rank runs the tournament on its rows
// [row0, row0+m); the winners (l rows + their global ids) are all-gathered and
// every rank runs the final GEPP on the same P·l rows — identical U, pivots and
// M everywhere — then applies L = Y·M to its own rows.
void lu_renorm_sharded(Ctx& c, double* Y, int64_t m, int64_t row0, int l, double* U_out, Arena& ar,
                       const double* mu) {
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
  const int64_t* cand = tournament(c, Y, m, l, false, nullptr, nullptr, nullptr, nullptr, ar, mu);
  pack_candidates_kernel<<<1, 256, 0, c.stream>>>(Y, l, row0, cand, mu, rows_send, ids_send);
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
  apply_l(c, Y, m, row0, l, M, Lp, piv, ar, mu);
}

}  // namespace rpca
