// gram.cu — G = Xᵀ·Y for thin row-major blocks (rows × l, l ≤ 64) on the fp64
// tensor cores.  Used by the Cholesky-QR steps of the last renormalisation
// (cholqr.cu: the Grams LᵀL and Q1ᵀQ1 of PAPER.md:406-425's orthonormal Q) and
// by the Nyström B2 = QᵀB1.
//
// B200 design: persistent CTAs own contiguous ranges of 64-row tiles (fixed
// assignment ⇒ deterministic partials).  A tile of X (and of Y when Y ≠ X) is
// staged into shared memory with cp.async, double-buffered, at a row stride s
// ≡ 4 (mod 16) doubles so the DMMA fragment loads (row k = lane&3, column
// lane>>2) hit 16 distinct bank pairs per half-warp.  The 8×8 blocks of G
// (only bi ≤ bj when Y = X) are spread over the 8 warps; each k-step of 4 rows
// is one mma.m8n8k4.f64 per block.  Per-CTA partials are summed in ascending
// CTA order.  Per row: l·8 bytes (X only) and l² (or l²/2) fp64 MACs — HBM-
// bound for l ≲ 32, fp64-tensor-bound above.
#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kRows = 64;  // rows per tile
constexpr int kWarps = 8;

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

int stride_for(int LP) {
  int s = LP;
  while (s % 16 != 4) ++s;
  return s;
}

// stage rows [r0, r0+64) of X (l columns) into T (64 × s); zeros past rows /
// past l (the padded columns up to LP are read by the fragments).  vec: l even
// and X 16-byte aligned — 16-byte copies (s is even, so T's rows stay aligned)
__device__ __forceinline__ void stage(double* T, const double* __restrict__ X, int64_t rows, int l, int LP, int s,
                                      int64_t r0, bool vec) {
  const int nr = (int)imin64(kRows, rows - r0);
  if (vec) {
    const int hp = LP / 2;
    for (int idx = threadIdx.x; idx < kRows * hp; idx += blockDim.x) {
      const int r = idx / hp, cc = 2 * (idx - r * hp);
      double* d = T + r * s + cc;
      if (r < nr && cc < l) cp_async16(d, X + (r0 + r) * l + cc);
      else d[0] = d[1] = 0.0;
    }
    return;
  }
  for (int idx = threadIdx.x; idx < kRows * LP; idx += blockDim.x) {
    const int r = idx / LP, cc = idx - r * LP;
    double* d = T + r * s + cc;
    if (r < nr && cc < l) cp_async8(d, X + (r0 + r) * l + cc);
    else *d = 0.0;
  }
}

__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  if (n <= 0) cp_async_wait<0>();
  else if (n == 1) cp_async_wait<1>();
  else cp_async_wait<2>();
}

// The 8×8 blocks of G (bi ≤ bj when Y = X) are split over BG warp groups
// (block q·BG + g to group g) and the 16 four-row k-steps of a tile over the
// KS = 8/BG warps of a group, so every warp issues the same number of DMMAs
// and one fragment load per block row serves all of its blocks.
template <int NB, bool SAME>
struct GramCfg {
  static constexpr int kPairs = SAME ? NB * (NB + 1) / 2 : NB * NB;
  static constexpr int BG = kPairs <= 18 ? 1 : (kPairs <= 36 ? 2 : 4);
  static constexpr int KS = kWarps / BG;
  static constexpr int kAcc = (kPairs + BG - 1) / BG;
};

template <int NB, bool SAME>
size_t gram_red_bytes() {
  using C = GramCfg<NB, SAME>;
  return (size_t)C::KS * C::kPairs * 64 * sizeof(double);
}

template <int NB, bool SAME>
__global__ void __launch_bounds__(256) gram_dmma_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                                        int64_t rows, int l, int s, int64_t ntiles, int nst, int vec,
                                                        double* __restrict__ part) {
  using C = GramCfg<NB, SAME>;
  constexpr int LP = 8 * NB;
  extern __shared__ __align__(16) double sm[];
  const int tile_elems = kRows * s;
  const int buf_elems = (SAME ? 1 : 2) * tile_elems;  // X tile, then Y tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = warp % C::BG, ksl = warp / C::BG;
  const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  auto stage_tile = [&](int b, int64_t t) {
    stage(sm + b * buf_elems, X, rows, l, LP, s, t * kRows, vec);
    if (!SAME) stage(sm + b * buf_elems + tile_elems, Y, rows, l, LP, s, t * kRows, vec);
  };
  double acc[C::kAcc][2];
#pragma unroll
  for (int q = 0; q < C::kAcc; ++q) acc[q][0] = acc[q][1] = 0.0;

  // ring of nst tiles: tile t's copy group is complete once at most nst − 2
  // younger groups are pending (one group is committed per tile, empty or not)
  for (int i = 0; i < nst - 1; ++i) {
    if (t0 + i < t1) stage_tile(i, t0 + i);
    cp_async_commit();
  }
  const int kr = lane & 3, kc = lane >> 2;
  for (int64_t t = t0; t < t1; ++t) {
    const int b = (int)((t - t0) % nst);
    cp_async_wait_dyn(nst - 2);
    __syncthreads();  // tile t visible; every warp is done with tile t − 1's buffer
    if (t + nst - 1 < t1) stage_tile((b + nst - 1) % nst, t + nst - 1);
    cp_async_commit();
    const double* xs = sm + b * buf_elems;
    const double* ys = SAME ? xs : xs + tile_elems;
#pragma unroll
    for (int kk = 0; kk < 16 / C::KS; ++kk) {
      const int k4 = 4 * (ksl + C::KS * kk);
      const double* xr = xs + (k4 + kr) * s + kc;
      const double* yr = ys + (k4 + kr) * s + kc;
      double fx[NB], fy[NB];
#pragma unroll
      for (int a = 0; a < NB; ++a) {
        fx[a] = xr[a * 8];
        fy[a] = SAME ? fx[a] : yr[a * 8];
      }
      int idx = 0;
#pragma unroll
      for (int a = 0; a < NB; ++a)
#pragma unroll
        for (int bb = SAME ? a : 0; bb < NB; ++bb, ++idx)
          if (idx % C::BG == g) dmma(acc[idx / C::BG], fx[a], fy[bb]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // fixed-order sum of the KS k-slices: red[(ksl·kPairs + p)·64 + lane·2 + e]
  double* red = sm;
#pragma unroll
  for (int q = 0; q < C::kAcc; ++q) {
    const int p = q * C::BG + g;
    if (p < C::kPairs) {
      red[(ksl * C::kPairs + p) * 64 + lane * 2] = acc[q][0];
      red[(ksl * C::kPairs + p) * 64 + lane * 2 + 1] = acc[q][1];
    }
  }
  __syncthreads();
  // partial G of this CTA (d = {D[kc][2kr], D[kc][2kr+1]}); mirrored when Y = X
  double* G = part + (int64_t)blockIdx.x * l * l;
  for (int idx = threadIdx.x; idx < C::kPairs * 64; idx += blockDim.x) {
    const int p = idx >> 6, ln = (idx >> 1) & 31, e = idx & 1;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < C::KS; ++k) v += red[(k * C::kPairs + p) * 64 + ln * 2 + e];
    int bi, bj;
    if (SAME) {  // row-major upper triangle
      int a = 0, rem = p;
      while (rem >= NB - a) { rem -= NB - a; ++a; }
      bi = a;
      bj = a + rem;
    } else {
      bi = p / NB;
      bj = p % NB;
    }
    const int i = bi * 8 + (ln >> 2), j = bj * 8 + 2 * (ln & 3) + e;
    if (i < l && j < l) {
      G[i * l + j] = v;
      if (SAME && bi != bj) G[j * l + i] = v;
    }
  }
}

// v[j] = Σ_b part[b][j]: 32 entries per CTA, the 8 warps take partials
// b ≡ warp (mod 8) in ascending order, then warp 0 adds the 8 sums in order
__global__ void sum_parts_kernel(const double* __restrict__ part, int64_t nparts, int w, double* __restrict__ v) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (j < w) {
    int64_t b = warp;
    for (; b + 56 < nparts; b += 64) {  // eight loads in flight, added in the same order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(b + 8 * u) * w + j];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; b < nparts; b += 8) s += part[b * w + j];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && j < w) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    v[j] = t;
  }
}

int gram_ctas(Ctx& c, int64_t rows) {
  const int64_t ntiles = std::max<int64_t>(1, cdiv(rows, kRows));
  return (int)std::min<int64_t>(ntiles, (int64_t)c.num_sms * 2);
}

template <int NB, bool SAME>
void launch_gram_nb(Ctx& c, const double* X, const double* Y, int64_t rows, int l, int s, int64_t ntiles, int& grid,
                    double* part) {
  const size_t buf = (size_t)(SAME ? 1 : 2) * kRows * s * sizeof(double);
  // deepest ring (≤ 4 tiles) that leaves two CTAs per SM, else one
  int nst = 4;
  while (nst > 2 && nst * buf > 110 * 1024) --nst;
  if (nst == 2 && 3 * buf <= 220 * 1024) nst = 3;
  const size_t smem = std::max(nst * buf, gram_red_bytes<NB, SAME>());
  const void* fn = (const void*)gram_dmma_kernel<NB, SAME>;
  ensure_smem(fn, (int)smem);
  int occ = 1;
  RPCA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
  grid = (int)std::min<int64_t>(grid, (int64_t)c.num_sms * std::max(1, occ));  // one wave: fixed tile ranges
  const int vec = (l % 2 == 0) && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  gram_dmma_kernel<NB, SAME><<<grid, 256, smem, c.stream>>>(X, Y, rows, l, s, ntiles, nst, vec, part);
}

// the partial count is returned through `grid` (≤ gram_ctas)
void launch_gram(Ctx& c, const double* X, const double* Y, int64_t rows, int l, int LP, int s, int64_t ntiles,
                 int& grid, double* part) {
  const bool same = X == Y;
#define RPCA_GRAM(NBV)                                                                            \
  case NBV:                                                                                       \
    if (same) launch_gram_nb<NBV, true>(c, X, Y, rows, l, s, ntiles, grid, part);                 \
    else launch_gram_nb<NBV, false>(c, X, Y, rows, l, s, ntiles, grid, part);                     \
    break;
  switch (LP / 8) {
    RPCA_GRAM(1)
    RPCA_GRAM(2)
    RPCA_GRAM(3)
    RPCA_GRAM(4)
    RPCA_GRAM(5)
    RPCA_GRAM(6)
    RPCA_GRAM(7)
    RPCA_GRAM(8)
    default: RPCA_REQUIRE(false, RPCA_E_SHAPE, "gram: l=%d", l);
  }
#undef RPCA_GRAM
}

}  // namespace

size_t gram_ws_bytes(Ctx& c, int64_t rows, int l) {
  Sizer s;
  s.add<double>((size_t)gram_ctas(c, rows) * l * l);
  return s.total;
}

void gram(Ctx& c, const double* X, const double* Y, int64_t rows, int l, double* G, Arena& ar) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "gram: l out of range");
  if (rows <= 0) {
    RPCA_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * l * l, c.stream));
    return;
  }
  const int LP = (l + 7) / 8 * 8, s = stride_for(LP);
  const int64_t ntiles = cdiv(rows, kRows);
  int grid = gram_ctas(c, rows);
  double* part = ar.get<double>((size_t)grid * l * l);
  launch_gram(c, X, Y, rows, l, LP, s, ntiles, grid, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "gram");
  sum_parts_kernel<<<(unsigned)cdiv(l * l, 32), 256, 0, c.stream>>>(part, grid, l * l, G);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "gram_sum");
}

}  // namespace rpca
