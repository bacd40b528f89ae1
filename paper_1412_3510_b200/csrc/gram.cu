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

// stage rows [r0, r0+64) of X (l columns) into T (128 × s); zeros past rows /
// past l (the padded columns up to LP are read by the fragments)
__device__ __forceinline__ void stage(double* T, const double* __restrict__ X, int64_t rows, int l, int LP, int s,
                                      int64_t r0) {
  const int nr = (int)imin64(kRows, rows - r0);
  for (int idx = threadIdx.x; idx < kRows * LP; idx += blockDim.x) {
    const int r = idx / LP, cc = idx - r * LP;
    double* d = T + r * s + cc;
    if (r < nr && cc < l) cp_async8(d, X + (r0 + r) * l + cc);
    else *d = 0.0;
  }
}

template <int NB>
__global__ void __launch_bounds__(256) gram_dmma_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                                        int64_t rows, int l, int s, int64_t ntiles,
                                                        double* __restrict__ part) {
  constexpr int LP = 8 * NB;
  constexpr int kMaxPairs = (NB * NB + kWarps - 1) / kWarps;
  extern __shared__ double sm[];
  const bool same = (X == Y);
  const int tile_elems = kRows * s;
  double* ybase = same ? sm : sm + 2 * tile_elems;  // buffers b at +b·tile_elems
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;

  // this warp's blocks of G: pairs p = warp, warp+8, … of the (bi, bj) list
  const int npairs = same ? NB * (NB + 1) / 2 : NB * NB;
  int bi[kMaxPairs], bj[kMaxPairs];
  int np = 0;
#pragma unroll
  for (int q = 0; q < kMaxPairs; ++q) {
    const int p = warp + q * kWarps;
    bi[q] = bj[q] = 0;
    if (p < npairs) {
      ++np;
      if (same) {  // row-major upper triangle
        int a = 0, rem = p;
        while (rem >= NB - a) { rem -= NB - a; ++a; }
        bi[q] = a;
        bj[q] = a + rem;
      } else {
        bi[q] = p / NB;
        bj[q] = p % NB;
      }
    }
  }
  double acc[kMaxPairs][2];
#pragma unroll
  for (int q = 0; q < kMaxPairs; ++q) acc[q][0] = acc[q][1] = 0.0;

  if (t0 < t1) {
    stage(sm, X, rows, l, LP, s, t0 * kRows);
    if (!same) stage(ybase, Y, rows, l, LP, s, t0 * kRows);
    cp_async_commit();
  }
  const int kr = lane & 3, kc = lane >> 2;
  for (int64_t t = t0; t < t1; ++t) {
    const int b = (int)((t - t0) & 1);
    if (t + 1 < t1) {
      stage(sm + (b ^ 1) * tile_elems, X, rows, l, LP, s, (t + 1) * kRows);
      if (!same) stage(ybase + (b ^ 1) * tile_elems, Y, rows, l, LP, s, (t + 1) * kRows);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xs = sm + b * tile_elems;
    const double* ys = ybase + b * tile_elems;
#pragma unroll 4
    for (int k4 = 0; k4 < kRows; k4 += 4) {
      const double* xr = xs + (k4 + kr) * s + kc;
      const double* yr = ys + (k4 + kr) * s + kc;
#pragma unroll
      for (int q = 0; q < kMaxPairs; ++q)
        if (q < np) dmma(acc[q], xr[bi[q] * 8], yr[bj[q] * 8]);
    }
    __syncthreads();
  }
  // partial G of this CTA (d = {D[kc][2kr], D[kc][2kr+1]}); mirrored when Y = X
  double* G = part + (int64_t)blockIdx.x * l * l;
#pragma unroll
  for (int q = 0; q < kMaxPairs; ++q) {
    if (q >= np) continue;
    const int i = bi[q] * 8 + kc;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = bj[q] * 8 + 2 * kr + e;
      if (i < l && j < l) {
        G[i * l + j] = acc[q][e];
        if (same && bi[q] != bj[q]) G[j * l + i] = acc[q][e];
      }
    }
  }
  (void)LP;
}

// v[j] = Σ_b part[b][j]: 32 entries per CTA, the 8 warps take partials
// b ≡ warp (mod 8) in ascending order, then warp 0 adds the 8 sums in order
__global__ void sum_parts_kernel(const double* __restrict__ part, int64_t nparts, int w, double* __restrict__ v) {
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (j < w)
    for (int64_t b = warp; b < nparts; b += 8) s += part[b * w + j];
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
  const int grid = gram_ctas(c, rows);
  double* part = ar.get<double>((size_t)grid * l * l);
  const size_t smem = (size_t)(X == Y ? 2 : 4) * kRows * s * sizeof(double);
#define RPCA_GRAM(NBV)                                                                                    \
  case NBV:                                                                                               \
    ensure_smem((const void*)gram_dmma_kernel<NBV>, 4 * kRows * 68 * 8);                                  \
    gram_dmma_kernel<NBV><<<grid, 256, smem, c.stream>>>(X, Y, rows, l, s, ntiles, part);                 \
    break;
  switch (LP / 8) {
    RPCA_GRAM(1)
    RPCA_GRAM(2)
    RPCA_GRAM(3)
    RPCA_GRAM(4)
    RPCA_GRAM(5)
    RPCA_GRAM(6)
    RPCA_GRAM(7)
    default: ensure_smem((const void*)gram_dmma_kernel<8>, 4 * kRows * 68 * 8);
      gram_dmma_kernel<8><<<grid, 256, smem, c.stream>>>(X, Y, rows, l, s, ntiles, part);
      break;
  }
#undef RPCA_GRAM
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "gram");
  sum_parts_kernel<<<(unsigned)cdiv(l * l, 32), 256, 0, c.stream>>>(part, grid, l * l, G);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "gram_sum");
}

}  // namespace rpca
