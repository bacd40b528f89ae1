// csr.cu — §8(a) row a9: sparse A in CSR.  PAPER.md:427-435 (§5): "A little
// care in the implementation ensures that the same code can efficiently handle
// both dense and sparse matrices" — A is applied as A*Q, its adjoint as
// (Q'*A)' and the centring as a rank-1 correction, so the sparsity is never
// destroyed.
//
// B200 design:
//   * A·X (X n×l row-major): one warp per row of A; lane j owns columns j and
//     j+32 of the output row, so every nonzero gathers one contiguous 8·l-byte
//     row of X (coalesced); the row's (colind, value) pairs are loaded 32 at a
//     time by the lanes and broadcast with shuffles.  Gather-bound: the bytes
//     are CSR + nnz·8·l (X rows, partly L2-resident) + m·8·l.
//   * Aᵀ·Y: the same kernel on CSR(Aᵀ).  The transpose is built on the device
//     by a STABLE radix sort of the column indices (entry order inside a column
//     = ascending row), so every Aᵀ·Y sum runs over rows in ascending order —
//     deterministic, no float atomics.  It is cached on the context, keyed by
//     the CSR pointers and shape (rpca_ctx_clear_cache drops it).
//   * column means: per-column sums over CSR(Aᵀ) (ascending row order) / m.
#include <cub/device/device_radix_sort.cuh>

#include <vector>

#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 256;

// lane-owned output columns (lane, lane+32) of Σ_{t0 ≤ t < t1} vals[t]·X[colind[t]]
template <class T>
__device__ __forceinline__ void row_dot(const int32_t* __restrict__ colind, const T* __restrict__ vals, int64_t t0,
                                        int64_t t1, const double* __restrict__ X, int l, int lane, double& a0,
                                        double& a1, double& vsum) {
  for (int64_t tb = t0; tb < t1; tb += 32) {
    const int cnt = (int)imin64(32, t1 - tb);
    int myc = 0;
    double myv = 0.0;
    if (lane < cnt) {
      myc = colind[tb + lane];
      myv = static_cast<double>(vals[tb + lane]);
    }
    vsum += myv;  // per-lane partial Σ vals (for a centred operand)
    int k = 0;
    for (; k + 4 <= cnt; k += 4) {  // four gathers in flight
      const int c0 = __shfl_sync(0xffffffffu, myc, k), c1 = __shfl_sync(0xffffffffu, myc, k + 1);
      const int c2 = __shfl_sync(0xffffffffu, myc, k + 2), c3 = __shfl_sync(0xffffffffu, myc, k + 3);
      const double v0 = __shfl_sync(0xffffffffu, myv, k), v1 = __shfl_sync(0xffffffffu, myv, k + 1);
      const double v2 = __shfl_sync(0xffffffffu, myv, k + 2), v3 = __shfl_sync(0xffffffffu, myv, k + 3);
      if (lane < l) {
        const double x0 = X[(int64_t)c0 * l + lane], x1 = X[(int64_t)c1 * l + lane];
        const double x2 = X[(int64_t)c2 * l + lane], x3 = X[(int64_t)c3 * l + lane];
        a0 += v0 * x0;
        a0 += v1 * x1;
        a0 += v2 * x2;
        a0 += v3 * x3;
      }
      if (lane + 32 < l) {
        const double x0 = X[(int64_t)c0 * l + lane + 32], x1 = X[(int64_t)c1 * l + lane + 32];
        const double x2 = X[(int64_t)c2 * l + lane + 32], x3 = X[(int64_t)c3 * l + lane + 32];
        a1 += v0 * x0;
        a1 += v1 * x1;
        a1 += v2 * x2;
        a1 += v3 * x3;
      }
    }
    for (; k < cnt; ++k) {
      const int cc = __shfl_sync(0xffffffffu, myc, k);
      const double vv = __shfl_sync(0xffffffffu, myv, k);
      if (lane < l) a0 += vv * X[(int64_t)cc * l + lane];
      if (lane + 32 < l) a1 += vv * X[(int64_t)cc * l + lane + 32];
    }
  }
}

// warp per row; rows with more than `heavy` nonzeros are left to the chunk kernels
template <class T>
__global__ void __launch_bounds__(kThreads) csr_spmm_kernel(const int64_t* __restrict__ rowptr,
                                                            const int32_t* __restrict__ colind,
                                                            const T* __restrict__ vals, int64_t rows,
                                                            const double* __restrict__ X, int l, int64_t heavy,
                                                            const double* __restrict__ xmean,
                                                            double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t i = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); i < rows; i += warps) {
    const int64_t t0 = rowptr[i], t1 = rowptr[i + 1];
    if (t1 - t0 > heavy) continue;
    double a0 = 0.0, a1 = 0.0, vs = 0.0;
    row_dot(colind, vals, t0, t1, X, l, lane, a0, a1, vs);
    if (xmean) {  // Σ v·(x − x̄) = Σ v·x − x̄·Σ v
      vs = warp_sum(vs);
      if (lane < l) a0 -= xmean[lane] * vs;
      if (lane + 32 < l) a1 -= xmean[lane + 32] * vs;
    }
    if (lane < l) Y[i * l + lane] = a0;
    if (lane + 32 < l) Y[i * l + lane + 32] = a1;
  }
}

// W lanes per row (W = 16 or 8) for l ≤ 2W·… even, l ≤ 32: C5's A·X has ~10
// nonzeros per row, where a warp per row leaves most of the memory
// parallelism unused.  Sub-lane s owns columns C·s … C·s+C−1 (C = 32/W, one
// or two 16-byte gathers per nonzero), eight nonzeros in flight per row,
// 32/W rows per warp.  Same summation order per output as csr_spmm_kernel
// (ascending t).
#ifndef CSR_PAIR_MINB
#define CSR_PAIR_MINB 5  // 5 CTAs per SM (≤ 51 registers): C5 A·X −5%, Aᵀ·Y −2% against 4 (64 registers)
#endif
#ifndef CSR_PAIR_B
#define CSR_PAIR_B 8
#endif
// Short rows (avg < 32 nonzeros: C5's A·X) take B = 4 gathers per batch at 6
// CTAs per SM (A·X −3.5% against 8 at 5, interleaved A/B; long rows, C5's
// Aᵀ·Y, unchanged).  The batch size does not change the order of the sums.
template <class T, int W, int B = CSR_PAIR_B, int MINB = CSR_PAIR_MINB>
__global__ void __launch_bounds__(kThreads, MINB) csr_spmm_pair_kernel(const int64_t* __restrict__ rowptr,
                                                                 const int32_t* __restrict__ colind,
                                                                 const T* __restrict__ vals, int64_t rows,
                                                                 const double* __restrict__ X, int l, int64_t heavy,
                                                                 const double* __restrict__ xmean,
                                                                 double* __restrict__ Y) {
  constexpr int C = 32 / W;  // columns per sub-lane (2 or 4)
  const int lane = threadIdx.x & 31, grp = lane / W, s = lane % W;
  const unsigned hm = (W == 32 ? 0xFFFFFFFFu : ((1u << W) - 1u)) << (W * grp);
  const bool act = C * s < l;
  const int64_t stride = (int64_t)gridDim.x * (kThreads / W);
  for (int64_t i = ((int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5)) * (32 / W) + grp; i < rows;
       i += stride) {
    const int64_t t0 = rowptr[i], t1 = rowptr[i + 1];
    if (t1 - t0 > heavy) continue;
    double a[C];
#pragma unroll
    for (int q = 0; q < C; ++q) a[q] = 0.0;
    double vs = 0.0;
    for (int64_t tb = t0; tb < t1; tb += W) {
      const int cnt = (int)imin64(W, t1 - tb);
      int myc = 0;
      double myv = 0.0;
      if (s < cnt) {
        myc = colind[tb + s];
        myv = static_cast<double>(vals[tb + s]);
      }
      vs += myv;
      int k = 0;
      for (; k + B <= cnt; k += B) {
        int c[B];
        double v[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          c[u] = __shfl_sync(hm, myc, k + u, W);
          v[u] = __shfl_sync(hm, myv, k + u, W);
        }
        if (act) {
          double2 x[B][C / 2];
#pragma unroll
          for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < C / 2; ++h)
              x[u][h] = *reinterpret_cast<const double2*>(X + (int64_t)c[u] * l + C * s + 2 * h);
#pragma unroll
          for (int u = 0; u < B; ++u)
#pragma unroll
            for (int h = 0; h < C / 2; ++h) {
              a[2 * h] += v[u] * x[u][h].x;
              a[2 * h + 1] += v[u] * x[u][h].y;
            }
        }
      }
      for (; k < cnt; ++k) {
        const int cc = __shfl_sync(hm, myc, k, W);
        const double vv = __shfl_sync(hm, myv, k, W);
        if (act)
#pragma unroll
          for (int h = 0; h < C / 2; ++h) {
            const double2 x = *reinterpret_cast<const double2*>(X + (int64_t)cc * l + C * s + 2 * h);
            a[2 * h] += vv * x.x;
            a[2 * h + 1] += vv * x.y;
          }
      }
    }
    if (xmean) {  // Σ v·(x − x̄) = Σ v·x − x̄·Σ v
#pragma unroll
      for (int o = W / 2; o > 0; o >>= 1) vs += __shfl_xor_sync(hm, vs, o, W);
      if (act)
#pragma unroll
        for (int q = 0; q < C; ++q) a[q] -= xmean[C * s + q] * vs;
    }
    if (act)
#pragma unroll
      for (int h = 0; h < C / 2; ++h)
        *reinterpret_cast<double2*>(Y + i * l + C * s + 2 * h) = make_double2(a[2 * h], a[2 * h + 1]);
  }
}

// warp per chunk of a heavy row → its partial row
template <class T>
__global__ void __launch_bounds__(kThreads) csr_chunk_kernel(const int32_t* __restrict__ colind,
                                                             const T* __restrict__ vals,
                                                             const int64_t* __restrict__ hc, int64_t nhc,
                                                             const double* __restrict__ X, int l,
                                                             const double* __restrict__ xmean,
                                                             double* __restrict__ hpart) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t c = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); c < nhc; c += warps) {
    double a0 = 0.0, a1 = 0.0, vs = 0.0;
    row_dot(colind, vals, hc[3 * c + 1], hc[3 * c + 2], X, l, lane, a0, a1, vs);
    if (xmean) {
      vs = warp_sum(vs);
      if (lane < l) a0 -= xmean[lane] * vs;
      if (lane + 32 < l) a1 -= xmean[lane + 32] * vs;
    }
    hpart[c * kMaxL + lane] = a0;
    hpart[c * kMaxL + lane + 32] = a1;
  }
}

// warp per heavy row: Y[row] = Σ of its chunks' partials, ascending chunk order
__global__ void csr_heavy_reduce_kernel(const int64_t* __restrict__ hr, int64_t nhr,
                                        const double* __restrict__ hpart, int l, double* __restrict__ Y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t k = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); k < nhr; k += warps) {
    const int64_t row = hr[2 * k], c0 = hr[2 * k + 1], c1 = hr[2 * k + 3];
    double a0 = 0.0, a1 = 0.0;
    for (int64_t c = c0; c < c1; ++c) {
      a0 += hpart[c * kMaxL + lane];
      a1 += hpart[c * kMaxL + lane + 32];
    }
    if (lane < l) Y[row * l + lane] = a0;
    if (lane + 32 < l) Y[row * l + lane + 32] = a1;
  }
}

__global__ void row_of_entry_kernel(const int64_t* __restrict__ rowptr, int64_t rows, int32_t* __restrict__ rowidx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < rows; i += warps)
    for (int64_t t = rowptr[i] + lane; t < rowptr[i + 1]; t += 32) rowidx[t] = (int32_t)i;
}

__global__ void iota_kernel(int64_t n, int64_t* __restrict__ v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

template <class T>
__global__ void permute_kernel(const int64_t* __restrict__ perm, const int32_t* __restrict__ rowidx,
                               const T* __restrict__ vals, int64_t nnz, int32_t* __restrict__ trow,
                               T* __restrict__ tvals) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = perm[p];
    trow[p] = rowidx[t];
    tvals[p] = vals[t];
  }
}

// colptr[c] = first position of column c in the sorted keys (lower bound)
__global__ void colptr_kernel(const int32_t* __restrict__ skeys, int64_t nnz, int64_t n, int64_t* __restrict__ colptr) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= n; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    colptr[c] = lo;
  }
}

template <class T>
__global__ void csr_rowsum_kernel(const int64_t* __restrict__ ptr, const T* __restrict__ v, int64_t rows,
                                  double scale, double* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t t = ptr[r]; t < ptr[r + 1]; ++t) s += static_cast<double>(v[t]);
    out[r] = s * scale;
  }
}

unsigned grid_cap(Ctx& c, int64_t work, int per) {
  int64_t b = cdiv(work, per);
  b = std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)c.num_sms * 32));
  return (unsigned)b;
}

}  // namespace

void csr_spmm(Ctx& c, const CsrA& A, const double* X, int l, double* Y, const double* xmean) {
  csr_spmm_rows(c, A, 0, A.rows, X, l, Y, xmean);
  csr_spmm_heavy(c, A, X, l, Y, xmean);
}

// rows [r0, r1) of A·X, heavy rows (> kHeavyNnz nonzeros, when A has a plan) excluded
void csr_spmm_rows(Ctx& c, const CsrA& Afull, int64_t r0, int64_t r1, const double* X, int l, double* Yfull,
                   const double* xmean) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "l out of range");
  if (r1 <= r0) return;
  CsrA A = Afull;  // the row range as a CSR of its own (row pointers stay absolute)
  A.ptr = Afull.ptr + r0;
  A.rows = r1 - r0;
  double* Y = Yfull + r0 * l;
  const unsigned grid = grid_cap(c, A.rows, kThreads / 32);
  const int64_t heavy = A.nhc ? kHeavyNnz : INT64_MAX;
  prof_pre(c);
#ifndef CSR_LANES
#define CSR_LANES 16
#endif
  // lanes per row: 16 × 2 columns (measured best on C5; 8 × 4 with CSR_LANES=8)
  const bool al = (reinterpret_cast<uintptr_t>(X) & 15) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  const int avg = (int)std::min<int64_t>(1 << 20, A.nnz / std::max<int64_t>(1, A.rows));
  const int W = (CSR_LANES == 8 && l % 4 == 0 && avg < 64) ? 8 : 16;
  const bool pair = al && l % 2 == 0 && l <= 32;
  if (pair && W == 8) {
    const unsigned gp = grid_cap(c, A.rows, kThreads / 8);
    if (A.dtype == RPCA_F64)
      csr_spmm_pair_kernel<double, 8><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const double*)A.vals, A.rows, X,
                                                                     l, heavy, xmean, Y);
    else
      csr_spmm_pair_kernel<float, 8><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const float*)A.vals, A.rows, X, l,
                                                                    heavy, xmean, Y);
  } else if (pair && avg < 32) {
    const unsigned gp = grid_cap(c, A.rows, kThreads / 16);
    if (A.dtype == RPCA_F64)
      csr_spmm_pair_kernel<double, 16, 4, 6><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const double*)A.vals, A.rows,
                                                                            X, l, heavy, xmean, Y);
    else
      csr_spmm_pair_kernel<float, 16, 4, 6><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const float*)A.vals, A.rows,
                                                                           X, l, heavy, xmean, Y);
  } else if (pair) {
    const unsigned gp = grid_cap(c, A.rows, kThreads / 16);
    if (A.dtype == RPCA_F64)
      csr_spmm_pair_kernel<double, 16><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const double*)A.vals, A.rows, X,
                                                                      l, heavy, xmean, Y);
    else
      csr_spmm_pair_kernel<float, 16><<<gp, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const float*)A.vals, A.rows, X,
                                                                     l, heavy, xmean, Y);
  } else if (A.dtype == RPCA_F64)
    csr_spmm_kernel<double><<<grid, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const double*)A.vals, A.rows, X, l, heavy,
                                                             xmean, Y);
  else
    csr_spmm_kernel<float><<<grid, kThreads, 0, c.stream>>>(A.ptr, A.idx, (const float*)A.vals, A.rows, X, l, heavy,
                                                            xmean, Y);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "csr_spmm");
}

// the heavy rows of A·X: one warp per 4096-nonzero chunk, chunks summed in order
void csr_spmm_heavy(Ctx& c, const CsrA& A, const double* X, int l, double* Y, const double* xmean) {
  if (A.nhc) {
    const unsigned g2 = grid_cap(c, A.nhc, kThreads / 32);
    if (A.dtype == RPCA_F64)
      csr_chunk_kernel<double><<<g2, kThreads, 0, c.stream>>>(A.idx, (const double*)A.vals, A.hc, A.nhc, X, l,
                                                              xmean, A.hpart);
    else
      csr_chunk_kernel<float><<<g2, kThreads, 0, c.stream>>>(A.idx, (const float*)A.vals, A.hc, A.nhc, X, l,
                                                             xmean, A.hpart);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "csr_spmm_heavy");
    csr_heavy_reduce_kernel<<<grid_cap(c, A.nhr, 8), 256, 0, c.stream>>>(A.hr, A.nhr, A.hpart, l, Y);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "csr_heavy_reduce");
  }
}

// at most 2·nnz/kHeavyNnz + 1 chunks over at most nnz/kHeavyNnz + 1 heavy rows
size_t csr_heavy_plan_bytes(const CsrA& A) {
  const int64_t C = 2 * (A.nnz / kHeavyNnz) + 1, H = A.nnz / kHeavyNnz + 2;
  return Arena::align((size_t)C * 3 * 8) + Arena::align((size_t)H * 2 * 8) + Arena::align((size_t)C * kMaxL * 8);
}

void csr_build_heavy_plan(Ctx& c, CsrA& A, char* mem, const int64_t* host_ptr) {
  A.hc = nullptr;
  A.hr = nullptr;
  A.nhc = A.nhr = 0;
  A.hpart = nullptr;
  if (A.rows == 0) return;
  std::vector<int64_t> buf;
  const int64_t* ptr = host_ptr;
  if (!ptr) {
    buf.resize((size_t)A.rows + 1);
    RPCA_CUDA(cudaMemcpyAsync(buf.data(), A.ptr, sizeof(int64_t) * buf.size(), cudaMemcpyDeviceToHost, c.stream));
    RPCA_CUDA(cudaStreamSynchronize(c.stream));
    ptr = buf.data();
  }
  std::vector<int64_t> hc, hr;
  for (int64_t i = 0; i < A.rows; ++i) {
    const int64_t t0 = ptr[i], t1 = ptr[i + 1];
    if (t1 - t0 <= kHeavyNnz) continue;
    hr.push_back(i);
    hr.push_back((int64_t)hc.size() / 3);
    for (int64_t t = t0; t < t1; t += kHeavyNnz) {
      hc.push_back(i);
      hc.push_back(t);
      hc.push_back(std::min(t1, t + kHeavyNnz));
    }
  }
  if (hr.empty()) return;
  const int64_t nhc = (int64_t)hc.size() / 3, nhr = (int64_t)hr.size() / 2;
  hr.push_back(-1);
  hr.push_back(nhc);
  const size_t b_hc = Arena::align(hc.size() * 8), b_hr = Arena::align(hr.size() * 8);
  RPCA_REQUIRE(b_hc + b_hr + Arena::align((size_t)nhc * kMaxL * 8) <= csr_heavy_plan_bytes(A), RPCA_E_WORKSPACE,
               "heavy-row plan exceeds its bound");
  RPCA_CUDA(cudaMemcpyAsync(mem, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice, c.stream));
  RPCA_CUDA(cudaMemcpyAsync(mem + b_hc, hr.data(), hr.size() * 8, cudaMemcpyHostToDevice, c.stream));
  RPCA_CUDA(cudaStreamSynchronize(c.stream));  // hc / hr are host temporaries
  A.hc = reinterpret_cast<const int64_t*>(mem);
  A.nhc = nhc;
  A.hr = reinterpret_cast<const int64_t*>(mem + b_hc);
  A.nhr = nhr;
  A.hpart = reinterpret_cast<double*>(mem + b_hc + b_hr);
}

namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// Σ_i mix(word_i, i, salt) mod 2^64 over the 4-byte words of an array:
// integer sums commute, so the result does not depend on the grid.  (Row
// shards of a CSR are often views at 4-byte offsets, so no wider alignment is
// assumed.)
__global__ void fingerprint_kernel(const uint32_t* __restrict__ w, int64_t nw, uint64_t salt,
                                   unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += stride)
    acc += mix64((uint64_t)w[i] ^ mix64((uint64_t)i + salt));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}
}  // namespace

uint64_t csr_fingerprint(Ctx& c, const CsrA& A) {
  unsigned long long* d = reinterpret_cast<unsigned long long*>(c.dscratch + 64);
  RPCA_CUDA(cudaMemsetAsync(d, 0, 8, c.stream));
  const int es = A.dtype == RPCA_F64 ? 8 : 4;
  const void* arrs[3] = {A.ptr, A.idx, A.vals};
  const size_t bytes[3] = {(size_t)(A.rows + 1) * 8, (size_t)A.nnz * 4, (size_t)A.nnz * es};
  for (int a = 0; a < 3; ++a) {
    if (bytes[a] == 0) continue;
    RPCA_REQUIRE((reinterpret_cast<uintptr_t>(arrs[a]) & 3) == 0, RPCA_E_ARG, "CSR arrays must be 4-byte aligned");
    const int64_t nw = (int64_t)(bytes[a] / 4);
    fingerprint_kernel<<<grid_cap(c, nw, 2048), 256, 0, c.stream>>>(reinterpret_cast<const uint32_t*>(arrs[a]), nw,
                                                                    0x51ED27ull * (a + 1), d);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "csr_fingerprint");
  }
  uint64_t h = 0;
  RPCA_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c.stream));
  RPCA_CUDA(cudaStreamSynchronize(c.stream));
  return h;
}

size_t csr_transpose_ws_bytes(const CsrA& A) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, (const int32_t*)nullptr, (int32_t*)nullptr, (const int64_t*)nullptr,
                                  (int64_t*)nullptr, (size_t)A.nnz);
  Sizer s;
  s.add<int32_t>(A.nnz);  // rowidx
  s.add<int32_t>(A.nnz);  // sorted keys
  s.add<int64_t>(A.nnz);  // iota
  s.add<int64_t>(A.nnz);  // perm
  s.add<char>(tmp + 256);
  return s.total;
}

void csr_transpose(Ctx& c, const CsrA& A, int64_t n, CsrA& T, Arena& scratch) {
  const int64_t nnz = A.nnz;
  const int es = A.dtype == RPCA_F64 ? 8 : 4;
  int32_t* rowidx = scratch.get<int32_t>(nnz);
  int32_t* skeys = scratch.get<int32_t>(nnz);
  int64_t* iota = scratch.get<int64_t>(nnz);
  int64_t* perm = scratch.get<int64_t>(nnz);
  size_t tmp = 0;
  RPCA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, A.idx, skeys, iota, perm, (size_t)nnz));
  void* tmpbuf = scratch.get<char>(tmp + 256);
  row_of_entry_kernel<<<grid_cap(c, A.rows, 8), 256, 0, c.stream>>>(A.ptr, A.rows, rowidx);
  RPCA_CHECK_LAUNCH();
  iota_kernel<<<grid_cap(c, nnz, 256), 256, 0, c.stream>>>(nnz, iota);
  RPCA_CHECK_LAUNCH();
  int bits = 1;
  while ((int64_t(1) << bits) < n && bits < 31) ++bits;
  RPCA_CUDA(cub::DeviceRadixSort::SortPairs(tmpbuf, tmp, A.idx, skeys, iota, perm, (size_t)nnz, 0, bits, c.stream));
  int64_t* colptr = const_cast<int64_t*>(T.ptr);
  colptr_kernel<<<grid_cap(c, n + 1, 256), 256, 0, c.stream>>>(skeys, nnz, n, colptr);
  RPCA_CHECK_LAUNCH();
  if (es == 8)
    permute_kernel<double><<<grid_cap(c, nnz, 256), 256, 0, c.stream>>>(
        perm, rowidx, (const double*)A.vals, nnz, const_cast<int32_t*>(T.idx), (double*)const_cast<void*>(T.vals));
  else
    permute_kernel<float><<<grid_cap(c, nnz, 256), 256, 0, c.stream>>>(
        perm, rowidx, (const float*)A.vals, nnz, const_cast<int32_t*>(T.idx), (float*)const_cast<void*>(T.vals));
  RPCA_CHECK_LAUNCH();
  count_launch(c, 5, "csr_transpose");
  T.rows = n;
  T.nnz = nnz;
  T.dtype = A.dtype;
}

void csr_colmeans(Ctx& c, const CsrA& T, int64_t m_total, double* cmean) {
  if (T.dtype == RPCA_F64)
    csr_rowsum_kernel<double><<<grid_cap(c, T.rows, 256), 256, 0, c.stream>>>(T.ptr, (const double*)T.vals, T.rows,
                                                                              1.0 / (double)m_total, cmean);
  else
    csr_rowsum_kernel<float><<<grid_cap(c, T.rows, 256), 256, 0, c.stream>>>(T.ptr, (const float*)T.vals, T.rows,
                                                                             1.0 / (double)m_total, cmean);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "csr_colmeans");
}

}  // namespace rpca
