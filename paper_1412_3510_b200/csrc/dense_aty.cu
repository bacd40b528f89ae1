// dense_aty.cu — §8(a) steps a4/a6: Z = Aᵀ·Y for a dense row-major A (m×n)
// and a thin Y (m×l): the "(Q'*A)'" of PAPER.md:432-435, which applies the
// adjoint "without ever forming the adjoint of A explicitly", with the
// centring correction Z −= cᵀ·(1ᵀY) (the adjoint of PAPER.md:430).
//
// fp64 design (B200, sm_100a):
//   * work units = (column block of 128 columns) × (chunk of 32 rows), laid
//     out column-block-major and split into equal contiguous ranges, one per
//     persistent CTA (stream-K style: every SM gets the same number of A
//     bytes whatever m and n are);
//   * a producer warp streams each unit's A chunk with eight 2-D TMA boxes
//     [32 rows × 16 doubles] (SWIZZLE_128B) and the unit's 32 rows of the
//     packed Y with one bulk copy; eight consumer warps run DMMA (M = 16
//     columns of A per warp, N = l, K = rows);
//   * when a CTA leaves a column block it writes its fp64 partial (128×l);
//     a second kernel sums, for each column, the partials of the CTAs that
//     touched it in ascending CTA order (no float atomics, bitwise
//     reproducible) and applies the centring correction.
// Row order inside an 8-row group is permuted ({0,2,4,6}, {1,3,5,7}) so the
// A-fragment loads from the swizzled boxes are bank-conflict-free; the packed
// Y (thin.cu pack_y) uses the same order.
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace rpca {
namespace {

constexpr int BN = 128;          // columns of A per column block
constexpr int BR = 32;           // rows of A per unit / stage
constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;

template <int NT>
struct AtyCfg {
  static constexpr int kABytes = BR * BN * 8;             // 32 KB: 8 boxes × 4 KB
  static constexpr int kYBytes = 4 * 2 * NT * 32 * 8;     // packed Y for 32 rows
  static constexpr int kStageBytes = kABytes + kYBytes;
  static constexpr int kStages = (212 * 1024) / kStageBytes > 8 ? 8 : (212 * 1024) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 2 * kStages * 8;
};

struct Split {
  int64_t U, P, cpc;  // units, CTAs, chunks per column block
  __host__ __device__ int64_t u0(int64_t p) const { return p * U / P; }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
    aty_f64_tma_kernel(const __grid_constant__ CUtensorMap tmA, const double* __restrict__ Yp, Split sp,
                       int maxslots, double* __restrict__ part) {
  using Cfg = AtyCfg<NT>;
  constexpr int LP = NT * 8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = blockIdx.x;
  const int64_t ub = sp.u0(p), ue = sp.u0(p + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      int s = 0;
      uint32_t ph = 0;
      int64_t cb = ub / sp.cpc, rc = ub - cb * sp.cpc;
      for (int64_t u = ub; u < ue; ++u, ++rc) {
        if (rc == sp.cpc) { rc = 0; ++cb; }
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * Cfg::kStageBytes;
        mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
#pragma unroll
        for (int b = 0; b < 8; ++b)
          tma_load_2d(st + b * (BR * 128), &tmA, (int32_t)(cb * BN + b * 16), (int32_t)(rc * BR), &full[s]);
        bulk_load(st + Cfg::kABytes, Yp + rc * (256 * NT), Cfg::kYBytes, &full[s]);
        if (++s == Cfg::kStages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  int s = 0;
  uint32_t ph = 0;
  const int csel = lane >> 2;
  const int64_t cb_first = ub / sp.cpc;
  double acc[2][NT][2];
  auto zero = [&]() {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  };
  zero();
  int64_t cb = cb_first, rc = ub - cb_first * sp.cpc;  // no 64-bit division per unit
  for (int64_t u = ub; u < ue; ++u) {
    mbar_wait(&full[s], ph);
    const uint8_t* box = smem + s * Cfg::kStageBytes + warp * (BR * 128);
    const double* Ys = reinterpret_cast<const double*>(smem + s * Cfg::kStageBytes + Cfg::kABytes);
#pragma unroll
    for (int g = 0; g < 4; ++g) {
#pragma unroll
      for (int ss = 0; ss < 2; ++ss) {
        const int r = 8 * g + 2 * (lane & 3) + ss;
        const double a0 = *reinterpret_cast<const double*>(box + swz128_off(r, csel));
        const double a1 = *reinterpret_cast<const double*>(box + swz128_off(r, 8 + csel));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const double b = Ys[((g * 2 + ss) * NT + nt) * 32 + lane];
          dmma(acc[0][nt], a0, b);
          dmma(acc[1][nt], a1, b);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == Cfg::kStages) { s = 0; ph ^= 1; }
    const bool last_of_cb = (u + 1 == ue) || (rc + 1 == sp.cpc);
    if (last_of_cb) {
      double* dst = part + ((p * maxslots + (cb - cb_first)) * BN) * LP;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int cl = warp * 16 + mt * 8 + csel;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int j = nt * 8 + 2 * (lane & 3);
          *reinterpret_cast<double2*>(dst + cl * LP + j) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      }
      zero();
    }
    if (++rc == sp.cpc) { rc = 0; ++cb; }
  }
}

// Z[c][j] = Σ_{p covering cb(c), ascending} part[p][slot][c mod 128][j] − cmean[c]·sy[j]
// One thread per output: the few CTAs covering column block cb(c) (stream-K
// ranges) are summed in ascending order — deterministic.
__global__ void aty_reduce_kernel(const double* __restrict__ part, Split sp, int maxslots, int64_t n, int l, int LP,
                                  const double* __restrict__ cmean, const double* __restrict__ sy,
                                  double* __restrict__ Z) {
  const int64_t total = n * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / l;
    const int j = (int)(idx - c * l);
    const int64_t cb = c / BN;
    const int cl = (int)(c - cb * BN);
    const int64_t ustart = cb * sp.cpc, uend = ustart + sp.cpc;
    int64_t p = (ustart * sp.P) / sp.U;  // first CTA whose range can reach ustart
    if (p > 0) --p;
    while (p < sp.P && sp.u0(p + 1) <= ustart) ++p;
    double s = 0.0;
    for (; p < sp.P && sp.u0(p) < uend; ++p) {
      const int64_t a = sp.u0(p), b = sp.u0(p + 1);
      if (b <= a) continue;
      const int64_t slot = cb - a / sp.cpc;
      s += part[((p * maxslots + slot) * BN + cl) * LP + j];
    }
    Z[idx] = cmean ? s - cmean[c] * sy[j] : s;
  }
}

// Generic CUDA-core fallback: CTA = (64-column block, row split); fp64 partials.
template <class T>
__global__ void __launch_bounds__(256) aty_generic_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                          const double* __restrict__ Y, int l, int64_t rows_per_split,
                                                          double* __restrict__ part) {
  __shared__ double As[32][65];
  __shared__ double Ys[32][kMaxL];
  const int64_t c0 = (int64_t)blockIdx.x * 64;
  const int64_t rb = (int64_t)blockIdx.y * rows_per_split, re = min(m, rb + rows_per_split);
  const int cl = threadIdx.x & 63, ph = threadIdx.x >> 6;
  double acc[kMaxL / 4];
#pragma unroll
  for (int t = 0; t < kMaxL / 4; ++t) acc[t] = 0.0;
  for (int64_t i0 = rb; i0 < re; i0 += 32) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * 64; idx += 256) {
      const int rr = idx >> 6, cc = idx & 63;
      const int64_t gi = i0 + rr, gc = c0 + cc;
      As[rr][cc] = (gi < re && gc < n) ? static_cast<double>(A[gi * lda + gc]) : 0.0;
    }
    for (int idx = threadIdx.x; idx < 32 * l; idx += 256) {
      const int rr = idx / l, j = idx % l;
      const int64_t gi = i0 + rr;
      Ys[rr][j] = gi < re ? Y[gi * l + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < 32; ++rr) {
      const double a = As[rr][cl];
#pragma unroll
      for (int t = 0; t < kMaxL / 4; ++t) {
        const int j = ph + 4 * t;
        if (j < l) acc[t] += a * Ys[rr][j];
      }
    }
  }
  const int64_t gc = c0 + cl;
  if (gc < n) {
#pragma unroll
    for (int t = 0; t < kMaxL / 4; ++t) {
      const int j = ph + 4 * t;
      if (j < l) part[((int64_t)blockIdx.y * n + gc) * l + j] = acc[t];
    }
  }
}

__global__ void aty_generic_reduce(const double* __restrict__ part, int64_t splits, int64_t n, int l,
                                   const double* __restrict__ cmean, const double* __restrict__ sy,
                                   double* __restrict__ Z) {
  const int64_t total = n * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < splits; ++b) s += part[b * total + idx];
    if (cmean) s -= cmean[idx / l] * sy[idx % l];
    Z[idx] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    RPCA_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    RPCA_REQUIRE(q == cudaDriverEntryPointSuccess && p, RPCA_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool tma_ok(const DenseA& A) {
  return A.dtype == RPCA_F64 && ((reinterpret_cast<uintptr_t>(A.a) & 15u) == 0) && ((A.lda * 8) % 16 == 0);
}

Split make_split(Ctx& c, const DenseA& A) {
  Split sp;
  sp.cpc = cdiv(A.m, BR);
  sp.U = cdiv(A.n, BN) * sp.cpc;
  // ≥ 16 units (512 KB of A) per CTA: small passes would otherwise spend
  // more in the reduction of many partials than in the pass
  sp.P = std::min<int64_t>({(int64_t)c.num_sms, sp.U, std::max<int64_t>(1, cdiv(sp.U, 16))});
  return sp;
}

int max_slots(const Split& sp) {
  int mx = 1;
  for (int64_t p = 0; p < sp.P; ++p) {
    const int64_t a = sp.u0(p), b = sp.u0(p + 1);
    if (b > a) mx = std::max<int>(mx, (int)((b - 1) / sp.cpc - a / sp.cpc + 1));
  }
  return mx;
}

int64_t generic_splits(Ctx& c, const DenseA& A) {
  const int64_t ncb = cdiv(A.n, 64);
  int64_t splits = std::max<int64_t>(1, (2 * c.num_sms + ncb - 1) / ncb);
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, cdiv(A.m, 256)));
  return splits;
}

template <int NT>
void launch_aty_tma(Ctx& c, const DenseA& A, const double* Yp, const Split& sp, int maxslots, double* part) {
  using Cfg = AtyCfg<NT>;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)A.n, (cuuint64_t)A.m};
  cuuint64_t strides[1] = {(cuuint64_t)A.lda * 8};
  cuuint32_t box[2] = {16, BR};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(A.a), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RPCA_REQUIRE(r == CUDA_SUCCESS, RPCA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  ensure_smem((const void*)aty_f64_tma_kernel<NT>, Cfg::kSmem);
  prof_pre(c);
  aty_f64_tma_kernel<NT><<<(unsigned)sp.P, kThreads, Cfg::kSmem, c.stream>>>(tm, Yp, sp, maxslots, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "aty_f64_dmma");
}

}  // namespace

void aty_reduce_partials(Ctx& c, const double* part, int64_t U, int64_t P, int64_t cpc, int maxslots, int64_t n,
                         int l, int LP, const double* cmean, const double* sy, double* Z) {
  Split sp;
  sp.U = U;
  sp.P = P;
  sp.cpc = cpc;
  const int64_t total = n * l;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 16);
  aty_reduce_kernel<<<grid, 256, 0, c.stream>>>(part, sp, maxslots, n, l, LP, cmean, sy, Z);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "aty_reduce");
}

size_t aty_ws_bytes(Ctx& c, const DenseA& A, int l) {
  Sizer s;
  s.add<double>(kMaxL);                                            // sy
  s.add<double>(std::max<int64_t>(1, cdiv(A.m, 2048)) * kMaxL);    // colsum partials
  if (f32_tc_ok(A)) {
    s.add<char>(aty_f32_ws_bytes(c, A, l));
  } else if (tma_ok(A)) {
    const Split sp = make_split(c, A);
    s.add<double>(packy_elems(A.m, l));
    s.add<double>(sp.P * (int64_t)max_slots(sp) * BN * cdiv(l, 8) * 8);
  } else {
    s.add<double>(generic_splits(c, A) * A.n * l);
    s.add<double>((size_t)A.m * l);  // centred copy of Y
  }
  return s.total;
}

void dense_aty(Ctx& c, const DenseA& A, const double* Y, int l, const double* cmean, double* Z, Arena& ar,
               const double* ymean) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "l=%d out of range [1,%d]", l, kMaxL);
  double* sy = nullptr;
  if (cmean) {
    sy = ar.get<double>(kMaxL);
    weighted_colsum(c, nullptr, Y, A.m, l, sy, ar);
  }
  if (f32_tc_ok(A) && A.m > 0) {
    const size_t mark = ar.off;
    dense_aty_f32(c, A, Y, l, cmean, sy, Z, ar, ymean);
    ar.off = mark;
    return;
  }
  if (tma_ok(A) && A.m > 0) {
    const Split sp = make_split(c, A);
    const int ms = max_slots(sp);
    const int NT = (int)cdiv(l, 8);
    double* Yp = ar.get<double>(packy_elems(A.m, l));
    double* part = ar.get<double>(sp.P * (int64_t)ms * BN * NT * 8);
    pack_y(c, Y, A.m, l, Yp, ymean);
    switch (NT) {
      case 1: launch_aty_tma<1>(c, A, Yp, sp, ms, part); break;
      case 2: launch_aty_tma<2>(c, A, Yp, sp, ms, part); break;
      case 3: launch_aty_tma<3>(c, A, Yp, sp, ms, part); break;
      case 4: launch_aty_tma<4>(c, A, Yp, sp, ms, part); break;
      case 5: launch_aty_tma<5>(c, A, Yp, sp, ms, part); break;
      case 6: launch_aty_tma<6>(c, A, Yp, sp, ms, part); break;
      case 7: launch_aty_tma<7>(c, A, Yp, sp, ms, part); break;
      default: launch_aty_tma<8>(c, A, Yp, sp, ms, part); break;
    }
    const int64_t total = A.n * l;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 16);
    aty_reduce_kernel<<<grid, 256, 0, c.stream>>>(part, sp, ms, A.n, l, NT * 8, cmean, sy, Z);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "aty_reduce");
    return;
  }
  if (ymean && A.m > 0) {  // generic kernel: centre a copy of Y first
    double* Yc = ar.get<double>((size_t)A.m * l);
    RPCA_CUDA(cudaMemcpyAsync(Yc, Y, sizeof(double) * A.m * l, cudaMemcpyDeviceToDevice, c.stream));
    sub_rank1(c, Yc, A.m, l, nullptr, ymean);
    Y = Yc;
  }
  const int64_t splits = A.m > 0 ? generic_splits(c, A) : 1;
  const int64_t rps = std::max<int64_t>(1, cdiv(A.m, splits));
  double* part = ar.get<double>(splits * A.n * l);
  if (A.m > 0) {
    dim3 grid((unsigned)cdiv(A.n, 64), (unsigned)splits);
    prof_pre(c);
    if (A.dtype == RPCA_F64)
      aty_generic_kernel<double><<<grid, 256, 0, c.stream>>>((const double*)A.a, A.m, A.n, A.lda, Y, l, rps, part);
    else
      aty_generic_kernel<float><<<grid, 256, 0, c.stream>>>((const float*)A.a, A.m, A.n, A.lda, Y, l, rps, part);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "aty_generic");
  } else {
    RPCA_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * A.n * l, c.stream));
  }
  const int64_t total = A.n * l;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 8);
  aty_generic_reduce<<<grid, 256, 0, c.stream>>>(part, splits, A.n, l, cmean, sy, Z);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "aty_reduce");
}

}  // namespace rpca
