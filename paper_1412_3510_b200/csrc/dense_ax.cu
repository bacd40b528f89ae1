// dense_ax.cu — §8(a) steps a2/a5: Y = A·X for a dense row-major A (m×n) and
// a thin X (n×l), the "A*Q" of PAPER.md:398/430 — the pass that streams A.
//
// fp64 design (B200, sm_100a):
//   * persistent CTAs (one per SM), each walks row tiles of BM = 128 rows;
//   * one producer warp streams A with 2-D TMA boxes [128 rows × 16 doubles]
//     (SWIZZLE_128B, zero fill past m and n) plus the matching 32-row chunk of
//     the packed X with a 1-D bulk copy into a STAGES-deep mbarrier ring;
//   * eight consumer warps run the fp64 tensor-core MMA (mma.m8n8k4 f64,
//     "DMMA"); each warp owns 16 rows × 8·NT columns in registers.  The k
//     order inside a 32-wide chunk is permuted so that every lane fetches its
//     two A values with one conflict-free 16-byte LDS (see the layout note);
//     X is pre-packed in exactly the fragment order (thin.cu pack_x).
//   Per element of A: 8 bytes and 2·l flops — at l = 22 the fp64 pipe (≈37
//   TF/s measured) and HBM (≈6.5-7.3 TB/s) bind together.
// Generic fallback (fp32 A until the tcgen05 path lands, or lda·8 not a
// multiple of 16): CUDA-core kernel with the same result contract.
#include <cudaTypedefs.h>

#include <type_traits>

#include "internal.cuh"

namespace rpca {
namespace {

constexpr int BM = 128;          // rows per tile
constexpr int BK = 32;           // k per stage (two TMA boxes of 16 doubles)
constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kMaxSms = 160;  // stream-K partial slots (≥ the SM count)

template <int NT>
struct AxCfg {
  static constexpr int kABytes = BM * BK * 8;             // 32 KB
  static constexpr int kXBytes = 8 * NT * 32 * 8;         // packed X chunk
  static constexpr int kStageBytes = kABytes + kXBytes;   // multiple of 1024
  static constexpr int kStages = (212 * 1024) / kStageBytes > 8 ? 8 : (212 * 1024) / kStageBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 2 * kStages * 8;
};

// Layout note.  Stage s holds A rows [tile·128, +128) × k [kb·32, +32) as
// two boxes (k 0-15, k 16-31), each 128 rows × 128 B, 128B-swizzled.  DMMA
// k-step st (0..7) gives lane (row r = lane>>2, kpos c = lane&3) the value
// A[r][kb·32 + 16·(q>>1) + 4c + 2(q&1) + (st&1)], q = st>>1: for st = 2q,
// 2q+1 both values sit in 16-byte chunk 2c + (q&1) of box q>>1, loaded once
// as a double2.  Within each 8-lane LDS.128 phase (rows r, r+1) the swizzled
// chunk positions (2c + (q&1)) ^ (r&7) are all distinct: conflict-free.
// Packed X holds X[that same k][nt·8 + (lane>>2)] at Xp[kb][st][nt][lane].
// Stream-K work split: unit u = tile·KB + kb; CTA p owns units
// [p·U/P, (p+1)·U/P).  A tile the CTA covers whole is written to Y directly;
// a tile cut by a CTA boundary leaves fp64 partial rows in part[p][slot]
// (slot 0 = the CTA's first tile, 1 = its last) that ax_fixup_kernel sums in
// ascending CTA order — every CTA gets the same number of k-blocks (no tail
// wave: C2's 782 tiles on 148 SMs left 12% idle) and the result is
// deterministic.
struct AxSplit {
  int64_t U, P;
  int KB;
  int whole_tiles;  // split at tile granularity (no tile is cut, no fixup)
  __host__ __device__ int64_t u0(int64_t p) const {
    return whole_tiles ? (p * (U / KB) / P) * KB : p * U / P;
  }
};

// UPPER: X is upper triangular (the thin products Y·U⁻¹ of the LU and the
// Cholesky-QR): a k-step whose smallest k exceeds an n-tile's last column
// only multiplies zeros there and is skipped (43% of the DMMAs at l = 52).
template <int NT, bool UPPER>
__global__ void __launch_bounds__(kThreads, 1)
    ax_f64_tma_kernel(const __grid_constant__ CUtensorMap tmA, const double* __restrict__ Xp, int64_t m, int l,
                      AxSplit sp, const double* __restrict__ cx, double* __restrict__ Y, double* __restrict__ part) {
  using Cfg = AxCfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* empty = full + Cfg::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = sp.KB;
  const int64_t ub = sp.u0(blockIdx.x), ue = sp.u0(blockIdx.x + 1);
  const int64_t tile_first = ub / KB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (ub >= ue) return;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      int s = 0;
      uint32_t ph = 0;
      int64_t tile = tile_first;
      int kb = (int)(ub - tile_first * KB);
      for (int64_t u = ub; u < ue; ++u) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * Cfg::kStageBytes;
        mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
        tma_load_2d(st, &tmA, kb * BK, (int32_t)(tile * BM), &full[s]);
        tma_load_2d(st + BM * 128, &tmA, kb * BK + 16, (int32_t)(tile * BM), &full[s]);
        bulk_load(st + Cfg::kABytes, Xp + (int64_t)kb * 256 * NT, Cfg::kXBytes, &full[s]);
        if (++s == Cfg::kStages) { s = 0; ph ^= 1; }
        if (++kb == KB) { kb = 0; ++tile; }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  int s = 0;
  uint32_t ph = 0;
  const int rsel = lane >> 2;
  int64_t tile = tile_first;
  int kb = (int)(ub - tile_first * KB);
  int64_t u = ub;
  while (u < ue) {
    const bool starts = (kb == 0);
    const int kend = (int)imin64(KB, kb + (ue - u));  // this CTA's k-blocks of the tile: [kb, kend)
    const bool whole = starts && kend == KB;
    double acc[2][NT][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

    // one k-block of DMMAs; KBS = the k-block index when it is static (the
    // UPPER kernels: K = l ≤ 64, two k-blocks), so the zero-block skips fold
    // at compile time, else −1
    auto kblock = [&](auto KBS) {
      constexpr int kbs = decltype(KBS)::value;
      mbar_wait(&full[s], ph);
      const uint8_t* As = smem + s * Cfg::kStageBytes;
      const double* Xs = reinterpret_cast<const double*>(As + Cfg::kABytes);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint8_t* box = As + (q >> 1) * (BM * 128);
        const int chunk = 2 * (lane & 3) + (q & 1);  // rows r, r+1 of a phase hit chunks of opposite parity
        double2 a[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int r = warp * 16 + mt * 8 + rsel;
          a[mt] = *reinterpret_cast<const double2*>(box + r * 128 + ((chunk ^ rsel) << 4));
        }
#pragma unroll
        for (int ss = 0; ss < 2; ++ss) {
          const int st = 2 * q + ss;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            // X[k][n-tile] = 0 for every k of this k-step (smallest k > the tile's last column)
            if (kbs >= 0 && kbs * BK + 16 * (q >> 1) + 2 * (q & 1) + ss > nt * 8 + 7) continue;
            const double b = Xs[(st * NT + nt) * 32 + lane];
            dmma(acc[0][nt], ss ? a[0].y : a[0].x, b);
            dmma(acc[1][nt], ss ? a[1].y : a[1].x, b);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == Cfg::kStages) { s = 0; ph ^= 1; }
    };
    for (; kb < kend; ++kb, ++u) {
      if constexpr (UPPER) {
        if (kb == 0) kblock(std::integral_constant<int, 0>{});
        else if (kb == 1) kblock(std::integral_constant<int, 1>{});
        else kblock(std::integral_constant<int, -1>{});
      } else {
        kblock(std::integral_constant<int, -1>{});
      }
    }
    // epilogue: D rows = lane>>2, cols 2·(lane&3) + {0,1}
    double* dst = Y;
    int64_t ld = l, rbase = tile * BM;
    if (!whole) {  // partial rows of a split tile → this CTA's slot
      dst = part + ((int64_t)blockIdx.x * 2 + (tile == tile_first ? 0 : 1)) * BM * (NT * 8);
      ld = NT * 8;
      rbase = 0;
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int rt = warp * 16 + mt * 8 + rsel;
      if (tile * BM + rt >= m) continue;
      const int64_t row = rbase + rt;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int col = nt * 8 + 2 * (lane & 3);
        double* y = dst + row * ld + col;
        if (!whole) {
          *reinterpret_cast<double2*>(y) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        } else {
          // the centring correction Y −= 1·cxᵀ folded into the store
          const double v0 = acc[mt][nt][0] - (cx && col < l ? cx[col] : 0.0);
          const double v1 = acc[mt][nt][1] - (cx && col + 1 < l ? cx[col + 1] : 0.0);
          if (col + 1 < l) {
            if ((l & 1) == 0)
              *reinterpret_cast<double2*>(y) = make_double2(v0, v1);
            else {
              y[0] = v0;
              y[1] = v1;
            }
          } else if (col < l) {
            y[0] = v0;
          }
        }
      }
    }
    if (kb == KB) { kb = 0; ++tile; }
  }
}

// Split tiles: block b looks at CTA boundary p = b+1; if it cuts a tile and is
// the first boundary inside it, the block sums that tile's partials over the
// covering CTAs in ascending order and writes its rows of Y.
__global__ void ax_fixup_kernel(AxSplit sp, int64_t m, int l, int LP, const double* __restrict__ part,
                                const double* __restrict__ cx, double* __restrict__ Y) {
  __shared__ int64_t t_s;
  __shared__ int nq_s;
  __shared__ const double* src[32];  // the covering CTAs' partial slots, ascending
  if (threadIdx.x == 0) {
    nq_s = 0;
    const int64_t p = blockIdx.x + 1;
    const int64_t KB = sp.KB;
    const int64_t b = sp.u0(p);
    const int64_t t = b / KB;
    // act only for the first boundary strictly inside a tile
    if (b % KB != 0 && b < sp.U && sp.u0(p - 1) <= t * KB) {
      int64_t q = p - 1;  // CTA holding unit t·KB
      int nq = 0;
      for (; q < sp.P && sp.u0(q) < (t + 1) * KB && nq < 32; ++q, ++nq) {
        const int slot = (sp.u0(q) / KB == t) ? 0 : 1;  // t is q's first tile, or its last
        src[nq] = part + (q * 2 + slot) * BM * LP;
      }
      nq_s = nq;
      t_s = t;
    }
  }
  __syncthreads();
  const int nq = nq_s;
  if (nq == 0) return;
  const int64_t t = t_s;
  const int nrow = (int)imin64(BM, m - t * BM);
  double* __restrict__ yt = Y + t * BM * l;
  // four outputs per thread in flight (the loads do not alias the stores)
  for (int idx0 = threadIdx.x; idx0 < nrow * l; idx0 += 4 * blockDim.x) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int off[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = idx0 + e * blockDim.x;
      const int r = idx / l, j = idx - r * l;
      off[e] = idx < nrow * l ? r * LP + j : -1;
    }
    for (int k = 0; k < nq; ++k) {
      const double* __restrict__ sk = src[k];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (off[e] >= 0) s[e] += __ldg(sk + off[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = idx0 + e * blockDim.x;
      if (idx < nrow * l) yt[idx] = cx ? s[e] - cx[idx % l] : s[e];
    }
  }
}

// Generic CUDA-core fallback: 64-row tiles, X and A chunks staged in smem (fp64).
template <class T>
__global__ void __launch_bounds__(256) ax_generic_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                         const double* __restrict__ X, int l,
                                                         double* __restrict__ Y) {
  __shared__ double As[64][33];
  __shared__ double Xs[32][kMaxL];
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  // thread → (row = tid & 63, column phase = tid >> 6): columns j = ph, ph+4, ...
  const int r = threadIdx.x & 63, ph = threadIdx.x >> 6;
  double acc[kMaxL / 4];
#pragma unroll
  for (int t = 0; t < kMaxL / 4; ++t) acc[t] = 0.0;
  for (int64_t k0 = 0; k0 < n; k0 += 32) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < 64 * 32; idx += 256) {
      const int rr = idx >> 5, kk = idx & 31;
      const int64_t gi = r0 + rr, gk = k0 + kk;
      As[rr][kk] = (gi < m && gk < n) ? static_cast<double>(A[gi * lda + gk]) : 0.0;
    }
    for (int idx = threadIdx.x; idx < 32 * l; idx += 256) {
      const int kk = idx / l, j = idx % l;
      const int64_t gk = k0 + kk;
      Xs[kk][j] = gk < n ? X[gk * l + j] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 32; ++kk) {
      const double a = As[r][kk];
#pragma unroll
      for (int t = 0; t < kMaxL / 4; ++t) {
        const int j = ph + 4 * t;
        if (j < l) acc[t] += a * Xs[kk][j];
      }
    }
  }
  const int64_t gi = r0 + r;
  if (gi < m) {
#pragma unroll
    for (int t = 0; t < kMaxL / 4; ++t) {
      const int j = ph + 4 * t;
      if (j < l) Y[gi * l + j] = acc[t];
    }
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

template <int NT>
void launch_ax_tma(Ctx& c, const DenseA& A, const double* Xp, int l, const double* cx, double* Y, double* part,
                   bool upper) {
  using Cfg = AxCfg<NT>;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)A.n, (cuuint64_t)A.m};
  cuuint64_t strides[1] = {(cuuint64_t)A.lda * 8};
  cuuint32_t box[2] = {16, BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(A.a), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RPCA_REQUIRE(r == CUDA_SUCCESS, RPCA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  ensure_smem((const void*)ax_f64_tma_kernel<NT, false>, Cfg::kSmem);
  ensure_smem((const void*)ax_f64_tma_kernel<NT, true>, Cfg::kSmem);
  const int64_t ntiles = cdiv(A.m, BM);
  const int KB = (int)cdiv(A.n, BK);
  AxSplit sp;
  sp.KB = KB;
  sp.U = ntiles * KB;
  sp.whole_tiles = 0;
  sp.P = std::min<int64_t>({sp.U, (int64_t)c.num_sms, ntiles * 16});  // a tile spans ≤ ~17 CTAs (fixup ≤ 32)
  // small passes (A mostly L2-resident, microseconds of work): ≥ 16 units
  // (512 KB of A) per CTA, so the fixup does not cost more than it saves
  sp.P = std::min<int64_t>(sp.P, std::max<int64_t>(1, cdiv(sp.U, 16)));
  // whole tiles when they balance already or K is short (the thin-block
  // products: K = l ≤ 64): the split is then at tile granularity, so no tile
  // is cut and no fixup runs — which also makes the in-place products
  // (apply_l's L = Y·M, the Cholesky-QR TRMMs) safe by construction: a tile's
  // rows are read and then written by the one CTA that owns the tile
  if (ntiles % sp.P == 0 || KB < 8) {
    sp.P = std::min<int64_t>(ntiles, c.num_sms);
    sp.whole_tiles = 1;
  }
  bool split = false;  // does any CTA boundary cut a tile?
  for (int64_t q = 1; q < sp.P && !split; ++q) split = sp.u0(q) % KB != 0;
  prof_pre(c);
  if (upper)
    ax_f64_tma_kernel<NT, true><<<(unsigned)sp.P, kThreads, Cfg::kSmem, c.stream>>>(tm, Xp, A.m, l, sp, cx, Y, part);
  else
    ax_f64_tma_kernel<NT, false><<<(unsigned)sp.P, kThreads, Cfg::kSmem, c.stream>>>(tm, Xp, A.m, l, sp, cx, Y, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "ax_f64_dmma");
  if (split && sp.P > 1) {
    ax_fixup_kernel<<<(unsigned)(sp.P - 1), 256, 0, c.stream>>>(sp, A.m, l, NT * 8, part, cx, Y);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "stream_k_fixup");
  }
}

bool tma_ok(const DenseA& A) {
  return A.dtype == RPCA_F64 && ((reinterpret_cast<uintptr_t>(A.a) & 15u) == 0) && ((A.lda * 8) % 16 == 0) &&
         A.n >= 1 && A.m >= 1 && A.lda * 8 < (int64_t(1) << 40);
}

}  // namespace

size_t ax_ws_bytes(const DenseA& A, int l) {
  if (f32_tc_ok(A)) return ax_f32_ws_bytes(A, l);
  Sizer s;
  s.add<double>(packx_elems(A.n, l));
  s.add<double>((size_t)kMaxSms * 2 * BM * ((l + 7) / 8 * 8));  // stream-K partial rows
  return std::max(s.total, emu_eligible(A, l) ? emu_ws_bytes(A, l) : (size_t)0);
}

void dense_ax(Ctx& c, const DenseA& A, const double* X, int l, double* Y, Arena& ar, const double* cx, bool upper) {
  RPCA_REQUIRE(l >= 1 && l <= kMaxL, RPCA_E_SHAPE, "l=%d out of range [1,%d]", l, kMaxL);
  if (A.m == 0) return;
  if (f32_tc_ok(A)) {
    dense_ax_f32(c, A, X, l, cx, Y, ar);  // centring folded into the epilogue
    return;
  }
  if (!cx && c.emu_E && A.a == c.emu_A && emu_eligible(A, l)) {  // the driver's A, row exponents known
    dense_ax_emu(c, A, c.emu_E, X, l, Y, ar);
    return;
  }
  if (cx && !tma_ok(A)) {  // generic kernel: the rank-1 correction as a separate thin pass
    dense_ax(c, A, X, l, Y, ar, nullptr, upper);
    sub_rank1(c, Y, A.m, l, nullptr, cx);
    return;
  }
  if (tma_ok(A)) {
    double* Xp = ar.get<double>(packx_elems(A.n, l));
    double* part = ar.get<double>((size_t)kMaxSms * 2 * BM * ((l + 7) / 8 * 8));
    pack_x(c, X, A.n, l, Xp);
    switch ((l + 7) / 8) {
      case 1: launch_ax_tma<1>(c, A, Xp, l, cx, Y, part, upper); break;
      case 2: launch_ax_tma<2>(c, A, Xp, l, cx, Y, part, upper); break;
      case 3: launch_ax_tma<3>(c, A, Xp, l, cx, Y, part, upper); break;
      case 4: launch_ax_tma<4>(c, A, Xp, l, cx, Y, part, upper); break;
      case 5: launch_ax_tma<5>(c, A, Xp, l, cx, Y, part, upper); break;
      case 6: launch_ax_tma<6>(c, A, Xp, l, cx, Y, part, upper); break;
      case 7: launch_ax_tma<7>(c, A, Xp, l, cx, Y, part, upper); break;
      default: launch_ax_tma<8>(c, A, Xp, l, cx, Y, part, upper); break;
    }
    return;
  }
  const unsigned grid = (unsigned)cdiv(A.m, 64);
  prof_pre(c);
  if (A.dtype == RPCA_F64)
    ax_generic_kernel<double><<<grid, 256, 0, c.stream>>>((const double*)A.a, A.m, A.n, A.lda, X, l, Y);
  else
    ax_generic_kernel<float><<<grid, 256, 0, c.stream>>>((const float*)A.a, A.m, A.n, A.lda, X, l, Y);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "ax_generic");
}

}  // namespace rpca
