// dense_f32_tc.cu — §8(a) steps a2/a4/a5/a6 for an fp32 A (the C4 workload):
// Y = A·X and Z = Aᵀ·Y on the 5th-generation tensor cores (tcgen05, TMEM
// accumulators, TMA), with 3×TF32 products.
//
// Why 3×TF32: one tf32 product keeps 11 bits of each operand; SURVEY.md §8(c)
// c.4 measured that 1×TF32 misses BASELINE's fp32 tolerances (σ 1e-4, angle
// 1e-3) by two orders of magnitude, while A_hi·X_hi + A_hi·X_lo + A_lo·X_hi
// (A_hi = tf32(A), A_lo = A − A_hi exactly in fp32) meets them with a 10×
// margin.  The tensor core TRUNCATES fp32 operands to tf32 (measured:
// tools/microbench/tc_tf32_probe.cu), so the raw fp32 tile is the "hi"
// operand as loaded and only A_lo = A − trunc13(A) has to be formed.
//
// A·X  (D[128 rows × N] += A[128 × K] · X[K × N]):
//   warp 0 — TMA producer: A box [128 rows × 32 fp32] (SWIZZLE_128B) and the
//            matching K-chunk of Xᵀ_hi / Xᵀ_lo ([N × 32], K-major) per stage;
//   warps 2-5 — split: thread t owns row t, reads its 128-byte row from the
//            swizzled tile and writes A_lo in the same layout (conflict-free
//            16-byte accesses), then the epilogue (tcgen05.ld → fp64 → Y);
//   warp 1 — one thread issues tcgen05.mma kind::tf32 (M=128, N = 16..64,
//            K=8) ×3 per k-step into a TMEM fp32 accumulator, and commits
//            stage releases / the tile to mbarriers.
// Aᵀ·Y (D[128 cols × N] += Aᵀ[128 × K rows] · Y[K × N]): the same roles on
//   (128-column block × 32-row chunk) units split evenly over the CTAs
//   (stream-K, as the fp64 kernel); the split warps transpose the tile into
//   K-major Aᵀ_hi / Aᵀ_lo, partial accumulators are flushed in fp64 and
//   reduced in ascending CTA order by dense_aty.cu's reducer.
// Per element of A: 4 bytes, 3·2·N tensor flops.  fp32 accumulation runs over
// the whole K of one tile (≤ 4096 for C4); everything across tiles, CTAs and
// ranks is fp64.
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kThreads = 192;  // 6 warps

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;          // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;  // SBO: 8-row atoms 1024 B apart
  d |= (uint64_t)1 << 46;          // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;          // SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// element (r, k) of a K-major tile with 32 fp32 per row, SWIZZLE_128B
__device__ __forceinline__ uint32_t kmaj(int r, int k) {
  return r * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + ((k & 3) << 2);
}

__device__ __forceinline__ float lo_part(float a) {
  return a - __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Stage layout: raw A tile (16 KB) | NT split tiles of 16 KB (AX: A_lo; AtY:
// Aᵀ_hi, Aᵀ_lo) | Xᵀ_hi chunk | Xᵀ_lo chunk (N rows × 128 B each).
template <int N, int NT>
struct F32Cfg {
  static constexpr int kA = 128 * 128;
  static constexpr int kAlo = 128 * 128;
  static constexpr int kX = N * 128;
  static constexpr int kXoff = kA + NT * kAlo;
  static constexpr int kStage = kXoff + 2 * kX;
  static constexpr int kStages = (216 * 1024) / kStage > 4 ? 4 : (216 * 1024) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024 + 256;
  static constexpr int kTmemCols = N <= 32 ? 32 : 64;
};

// ---------------------------------------------------------------- Y = A·X
template <int N>
__global__ void __launch_bounds__(kThreads, 1)
    ax_f32_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                     const __grid_constant__ CUtensorMap tmXl, int64_t m, int l, int64_t ntiles, int KB,
                     double* __restrict__ Y) {
  using Cfg = F32Cfg<N, 1>;
  constexpr int kStagesF = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesF * Cfg::kStage);
  uint64_t* lo_full = full + kStagesF;
  uint64_t* empty = lo_full + kStagesF;
  uint64_t* acc_full = empty + kStagesF;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesF; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lo_full[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------ producer
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmXh);
      prefetch_tmap(&tmXl);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * Cfg::kStage;
          mbar_arrive_expect_tx(&full[s], Cfg::kA + 2 * Cfg::kX);
          tma_load_2d(st, &tmA, kb * 32, (int32_t)(tile * 128), &full[s]);
          tma_load_2d(st + Cfg::kXoff, &tmXh, kb * 32, 0, &full[s]);
          tma_load_2d(st + Cfg::kXoff + Cfg::kX, &tmXl, kb * 32, 0, &full[s]);
          if (++s == kStagesF) { s = 0; ph ^= 1; }
        }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_tf32(128, N);
      int s = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(acc_empty, aph ^ 1);
        aph ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&lo_full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a0 = smem_u32(smem + s * Cfg::kStage);
          const uint32_t al = a0 + Cfg::kA;
          const uint32_t xh = a0 + Cfg::kXoff, xl = xh + Cfg::kX;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t acc = (kb | ks) != 0;
            mma_tf32(tmem, desc_sw128(a0 + ks * 32), desc_sw128(xh + ks * 32), idesc, acc);
            mma_tf32(tmem, desc_sw128(a0 + ks * 32), desc_sw128(xl + ks * 32), idesc, 1);
            mma_tf32(tmem, desc_sw128(al + ks * 32), desc_sw128(xh + ks * 32), idesc, 1);
          }
          mma_commit(&empty[s]);
          if (kb == KB - 1) mma_commit(acc_full);
          if (++s == kStagesF) { s = 0; ph ^= 1; }
        }
      }
    }
  } else {  // ---------------------------------------------------- split + epilogue
    const int t = threadIdx.x - 64;  // row of the tile, 0..127
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    int s = 0;
    uint32_t ph = 0, aph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      for (int kb = 0; kb < KB; ++kb) {
        mbar_wait(&full[s], ph);
        const uint8_t* a = smem + s * Cfg::kStage;
        uint8_t* al = smem + s * Cfg::kStage + Cfg::kA;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = kmaj(t, 4 * c);
          float4 v = *reinterpret_cast<const float4*>(a + off);
          v.x = lo_part(v.x);
          v.y = lo_part(v.y);
          v.z = lo_part(v.z);
          v.w = lo_part(v.w);
          *reinterpret_cast<float4*>(al + off) = v;
        }
        fence_proxy_async();  // generic-proxy writes → visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full[s]);
        if (++s == kStagesF) { s = 0; ph ^= 1; }
      }
      // epilogue: rows 32q..32q+31 of the accumulator live in TMEM lanes of quarter q
      mbar_wait(acc_full, aph);
      aph ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = tile * 128 + 32 * q + lane;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
        if (row < m) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < l) Y[row * l + c0 + j] = (double)v[j];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::kTmemCols));
  }
}

// ---------------------------------------------------------------- Z = Aᵀ·Y
struct SplitF {
  int64_t U, P, cpc;  // units, CTAs, 32-row chunks per 128-column block
  __host__ __device__ int64_t u0(int64_t p) const { return p * U / P; }
};

template <int N>
__global__ void __launch_bounds__(kThreads, 1)
    aty_f32_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmYh,
                      const __grid_constant__ CUtensorMap tmYl, SplitF sp, int maxslots, int LP,
                      double* __restrict__ part) {
  using Cfg = F32Cfg<N, 2>;
  constexpr int kStagesF = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesF * Cfg::kStage);
  uint64_t* lo_full = full + kStagesF;
  uint64_t* empty = lo_full + kStagesF;
  uint64_t* acc_full = empty + kStagesF;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t p = blockIdx.x;
  const int64_t ub = sp.u0(p), ue = sp.u0(p + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesF; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&lo_full[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmYh);
      prefetch_tmap(&tmYl);
      int s = 0;
      uint32_t ph = 0;
      for (int64_t u = ub; u < ue; ++u) {
        const int64_t cb = u / sp.cpc, rc = u - cb * sp.cpc;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * Cfg::kStage;
        mbar_arrive_expect_tx(&full[s], Cfg::kA + 2 * Cfg::kX);
#pragma unroll
        for (int b = 0; b < 4; ++b)  // four [32 rows × 32 cols] boxes = the 32×128 tile
          tma_load_2d(st + b * 4096, &tmA, (int32_t)(cb * 128 + b * 32), (int32_t)(rc * 32), &full[s]);
        tma_load_2d(st + Cfg::kXoff, &tmYh, (int32_t)(rc * 32), 0, &full[s]);
        tma_load_2d(st + Cfg::kXoff + Cfg::kX, &tmYl, (int32_t)(rc * 32), 0, &full[s]);
        if (++s == kStagesF) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(128, N);
      int s = 0;
      uint32_t ph = 0, aph = 0;
      bool first = true;
      for (int64_t u = ub; u < ue; ++u) {
        const int64_t cb = u / sp.cpc;
        if (first) {
          mbar_wait(acc_empty, aph ^ 1);
          aph ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        mbar_wait(&lo_full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t th = smem_u32(smem + s * Cfg::kStage) + Cfg::kA;  // Aᵀ_hi (128 cols × 32 rows)
        const uint32_t tl = th + Cfg::kAlo;                              // Aᵀ_lo
        const uint32_t yh = smem_u32(smem + s * Cfg::kStage) + Cfg::kXoff, yl = yh + Cfg::kX;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t acc = (!first || ks) ? 1u : 0u;
          mma_tf32(tmem, desc_sw128(th + ks * 32), desc_sw128(yh + ks * 32), idesc, acc);
          mma_tf32(tmem, desc_sw128(th + ks * 32), desc_sw128(yl + ks * 32), idesc, 1);
          mma_tf32(tmem, desc_sw128(tl + ks * 32), desc_sw128(yh + ks * 32), idesc, 1);
        }
        mma_commit(&empty[s]);
        const bool last_of_cb = (u + 1 == ue) || ((u + 1) / sp.cpc != cb);
        if (last_of_cb) mma_commit(acc_full);
        first = last_of_cb;
        if (++s == kStagesF) { s = 0; ph ^= 1; }
      }
    }
  } else {
    const int t = threadIdx.x - 64;  // column of the 128-column block, 0..127
    const int q = warp & 3;
    int s = 0;
    uint32_t ph = 0, aph = 0;
    const int64_t cb_first = ub / sp.cpc;
    for (int64_t u = ub; u < ue; ++u) {
      const int64_t cb = u / sp.cpc;
      mbar_wait(&full[s], ph);
      const uint8_t* a = smem + s * Cfg::kStage;
      uint8_t* th = smem + s * Cfg::kStage + Cfg::kA;
      uint8_t* tl = th + Cfg::kAlo;
      const uint8_t* slab = a + (t >> 5) * 4096;
      const int cc = t & 31;
#pragma unroll
      for (int g = 0; g < 8; ++g) {  // rows 4g..4g+3 of column t → one 16-byte chunk of row t of Aᵀ
        float4 h, lo;
        h.x = *reinterpret_cast<const float*>(slab + kmaj(4 * g + 0, cc));
        h.y = *reinterpret_cast<const float*>(slab + kmaj(4 * g + 1, cc));
        h.z = *reinterpret_cast<const float*>(slab + kmaj(4 * g + 2, cc));
        h.w = *reinterpret_cast<const float*>(slab + kmaj(4 * g + 3, cc));
        lo.x = lo_part(h.x);
        lo.y = lo_part(h.y);
        lo.z = lo_part(h.z);
        lo.w = lo_part(h.w);
        const uint32_t off = kmaj(t, 4 * g);
        *reinterpret_cast<float4*>(th + off) = h;
        *reinterpret_cast<float4*>(tl + off) = lo;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&lo_full[s]);
      if (++s == kStagesF) { s = 0; ph ^= 1; }
      const bool last_of_cb = (u + 1 == ue) || ((u + 1) / sp.cpc != cb);
      if (last_of_cb) {  // flush: column 32q+lane of the block ← TMEM lane 32q+lane
        mbar_wait(acc_full, aph);
        aph ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        double* dst = part + ((p * maxslots + (cb - cb_first)) * 128 + 32 * q + lane) * LP;
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + c0, v);
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c0 + j < LP) dst[c0 + j] = (double)v[j];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::kTmemCols));
  }
}

// Xᵀ split: Xt_hi[j][k] = tf32(X[k][j]) (as fp32 with the low 13 bits cleared),
// Xt_lo[j][k] = fp32(X[k][j] − Xt_hi[j][k]); zero padding to (Npad × Kpad).
// 64-row tiles go through shared memory so both the read of X (rows of l
// doubles) and the writes of Xᵀ (runs of 64 k) are coalesced.
__global__ void __launch_bounds__(256) split_transpose_kernel(const double* __restrict__ X, int64_t K, int l, int Npad,
                                                              int64_t Kpad, float* __restrict__ hi,
                                                              float* __restrict__ lo) {
  __shared__ double tile[64][kMaxL + 1];
  for (int64_t k0 = (int64_t)blockIdx.x * 64; k0 < Kpad; k0 += (int64_t)gridDim.x * 64) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < 64 * l; idx += 256) {
      const int r = idx / l, j = idx - r * l;
      const int64_t k = k0 + r;
      tile[r][j] = k < K ? X[k * l + j] : 0.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 64 * Npad; idx += 256) {
      const int j = idx >> 6, r = idx & 63;
      const double x = j < l ? tile[r][j] : 0.0;
      const float h = __uint_as_float(__float_as_uint((float)x) & 0xFFFFE000u);
      hi[(int64_t)j * Kpad + k0 + r] = h;
      lo[(int64_t)j * Kpad + k0 + r] = (float)(x - (double)h);
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

CUtensorMap tmap_f32(const void* base, int64_t inner, int64_t outer, int64_t ld_elems, int box_inner, int box_outer) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RPCA_REQUIRE(r == CUDA_SUCCESS, RPCA_E_CUDA, "cuTensorMapEncodeTiled(f32) failed (%d)", (int)r);
  return tm;
}

int npad_for(int l) { return l <= 16 ? 16 : (l <= 32 ? 32 : (l <= 48 ? 48 : 64)); }

void split_transpose(Ctx& c, const double* X, int64_t K, int l, int Npad, int64_t Kpad, float* hi, float* lo) {
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(Kpad, 64), (int64_t)c.num_sms * 8);
  split_transpose_kernel<<<grid, 256, 0, c.stream>>>(X, K, l, Npad, Kpad, hi, lo);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "split_tf32");
}

template <int N>
void launch_ax(Ctx& c, const DenseA& A, const float* hi, const float* lo, int64_t Kpad, int l, double* Y) {
  using Cfg = F32Cfg<N, 1>;
  const CUtensorMap tA = tmap_f32(A.a, A.n, A.m, A.lda, 32, 128);
  const CUtensorMap tH = tmap_f32(hi, Kpad, N, Kpad, 32, N);
  const CUtensorMap tL = tmap_f32(lo, Kpad, N, Kpad, 32, N);
  ensure_smem((const void*)ax_f32_tc_kernel<N>, Cfg::kSmem);
  const int64_t ntiles = cdiv(A.m, 128);
  const int grid = (int)std::min<int64_t>(ntiles, c.num_sms);
  ax_f32_tc_kernel<N><<<grid, kThreads, Cfg::kSmem, c.stream>>>(tA, tH, tL, A.m, l, ntiles, (int)(Kpad / 32), Y);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "ax_f32_tc");
}

template <int N>
void launch_aty(Ctx& c, const DenseA& A, const float* hi, const float* lo, int64_t Kpad, const SplitF& sp,
                int maxslots, double* part) {
  using Cfg = F32Cfg<N, 2>;
  const CUtensorMap tA = tmap_f32(A.a, A.n, A.m, A.lda, 32, 32);
  const CUtensorMap tH = tmap_f32(hi, Kpad, N, Kpad, 32, N);
  const CUtensorMap tL = tmap_f32(lo, Kpad, N, Kpad, 32, N);
  ensure_smem((const void*)aty_f32_tc_kernel<N>, Cfg::kSmem);
  aty_f32_tc_kernel<N><<<(unsigned)sp.P, kThreads, Cfg::kSmem, c.stream>>>(tA, tH, tL, sp, maxslots, N, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "aty_f32_tc");
}

SplitF make_split(Ctx& c, const DenseA& A) {
  SplitF sp;
  sp.cpc = cdiv(A.m, 32);
  sp.U = cdiv(A.n, 128) * sp.cpc;
  sp.P = std::min<int64_t>(c.num_sms, sp.U);
  return sp;
}

int max_slots(const SplitF& sp) {
  int mx = 1;
  for (int64_t p = 0; p < sp.P; ++p) {
    const int64_t a = sp.u0(p), b = sp.u0(p + 1);
    if (b > a) mx = std::max<int>(mx, (int)((b - 1) / sp.cpc - a / sp.cpc + 1));
  }
  return mx;
}

}  // namespace

bool f32_tc_ok(const DenseA& A) {
  return A.dtype == RPCA_F32 && ((reinterpret_cast<uintptr_t>(A.a) & 15u) == 0) && ((A.lda * 4) % 16 == 0) &&
         A.m >= 1 && A.n >= 1;
}

size_t ax_f32_ws_bytes(const DenseA& A, int l) {
  Sizer s;
  const int64_t Kpad = cdiv(A.n, 64) * 64;
  s.add<float>((size_t)npad_for(l) * Kpad);
  s.add<float>((size_t)npad_for(l) * Kpad);
  return s.total;
}

void dense_ax_f32(Ctx& c, const DenseA& A, const double* X, int l, double* Y, Arena& ar) {
  const int Np = npad_for(l);
  const int64_t Kpad = cdiv(A.n, 64) * 64;
  float* hi = ar.get<float>((size_t)Np * Kpad);
  float* lo = ar.get<float>((size_t)Np * Kpad);
  split_transpose(c, X, A.n, l, Np, Kpad, hi, lo);
  switch (Np) {
    case 16: launch_ax<16>(c, A, hi, lo, Kpad, l, Y); break;
    case 32: launch_ax<32>(c, A, hi, lo, Kpad, l, Y); break;
    case 48: launch_ax<48>(c, A, hi, lo, Kpad, l, Y); break;
    default: launch_ax<64>(c, A, hi, lo, Kpad, l, Y); break;
  }
}

size_t aty_f32_ws_bytes(Ctx& c, const DenseA& A, int l) {
  const SplitF sp = make_split(c, A);
  Sizer s;
  const int64_t Kpad = cdiv(A.m, 64) * 64;
  s.add<float>((size_t)npad_for(l) * Kpad);
  s.add<float>((size_t)npad_for(l) * Kpad);
  s.add<double>((size_t)sp.P * max_slots(sp) * 128 * npad_for(l));
  return s.total;
}

// Z partials; the caller reduces them with aty_reduce (dense_aty.cu)
void dense_aty_f32_partials(Ctx& c, const DenseA& A, const double* Y, int l, double** part_out, int64_t* P,
                            int* maxslots, int64_t* cpc, int* LP, Arena& ar) {
  const int Np = npad_for(l);
  const int64_t Kpad = cdiv(A.m, 64) * 64;
  float* hi = ar.get<float>((size_t)Np * Kpad);
  float* lo = ar.get<float>((size_t)Np * Kpad);
  split_transpose(c, Y, A.m, l, Np, Kpad, hi, lo);
  const SplitF sp = make_split(c, A);
  const int ms = max_slots(sp);
  double* part = ar.get<double>((size_t)sp.P * ms * 128 * Np);
  *part_out = part;
  switch (Np) {
    case 16: launch_aty<16>(c, A, hi, lo, Kpad, sp, ms, part); break;
    case 32: launch_aty<32>(c, A, hi, lo, Kpad, sp, ms, part); break;
    case 48: launch_aty<48>(c, A, hi, lo, Kpad, sp, ms, part); break;
    default: launch_aty<64>(c, A, hi, lo, Kpad, sp, ms, part); break;
  }
  *P = sp.P;
  *maxslots = ms;
  *cpc = sp.cpc;
  *LP = Np;
}

}  // namespace rpca
