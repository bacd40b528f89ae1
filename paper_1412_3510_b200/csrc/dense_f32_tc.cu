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
// Both kernels move A through TMEM: split warps read the A tile from shared
// memory once, store A_hi = trunc13(A) and A_lo = A − A_hi to TMEM (one
// 32-bit TMEM column per k, lane = the M index), and every product reads its
// A operand from TMEM (tcgen05.mma TS form) — shared memory carries the tile
// once plus the thin operand (ablations: both passes were shared-memory
// bound with the A_hi operand read from shared memory).
//
// A·X  (D[128 rows × N] += A[128 × K] · Xᵀ[N × K]ᵀ, both K-major):
//   warp 0 producer (TMA A box [128 rows × 32 fp32] + Xᵀ_hi/lo chunks),
//   warp 1 MMA issuer (A_hi·[X_hi | X_lo] as one N = 2N MMA, A_lo·X_hi into
//   the first N columns), warps 2-5 split, warps 6-9 epilogue.  Units are
//   (128-row tile, ≤ 4096-wide K chunk) — fp32 accumulation never runs over
//   more than 4096 products; two TMEM accumulators
//   alternate so the epilogue of unit u overlaps the MMAs of unit u+1; the
//   epilogue writes (first chunk) or adds (later chunks) fp64 into Y and
//   folds the centring correction −1·(c·X) of PAPER.md:430.
// Aᵀ·Y (D[128 cols × N] += Aᵀ[128 cols × K rows] · Y[K × N]): the split
//   warps read the row-major A tile (thread = column) and store A_hi and A_lo
//   into TMEM (lane = column of A, one TMEM column per row), so all three
//   products take their A operand from TMEM and only Yᵀ from shared memory.
//   A CTA owns a group of ≤ 512/N column blocks (all accumulators live in
//   TMEM) and a contiguous row range; each 32-row chunk of Yᵀ_hi/lo is loaded
//   once and used for every column block of the group, so Y is read
//   ⌈n/(128·group)⌉ times instead of once per column block.  Every 4096 rows
//   the accumulators are flushed (fp64 adds into the CTA's partial); the
//   partials are reduced over the row ranges in ascending order.
// Per element of A: 4 bytes, 3·2·N tensor flops.
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace rpca {
namespace {


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


// (An MN-major tf32 shared-memory operand would need SWIZZLE_128B_BASE32B —
// descriptor layout type 1, TMA mode 128B_ATOM_32B, LBO 4096 / SBO 512; the
// Aᵀ·Y kernel avoids it by moving A through TMEM.)

// D[tmem] (+)= A[tmem] · B[smem]: the A operand read from TMEM (lane = M row,
// one 32-bit column per K element)
__device__ __forceinline__ void mma_tf32_ts(uint32_t dt, uint32_t at, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
      "r"(at), "l"(db), "r"(idesc), "r"(acc));
}

// this thread's 32 consecutive TMEM columns of its lane ← v
__device__ __forceinline__ void tmem_st32(uint32_t addr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// this thread's 16 consecutive TMEM columns of its lane ← v (no wait)
__device__ __forceinline__ void tmem_st16_nowait(uint32_t addr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Release a shared-memory stage only after its loads have RETURNED.  An
// mbarrier arrive is a volatile asm that stays in program order with other
// volatile asms, but the register arithmetic on the loaded values (the first
// instructions that wait for the loads' data) may be scheduled below it, so
// the TMA could refill the stage under loads still in flight.  Pass this
// empty volatile asm values COMPUTED from the loads (it emits no instruction
// itself, so raw load results would not do): the arithmetic producing them,
// and with it the wait for every load, must then come before the arrive.
__device__ __forceinline__ void loads_done16(const float* v) {
  asm volatile("" ::"f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
               "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
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

__device__ __forceinline__ void tmem_ld8(uint32_t addr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive TMEM columns starting at a column that is only 8-aligned
// (the second accumulator half when N = 56)
template <int N>
__device__ __forceinline__ void tmem_ld16_at(uint32_t addr, float (&v)[16]) {
  if constexpr (N % 16 == 0) {
    tmem_ld16(addr, v);
  } else {
    tmem_ld8(addr, v);
    tmem_ld8(addr + 8, v + 8);
  }
}

// one lane of a converged warp (the same one every time) — the issuing lane of
// TMA / tcgen05.mma / tcgen05.commit; the rest of the warp keeps the loop
// state uniform so operands stay in uniform registers
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

#ifndef ATY_F32_MAX_STAGES
#define ATY_F32_MAX_STAGES 8
#endif
#ifndef ATY_SLOTS
#define ATY_SLOTS 2
#endif
constexpr int kTileBytes = 128 * 128;  // 16 KB A tile
constexpr int kKChunk = 4096;          // max products per fp32 accumulation (Q15)

// stage index + phase of an S-deep mbarrier ring, advanced without division
template <int S>
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == S) { s = 0; ph ^= 1u; }
  }
};

template <int N>
struct AxCfg {
  static constexpr int kX = N * 128;  // one Xᵀ chunk: N rows × 32 fp32
  static constexpr int kStage = kTileBytes + 2 * kX;
  static constexpr int kStages = (212 * 1024) / kStage > 8 ? 8 : (212 * 1024) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024 + 512;
  // TMEM per accumulator: [0, N) A_hi·X_hi + A_lo·X_hi, [N, 2N) A_hi·X_lo
  // (one N = 2N MMA over the adjacent X_hi, X_lo chunks); two accumulators,
  // then 64-column A slots (32 columns A_hi, 32 columns A_lo)
  static constexpr int kW = (2 * N + 31) / 32 * 32;
  static constexpr int kSlot0 = 2 * kW;
  static constexpr int kNS = (512 - kSlot0) / 64 >= 4 ? 4 : 2;
};
constexpr int kThreadsAx = 320;  // 10 warps: producer, MMA, 4 split, 4 epilogue

// ---------------------------------------------------------------- Y = A·X
// warps: 0 TMA producer, 1 MMA issuer, 2-5 split (A → A_hi, A_lo in TMEM,
// thread = row = TMEM lane), 6-9 epilogue.  Both products of A take their
// A operand from TMEM (TS form), so shared memory carries the A tile once
// (TMA write, split read) plus the Xᵀ operand reads — 56 KB per 16 KB tile
// instead of 72 KB with the A_hi MMA reading A from shared memory (the
// ablation showed the pass shared-memory bound there).
template <int N>
__global__ void __launch_bounds__(kThreadsAx, 1)
    ax_f32_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmXh,
                     const __grid_constant__ CUtensorMap tmXl, int64_t m, int l, int64_t ntiles, int KB,
                     const double* __restrict__ cx, double* __restrict__ Y, double* __restrict__ colpart) {
  using Cfg = AxCfg<N>;
  constexpr int S = Cfg::kStages, NS = Cfg::kNS;
  constexpr int KC = kKChunk / 32;  // k-blocks per unit
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStage);
  uint64_t* empty = full + S;        // 4 split warps (A read) + MMA commit (Xᵀ read)
  uint64_t* afull = empty + S;       // [NS] 4 split warps (A_hi, A_lo in TMEM)
  uint64_t* tfree = afull + NS;      // [NS] MMA commit
  uint64_t* acc_full = tfree + NS;   // [2] MMA commit
  uint64_t* acc_empty = acc_full + 2;  // [2] 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkc = (KB + KC - 1) / KC;  // K chunks per tile

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 5);
    }
    for (int a = 0; a < NS; ++a) {
      mbar_init(&afull[a], 4);
      mbar_init(&tfree[a], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ----------------------------------------------- producer
    const bool leader = elect_one();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmXh);
    prefetch_tmap(&tmXl);
    Ring<S> rg;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < KB; ++kb, rg.next()) {
        mbar_wait(&empty[rg.s], rg.ph ^ 1u);
        uint8_t* st = smem + rg.s * Cfg::kStage;
        if (leader) {
          mbar_arrive_expect_tx(&full[rg.s], kTileBytes + 2 * Cfg::kX);
          tma_load_2d(st, &tmA, kb * 32, (int32_t)(tile * 128), &full[rg.s]);
          tma_load_2d(st + kTileBytes, &tmXh, kb * 32, 0, &full[rg.s]);
          tma_load_2d(st + kTileBytes + Cfg::kX, &tmXl, kb * 32, 0, &full[rg.s]);
        }
        __syncwarp();
      }
  } else if (warp == 1) {  // ------------------------------------------- MMA issuer
    // D[:, 0:2N] += A_hi·[X_hi | X_lo]; D[:, 0:N] += A_lo·X_hi (A from TMEM)
    const bool leader = elect_one();
    // N = 56 (l ≤ 56): the lo·hi product runs at N = 64, whose extra 8
    // columns add A_lo·X_lo[0..7] into the A_hi·X_lo accumulator of output
    // columns 0-7 (a fourth, more accurate term), and [X_hi | X_lo] is one
    // 112-row operand — 176 MMA columns per k-step instead of 192 at N = 64
    constexpr uint32_t idesc2 = idesc_tf32(128, 2 * N), idesc1 = idesc_tf32(128, (N + 15) / 16 * 16);
    Ring<S> rg;
    Ring<NS> rt;
    int64_t u = -1;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < KB; ++kb, rg.next(), rt.next()) {
        const int kin = kb & (KC - 1);
        if (kin == 0) {  // first stage of a unit: its accumulator must have been drained
          ++u;
          mbar_wait(&acc_empty[u & 1], (uint32_t)((u >> 1) & 1) ^ 1u);
          tc_fence_after();
        }
        mbar_wait(&afull[rt.s], rt.ph);
        mbar_wait(&full[rg.s], rg.ph);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((u & 1) * Cfg::kW);
        const uint32_t ah = tmem + (uint32_t)(Cfg::kSlot0 + 64 * rt.s), al = ah + 32;
        const uint64_t dx = desc_sw128(smem_u32(smem + rg.s * Cfg::kStage) + kTileBytes);
        if (leader) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            mma_tf32_ts(d, ah + 8 * ks, dx + 2 * ks, idesc2, (kin != 0 || ks != 0) ? 1u : 0u);
            mma_tf32_ts(d, al + 8 * ks, dx + 2 * ks, idesc1, 1u);
          }
          mma_commit(&tfree[rt.s]);
          mma_commit(&empty[rg.s]);
          if (kb == KB - 1 || kin == KC - 1) mma_commit(&acc_full[u & 1]);
        }
        __syncwarp();
      }
  } else if (warp < 6) {  // ---------------------------------------- split: A → A_hi, A_lo in TMEM
    const int q = warp & 3;
    const int t = 32 * q + lane;  // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    Ring<S> rg;
    Ring<NS> rt;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int kb = 0; kb < KB; ++kb, rg.next(), rt.next()) {
        mbar_wait(&full[rg.s], rg.ph);
        const uint8_t* row = smem + rg.s * Cfg::kStage + t * 128;
        float hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // logical 16-byte chunk c (k = 4c..4c+3) sits at c ^ (t mod 8)
          const float4 x = *reinterpret_cast<const float4*>(row + ((c ^ (t & 7)) << 4));
          hi[4 * c] = x.x;
          hi[4 * c + 1] = x.y;
          hi[4 * c + 2] = x.z;
          hi[4 * c + 3] = x.w;
        }
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const float a = hi[k];
          hi[k] = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
          lo[k] = a - hi[k];
        }
        loads_done16(lo);  // the row is in registers (see loads_done16)
        loads_done16(lo + 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rg.s]);
        mbar_wait(&tfree[rt.s], rt.ph ^ 1u);
        tc_fence_after();
        const uint32_t at = tmem + lane_off + (uint32_t)(Cfg::kSlot0 + 64 * rt.s);
        tmem_st32(at, hi);
        tmem_st32(at + 32, lo);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[rt.s]);
      }
  } else {  // ---------------------------------------------------- epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int64_t lt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      const int64_t row = tile * 128 + 32 * q + lane;
      for (int kc = 0; kc < nkc; ++kc) {
        const int64_t u = lt * nkc + kc;
        mbar_wait(&acc_full[u & 1], (uint32_t)((u >> 1) & 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)((u & 1) * Cfg::kW) + ((uint32_t)(32 * q) << 16);
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
          float v[16], w[16];
          double fin[16];  // the values stored (final after the last chunk)
          tmem_ld16(d + c0, v);
          tmem_ld16_at<N>(d + N + c0, w);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            fin[j] = 0.0;
            if (row < m && c0 + j < l) {
              double* y = Y + row * l + c0 + j;
              const double a = (double)v[j] + (double)w[j];
              fin[j] = kc == 0 ? (cx ? a - cx[c0 + j] : a) : *y + a;
              *y = fin[j];
            }
          }
          if (colpart && kc == nkc - 1) {  // column sums of this quarter's 32 rows
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const double sv = warp_sum(fin[j]);
              if (lane == 0 && c0 + j < l) colpart[(tile * 4 + q) * l + c0 + j] = sv;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[u & 1]);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- Z = Aᵀ·Y
// Work plan: column blocks (128 columns) in groups of ≤ CBG; CTA p = g·Pg + r
// owns group g and row chunks [r·R/Pg, (r+1)·R/Pg) (32-row chunks).
struct AtyPlan {
  int64_t nb, R;  // column blocks, 32-row chunks
  int CBG, Gc, Pg;
  __host__ __device__ int64_t rc0(int r) const { return (int64_t)r * R / Pg; }
};

template <int N>
struct AtyCfg {
  static constexpr int kX = N * 128;  // one Yᵀ chunk: N rows × 32 fp32
  // [0, N) A_hi·Y_hi + A_lo·Y_hi, [N, 2N) A_hi·Y_lo (one N = 2N MMA)
  static constexpr int kTN = 2 * N <= 32 ? 32 : (2 * N <= 64 ? 64 : 128);
#ifndef ATY_YS
#define ATY_YS 3
#endif
  static constexpr int kYS = ATY_YS;  // Yᵀ chunk buffers
  static constexpr int kYBytes = kYS * 2 * kX;
  static constexpr int kFit = (227 * 1024 - 1536 - kYBytes) / kTileBytes;  // 227 KB per CTA
  static constexpr int kStages = kFit > ATY_F32_MAX_STAGES ? ATY_F32_MAX_STAGES : kFit;
  static constexpr int kSmem = kStages * kTileBytes + kYBytes + 1024 + 512;
  static constexpr int kNS = ATY_SLOTS;  // A slots after the accumulators: 32 columns A_hi + 32 columns A_lo
  static constexpr int kSlot0 = 512 - 64 * kNS;
  static constexpr int kMaxCB = kSlot0 / kTN;
};
constexpr int kSplitWarps = 8;    // two per TMEM lane quarter, 16 rows of the tile each
constexpr int kThreadsAty = 32 * (2 + kSplitWarps + 4);  // producer, MMA, split, 4 epilogue

// warps: 0 TMA producer, 1 MMA issuer, 2-9 split (A → A_hi, A_lo in TMEM;
// warps w and w+4 share a TMEM lane quarter and take 16 rows each), 10-13
// epilogue (fp64 flush per accumulation chunk).  Every product reads its
// A operand from TMEM (the "TS" form) and only Yᵀ from shared memory: per
// 16 KB A tile the SM moves 16 KB (TMA) + 16 KB (split reads) + 24 KB (three
// N-wide Yᵀ operands per k-step) through shared memory, not 88 KB as with the
// MN-major shared-memory A operand read twice.
template <int N>
__global__ void __launch_bounds__(kThreadsAty, 1)
    aty_f32_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmYh,
                      const __grid_constant__ CUtensorMap tmYl, AtyPlan pl, double* __restrict__ part) {
  using Cfg = AtyCfg<N>;
  constexpr int S = Cfg::kStages, YS = Cfg::kYS, NS = Cfg::kNS;
  constexpr int RC = kKChunk / 32;  // row chunks per fp32 accumulation
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* ybuf = smem + S * kTileBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ybuf + Cfg::kYBytes);
  uint64_t* empty = full + S;        // kSplitWarps (tile read into registers)
  uint64_t* yfull = empty + S;       // [YS]
  uint64_t* yempty = yfull + YS;     // [YS] MMA commit
  uint64_t* afull = yempty + YS;     // [NS] kSplitWarps (A_hi, A_lo in TMEM)
  uint64_t* tfree = afull + NS;      // [NS] MMA commit
  uint64_t* acc_full = tfree + NS;   // MMA commit
  uint64_t* acc_empty = acc_full + 1;  // [kMaxCB] 4 epilogue warps (that block's accumulator read out)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + Cfg::kMaxCB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x, g = p / pl.Pg, r = p - g * pl.Pg;
  const int64_t cb0 = (int64_t)g * pl.CBG;
  const int ncb = (int)imin64(pl.CBG, pl.nb - cb0);
  const int64_t rb = pl.rc0(r), re = pl.rc0(r + 1);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSplitWarps);
    }
    for (int y = 0; y < YS; ++y) {
      mbar_init(&yfull[y], 1);
      mbar_init(&yempty[y], 1);
    }
    for (int a = 0; a < NS; ++a) {
      mbar_init(&afull[a], kSplitWarps);
      mbar_init(&tfree[a], 1);
    }
    mbar_init(acc_full, 1);
    for (int cb = 0; cb < Cfg::kMaxCB; ++cb) mbar_init(&acc_empty[cb], 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ----------------------------------------------- producer
    const bool leader = elect_one();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmYh);
    prefetch_tmap(&tmYl);
    Ring<S> rg;
    Ring<YS> ry;
    // A is streamed once: evict-first, so it does not push out the Yᵀ chunks
    // the other column-block groups re-read from L2 (evict-last)
    const uint64_t pol_a = policy_evict_first(), pol_y = policy_evict_last();
    for (int64_t rc = rb; rc < re; ++rc, ry.next()) {
      mbar_wait(&yempty[ry.s], ry.ph ^ 1u);
      uint8_t* yb = ybuf + ry.s * 2 * Cfg::kX;
      if (leader) {
        mbar_arrive_expect_tx(&yfull[ry.s], 2 * Cfg::kX);
        tma_load_2d_hint(yb, &tmYh, (int32_t)(rc * 32), 0, &yfull[ry.s], pol_y);
        tma_load_2d_hint(yb + Cfg::kX, &tmYl, (int32_t)(rc * 32), 0, &yfull[ry.s], pol_y);
      }
      __syncwarp();
      for (int cbi = 0; cbi < ncb; ++cbi, rg.next()) {
        mbar_wait(&empty[rg.s], rg.ph ^ 1u);
        if (leader) {  // one box: 32 rows × 128 columns, row-major, no swizzle
          mbar_arrive_expect_tx(&full[rg.s], kTileBytes);
          tma_load_2d_hint(smem + rg.s * kTileBytes, &tmA, (int32_t)((cb0 + cbi) * 128), (int32_t)(rc * 32),
                           &full[rg.s], pol_a);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // ------------------------------------------- MMA issuer
    // D_cb += A_hi·Y_hi + A_hi·Y_lo + A_lo·Y_hi, A_hi/A_lo from TMEM (lane =
    // column of A, one TMEM column per row of A)
    const bool leader = elect_one();
    constexpr uint32_t idesc = idesc_tf32(128, (N + 15) / 16 * 16), idesc2 = idesc_tf32(128, 2 * N);  // (as A·X)
    Ring<YS> ry;
    Ring<NS> rt;
    int kin = 0;        // row chunks into the current accumulation chunk
    uint32_t chph = 0;  // acc_empty phase
    for (int64_t rc = rb; rc < re; ++rc, ry.next()) {
      const bool chunk_end = (kin == RC - 1) || (rc + 1 == re);
      mbar_wait(&yfull[ry.s], ry.ph);
      tc_fence_after();
      const uint32_t yh = smem_u32(ybuf + ry.s * 2 * Cfg::kX);
      const uint64_t dh = desc_sw128(yh);  // Y_hi rows [0, N) then Y_lo rows [N, 2N): one 2N-row operand
      for (int cbi = 0; cbi < ncb; ++cbi, rt.next()) {
        // a new accumulation chunk overwrites block cbi: its previous sums
        // must have been read out (per block, so the flush of the last blocks
        // overlaps the first MMAs of the next chunk)
        if (kin == 0) mbar_wait(&acc_empty[cbi], chph ^ 1u);
        mbar_wait(&afull[rt.s], rt.ph);
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(cbi * Cfg::kTN);
        const uint32_t ah = tmem + (uint32_t)(Cfg::kSlot0 + 64 * rt.s), al = ah + 32;
        if (leader) {
#ifndef ATY_NO_MMA  // ablation: the pipeline without the tensor-core products
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            mma_tf32_ts(d, ah + 8 * ks, dh + 2 * ks, idesc2, (kin != 0 || ks != 0) ? 1u : 0u);
            mma_tf32_ts(d, al + 8 * ks, dh + 2 * ks, idesc, 1u);
          }
#endif
          mma_commit(&tfree[rt.s]);
          if (cbi == ncb - 1) {
            mma_commit(&yempty[ry.s]);
            if (chunk_end) mma_commit(acc_full);
          }
        }
        __syncwarp();
      }
      if (kin == 0) chph ^= 1u;
      if (++kin == RC) kin = 0;
    }
  } else if (warp < 2 + kSplitWarps) {  // ------------------------- split: A → A_hi, A_lo in TMEM
    const int q = warp & 3;        // this warp's TMEM lane quarter
    const int h = (warp - 2) >> 2;  // which 16 rows of the tile
    const int t = 32 * q + lane;   // column of the block = TMEM lane
    const int64_t total = (re - rb) * ncb;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    Ring<S> rg;
    Ring<NS> rt;
    for (int64_t i = 0; i < total; ++i, rg.next(), rt.next()) {
      mbar_wait(&full[rg.s], rg.ph);
      const float* tile = reinterpret_cast<const float*>(smem + rg.s * kTileBytes) + 16 * h * 128 + t;
      float hi[16], lo[16];
#pragma unroll
      for (int rho = 0; rho < 16; ++rho) hi[rho] = tile[rho * 128];  // a warp reads 128 contiguous bytes
      // the stage may be refilled only once the loads have RETURNED
      // (loads_done16): arriving right after issuing them let the TMA
      // overwrite the stage under loads still in flight — stale A values in
      // some TMEM lanes, Z rows off by ~1e-3 relative, in 11 of 60 calls
      // (l = 40-64, 400000 × 600) and in every call with 4 stages
      // (tools/gpu/aty_f32_diag.py; 0 of 600 after this change)
#pragma unroll
      for (int rho = 0; rho < 16; ++rho) {
        const float a = hi[rho];
        hi[rho] = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
        lo[rho] = a - hi[rho];
      }
      loads_done16(hi);
      loads_done16(lo);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[rg.s]);
      mbar_wait(&tfree[rt.s], rt.ph ^ 1u);
      tc_fence_after();
      const uint32_t at = tmem + lane_off + (uint32_t)(Cfg::kSlot0 + 64 * rt.s + 16 * h);
#ifndef ATY_NO_TMEM_ST  // ablation: the split without its TMEM stores
      tmem_st16_nowait(at, hi);
      tmem_st16_nowait(at + 32, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
#else
      if (hi[0] == 12345.0f && lo[0] == 1.0f) asm volatile("trap;");  // keep the split live
      (void)at;
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[rt.s]);
    }
  } else {  // ---------------------------------------------------- epilogue: fp64 flush per chunk
    const int q = warp & 3;
    const int64_t nch = (re - rb + RC - 1) / RC;
    for (int64_t ch = 0; ch < nch; ++ch) {
      mbar_wait(acc_full, (uint32_t)(ch & 1));
      tc_fence_after();
      for (int cbi = 0; cbi < ncb; ++cbi) {
        double* dst = part + (((int64_t)p * pl.CBG + cbi) * 128 + 32 * q + lane) * N;
        const uint32_t d = tmem + (uint32_t)(cbi * Cfg::kTN) + ((uint32_t)(32 * q) << 16);
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
          float v[16], w[16];
          tmem_ld16(d + c0, v);
          tmem_ld16_at<N>(d + N + c0, w);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (c0 + j >= N) break;  // N = 56: the last group is half used
            const double a = (double)v[j] + (double)w[j];
            dst[c0 + j] = ch == 0 ? a : dst[c0 + j] + a;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[cbi]);
      }
    }
    if (nch == 0) {  // no rows: zero partial
      for (int cbi = 0; cbi < ncb; ++cbi) {
        double* dst = part + (((int64_t)p * pl.CBG + cbi) * 128 + 32 * q + lane) * N;
        for (int j = 0; j < N; ++j) dst[j] = 0.0;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Z[c][j] = Σ_{r ascending} part[g·Pg + r][c/128 − g·CBG][c mod 128][j] − cmean[c]·sy[j]
// (g = ⌊c/128⌋ / CBG), in ascending r — deterministic.
__global__ void aty_f32_reduce_kernel(const double* __restrict__ part, AtyPlan pl, int LP, int64_t n, int l,
                                      const double* __restrict__ cmean, const double* __restrict__ sy,
                                      double* __restrict__ Z) {
  // one thread per output (adjacent threads: adjacent j, coalesced reads),
  // eight loads in flight
  const int64_t total = n * l;
  const int64_t stride = (int64_t)pl.CBG * 128 * LP;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = idx / l;
    const int j = (int)(idx - c * l);
    const int64_t cb = c >> 7;
    const int g = (int)(cb / pl.CBG), cbi = (int)(cb - (int64_t)g * pl.CBG);
    const double* p = part + ((((int64_t)g * pl.Pg) * pl.CBG + cbi) * 128 + (c & 127)) * LP + j;
    double s = 0.0;
    int r = 0;
    for (; r + 8 <= pl.Pg; r += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p[(r + u) * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; r < pl.Pg; ++r) s += p[r * stride];
    Z[idx] = cmean ? s - cmean[c] * sy[j] : s;
  }
}

// Xᵀ split: Xt_hi[j][k] = tf32(X[k][j]) (as fp32 with the low 13 bits cleared),
// Xt_lo[j][k] = fp32(X[k][j] − Xt_hi[j][k]); rows j < l only (the TMA boxes
// read rows l … Npad−1 out of bounds, i.e. as zeros), k zero-padded to Kpad.
// 64-row tiles go through shared memory so both the read of X (64·l
// contiguous doubles, all in flight: 16 loads per thread) and the writes of
// Xᵀ (runs of 64 k) are coalesced.
__global__ void __launch_bounds__(256, 2) split_transpose_kernel(const double* __restrict__ X, int64_t K, int l,
                                                              uint32_t lmagic, int64_t Kpad,
                                                              const double* __restrict__ xmean,
                                                              float* __restrict__ hi, float* __restrict__ lo) {
  __shared__ double tile[64][kMaxL + 1];
  // the next tile's 16 loads per thread are issued before this tile's
  // stores, so they are in flight while the stores run (the kernel was
  // latency-bound on alternating load and store phases: ncu long scoreboard)
  double v[16];
  auto load = [&](int64_t k0) {
    const int nrow = (int)imin64(64, K - k0 > 0 ? K - k0 : 0);
    const int cnt = nrow * l;  // ≤ 64·64 = 16·256
    const double* src = X + k0 * l;  // 512-byte aligned (k0 is a multiple of 64)
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // 16-byte loads: elements e, e+1 with e = 2·(tid + 256u)
      const int e = 2 * (threadIdx.x + u * 256);
      if (e + 1 < cnt) {
        const double2 d = *reinterpret_cast<const double2*>(src + e);
        v[2 * u] = d.x;
        v[2 * u + 1] = d.y;
      } else {
        v[2 * u] = e < cnt ? src[e] : 0.0;
        v[2 * u + 1] = 0.0;
      }
    }
    return cnt;
  };
  int64_t k0 = (int64_t)blockIdx.x * 64;
  int cnt = k0 < Kpad ? load(k0) : 0;
  for (; k0 < Kpad; k0 += (int64_t)gridDim.x * 64) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = 2 * (threadIdx.x + (u >> 1) * 256) + (u & 1);
      if (idx < 64 * l) {
        // idx / l by multiply-high (exact for idx < 2^32/l; the kernel was
        // instruction-bound on the integer division: ncu issue 67%)
        const int r = l == 1 ? idx : (int)__umulhi((uint32_t)idx, lmagic), j = idx - r * l;
        tile[r][j] = idx < cnt ? v[u] - (xmean ? xmean[j] : 0.0) : 0.0;
      }
    }
    __syncthreads();
    const int64_t kn = k0 + (int64_t)gridDim.x * 64;
    if (kn < Kpad) cnt = load(kn);
    for (int idx = threadIdx.x; idx < 64 * l; idx += 256) {
      const int j = idx >> 6, r = idx & 63;
      const double x = tile[r][j];
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

CUtensorMap tmap_f32(const void* base, int64_t inner, int64_t outer, int64_t ld_elems, int box_inner, int box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld_elems * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RPCA_REQUIRE(r == CUDA_SUCCESS, RPCA_E_CUDA, "cuTensorMapEncodeTiled(f32) failed (%d)", (int)r);
  return tm;
}

int npad_for(int l) { return l <= 16 ? 16 : (l <= 32 ? 32 : (l <= 48 ? 48 : (l <= 56 ? 56 : 64))); }

void split_transpose(Ctx& c, const double* X, int64_t K, int l, int64_t Kpad, float* hi, float* lo,
                     const double* xmean = nullptr) {
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(Kpad, 64), (int64_t)c.num_sms * 8);
  const uint32_t lmagic = l > 1 ? (uint32_t)(((uint64_t(1) << 32) + l - 1) / l) : 0u;  // ⌈2^32 / l⌉
  split_transpose_kernel<<<grid, 256, 0, c.stream>>>(X, K, l, lmagic, Kpad, xmean, hi, lo);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "split_tf32");
}

template <int N>
void launch_ax(Ctx& c, const DenseA& A, const float* hi, const float* lo, int64_t Kpad, int l, const double* cx,
               double* Y) {
  using Cfg = AxCfg<N>;
  const CUtensorMap tA = tmap_f32(A.a, A.n, A.m, A.lda, 32, 128);
  const CUtensorMap tH = tmap_f32(hi, Kpad, l, Kpad, 32, N);  // rows l … N−1: out of bounds ⇒ zero fill
  const CUtensorMap tL = tmap_f32(lo, Kpad, l, Kpad, 32, N);
  ensure_smem((const void*)ax_f32_tc_kernel<N>, Cfg::kSmem);
  const int64_t ntiles = cdiv(A.m, 128);
  const int grid = (int)std::min<int64_t>(ntiles, c.num_sms);
  prof_pre(c);
  ax_f32_tc_kernel<N><<<grid, kThreadsAx, Cfg::kSmem, c.stream>>>(tA, tH, tL, A.m, l, ntiles, (int)(Kpad / 32), cx,
                                                                   Y, c.ax_colpart);
  if (c.ax_colpart) c.ax_colpart_n = ntiles * 4;
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "ax_f32_tc");
}

template <int N>
AtyPlan make_plan(Ctx& c, const DenseA& A) {
  AtyPlan pl;
  pl.nb = cdiv(A.n, 128);
  pl.R = cdiv(A.m, 32);
  pl.CBG = (int)std::min<int64_t>(pl.nb, AtyCfg<N>::kMaxCB);
  pl.Gc = (int)cdiv(pl.nb, pl.CBG);
  pl.Pg = (int)std::max<int64_t>(1, std::min<int64_t>(pl.R, c.num_sms / pl.Gc));
  return pl;
}

template <int N>
void launch_aty(Ctx& c, const DenseA& A, const float* hi, const float* lo, int64_t Kpad, int l, const AtyPlan& pl,
                double* part) {
  using Cfg = AtyCfg<N>;
  const CUtensorMap tA = tmap_f32(A.a, A.n, A.m, A.lda, 128, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
  const CUtensorMap tH = tmap_f32(hi, Kpad, l, Kpad, 32, N);  // rows l … N−1: out of bounds ⇒ zero fill
  const CUtensorMap tL = tmap_f32(lo, Kpad, l, Kpad, 32, N);
  ensure_smem((const void*)aty_f32_tc_kernel<N>, Cfg::kSmem);
  prof_pre(c);
  aty_f32_tc_kernel<N><<<(unsigned)(pl.Gc * pl.Pg), kThreadsAty, Cfg::kSmem, c.stream>>>(tA, tH, tL, pl, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "aty_f32_tc");
}

template <int N>
void aty_f32_run(Ctx& c, const DenseA& A, const float* hi, const float* lo, int64_t Kpad, int l,
                 const double* cmean, const double* sy, double* Z, Arena& ar) {
  const AtyPlan pl = make_plan<N>(c, A);
  double* part = ar.get<double>((size_t)pl.Gc * pl.Pg * pl.CBG * 128 * N);
  launch_aty<N>(c, A, hi, lo, Kpad, l, pl, part);
  const int64_t total = A.n * l;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 16);
  aty_f32_reduce_kernel<<<grid, 256, 0, c.stream>>>(part, pl, N, A.n, l, cmean, sy, Z);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "aty_reduce");
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

void dense_ax_f32(Ctx& c, const DenseA& A, const double* X, int l, const double* cx, double* Y, Arena& ar) {
  const int Np = npad_for(l);
  const int64_t Kpad = cdiv(A.n, 64) * 64;
  float* hi = ar.get<float>((size_t)Np * Kpad);
  float* lo = ar.get<float>((size_t)Np * Kpad);
  split_transpose(c, X, A.n, l, Kpad, hi, lo);
  switch (Np) {
    case 16: launch_ax<16>(c, A, hi, lo, Kpad, l, cx, Y); break;
    case 32: launch_ax<32>(c, A, hi, lo, Kpad, l, cx, Y); break;
    case 48: launch_ax<48>(c, A, hi, lo, Kpad, l, cx, Y); break;
    case 56: launch_ax<56>(c, A, hi, lo, Kpad, l, cx, Y); break;
    default: launch_ax<64>(c, A, hi, lo, Kpad, l, cx, Y); break;
  }
}

size_t aty_f32_ws_bytes(Ctx& c, const DenseA& A, int l) {
  const int Np = npad_for(l);
  Sizer s;
  const int64_t Kpad = cdiv(A.m, 64) * 64;
  s.add<float>((size_t)Np * Kpad);
  s.add<float>((size_t)Np * Kpad);
  AtyPlan pl;
  switch (Np) {
    case 16: pl = make_plan<16>(c, A); break;
    case 32: pl = make_plan<32>(c, A); break;
    case 48: pl = make_plan<48>(c, A); break;
    case 56: pl = make_plan<56>(c, A); break;
    default: pl = make_plan<64>(c, A); break;
  }
  s.add<double>((size_t)pl.Gc * pl.Pg * pl.CBG * 128 * Np);
  return s.total;
}

void dense_aty_f32(Ctx& c, const DenseA& A, const double* Y, int l, const double* cmean, const double* sy,
                   double* Z, Arena& ar, const double* ymean) {
  const int Np = npad_for(l);
  const int64_t Kpad = cdiv(A.m, 64) * 64;
  float* hi = ar.get<float>((size_t)Np * Kpad);
  float* lo = ar.get<float>((size_t)Np * Kpad);
  split_transpose(c, Y, A.m, l, Kpad, hi, lo, ymean);
  switch (Np) {
    case 16: aty_f32_run<16>(c, A, hi, lo, Kpad, l, cmean, sy, Z, ar); break;
    case 32: aty_f32_run<32>(c, A, hi, lo, Kpad, l, cmean, sy, Z, ar); break;
    case 48: aty_f32_run<48>(c, A, hi, lo, Kpad, l, cmean, sy, Z, ar); break;
    case 56: aty_f32_run<56>(c, A, hi, lo, Kpad, l, cmean, sy, Z, ar); break;
    default: aty_f32_run<64>(c, A, hi, lo, Kpad, l, cmean, sy, Z, ar); break;
  }
}

}  // namespace rpca
