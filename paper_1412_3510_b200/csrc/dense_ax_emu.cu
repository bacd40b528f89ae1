// dense_ax_emu.cu — §8(a) steps a2/a5/a8: Y = A·X for a dense fp64 A and a
// thin X on the INT8 tensor cores (tcgen05 kind::i8), an Ozaki-scheme-I
// emulation of the fp64 product.
//
// Why: at l ≳ 24 an fp64 pass is bound by the fp64 tensor pipe, not by HBM
// (2·LP flops per 8-byte element; C3, l = 42: 3.0 TB/s of 6.5, SURVEY.md §8(d)
// "≥ 70% needs FP64 emulation on INT8 tensor cores").  The int8 pipe has
// ~100× the fp64 MMA rate, so eight int8 digits per operand are affordable.
//
// Representation.  Row i of A has a common exponent E_i (2^E_i > max_k |a_ik|,
// one read of A per call: row_exp_kernel), column j of X its own G_j.  Then
//   T = trunc(a·2^(62−E_i)) (int64, |T| < 2^62),  U = T + 0x8080…80 (mod 2^64),
// and the bytes u_p of U give T = Σ_{p=0..7} (u_p − 128)·256^p exactly
// (balanced base-256 digits in [−128, 127]: byte p of U with its top bit
// flipped, read as int8).  Dropping p = 0 and naming D_s the digit of byte
// 7 − s (s = 0 most significant):  a ≈ 2^(E_i−6)·Σ_{s=0..6} D_s·2^(−8s), to
// 2^(E_i−55).  Likewise x ≈ 2^(G_j−6)·Σ_t X_t·2^(−8t).  So
//   (A·X)_ij ≈ 2^(E_i+G_j−12) · Σ_{L=0..6} 2^(−8L) · Σ_{s+t=L} (D_s·X_t)_ij,
// keeping the 28 digit products with s + t ≤ 6 (the rest lie below 2^−56 of
// the leading term).  Each D_s·X_t is an exact int32 product; a level sum has
// ≤ 7 terms of |·| ≤ 2^14·K, so K-chunks of 8192 keep it below 2^30 (exact),
// and the chunk results are combined in fp64.  Error: ~2^−55·2^E_i·2^G_j per
// product term — relative to the row/column maxima, not elementwise
// (DESIGN.md §6).  Extracting the digits is one DMUL, one F2I.S64, one 64-bit
// add and byte permutes (PRMT) per element.
//
// Kernel (one CTA per SM, 448 threads): warp 0 streams A in 128-row × 32-k
// fp64 tiles (two SWIZZLE_128B TMA boxes) plus the matching 32-k block of X's
// digit planes (pre-built by x_slices_kernel, one 1-D bulk copy); warps 2-9
// (two per TMEM lane quarter, 16 k each) turn their row (thread = row = TMEM
// lane) into 7 digit planes and store them to TMEM (8 columns of 4 int8 per
// plane); warp 1 issues, per plane s, a kind::i8 MMA with A = plane s from
// TMEM (TS form) and B = the X planes t = 0..6−s stacked along N, so its
// products land in the level accumulators s..6 (TMEM columns [s·LPn, 7·LPn));
// warps 10-13 fold the 7 int32 levels into fp64 (Horner in 2^−8) at the end
// of every K-chunk, scale by 2^(E_i+G_j−12) and write / add Y.
#include <cudaTypedefs.h>

#include <type_traits>

#include "internal.cuh"

namespace rpca {
namespace {

constexpr int kDigits = 7;                // digit planes per operand = levels kept
constexpr int kKChunkEmu = 8192;          // products per int32 level sum
#ifndef EMU_SPLIT_WARPS
#define EMU_SPLIT_WARPS 16
#endif
constexpr int kSplitW = EMU_SPLIT_WARPS;   // split warps: kSplitW/4 per TMEM lane quarter
constexpr int kGroups = 32 / kSplitW;      // 4-element k groups per split warp and stage
constexpr int kThreadsEmu = 32 * (2 + kSplitW + 4);  // producer, MMA, split, 4 epilogue
constexpr int kATile = 128 * 32 * 8;      // fp64 A stage: 128 rows × 32 k

template <int LPn>
struct EmuCfg {
  static constexpr int kNc = kDigits * LPn;      // level accumulator columns
  static constexpr int kBraw = kDigits * LPn * 32;  // X planes of one 32-k block: 7·LPn rows × 32 B
  static constexpr int kB = (kBraw + 1023) / 1024 * 1024;  // stages stay 1024-aligned (SW128 TMA)
  // separate rings: A tiles (released by the split warps once in registers)
  // and X planes (released by the MMA commit), so A streams ahead of the MMAs
#ifndef EMU_SB
#define EMU_SB 8
#endif
  static constexpr int kStagesB = EMU_SB;
  static constexpr int kStages = (210 * 1024 - kStagesB * kB) / kATile;  // A ring
  static constexpr int kSmem = kStages * kATile + kStagesB * kB + 1024 + 512;
  static constexpr int kSlot0 = kNc;             // then kSets digit sets of 8·kDigits columns
  static constexpr int kSet = 8 * kDigits;
  static constexpr int kSets = (512 - kNc) / kSet >= 3 ? 3 : 2;
  static_assert(kNc + 2 * kSet <= 512, "TMEM: levels + two digit sets");
};

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// K-major no-swizzle operand: 8-row × 16-byte core matrices, (row group g,
// k-chunk c) at (2g + c)·128 bytes: LBO (k direction) 128, SBO (rows) 256
__device__ __forceinline__ uint64_t desc_core(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ void mma_i8_ts(uint32_t dt, uint32_t at, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dt),
      "r"(at), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ bool elect() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

template <int S>
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++s == S) { s = 0; ph ^= 1u; }
  }
};

// 2^e as a double for −1022 ≤ e ≤ 1023
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

// exponent E with 2^E > |a| for every a whose biased exponent field is ≤ f;
// a non-finite value (field 2047) gives kNonFinite: its row / column of the
// product is NaN
constexpr int kNonFinite = 4096;
__host__ __device__ __forceinline__ int exp_of_field(int f) {
  if (f >= 2047) return kNonFinite;
  return f ? f - 1022 : -1021;  // f = 0: zeros and subnormals, all below 2^-1021
}
// 2^(62−E), capped at 2^1022 (E < −960 needs the pre-scale 2^(−960−E) too)
__device__ __forceinline__ double scale_of(int E) { return E >= kNonFinite ? 0.0 : pow2(E < -960 ? 1022 : 62 - E); }

// U = trunc(a·scale) + 0x8080…80 (two 32-bit halves): byte p of U, top bit
// flipped, is the balanced base-256 digit of weight 256^p
__device__ __forceinline__ void biased(double a, double scale, uint32_t& lo, uint32_t& hi) {
  const unsigned long long U = (unsigned long long)__double2ll_rz(a * scale) + 0x8080808080808080ull;
  lo = (uint32_t)U;
  hi = (uint32_t)(U >> 32);
}

// biased() with a·2^(62−E) formed by adding dexp = (62−E)<<20 to the high
// word (a normal, E ≥ −960): fields below flo = E − 61 give 0
__device__ __forceinline__ void biased_exp(double a, uint32_t dexp, int flo, uint32_t& lo, uint32_t& hi) {
  const uint32_t h = (uint32_t)__double2hiint(a);
  const int f = (int)((h >> 20) & 0x7FFu);
  const bool keep = f >= flo && f != 0;
  const double t = __hiloint2double(keep ? (int)(h + dexp) : 0, keep ? __double2loint(a) : 0);
  const unsigned long long U = (unsigned long long)__double2ll_rz(t) + 0x8080808080808080ull;
  lo = (uint32_t)U;
  hi = (uint32_t)(U >> 32);
}

// plane words of four consecutive elements (U halves lo[e], hi[e]): w[s] holds
// digit s (byte 7 − s of U) of elements 0..3 in bytes 0..3, as int8
__device__ __forceinline__ void planes4(const uint32_t (&lo)[4], const uint32_t (&hi)[4], uint32_t (&w)[kDigits]) {
  // pairs of planes from the same 32-bit half: PRMT bytes (b, b−1) of elements
  // (0,1) and (2,3), then split into the two plane words
  const uint32_t h01a = __byte_perm(hi[0], hi[1], 0x6273);  // {e0.b3, e1.b3, e0.b2, e1.b2}
  const uint32_t h23a = __byte_perm(hi[2], hi[3], 0x6273);
  const uint32_t h01b = __byte_perm(hi[0], hi[1], 0x4051);  // {e0.b1, e1.b1, e0.b0, e1.b0}
  const uint32_t h23b = __byte_perm(hi[2], hi[3], 0x4051);
  const uint32_t l01a = __byte_perm(lo[0], lo[1], 0x6273);
  const uint32_t l23a = __byte_perm(lo[2], lo[3], 0x6273);
  const uint32_t l01b = __byte_perm(lo[0], lo[1], 0x0051);  // {e0.b1, e1.b1, -, -}
  const uint32_t l23b = __byte_perm(lo[2], lo[3], 0x0051);
  w[0] = __byte_perm(h01a, h23a, 0x5410) ^ 0x80808080u;  // byte 7
  w[1] = __byte_perm(h01a, h23a, 0x7632) ^ 0x80808080u;  // byte 6
  w[2] = __byte_perm(h01b, h23b, 0x5410) ^ 0x80808080u;  // byte 5
  w[3] = __byte_perm(h01b, h23b, 0x7632) ^ 0x80808080u;  // byte 4
  w[4] = __byte_perm(l01a, l23a, 0x5410) ^ 0x80808080u;  // byte 3
  w[5] = __byte_perm(l01a, l23a, 0x7632) ^ 0x80808080u;  // byte 2
  w[6] = __byte_perm(l01b, l23b, 0x5410) ^ 0x80808080u;  // byte 1
}

// E[i] = exponent of row i's largest |a_ik| (+1): one warp per row.  With
// `wide` given, the same read also sets *wide = 1 for a row whose largest
// |a_ik| exceeds 1/8 of Σ_k |a_ik| (emulation guard): such a row
// would meet the emulation's row-max-relative truncation (≈ 2^-55·2^E per
// term) on terms far below its maximum, so the call keeps the fp64 DMMA pass.
__global__ void row_exp_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, int* __restrict__ E,
                               int* __restrict__ wide) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
    const double* row = A + i * lda;
    unsigned f = 0;
    double amax = 0.0, s0 = 0.0, s1 = 0.0;
    int64_t k = lane;
    for (; k + 32 < n; k += 64) {
      const double a0 = row[k], a1 = row[k + 32];
      f = max(f, max((unsigned)(__double_as_longlong(a0) >> 52) & 0x7FFu,
                     (unsigned)(__double_as_longlong(a1) >> 52) & 0x7FFu));
      if (wide) {
        amax = fmax(amax, fmax(fabs(a0), fabs(a1)));
        s0 += fabs(a0);
        s1 += fabs(a1);
      }
    }
    for (; k < n; k += 32) {
      const double a0 = row[k];
      f = max(f, (unsigned)(__double_as_longlong(a0) >> 52) & 0x7FFu);
      if (wide) {
        amax = fmax(amax, fabs(a0));
        s0 += fabs(a0);
      }
    }
    f = __reduce_max_sync(0xffffffffu, f);
    if (lane == 0) E[i] = exp_of_field((int)f);
    if (wide) {
      double s = warp_sum(s0 + s1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0 && 8.0 * amax > s) *wide = 1;
    }
  }
}

// Gf[j] = max biased exponent field of column j of X (K × l): per-block
// maxima in shared memory, then one atomicMax per block and column (max is
// order-independent, so deterministic); Gf zeroed before
__global__ void col_field_kernel(const double* __restrict__ X, int64_t K, int l, int* __restrict__ Gf) {
  __shared__ int bm[64];
  for (int j = threadIdx.x; j < 64; j += blockDim.x) bm[j] = 0;
  __syncthreads();
  const int64_t total = K * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)((__double_as_longlong(X[idx]) >> 52) & 0x7FF);
    if (f) atomicMax(bm + (int)(idx % l), f);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < l; j += blockDim.x)
    if (bm[j]) atomicMax(Gf + j, bm[j]);
}

// X digit planes, block b of 32 k (kB bytes apart): rows n' = t·LPn + j
// (plane t, column j), K-major core-matrix layout of desc_core; zero past K
// and past l.  Thread = (column j, 16-k half c of block b): it digitises 16
// elements of column j and writes one 16-byte core-matrix row per plane.
__global__ void x_slices_kernel(const double* __restrict__ X, int64_t K, int l, int LPn, int64_t KB, int kB,
                                const int* __restrict__ Gf, int8_t* __restrict__ Xs) {
  const int64_t total = KB * 2 * LPn;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % LPn);
    const int64_t bc = idx / LPn, b = bc >> 1;
    const int c = (int)(bc & 1);
    const int G = exp_of_field(j < l ? Gf[j] : 0);
    const double pre = G < -960 ? pow2(-960 - G) : 1.0, scale = scale_of(G);
    uint32_t w[kDigits][4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint32_t lo[4], hi[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t k = b * 32 + c * 16 + 4 * g + e;
        const double x = (k < K && j < l) ? X[k * l + j] : 0.0;
        biased(x * pre, scale, lo[e], hi[e]);
      }
      uint32_t pw[kDigits];
      planes4(lo, hi, pw);
#pragma unroll
      for (int t = 0; t < kDigits; ++t) w[t][g] = pw[t];
    }
    int8_t* blk = Xs + b * (int64_t)kB;
#pragma unroll
    for (int t = 0; t < kDigits; ++t) {
      const int np = t * LPn + j;
      *reinterpret_cast<uint4*>(blk + ((np >> 3) * 2 + c) * 128 + (np & 7) * 16) =
          make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]);
    }
  }
}

template <int LPn>
__global__ void __launch_bounds__(kThreadsEmu, 1)
    ax_f64_emu_kernel(const __grid_constant__ CUtensorMap tmA, const int8_t* __restrict__ Xs,
                      const int* __restrict__ E, const int* __restrict__ Gf, int64_t m, int l, int64_t ntiles,
                      int KB, double* __restrict__ Y, double* __restrict__ part) {
  using Cfg = EmuCfg<LPn>;
  constexpr int S = Cfg::kStages, SB = Cfg::kStagesB;
  constexpr int KCH = kKChunkEmu / 32;  // k-blocks per int32 accumulation
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* bring = smem + S * kATile;  // X-plane ring
  uint64_t* full = reinterpret_cast<uint64_t*>(bring + SB * Cfg::kB);
  uint64_t* empty = full + S;       // split warps (A read into registers)
  uint64_t* bfull = empty + S;      // [SB] X planes landed
  uint64_t* bempty = bfull + SB;    // [SB] MMA commit
  uint64_t* sfull = bempty + SB;    // [kSets] split warps (digits in TMEM)
  uint64_t* sfree = sfull + Cfg::kSets;  // [kSets] MMA commit
  uint64_t* acc_full = sfree + Cfg::kSets;  // MMA commit
  uint64_t* acc_empty = acc_full + 1;  // 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // units (tile, K-chunk of KCH k-blocks), dealt round-robin over the CTAs:
  // with several K-chunks per tile every unit writes its own partial (part,
  // 128 × l fp64) and ax_emu_reduce_kernel sums them in chunk order
  const int nkc = (KB + KCH - 1) / KCH;
  const int64_t nunits = ntiles * nkc;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSplitW);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int b = 0; b < Cfg::kSets; ++b) {
      mbar_init(&sfull[b], kSplitW);
      mbar_init(&sfree[b], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // ----------------------------------------------- producer
    const bool leader = elect();
    prefetch_tmap(&tmA);
    Ring<S> rg;
    Ring<SB> rx;
    for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x) {
      const int64_t tile = un / nkc;
      const int kc = (int)(un - tile * nkc);
      for (int kb = kc * KCH; kb < KB && kb < (kc + 1) * KCH; ++kb, rg.next(), rx.next()) {
        mbar_wait(&empty[rg.s], rg.ph ^ 1u);
        uint8_t* st = smem + rg.s * kATile;
        if (leader) {
          mbar_arrive_expect_tx(&full[rg.s], kATile);
          tma_load_2d(st, &tmA, kb * 32, (int32_t)(tile * 128), &full[rg.s]);
          tma_load_2d(st + 16384, &tmA, kb * 32 + 16, (int32_t)(tile * 128), &full[rg.s]);
        }
        __syncwarp();
        mbar_wait(&bempty[rx.s], rx.ph ^ 1u);
        if (leader) {
          mbar_arrive_expect_tx(&bfull[rx.s], Cfg::kBraw);
          bulk_load(bring + rx.s * Cfg::kB, Xs + (int64_t)kb * Cfg::kB, Cfg::kBraw, &bfull[rx.s]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // ------------------------------------------- MMA issuer
    const bool leader = elect();
    Ring<SB> rg;
    Ring<Cfg::kSets> rb;
    int64_t u = 0;  // units issued
    for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x, ++u) {
      const int64_t tile = un / nkc;
      const int kc = (int)(un - tile * nkc);
      const int kb0 = kc * KCH, kb1 = KB < kb0 + KCH ? KB : kb0 + KCH;
      for (int kb = kb0; kb < kb1; ++kb, rg.next(), rb.next()) {
        const int kin = kb - kb0;
        if (kin == 0) {  // the level accumulators of the last unit must have been read out
          mbar_wait(acc_empty, (uint32_t)(u & 1) ^ 1u);
          fence_after();
        }
        mbar_wait(&sfull[rb.s], rb.ph);
        mbar_wait(&bfull[rg.s], rg.ph);
        fence_after();
        const uint32_t xb = smem_u32(bring + rg.s * Cfg::kB);
        const uint32_t ad = tmem + (uint32_t)(Cfg::kSlot0 + Cfg::kSet * rb.s);
        if (leader) {
#ifndef EMU_NO_MMA
#pragma unroll
          for (int p = 0; p < kDigits; ++p) {
            const int np = (kDigits - p) * LPn;  // X planes t = 0..6−p, levels p..6
#pragma unroll
            for (int n0 = 0; n0 < np; n0 += 256) {
              const int nc = np - n0 < 256 ? np - n0 : 256;
              mma_i8_ts(tmem + (uint32_t)(p * LPn + n0), ad + 8 * p, desc_core(xb + n0 * 32), idesc_i8(128, nc),
                        (kin != 0 || p != 0) ? 1u : 0u);
            }
          }
#endif
          commit(&sfree[rb.s]);
          commit(&bempty[rg.s]);
          if (kb == kb1 - 1) commit(acc_full);
        }
        __syncwarp();
      }
    }
  } else if (warp < 2 + kSplitW) {  // -------------------------------- split: digits → TMEM
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;  // k = 4·kGroups·h .. of the stage's 32
    const int t = 32 * q + lane;    // tile row = TMEM lane
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    Ring<S> rg;
    Ring<Cfg::kSets> rb;
    for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x) {
      const int64_t tile = un / nkc;
      const int kc = (int)(un - tile * nkc);
      const int64_t row = tile * 128 + t;
      const int Erow = row < m ? E[row] : 0;
      const double scale = scale_of(Erow);
      // rows below 2^-960: 2^(62−E) is not a double — pre-scale by 2^(−960−E)
      const bool tiny = Erow < -960;
      const double pre = tiny ? pow2(-960 - Erow) : 1.0;
      const uint32_t dexp = (uint32_t)(62 - Erow) << 20;  // exponent-field increment of 2^(62−E)
      const int flo = Erow - 61;                            // smallest field kept
      // two instantiations of the k loop: rows below 2^-960 in this warp need
      // the extra pre-scale (warp-uniform choice, once per unit)
      auto kloop = [&](auto tiny_tag) {
      constexpr bool kTiny = decltype(tiny_tag)::value;
      for (int kb = kc * KCH; kb < KB && kb < (kc + 1) * KCH; ++kb, rg.next(), rb.next()) {
        mbar_wait(&full[rg.s], rg.ph);
        const uint8_t* st = smem + rg.s * kATile + t * 128;
        uint32_t w[kGroups][kDigits];  // group g (k = 4·(kGroups·h + g) .. +3), plane s
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
          uint32_t lo[4], hi[4];
          const int k0 = 4 * (kGroups * h + g);  // box k0/16, logical chunks (k0 mod 16)/2 + cc
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {  // logical 16-byte chunk c sits at c ^ (t mod 8)
            const int c = ((k0 & 15) >> 1) + cc;
            const double2 v = *reinterpret_cast<const double2*>(st + (k0 >> 4) * 16384 + ((c ^ (t & 7)) << 4));
#ifdef EMU_NO_SPLIT
            lo[2 * cc] = __double2loint(v.x); hi[2 * cc] = __double2hiint(v.x);
            lo[2 * cc + 1] = __double2loint(v.y); hi[2 * cc + 1] = __double2hiint(v.y);
          }
#pragma unroll
          for (int p = 0; p < kDigits; ++p) w[g][p] = lo[p & 3] ^ hi[(p + 1) & 3];
#else
#if !defined(EMU_NO_FP64) && !defined(EMU_DMUL)
            // the power-of-two scaling as an integer add to the exponent field
            // (exact: the field stays in [1, 1084]; elements below 2^(E−1083)
            // would give T = 0 and are zeroed) — the fp64 pipe, shared with
            // the tensor cores, then runs only the conversion
            if constexpr (kTiny) {
              biased(v.x * pre, scale, lo[2 * cc], hi[2 * cc]);
              biased(v.y * pre, scale, lo[2 * cc + 1], hi[2 * cc + 1]);
            } else {
              biased_exp(v.x, dexp, flo, lo[2 * cc], hi[2 * cc]);
              biased_exp(v.y, dexp, flo, lo[2 * cc + 1], hi[2 * cc + 1]);
            }
#elif defined(EMU_NO_FP64)  // ablation: the digit arithmetic without its fp64-pipe instructions
            lo[2 * cc] = __double2loint(v.x) + 0x80808080u; hi[2 * cc] = __double2hiint(v.x) + 0x80808080u;
            lo[2 * cc + 1] = __double2loint(v.y) + 0x80808080u; hi[2 * cc + 1] = __double2hiint(v.y) + 0x80808080u;
#else
            biased(kTiny ? v.x * pre : v.x, scale, lo[2 * cc], hi[2 * cc]);
            biased(kTiny ? v.y * pre : v.y, scale, lo[2 * cc + 1], hi[2 * cc + 1]);
#endif
          }
          planes4(lo, hi, w[g]);
#endif
        }
        // the digits (computed from every loaded value) must exist before the
        // stage is released, else the arithmetic — and the wait for the loads
        // — may be scheduled after the arrive and the TMA refill the stage
        // under loads in flight (as found in dense_f32_tc.cu's Aᵀ·Y split)
#pragma unroll
        for (int g = 0; g < kGroups; ++g)
#pragma unroll
          for (int p = 0; p < kDigits; ++p) asm volatile("" ::"r"(w[g][p]) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[rg.s]);  // the row is in registers
        mbar_wait(&sfree[rb.s], rb.ph ^ 1u);
        fence_after();
        const uint32_t at = tmem + lane_off + (uint32_t)(Cfg::kSlot0 + Cfg::kSet * rb.s + kGroups * h);
#pragma unroll
        for (int p = 0; p < kDigits; ++p) {
          if constexpr (kGroups == 4)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(at + 8 * p),
                         "r"(w[0][p]), "r"(w[1][p]), "r"(w[2][p]), "r"(w[3][p])
                         : "memory");
          else if constexpr (kGroups == 2)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(at + 8 * p), "r"(w[0][p]),
                         "r"(w[1][p])
                         : "memory");
          else
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(at + 8 * p), "r"(w[0][p])
                         : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfull[rb.s]);
      }
      };
      if (__any_sync(0xffffffffu, tiny)) kloop(std::true_type{});
      else kloop(std::false_type{});
    }
  } else {  // ---------------------------------------------------- epilogue
    const int q = warp & 3;
    const int t = 32 * q + lane;
    int64_t u = 0;
    for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x, ++u) {
      const int64_t tile = un / nkc;
      const int64_t row = tile * 128 + t;
      const int Er = row < m ? E[row] : 0;
      {
        mbar_wait(acc_full, (uint32_t)(u & 1));
        fence_after();
#pragma unroll
        for (int c0 = 0; c0 < LPn; c0 += 16) {  // 16 output columns at a time
          double s[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) s[j] = 0.0;
#pragma unroll
          for (int L = kDigits - 1; L >= 0; --L) {  // Horner in 2^−8 over the levels
            uint32_t v[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(L * LPn + c0)));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j) s[j] = fma(s[j], 0x1p-8, (double)(int)v[j]);
          }
          if (row < m) {
            double* y = nkc == 1 ? Y + row * l : part + (un * 128 + t) * l;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (c0 + j < l) {
                const int Gj = exp_of_field(__ldg(Gf + c0 + j));
                const int e = Er + Gj - 12;
                double v = (e >= -1022 && e <= 1023) ? s[j] * pow2(e) : ldexp(s[j], e);
                if (Er >= kNonFinite || Gj >= kNonFinite) v = __longlong_as_double(0x7FF8000000000000LL);
                y[c0 + j] = v;
              }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Y[row][j] = Σ_{kc ascending} part[tile·nkc + kc][row mod 128][j]
__global__ void ax_emu_reduce_kernel(const double* __restrict__ part, int64_t m, int l, int nkc,
                                     double* __restrict__ Y) {
  const int64_t total = m * l;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / l, tile = row >> 7;
    const int64_t off = ((row & 127) * l) + (idx - row * l);
    double s = 0.0;
    for (int kc = 0; kc < nkc; ++kc) s += part[(tile * nkc + kc) * 128 * l + off];
    Y[idx] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

int lpn_of(int l) { return (l + 15) / 16 * 16; }

template <int LPn>
void launch_emu(Ctx& c, const DenseA& A, const int8_t* Xs, const int* E, const int* Gf, int l, int KB, double* Y,
                double* part) {
  using Cfg = EmuCfg<LPn>;
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)A.n, (cuuint64_t)A.m};
  cuuint64_t strides[1] = {(cuuint64_t)A.lda * 8};
  cuuint32_t box[2] = {16, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(A.a), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  RPCA_REQUIRE(r == CUDA_SUCCESS, RPCA_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  ensure_smem((const void*)ax_f64_emu_kernel<LPn>, Cfg::kSmem);
  const int64_t ntiles = cdiv(A.m, 128);
  const int nkc = (int)cdiv(KB, kKChunkEmu / 32);
  const int grid = (int)std::min<int64_t>(ntiles * nkc, c.num_sms);
  prof_pre(c);
  ax_f64_emu_kernel<LPn><<<grid, kThreadsEmu, Cfg::kSmem, c.stream>>>(tm, Xs, E, Gf, A.m, l, ntiles, KB, Y, part);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, c.tag ? c.tag : "ax_f64_emu");
  if (nkc > 1) {
    const unsigned g2 = (unsigned)std::min<int64_t>(cdiv(A.m * l, 256), (int64_t)c.num_sms * 8);
    ax_emu_reduce_kernel<<<g2, 256, 0, c.stream>>>(part, A.m, l, nkc, Y);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "emu_reduce");
  }
}

}  // namespace

bool emu_eligible(const DenseA& A, int l) {
  // the fp64 tensor pipe binds from LP = 32 on (2·LP flops per 8 bytes); the
  // level accumulators plus two digit sets must fit TMEM (LPn ≤ 48)
  return A.dtype == RPCA_F64 && (reinterpret_cast<uintptr_t>(A.a) & 15u) == 0 && (A.lda * 8) % 16 == 0 && l > 24 &&
         lpn_of(l) <= 48 && A.m >= 128 && A.n >= 32;
}

void row_exponents(Ctx& c, const DenseA& A, int* E, int* wide) {
  if (A.m == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(A.m, 8), (int64_t)c.num_sms * 16);
  row_exp_kernel<<<grid, 256, 0, c.stream>>>(static_cast<const double*>(A.a), A.m, A.n, A.lda, E, wide);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "emu_row_exp");
}

size_t emu_ws_bytes(const DenseA& A, int l) {
  Sizer s;
  s.add<int>(64);
  s.add<int8_t>((size_t)cdiv(A.n, 32) * (lpn_of(l) == 32 ? EmuCfg<32>::kB : EmuCfg<48>::kB));
  s.add<double>((size_t)cdiv(A.m, 128) * cdiv(A.n, kKChunkEmu) * 128 * l);  // per-unit partials
  return s.total;
}

void dense_ax_emu(Ctx& c, const DenseA& A, const int* E, const double* X, int l, double* Y, Arena& ar) {
  const int LPn = lpn_of(l);
  const int KB = (int)cdiv(A.n, 32);
  int* Gf = ar.get<int>(64);
  const int kB = LPn == 32 ? EmuCfg<32>::kB : EmuCfg<48>::kB;
  int8_t* Xs = ar.get<int8_t>((size_t)KB * kB);
  const int64_t nkc = cdiv(KB, kKChunkEmu / 32);
  double* part = nkc > 1 ? ar.get<double>((size_t)cdiv(A.m, 128) * nkc * 128 * l) : nullptr;
  RPCA_CUDA(cudaMemsetAsync(Gf, 0, sizeof(int) * 64, c.stream));
  {
    const int64_t total = A.n * (int64_t)l;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 8);
    col_field_kernel<<<grid, 256, 0, c.stream>>>(X, A.n, l, Gf);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "emu_x_exp");
  }
  {
    const int64_t total = (int64_t)KB * 2 * LPn;
    const unsigned grid = (unsigned)std::min<int64_t>(cdiv(total, 256), (int64_t)c.num_sms * 8);
    x_slices_kernel<<<grid, 256, 0, c.stream>>>(X, A.n, l, LPn, KB, kB, Gf, Xs);
    RPCA_CHECK_LAUNCH();
    count_launch(c, 1, "emu_x_slices");
  }
  switch (LPn) {
    case 32: launch_emu<32>(c, A, Xs, E, Gf, l, KB, Y, part); break;
    default: launch_emu<48>(c, A, Xs, E, Gf, l, KB, Y, part); break;
  }
}

}  // namespace rpca
