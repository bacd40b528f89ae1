// Probe of the tcgen05 kind::i8 encodings an int8-slice (Ozaki) fp64 pass
// would use:
//   * the instruction descriptor (M=128, N=48, s8 × s8 → s32),
//   * K-major operands in the no-swizzle "core matrix" layout (8 rows × 16 B
//     blocks; LBO/SBO tried both ways) and in the 128B-swizzled layout
//     (128-byte rows = 128 int8 k, 32-byte k-steps, as for tf32),
//   * the s32 accumulator read back with tcgen05.ld 32x32b.
// Prints one JSON line with the max |error| of each layout (0 = exact).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_i8_probe tc_i8_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4)     // c_format S32
       | (1u << 7)     // a_format signed 8-bit
       | (1u << 10)    // b_format signed 8-bit
       | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int M = 128, N = 48;

// mode 0/1: no swizzle, K = 32 (two 16-byte core-matrix columns), core matrix
//   (group g of 8 rows, k-chunk c) at (g·2 + c)·128 bytes; mode 0 passes
//   LBO = 128 (k direction), SBO = 256 (row-group direction); mode 1 swaps them.
// mode 2: 128B swizzle, K = 128 per row (4 k-steps of 32), SBO 1024.
// mode 3: A from TMEM (TS form, 8 columns of 4 int8 per lane), B as mode 0.
__global__ void probe(const int8_t* A, const int8_t* B, int* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  uint8_t* As = base;           // ≤ 16 KB
  uint8_t* Bs = base + 16384;   // ≤ 6 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  const int K = mode == 2 ? 128 : 32;
  auto off = [&](int r, int k) -> uint32_t {
    if (mode == 2) return r * 128 + ((((k >> 4) ^ (r & 7)) & 7) << 4) + (k & 15);
    return ((r >> 3) * 2 + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15);
  };
  for (int i = tid; i < M * K; i += blockDim.x) As[off(i / K, i % K)] = A[i];
  for (int i = tid; i < N * K; i += blockDim.x) Bs[off(i / K, i % K)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (mode == 3) {  // row tid of A → TMEM lane tid, columns 64..71 (4 int8 per column, k ascending)
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) v |= (uint32_t)(uint8_t)A[tid * 32 + 4 * c + b] << (8 * b);
      w[c] = v;
    }
    const uint32_t addr = tmem + ((uint32_t)((tid >> 5) * 32) << 16) + 64;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(M, N);
    const int steps = K / 32;
    if (mode == 3) {
      const uint64_t db = make_desc(smem_u32(Bs), 128, 256, 0);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + 64), "l"(db), "r"(idesc), "r"(0u));
    } else
    for (int ks = 0; ks < steps; ++ks) {
      uint64_t da, db;
      if (mode == 2) {
        da = make_desc(smem_u32(As) + ks * 32, 16, 1024, 2);
        db = make_desc(smem_u32(Bs) + ks * 32, 16, 1024, 2);
      } else {
        const uint32_t lbo = mode == 0 ? 128 : 256, sbo = mode == 0 ? 256 : 128;
        da = make_desc(smem_u32(As), lbo, sbo, 0);
        db = make_desc(smem_u32(Bs), lbo, sbo, 0);
      }
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
  }
  {
    const uint32_t a = smem_u32(&bar);
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(a) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = tid >> 5, lane = tid & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * N + c0 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  static int8_t A[M * 128], B[N * 128];
  static int D[M * N];
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int)((s >> 8) & 0xFF) - 128; };
  for (auto& x : A) x = (int8_t)rnd();
  for (auto& x : B) x = (int8_t)rnd();
  int8_t *dA, *dB;
  int* dD;
  CK(cudaMalloc(&dA, sizeof(A)));
  CK(cudaMalloc(&dB, sizeof(B)));
  CK(cudaMalloc(&dD, sizeof(D)));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
  printf("{");
  for (int mode = 0; mode < 4; ++mode) {
    const int K = mode == 2 ? 128 : 32;
    static int8_t Ak[M * 128], Bk[N * 128];
    for (int i = 0; i < M; ++i) for (int k = 0; k < K; ++k) Ak[i * K + k] = A[i * 128 + k];
    for (int j = 0; j < N; ++j) for (int k = 0; k < K; ++k) Bk[j * K + k] = B[j * 128 + k];
    CK(cudaMemcpy(dA, Ak, M * K, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, Bk, N * K, cudaMemcpyHostToDevice));
    CK(cudaMemset(dD, 0, sizeof(D)));
    probe<<<1, 128, 32768>>>(dA, dB, dD, mode);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost));
    long long err = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        long long r = 0;
        for (int k = 0; k < K; ++k) r += (int)Ak[i * K + k] * (int)Bk[j * K + k];
        err = std::max(err, std::llabs(r - (long long)D[i * N + j]));
      }
    printf("%s\"mode%d\": %lld", mode ? ", " : "", mode, err);
  }
  printf(", \"sample\": %d}\n", D[5 * N + 7]);
  return 0;
}
