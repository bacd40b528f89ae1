// Probe of the tcgen05 kind::tf32 encodings used by dense_f32_tc.cu:
//   * K-major SWIZZLE_128B smem descriptors for A (128×32) and B (N×32),
//   * the instruction descriptor (M=128, N=64, fp32 accumulate),
//   * TMEM allocation and the 32x32b tcgen05.ld layout of the accumulator,
//   * whether the tensor core truncates or rounds fp32 inputs to tf32,
//   * an MN-major B operand (K rows × N cols, row-major 128B-swizzled slabs).
// Prints one JSON line.  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;   // version (Blackwell)
  d |= (uint64_t)2 << 61;   // SWIZZLE_128B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)            // c_format F32
       | (2u << 7)            // a_format TF32
       | (2u << 10)           // b_format TF32
       | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16)
       | ((uint32_t)(N >> 3) << 17)
       | ((uint32_t)(M >> 4) << 24);
}

// K-major SW128 offset (bytes) of element (r, k) in a tile of 32 fp32 per row
__device__ __forceinline__ uint32_t kmaj_off(int r, int k) {
  return r * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + ((k & 3) << 2);
}

template <int BMN>
__global__ void probe(const float* A, const float* B, float* D, int bmn, uint32_t lbo, uint32_t sbo) {
  // A: 128×32 (row-major, K contiguous); B: 64×32 (K-major, row = n) or, if bmn, 32×64 (row = k)
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  uint8_t* As = base;            // 16 KB
  uint8_t* Bs = base + 16384;    // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * 32; i += blockDim.x) {
    const int r = i / 32, k = i % 32;
    *reinterpret_cast<float*>(As + kmaj_off(r, k)) = A[i];
  }
  if (!bmn) {
    for (int i = tid; i < 64 * 32; i += blockDim.x) {
      const int n = i / 32, k = i % 32;
      *reinterpret_cast<float*>(Bs + kmaj_off(n, k)) = B[n * 32 + k];
    }
  } else {
    // MN-major: two slabs of 32 columns; slab s holds rows k = 0..31 of columns 32s..32s+31,
    // each row 128 B, 128B-swizzled: element (k, n) at s*4096 + kmaj_off(k, n % 32)
    for (int i = tid; i < 32 * 64; i += blockDim.x) {
      const int k = i / 64, n = i % 64;
      *reinterpret_cast<float*>(Bs + (n / 32) * 4096 + kmaj_off(k, n % 32)) = B[k * 64 + n];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(128, 64, 0, bmn);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t da = desc_sw128(smem_u32(As) + ks * 32, 16, 1024);
      uint64_t db;
      if (!bmn) db = desc_sw128(smem_u32(Bs) + ks * 32, 16, 1024);
      else db = desc_sw128(smem_u32(Bs) + ks * 1024, lbo, sbo);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
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
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t v[16];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 16; ++j) D[(warp * 32 + lane) * 64 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
static float rn_tf32(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  uint32_t lsb = (u >> 13) & 1u; u += 0xFFFu + lsb; u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}

int main() {
  const int M = 128, N = 64, K = 32;
  static float A[M * K], B[N * K], Bmn[K * N], D[M * N];
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; };
  for (int i = 0; i < M * K; ++i) A[i] = 1.0f + rnd() * 0.01f + ((i % 3) ? 0.0f : 0x1p-11f + 0x1p-20f);
  for (int i = 0; i < N * K; ++i) B[i] = rnd();
  for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) Bmn[k * N + n] = B[n * K + k];
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, sizeof(A))); CK(cudaMalloc(&dB, sizeof(B))); CK(cudaMalloc(&dD, sizeof(D)));
  CK(cudaMemcpy(dA, A, sizeof(A), cudaMemcpyHostToDevice));
  double err_trunc[6], err_rn[6];
  const uint32_t L[6] = {4096, 1024, 4096, 16, 4096, 8192}, S[6] = {1024, 4096, 4096, 4096, 16, 1024};
  for (int mode = 0; mode < 6; ++mode) {
    CK(cudaMemcpy(dB, mode ? Bmn : B, sizeof(B), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    probe<0><<<1, 128, 32768>>>(dA, dB, dD, mode ? 1 : 0, mode ? L[mode - 1] : 16, mode ? S[mode - 1] : 1024);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(D, dD, sizeof(D), cudaMemcpyDeviceToHost));
    double et = 0, er = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double st = 0, sr = 0;
        for (int k = 0; k < K; ++k) {
          st += (double)trunc_tf32(A[i * K + k]) * trunc_tf32(B[j * K + k]);
          sr += (double)rn_tf32(A[i * K + k]) * rn_tf32(B[j * K + k]);
        }
        et = fmax(et, fabs(D[i * N + j] - st));
        er = fmax(er, fabs(D[i * N + j] - sr));
      }
    err_trunc[mode] = et;
    err_rn[mode] = er;
  }
  printf("{\"kmajor_err_vs_trunc\": %.3e, \"kmajor_err_vs_round\": %.3e", err_trunc[0], err_rn[0]);
  for (int mode = 1; mode < 6; ++mode) printf(", \"mn lbo=%u sbo=%u\": %.3e", L[mode - 1], S[mode - 1], err_trunc[mode]);
  printf("}\n");
  return 0;
}
