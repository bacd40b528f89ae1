// common.cuh — device/host helpers shared by the sm_100a kernels of the
// randomized-PCA hot path (arXiv 1412.3510).  PTX wrappers for mbarrier,
// TMA (cp.async.bulk[.tensor]) and the fp64 tensor-core MMA (DMMA), plus the
// status plumbing of the C ABI (include/rpca.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../include/rpca.h"

namespace rpca {

// ---------------------------------------------------------------- host errors
struct Error {
  rpca_status code;
};

void set_last_error(const char* fmt, ...);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel, size increase)
void ensure_smem(const void* kernel, int bytes);

#define RPCA_CUDA(call)                                                              \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      ::rpca::set_last_error("%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                             cudaGetErrorString(e_));                                \
      throw ::rpca::Error{RPCA_E_CUDA};                                              \
    }                                                                                \
  } while (0)

#define RPCA_CHECK_LAUNCH() RPCA_CUDA(cudaGetLastError())

#define RPCA_REQUIRE(cond, code, ...)                                                \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      ::rpca::set_last_error(__VA_ARGS__);                                           \
      throw ::rpca::Error{code};                                                     \
    }                                                                                \
  } while (0)

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------- device PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Wait for the phase with parity `parity` to complete.  The suspend-time hint
// lets the waiting warp sleep in hardware until the phase flips instead of
// spinning: a spinning warp costs issue slots the working warps need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(0x989680u)
      : "memory");
}

// 2-D TMA tile load global → shared, completion counted on an mbarrier.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// The same with an L2 cache-policy hint (createpolicy: evict_first for data
// streamed once, evict_last for operands many CTAs re-read).
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 3-D TMA tile load global → shared.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, int32_t z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// 1-D bulk copy global → shared (16-byte aligned, size multiple of 16).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// D(8x8) += A(8x4, row) · B(4x8, col), fp64 tensor core.
// Fragments: a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d = {D[lane>>2][2(lane&3)], D[lane>>2][2(lane&3)+1]}.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// 1/u: MUFU seed + two Newton steps (≤ 1 ulp); 0 for u = 0, the exact
// reciprocal for |u| < 2^-1000 (where the flush-to-zero seed is not usable)
__device__ __forceinline__ double rcp_nr(double u) {
  if (fabs(u) < 0x1p-1000) return u != 0.0 ? 1.0 / u : 0.0;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(u));
  double e = fma(-u, r, 1.0);
  r = fma(r, e, r);
  e = fma(-u, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Offset of element (r, c) inside a TMA box of 16 doubles per 128-byte row,
// SWIZZLE_128B (16-byte chunk index XOR row mod 8; box base 1024-aligned).
__device__ __forceinline__ uint32_t swz128_off(uint32_t r, uint32_t c) {
  return r * 128u + ((((c >> 1) ^ (r & 7u)) & 7u) << 4) + ((c & 1u) << 3);
}

}  // namespace rpca
