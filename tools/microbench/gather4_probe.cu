// TMA tile::gather4 on this GPU: four rows of a 2-D fp64 tensor (box {l, 1})
// into shared memory, checked against the source.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int l, const int* rows, double* out) {
  __shared__ __align__(128) double buf[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(su(&bar)),
                 "r"(4 * l * 8) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5, %6}], [%7];" ::"r"(su(buf)), "l"(&tm), "r"(0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]),
        "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
                   su(&bar)) : "memory");
  for (int i = threadIdx.x; i < 4 * l; i += blockDim.x) out[i] = buf[i];
}
int main() {
  const int n = 1000;
  for (int l : {32, 22, 8}) {
    double* h = new double[n * l];
    for (int i = 0; i < n * l; ++i) h[i] = i;
    double *d, *o;
    int* r;
    cudaMalloc(&d, n * l * 8); cudaMalloc(&o, 4 * l * 8); cudaMalloc(&r, 16);
    cudaMemcpy(d, h, n * l * 8, cudaMemcpyHostToDevice);
    int rows[4] = {5, 17, 900, 3};
    cudaMemcpy(r, rows, 16, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)l, (cuuint64_t)n};
    cuuint64_t str[1] = {(cuuint64_t)l * 8};
    cuuint32_t box[2] = {(cuuint32_t)l, 1}, es[2] = {1, 1};
    CUresult e = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 128>>>(tm, l, r, o);
    cudaError_t ce = cudaDeviceSynchronize();
    double g[4 * 64];
    cudaMemcpy(g, o, 4 * l * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int j = 0; j < 4; ++j)
      for (int c = 0; c < l; ++c) bad += g[j * l + c] != h[rows[j] * l + c];
    printf("l=%d encode=%d kernel=%s mismatches=%d  first row %g %g\n", l, (int)e, cudaGetErrorString(ce), bad, g[0], g[1]);
    if (ce != cudaSuccess) return 1;
  }
  return 0;
}
