// Step-0 microbenchmarks: the ALU and HBM ceilings that
// bound the skinny A·X / Aᵀ·Y passes. Not part of the product; prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void read_stream(const double2* __restrict__ a, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + stride), v2 = __ldcs(a + i + 2 * stride), v3 = __ldcs(a + i + 3 * stride);
    s0 += v0.x + v1.x + v2.x + v3.x; s1 += v0.y + v1.y + v2.y + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = a[i]; s0 += v.x; s1 += v.y; }
  if (s0 + s1 == 12345.678) out[0] = s0;
}

__global__ void dfma_peak(double* out, int iters, double x) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = x + j + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.999999, 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 0.123) out[0] = s;
}

__global__ void ffma_peak(float* out, int iters, float x) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = x + j + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.9999f, 1e-7f);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 0.123f) out[0] = s;
}

__global__ void dmma_peak(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[4][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 0.123) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double* dout; CK(cudaMalloc(&dout, 64));
  size_t bytes = (size_t)4 << 30;
  double2* a; CK(cudaMalloc(&a, bytes)); CK(cudaMemset(a, 0, bytes));
  float best_rd = 1e30f, ms;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); read_stream<<<p.multiProcessorCount * 8, 512>>>(a, bytes / 16, dout);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best_rd) best_rd = ms;
  }
  CK(cudaGetLastError());
  int iters = 1 << 16;
  float best_dfma = 1e30f, best_ffma = 1e30f, best_dmma = 1e30f;
  int blocks = p.multiProcessorCount * 8, thr = 256;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); dfma_peak<<<blocks, thr>>>(dout, iters, 1.0); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best_dfma) best_dfma = ms;
    cudaEventRecord(e0); ffma_peak<<<blocks, thr>>>((float*)dout, iters * 4, 1.0f); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best_ffma) best_ffma = ms;
    cudaEventRecord(e0); dmma_peak<<<blocks, thr>>>(dout, iters / 4); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best_dmma) best_dmma = ms;
  }
  CK(cudaGetLastError());
  double nthr = (double)blocks * thr;
  double dfma_tf = nthr * iters * 8 * 2 / (best_dfma * 1e-3) / 1e12;
  double ffma_tf = nthr * iters * 4 * 8 * 2 / (best_ffma * 1e-3) / 1e12;
  double dmma_tf = (double)blocks * (thr / 32) * (iters / 4) * 4 * 512.0 / (best_dmma * 1e-3) / 1e12;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"sm_clock_khz\": %d, "
         "\"mem_clock_khz\": %d, \"bus_bits\": %d, \"read_stream_gbs\": %.1f, \"dfma_tflops\": %.2f, "
         "\"dmma_tflops\": %.2f, \"ffma_tflops\": %.2f}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, clk, memclk, p.memoryBusWidth,
         bytes / (best_rd * 1e-3) / 1e9, dfma_tf, dmma_tf, ffma_tf);
  return 0;
}
