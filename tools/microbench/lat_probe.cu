// Dependent-chain latencies (cycles per operation, clock64) of the operations
// on the latency-bound l×l / LU paths: DFMA, DADD, FFMA, double rsqrt/sqrt,
// the Newton reciprocal seed (MUFU.RCP64H), a 64-bit shuffle, a shared-memory
// load and a one-warp-CTA vs 8-warp __syncthreads round trip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void probe(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  __shared__ int idx[64];
  const int t = threadIdx.x;
  if (t < 64) { sm[t] = seed + t; idx[t] = (t + 1) & 63; }
  __syncthreads();
  double x = seed, y = 1.0000001;
  float xf = (float)seed;
  long long c0, c1;
  // DFMA
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-300);
  c1 = clock64(); if (t == 0) cyc[0] = c1 - c0;
  // DADD
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x + y;
  c1 = clock64(); if (t == 0) cyc[1] = c1 - c0;
  // FFMA
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) xf = fmaf(xf, 1.0000001f, 1e-30f);
  c1 = clock64(); if (t == 0) cyc[2] = c1 - c0;
  // double rsqrt
  c0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) x = rsqrt(x + 2.0);
  c1 = clock64(); if (t == 0) cyc[3] = (c1 - c0) * 16;
  // double sqrt
  c0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N / 16; ++i) x = sqrt(x + 2.0);
  c1 = clock64(); if (t == 0) cyc[4] = (c1 - c0) * 16;
  // MUFU.RCP64H seed (approximate reciprocal, top word)
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    x = r + 1.0;
  }
  c1 = clock64(); if (t == 0) cyc[5] = c1 - c0;
  // 64-bit shuffle
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (t + 1) & 31);
  c1 = clock64(); if (t == 0) cyc[6] = c1 - c0;
  // shared-memory pointer chase
  int p = t & 63;
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) p = idx[p];
  c1 = clock64(); if (t == 0) cyc[7] = c1 - c0;
  // __syncthreads round trip (blockDim warps)
  c0 = clock64();
  for (int i = 0; i < N / 16; ++i) { sm[t & 63] += 1.0; __syncthreads(); }
  c1 = clock64(); if (t == 0) cyc[8] = (c1 - c0) * 16;
  // redux.sync max (u32)
  unsigned u = t;
  c0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) u = __reduce_max_sync(0xffffffffu, u) + (unsigned)i;
  c1 = clock64(); if (t == 0) cyc[9] = c1 - c0;
  out[t] = x + xf + p + u + sm[t & 63];
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 16 * 8);
  const char* names[] = {"dfma", "dadd", "ffma", "rsqrt_f64", "sqrt_f64", "rcp_approx_f64", "shfl_64", "lds_chase", "syncthreads", "redux_max"};
  for (int threads : {32, 256}) {
    probe<<<1, threads>>>(out, cyc, 1.5);
    probe<<<1, threads>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"threads\": %d", threads);
    for (int i = 0; i < 10; ++i) printf(", \"%s\": %.1f", names[i], (double)h[i] / N);
    printf("}\n");
  }
  return 0;
}
