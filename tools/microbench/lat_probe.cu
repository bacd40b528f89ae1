// Dependent-chain latencies on this GPU (one thread): DFMA, FFMA, DMUL, LDS,
// MUFU.RCP64H, fp64 division.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o /tmp/lat lat_probe.cu && /tmp/lat
#include <cstdio>
__global__ void k(double* out, float* outf, long long* cyc, double a, double b, float fa, float fb) {
  __shared__ double sh[64];
  if (threadIdx.x < 64) sh[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x) return;
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  float y = fa;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) y = fmaf(y, fb, fa);
  long long t2 = clock64();
  int idx = (int)x & 63;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = ((int)sh[idx]) & 63;
  long long t3 = clock64();
  double z = a + idx;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) z = 1.0 / (z + b);
  long long t4 = clock64();
  double w = a;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) w = w * b;
  long long t5 = clock64();
  out[0] = x + z + w;
  outf[0] = y;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
  double* o; float* of; long long* c;
  cudaMalloc(&o, 8); cudaMalloc(&of, 4); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 64>>>(o, of, c, 1.0000001, 0.9999999, 1.0001f, 0.9999f); cudaDeviceSynchronize(); }
  printf("cycles per dependent op (incl. loop overhead): DFMA %.1f  FFMA %.1f  LDS.64+cvt %.1f  fp64 div %.1f  DMUL %.1f\n",
         c[0] / 1024.0, c[1] / 1024.0, c[2] / 1024.0, c[3] / 1024.0, c[4] / 1024.0);
  return 0;
}
