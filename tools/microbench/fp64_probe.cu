// DFMA / FFMA dependent latency (unrolled chains, one thread) and DFMA
// throughput (8 independent chains per thread, 1024 threads per SM).
#include <cstdio>
template <class T>
__global__ void lat(T* out, long long* cyc, T a, T b) {
  T x = a;
  long long t0 = clock64();
#pragma unroll
  for (int i = 0; i < 256; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}
template <class T>
__global__ void thr(T* out, long long* cyc, T a, T b) {
  T x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) x[u] = a + u;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = fma(x[u], b, a);
  __syncthreads();
  long long t1 = clock64();
  T s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += x[u];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* od; float* of; long long* c;
  cudaMalloc(&od, 8192); cudaMalloc(&of, 8192); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) {
    lat<double><<<1, 1>>>(od, c, 1.0000001, 0.9999999); cudaDeviceSynchronize(); long long dl = c[0];
    lat<float><<<1, 1>>>(of, c, 1.0001f, 0.9999f); cudaDeviceSynchronize(); long long fl = c[0];
    thr<double><<<1, 1024>>>(od, c, 1.0000001, 0.9999999); cudaDeviceSynchronize(); long long dt = c[0];
    thr<float><<<1, 1024>>>(of, c, 1.0001f, 0.9999f); cudaDeviceSynchronize(); long long ft = c[0];
    const double ops = 64.0 * 64 * 1024;  // FMAs per SM
    if (r) printf("latency: DFMA %.1f FFMA %.1f cycles;  throughput per SM: DFMA %.1f FFMA %.1f per cycle\n",
                  dl / 256.0, fl / 256.0, ops / dt, ops / ft);
  }
  return 0;
}
