// Cost of a kernel boundary when consecutive kernels need different shared-
// memory carve-outs: an empty 256-thread kernel with 0 / 48 KB / 200 KB of
// dynamic shared memory launched after a 200 KB kernel, timed with events
// over many back-to-back launches (and via ncu's gpu__time_duration).
#include <cstdio>
__global__ void k_empty(int* p) { if (threadIdx.x == 9999) p[0] = 1; }
__global__ void k_smem(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 9999) { s[0] = 1; p[0] = s[1]; }
}
int main() {
  int* p; cudaMalloc(&p, 4);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int N = 2000;
  auto run = [&](const char* name, int s1, int s2) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a);
      for (int i = 0; i < N; ++i) {
        k_smem<<<148, 256, s1>>>(p);
        k_smem<<<8, 256, s2>>>(p);
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (w) printf("%-40s %.2f us per pair\n", name, 1e3 * ms / N);
    }
  };
  run("200KB then 200KB", 200 * 1024, 200 * 1024);
  run("200KB then 48KB", 200 * 1024, 48 * 1024);
  run("200KB then 0", 200 * 1024, 0);
  run("0 then 0", 0, 0);
  run("48KB then 48KB", 48 * 1024, 48 * 1024);
  return 0;
}
