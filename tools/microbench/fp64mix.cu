// Does DFMA (fp64 pipe) run concurrently with DMMA (tensor fp64 subpipe)?
#include <cstdio>
#include <cuda_runtime.h>
template <int ND, int NF>
__global__ void mix(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[ND > 0 ? ND : 1][2] = {};
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int j = 0; j < (NF > 0 ? NF : 1); ++j) f[j] = j + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ND; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int j = 0; j < NF; ++j) f[j] = fma(f[j], 0.999999, 1e-7);
  }
  double s = 0;
  for (int j = 0; j < ND; ++j) s += c[j][0] + c[j][1];
  for (int j = 0; j < NF; ++j) s += f[j];
  if (s == 0.123) out[0] = s;
}
template <int ND, int NF>
void run(const char* name, double* d, int blocks) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 1 << 14; float best = 1e30f, ms;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); mix<ND, NF><<<blocks, 256>>>(d, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double thr = (double)blocks * 256;
  double dmma_fl = thr / 32 * iters * ND * 512.0;  // 256 FMA per DMMA
  double dfma_fl = thr * iters * NF * 2.0;
  printf("%s: %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", name, best, dmma_fl / best / 1e9,
         dfma_fl / best / 1e9, (dmma_fl + dfma_fl) / best / 1e9);
}
int main() {
  double* d; cudaMalloc(&d, 64);
  int blocks = 148 * 8;
  run<4, 0>("dmma only  ", d, blocks);
  run<0, 8>("dfma only  ", d, blocks);
  run<4, 8>("4 dmma+8 dfma", d, blocks);
  run<4, 16>("4 dmma+16dfma", d, blocks);
  run<2, 16>("2 dmma+16dfma", d, blocks);
  return 0;
}
