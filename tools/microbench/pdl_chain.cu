// pdl_chain.cu — cost of a kernel boundary inside a CUDA graph, with and
// without programmatic dependent launch (PDL): a chain of K dependent small
// kernels (each reads its predecessor's output), captured once, replayed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_chain pdl_chain.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(const double* __restrict__ x, double* __restrict__ y, int n, int wait) {
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] = x[i] * 1.0000001 + 1.0;
}

float run(int K, int n, int grid, bool pdl) {
  double *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = 256;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    const double* x = (k & 1) ? b : a;
    double* y = (k & 1) ? a : b;
    cudaLaunchKernelEx(&cfg, step, x, y, n, pdl ? 1 : 0);
  }
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  cudaFree(a);
  cudaFree(b);
  return ms / 20 / K * 1e3;  // us per kernel
}

int main() {
  for (int n : {1 << 10, 1 << 16, 1 << 20})
    for (int grid : {1, 148, 592})
      printf("n=%8d grid=%4d: %.2f us/kernel plain, %.2f us/kernel PDL\n", n, grid, run(80, n, grid, false),
             run(80, n, grid, true));
  return 0;
}
