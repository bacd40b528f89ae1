// gepp_step.cu — where does one column step of the register-resident GEPP of
// tslu.cu spend its time?  A stand-alone copy of the step loop (R = 1 row per
// thread, 256 threads) with clock64 stamps taken by thread 0 at the phase
// boundaries: candidate+warp argmax | winner publication | barrier |
// cross-warp max + pivot fetch | elimination.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gepp_step gepp_step.cu
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int kThreads = 256, kWarps = 8;

__device__ __forceinline__ uint32_t piv_key(double v) { return ((uint32_t)__double2hiint(v) & 0x7FFFFFFFu) + 1u; }

template <int LP, int MODE>
__global__ void __launch_bounds__(kThreads, 1) gepp(const double* __restrict__ Y, int steps, long long* __restrict__ t,
                                                     int* __restrict__ piv_out) {
  __shared__ uint2 slot[2][kWarps];
  __shared__ double suinv[2][kWarps];
  __shared__ __align__(16) double buf[2][kWarps][LP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double w[LP];
#pragma unroll
  for (int c = 0; c < LP; ++c) w[c] = Y[((size_t)blockIdx.x * kThreads + tid) * LP + c];
  bool act = true;
  long long acc[5] = {0, 0, 0, 0, 0};
  int pv = 0;
  __syncthreads();
  for (int j = 0; j < steps; ++j) {
    long long c0 = clock64();
    const uint32_t best = act ? piv_key(w[0]) : 0u;
    const uint32_t mk = __reduce_max_sync(0xffffffffu, best);
    const int wl = __ffs(__ballot_sync(0xffffffffu, best == mk)) - 1;
    long long c1 = clock64();
    if (MODE == 2) {
      double2* dst = reinterpret_cast<double2*>(buf[j & 1][warp]);
#pragma unroll
      for (int c = 0; c < LP; c += 2) {
        const double a = __shfl_sync(0xffffffffu, w[c], wl), b = __shfl_sync(0xffffffffu, w[c + 1], wl);
        if (lane == ((c >> 1) & 31)) dst[c >> 1] = make_double2(a, b);
      }
      if (lane == wl) {
        const double u = w[0];
        slot[j & 1][warp] = make_uint2(mk, (uint32_t)tid);
        suinv[j & 1][warp] = (u != 0.0) ? __drcp_rn(u) : 0.0;
      }
    } else if (lane == wl) {
      const double u = w[0];
      slot[j & 1][warp] = make_uint2(mk, (uint32_t)tid);
      suinv[j & 1][warp] = (u != 0.0) ? __drcp_rn(u) : 0.0;
      double2* dst = reinterpret_cast<double2*>(buf[j & 1][warp]);
      if (MODE == 0) {
#pragma unroll
        for (int c = 0; c < LP; c += 2) dst[c >> 1] = make_double2(w[c], w[c + 1]);
      } else if (MODE == 3) {
#pragma unroll
        for (int c = 0; c < 8; c += 2) dst[c >> 1] = make_double2(w[c], w[c + 1]);
      } else {  // only the LP − j live values (Duff-style fallthrough over pairs)
        const int npair = (LP - j + 1) >> 1;
#pragma unroll
        for (int c = 0; c < LP; c += 2)
          if ((c >> 1) < npair) dst[c >> 1] = make_double2(w[c], w[c + 1]);
      }
    }
    long long c2 = clock64();
    __syncthreads();
    long long c3 = clock64();
    uint2 k[kWarps];
    int wi[kWarps];
#pragma unroll
    for (int i = 0; i < kWarps; ++i) {
      k[i] = slot[j & 1][i];
      wi[i] = i;
    }
#pragma unroll
    for (int st = 1; st < kWarps; st <<= 1)
#pragma unroll
      for (int i = 0; i < kWarps; i += 2 * st)
        if (k[i + st].x > k[i].x) { k[i] = k[i + st]; wi[i] = wi[i + st]; }
    const int p = (int)k[0].y;
    const double uinv = suinv[j & 1][wi[0]];
    const double* prow = buf[j & 1][wi[0]];
    pv += p;
    long long c4 = clock64();
    if (act) {
      if (tid == p) {
        act = false;
      } else {
        const double mult = w[0] * uinv;
        if (MODE == 3) {
#pragma unroll
          for (int c = 1; c < 8; ++c) w[c - 1] = fma(-mult, prow[c], w[c]);
          w[7] = w[8];
        } else {
#pragma unroll
          for (int c = 1; c < LP; ++c) w[c - 1] = fma(-mult, prow[c], w[c]);
          w[LP - 1] = 0.0;
        }
      }
    }
    long long c5 = clock64();
    acc[0] += c1 - c0;
    acc[1] += c2 - c1;
    acc[2] += c3 - c2;
    acc[3] += c4 - c3;
    acc[4] += c5 - c4;
  }
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 5; ++i) t[i] = acc[i];
  if (tid == 0) piv_out[blockIdx.x] = pv;
}

template <int LP, int MODE>
void run(int blocks) {
  const int steps = LP - 2;
  std::vector<double> h((size_t)blocks * kThreads * LP);
  uint64_t s = 88172645463325252ull;
  for (auto& x : h) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    x = (double)(s % 2000001) / 1e6 - 1.0;
  }
  double* d;
  long long* t;
  int* pv;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&t, 5 * 8);
  cudaMalloc(&pv, blocks * 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  gepp<LP, MODE><<<blocks, kThreads>>>(d, steps, t, pv);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  gepp<LP, MODE><<<blocks, kThreads>>>(d, steps, t, pv);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long ht[5];
  cudaMemcpy(ht, t, 40, cudaMemcpyDeviceToHost);
  printf("mode %d LP=%d blocks=%d: %.1f us total, %.3f us/step; clocks/step (thread 0): argmax %lld publish %lld barrier %lld "
         "xwarp %lld elim %lld\n",
         MODE, LP, blocks, ms * 1e3, ms * 1e3 / steps, ht[0] / steps, ht[1] / steps, ht[2] / steps, ht[3] / steps,
         ht[4] / steps);
  cudaFree(d);
  cudaFree(t);
  cudaFree(pv);
}

int main() {
  for (int b : {1, 1184}) {
    run<24, 1>(b); run<24, 3>(b);
    run<32, 1>(b); run<32, 3>(b);
    run<56, 1>(b); run<56, 3>(b);
  }
  return 0;
}
