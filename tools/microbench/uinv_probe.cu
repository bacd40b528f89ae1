// Cycles of M = U⁻¹ (l×l upper triangular, fp64, shared memory) inside one
// 256-thread CTA: the column-serial back substitution (thread j walks column
// j) against the row sweep (one barrier per row).  Tuning aid for the last
// tournament level of tslu.cu.
#include <cstdio>
constexpr int LP = 56;
template <int V>
__global__ void k(const double* Ug, double* Mg, int l, long long* cyc) {
  __shared__ double U[LP * LP], Ms[52 * 52], udr[LP];
  const int tid = threadIdx.x;
  for (int i = tid; i < l * l; i += 256) U[(i / l) * LP + i % l] = Ug[i];
  __syncthreads();
  for (int j = tid; j < l; j += 256) udr[j] = 1.0 / U[j * LP + j];
  __syncthreads();
  long long t0 = clock64();
  if (V == 0) {
    if (tid < l) {
      const int j = tid;
      for (int i = l - 1; i > j; --i) Ms[i * l + j] = 0.0;
      for (int i = j; i >= 0; --i) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* ui = U + i * LP;
        int t = i + 1;
        for (; t + 3 <= j; t += 4) {
          a0 = fma(ui[t], Ms[t * l + j], a0);
          a1 = fma(ui[t + 1], Ms[(t + 1) * l + j], a1);
          a2 = fma(ui[t + 2], Ms[(t + 2) * l + j], a2);
          a3 = fma(ui[t + 3], Ms[(t + 3) * l + j], a3);
        }
        for (; t <= j; ++t) a0 = fma(ui[t], Ms[t * l + j], a0);
        Ms[i * l + j] = ((i == j ? 1.0 : 0.0) - ((a0 + a1) + (a2 + a3))) * udr[i];
      }
    }
  } else if (V == 4) {
    // as V == 3, M stored straight to global memory
    if (tid < l) {
      const int j = tid;
      double acc[LP];
#pragma unroll
      for (int i = 0; i < LP; ++i) acc[i] = 0.0;
#pragma unroll
      for (int t = LP - 1; t >= 0; --t) {
        if (t >= l) continue;
        const double mt = j >= t ? ((t == j ? 1.0 : 0.0) - acc[t]) * udr[t] : 0.0;
        Mg[t * l + j] = mt;
#pragma unroll
        for (int i = 0; i < t; ++i) acc[i] = fma(U[i * LP + t], mt, acc[i]);
      }
    }
  } else if (V == 3) {
    // right-looking: as soon as M[t][j] is known it updates every row above,
    // acc[i] += U_it·M[t][j] (independent across i): the critical path is one
    // FMA + the division per row
    if (tid < l) {
      const int j = tid;
      double acc[LP];
#pragma unroll
      for (int i = 0; i < LP; ++i) acc[i] = 0.0;
#pragma unroll
      for (int t = LP - 1; t >= 0; --t) {
        const double mt = (t < l && j >= t) ? ((t == j ? 1.0 : 0.0) - acc[t]) * udr[t] : 0.0;
        if (t < l) Ms[t * l + j] = mt;
#pragma unroll
        for (int i = 0; i < t; ++i) acc[i] = fma(U[i * LP + t], mt, acc[i]);
      }
    }
  } else if (V == 2) {
    // thread j keeps column j of M in registers; rows from the bottom, all
    // indices static (i, t unrolled), no barrier: M[i][j] = (δ_ij − Σ_{t=i+1..j} U_it M_tj)/U_ii
    if (tid < l) {
      const int j = tid;
      double mc[LP];
#pragma unroll
      for (int i = LP - 1; i >= 0; --i) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        const double* ui = U + i * LP;
#pragma unroll
        for (int t = i + 1; t < LP; ++t) {
          if (t <= j) {
            const double p = ui[t] * 1.0;
            switch ((t - i - 1) & 3) {
              case 0: a0 = fma(p, mc[t], a0); break;
              case 1: a1 = fma(p, mc[t], a1); break;
              case 2: a2 = fma(p, mc[t], a2); break;
              default: a3 = fma(p, mc[t], a3); break;
            }
          }
        }
        mc[i] = (i < l && j >= i) ? ((i == j ? 1.0 : 0.0) - ((a0 + a1) + (a2 + a3))) * udr[i] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < LP; ++t)
        if (t < l) Ms[t * l + j] = mc[t];
    }
  } else {
    // row sweep, the dot product split over 4 threads per column (lanes 4j..4j+3)
    const int j = tid >> 2, part = tid & 3;
    for (int i = l - 1; i >= 0; --i) {
      double a = 0.0;
      if (j < l && j > i) {
        const double* ui = U + i * LP;
        for (int t = i + 1 + part; t <= j; t += 4) a = fma(ui[t], Ms[t * l + j], a);
      }
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      if (j < l && part == 0) Ms[i * l + j] = j >= i ? ((i == j ? 1.0 : 0.0) - a) * udr[i] : 0.0;
      __syncthreads();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (V != 4)
    for (int i = tid; i < l * l; i += 256) Mg[i] = Ms[i];
  if (tid == 0) cyc[V] = t1 - t0;
}
int main() {
  const int l = 52;
  double h[l * l];
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) h[i * l + j] = j < i ? 0.0 : (j == i ? 1.0 + 0.01 * i : 0.3 / (1 + j - i));
  double *U, *M0, *M1, *M2, *M3;
  long long* c;
  cudaMalloc(&U, sizeof h); cudaMalloc(&M0, sizeof h); cudaMalloc(&M1, sizeof h); cudaMallocManaged(&c, 64); cudaMalloc(&M2, sizeof h); cudaMalloc(&M3, sizeof h);
  cudaMemcpy(U, h, sizeof h, cudaMemcpyHostToDevice);
  for (int r = 0; r < 3; ++r) {
    k<0><<<1, 256>>>(U, M0, l, c);
    k<1><<<1, 256>>>(U, M1, l, c);
    k<2><<<1, 256>>>(U, M2, l, c);
    k<3><<<1, 256>>>(U, M3, l, c);
    k<4><<<1, 256>>>(U, M0, l, c);
    cudaDeviceSynchronize();
  }
  double a[l * l], b[l * l];
  cudaMemcpy(a, M0, sizeof a, cudaMemcpyDeviceToHost);
  cudaMemcpy(b, M1, sizeof b, cudaMemcpyDeviceToHost);
  double d = 0, d2 = 0;
  for (int i = 0; i < l * l; ++i) d = fmax(d, fabs(a[i] - b[i]));
  cudaMemcpy(b, M2, sizeof b, cudaMemcpyDeviceToHost);
  for (int i = 0; i < l * l; ++i) d2 = fmax(d2, fabs(a[i] - b[i]));
  double d3 = 0;
  cudaMemcpy(b, M3, sizeof b, cudaMemcpyDeviceToHost);
  for (int i = 0; i < l * l; ++i) d3 = fmax(d3, fabs(a[i] - b[i]));
  printf("right-looking %lld cycles (max diff %.2e); with global stores %lld cycles\n", c[3], d3, c[4]);
  printf("U^-1 l=%d: column-serial %lld cycles, row sweep (4 threads/column) %lld cycles (max diff %.2e), column in registers %lld cycles (max diff %.2e)\n", l, c[0],
         c[1], d, c[2], d2);
  return 0;
}
