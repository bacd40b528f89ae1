// omega.cu — §8(a) step a1: the random test block Ω.
//
// PAPER.md:163-168 (§2): "apply A to k random vectors ... entries i.i.d. ...
// drawn from a standard normal distribution"; PAPER.md:437-440 (§5): uniform
// on [-1,1] is enough ("robust to the quality of the random numbers").
// Generator: Philox4x32-10 (Salmon et al., SC'11), counter-based so every
// element is computed independently and every rank regenerates the same Ω.
// Counter layout (reading Q7): element e = i·cols + j uses call
// p = e >> 1, counter (lo32 p, hi32 p, 0, stream_id), key (lo32 seed,
// hi32 seed); a, b = the call's two 53-bit uniforms; Box–Muller
// r = sqrt(-2 ln(1-a)), e even → r·cos(2πb), e odd → r·sin(2πb).
// One thread per Philox call; HBM-write bound (16 bytes per call).
#include "internal.cuh"

namespace rpca {
namespace {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0;
  c1 = lo1;
  c2 = n2;
  c3 = lo0;
}

// elements [e0, e0 + total) of the row-major Ω stream (e = i·l + j); pair p
// covers elements 2p and 2p+1
__global__ void omega_kernel(uint64_t seed, uint32_t sid, int64_t e0, int64_t total, int dist, int round32,
                             double* __restrict__ out) {
  const int64_t p0 = e0 >> 1, calls = ((e0 + total + 1) >> 1) - p0;
  const uint32_t key0 = static_cast<uint32_t>(seed), key1 = static_cast<uint32_t>(seed >> 32);
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < calls; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = p0 + q;
    uint32_t c0 = static_cast<uint32_t>(p), c1 = static_cast<uint32_t>(static_cast<uint64_t>(p) >> 32), c2 = 0u,
             c3 = sid;
    uint32_t k0 = key0, k1 = key1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) {
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      philox_round(c0, c1, c2, c3, k0, k1);
    }
    const uint64_t ua = ((static_cast<uint64_t>(c0) << 32) | c1) >> 11;
    const uint64_t ub = ((static_cast<uint64_t>(c2) << 32) | c3) >> 11;
    const double a = static_cast<double>(ua) * 0x1p-53, b = static_cast<double>(ub) * 0x1p-53;
    double v0, v1;
    if (dist == RPCA_GAUSSIAN) {
      const double r = sqrt(-2.0 * log(1.0 - a));
      double s, co;
      sincos(2.0 * 3.141592653589793 * b, &s, &co);
      v0 = r * co;
      v1 = r * s;
    } else {
      v0 = 2.0 * a - 1.0;
      v1 = 2.0 * b - 1.0;
    }
    if (round32) {
      v0 = static_cast<double>(static_cast<float>(v0));
      v1 = static_cast<double>(static_cast<float>(v1));
    }
    const int64_t e = (p << 1) - e0;  // local index of element 2p
    if (e >= 0 && e + 1 < total && ((reinterpret_cast<uintptr_t>(out + e) & 15u) == 0)) {
      *reinterpret_cast<double2*>(out + e) = make_double2(v0, v1);
    } else {
      if (e >= 0) out[e] = v0;
      if (e + 1 < total) out[e + 1] = v1;
    }
  }
}

}  // namespace

void omega(Ctx& c, uint64_t seed, uint32_t sid, int64_t rows, int64_t cols, int dist, int round32, double* out,
           int64_t row0) {
  const int64_t total = rows * cols, e0 = row0 * cols;
  if (total <= 0) return;
  const int64_t calls = ((e0 + total + 1) >> 1) - (e0 >> 1);
  int64_t blocks = cdiv(calls, 256);
  const int64_t cap = (int64_t)c.num_sms * 8;
  if (blocks > cap) blocks = cap;
  omega_kernel<<<(unsigned)blocks, 256, 0, c.stream>>>(seed, sid, e0, total, dist, round32, out);
  RPCA_CHECK_LAUNCH();
  count_launch(c, 1, "omega");
}

}  // namespace rpca
