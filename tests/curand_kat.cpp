// Known-answer source for Philox4x32-10: the host path of cuRAND's own header
// (/usr/local/cuda/include/curand_philox4x32_x.h, a library routine in the image).
// Reads "c0 c1 c2 c3 k0 k1" lines, prints the four output words.  Test-only.
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#define QUALIFIERS static inline
#include <curand_philox4x32_x.h>
int main(int argc, char** argv) {
  unsigned a[6];
  while (scanf("%u %u %u %u %u %u", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
    uint4 c = {a[0], a[1], a[2], a[3]}; uint2 k = {a[4], a[5]};
    uint4 r = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
}
