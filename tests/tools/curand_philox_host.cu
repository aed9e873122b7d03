// Host-compiled CUDA-toolkit Philox4x32-10 (curand_philox4x32_x.h), used ONLY as an independent
// library known-answer source for the oracle's Philox (tests/test_oracle_philox.py).
// The header's QUALIFIERS macro is overridden so that curand_Philox4x32_10 compiles for the host.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdlib>

int main(int argc, char** argv) {
  // stdin: lines "c0 c1 c2 c3 k0 k1" (decimal); stdout: "x y z w"
  unsigned a[6];
  while (scanf("%u %u %u %u %u %u", &a[0], &a[1], &a[2], &a[3], &a[4], &a[5]) == 6) {
    uint4 c = make_uint4(a[0], a[1], a[2], a[3]);
    uint2 k = make_uint2(a[4], a[5]);
    uint4 o = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
