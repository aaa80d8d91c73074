// Test tool: prints curand's Philox4x32-10 (a LIBRARY routine, curand_philox4x32_x.h)
// for the counters/keys given on stdin, so tests can pin both Philox implementations
// (oracle/ and the CUDA product path) against it.  Host-side only: QUALIFIERS is
// overridden so the header's functions compile for the host.
#define QUALIFIERS static inline __host__ __device__
#include <cstdio>
#include <vector_types.h>
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3);
    uint2 k = make_uint2(k0, k1);
    uint4 r = curand_Philox4x32_10(c, k);
    printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
