// philox.cuh -- counter-based uniforms for the sampler's Bernoulli draws (device side).
//
// PAPER.md:437 only says "Bernoulli(A_j)"; reading R2 fixes the
// generator so that the oracle and the GPU draw identical u_j:
//   Philox4x32-10 (Salmon et al., SC'11): 10 rounds of
//     (c0,c1,c2,c3) <- (hi(M1*c2) ^ c1 ^ k0, lo(M1*c2), hi(M0*c0) ^ c3 ^ k1, lo(M0*c0))
//   with M0 = 0xD2511F53, M1 = 0xCD9E8D57 and key bumps (0x9E3779B9, 0xBB67AE85);
//   counter = (lo32 j, hi32 j, lo32 b, hi32 b), key = (lo32 seed, hi32 seed);
//   x = (r1 << 32) | r0;  u = (2 (x >> 12) + 1) * 2^-53  in (0, 1), exact in fp64.
#pragma once
#include <cstdint>

namespace dpp {

__device__ __forceinline__ uint4 philox_4x32_10(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * ctr.x, hi0 = __umulhi(0xD2511F53u, ctr.x);
    const uint32_t lo1 = 0xCD9E8D57u * ctr.z, hi1 = __umulhi(0xCD9E8D57u, ctr.z);
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}

__device__ __forceinline__ double uniform_u(uint64_t seed, uint64_t j, uint64_t b) {
  const uint4 r = philox_4x32_10(make_uint4((uint32_t)j, (uint32_t)(j >> 32), (uint32_t)b, (uint32_t)(b >> 32)),
                                 make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const uint64_t x = ((uint64_t)r.y << 32) | (uint64_t)r.x;
  return (double)(((x >> 12) << 1) | 1ull) * 0x1.0p-53;
}

}  // namespace dpp
