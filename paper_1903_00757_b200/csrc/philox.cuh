// philox.cuh — counter-based RNG of the product path (host + device).
//
// Philox4x32-10 of Salmon et al., "Parallel random numbers: as easy as 1, 2,
// 3" (SC'11). Counter-based, so every random number the method draws is a
// pure function of (counter, key): negatives of sample q in block (i,j) of
// pool e use counter {q, (i<<16)|j, e, k} (reading R-RNG), the
// walks of the host augmentation use {walk, step, thread, 'WALK'}
// (R-AUG), the embedding init uses {orig_id, k/4, 0, 'INIT'} (R-INIT).
// This file is the product's own implementation; the oracle has its own.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define GV_HD __host__ __device__ __forceinline__
#else
#define GV_HD inline
#endif

namespace gv {

struct u32x4 {
  uint32_t x, y, z, w;
};

GV_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

// Ten rounds; the key is bumped by the Weyl constants between rounds.
GV_HD u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
  constexpr uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(kM0, c.x), lo0 = kM0 * c.x;
    const uint32_t hi1 = mulhi32(kM1, c.z), lo1 = kM1 * c.z;
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += kW0;
    k1 += kW1;
  }
  return c;
}

// floor(x * m / 2^64): maps 64 random bits to a slot in [0, m).
GV_HD uint32_t slot_of(uint64_t x, uint32_t m) {
#if defined(__CUDA_ARCH__)
  return static_cast<uint32_t>(__umul64hi(x, static_cast<uint64_t>(m)));
#else
  return static_cast<uint32_t>((static_cast<unsigned __int128>(x) * m) >> 64);
#endif
}

// One categorical draw from an integer alias table {prob, alias} of m slots
// using words (a, b, c) of a Philox output: slot from (a:b), accept if c < prob.
GV_HD uint32_t alias_pick(uint32_t prob, uint32_t alias, uint32_t slot, uint32_t c) {
  return c < prob ? slot : alias;
}

constexpr uint32_t kTagInit = 0x494E4954u;  // 'INIT'
constexpr uint32_t kTagWalk = 0x57414C4Bu;  // 'WALK'
constexpr uint32_t kTagShuf = 0x53485546u;  // 'SHUF'

}  // namespace gv
