// philox.cuh — Philox4x32-10 block function for sm_100a (R1).
//
// The paper names no generator (PAPER.md is silent on random numbers); the
// counter-based Philox4x32-10 of Salmon et al. (SC'11) makes every tree
// reproducible independently of launch geometry: counter = (tree j, node i,
// particle label lo32, label hi24 | call << 24), key = seed.  The ten round
// keys are precomputed on the host and read from the kernel-parameter
// constant bank, so each round is 2 IMAD.WIDE.U32 + 2 LOP3 with a constant
// operand and no key-schedule arithmetic in the loop.
#pragma once
#include <cstdint>

namespace rtk {

constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

struct RoundKeys {
  uint32_t k[10][2];
};

inline RoundKeys make_round_keys(uint64_t seed) {
  RoundKeys rk;
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    rk.k[r][0] = k0;
    rk.k[r][1] = k1;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  return rk;
}

__device__ __forceinline__ uint4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3, const RoundKeys& rk) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = static_cast<uint64_t>(kPhiloxM0) * c0;   // IMAD.WIDE.U32
    const uint64_t p1 = static_cast<uint64_t>(kPhiloxM1) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ rk.k[r][0];
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ rk.k[r][1];
    c1 = static_cast<uint32_t>(p1);
    c3 = static_cast<uint32_t>(p0);
    c0 = n0;
    c2 = n2;
  }
  return make_uint4(c0, c1, c2, c3);
}

// Uniform in (0,1): (2*(x>>12)+1)·2^-53 with x = hi:lo.  Built exactly from
// the bits: d = 1 + (x>>12)·2^-52 ∈ [1,2); d − (1 − 2^-53) is exact.
__device__ __forceinline__ double unif53(uint32_t lo, uint32_t hi) {
  const uint32_t mlo = __funnelshift_r(lo, hi, 12);
  const uint32_t mhi = (hi >> 12) | 0x3FF00000u;
  const double d = __hiloint2double(static_cast<int>(mhi), static_cast<int>(mlo));
  return d - 0x1.fffffffffffffp-1;
}

// Uniform in (0,1) from 32 random bits: (2w+1)·2^-33, exactly, via
// d = 1 + w·2^-32 and d − (1 − 2^-33).
__device__ __forceinline__ double unif32(uint32_t w) {
  // (2w+1)·2^-33 = w·2^-32 + 2^-33, exact (33 significant bits): one
  // conversion (XU pipe) and one DFMA with power-of-two immediates
  return fma(static_cast<double>(w), 0x1p-32, 0x1p-33);
}

}  // namespace rtk
