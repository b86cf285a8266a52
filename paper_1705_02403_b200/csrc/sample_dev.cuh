// sample_dev.cuh -- PCG32 (rng.hpp:11-33) and prime helpers shared by the
// single-instance and the batched sample_free (sample.cu, batch_build.cu).
#pragma once

#include <cstdint>

namespace gmtb {

constexpr uint64_t kPcgMult = 6364136223846793005ULL;
constexpr uint64_t kPcgInc = 1ULL;  // Pcg32(seed) uses seq = 0 -> inc = 1 (rng.hpp:16-22)

// PCG-XSH-RR output of state `old` (rng.hpp:23-30).
__device__ __forceinline__ uint32_t pcg_out(uint64_t old) {
  const uint32_t xorshifted = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  const uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xorshifted >> rot) | (xorshifted << ((32u - rot) & 31u));
}

// LCG jump-ahead: the state after `delta` steps from `state`.
__device__ __forceinline__ uint64_t pcg_advance(uint64_t state, uint64_t delta) {
  uint64_t acc_mult = 1u, acc_plus = 0u, cur_mult = kPcgMult, cur_plus = kPcgInc;
  while (delta > 0) {
    if (delta & 1u) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1u) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1u;
  }
  return acc_mult * state + acc_plus;
}


inline bool is_prime_h(uint32_t v) {
  if (v < 2) return false;
  for (uint32_t p = 2; p * p <= v; ++p)
    if (v % p == 0) return false;
  return true;
}

inline uint32_t nth_prime_h(int k) {  // sampling.cpp:36-44
  uint32_t c = 1;
  for (int found = 0; found < k;) {
    ++c;
    if (is_prime_h(c)) ++found;
  }
  return c;
}

inline uint64_t pcg_seed_state(uint64_t seed) {  // Pcg32(seed) (rng.hpp:16-22)
  uint64_t state = 0u;
  state = state * kPcgMult + kPcgInc;
  state += seed;
  state = state * kPcgMult + kPcgInc;
  return state;
}


}  // namespace gmtb
