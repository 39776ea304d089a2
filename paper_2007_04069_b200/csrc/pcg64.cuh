// numpy's PCG64 bit generator on the device (numpy/random/src/pcg64: XSL-RR
// 128/64), and the Generator methods the reference planner draws through:
//   random()        next_double: (next64 >> 11) * 2^-53
//   integers(n)     next_uint32 (the bit generator's own buffered 32-bit halves:
//                   has_uint32 / uinteger persist across calls) fed to Lemire's
//                   bounded rejection (numpy distributions.c
//                   buffered_bounded_lemire_uint32); n == 1 draws nothing
//   uniform(lo,hi)  lo + (hi - lo) * random()
// Each 64-bit draw steps the 128-bit LCG (state = state * M + inc) and outputs
// rotr64(hi ^ lo, state >> 122) of the new state.
#pragma once

#include <cstdint>

namespace apb {

using u128 = unsigned __int128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// state after `delta` steps (PCG advance: repeated squaring of the affine map)
__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__host__ __device__ __forceinline__ uint64_t pcg_next64(u128& state, u128 inc) {
  state = state * pcg_mult() + inc;
  const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  const unsigned rot = (unsigned)(state >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ __forceinline__ double pcg_next_double(u128& state, u128 inc) {
  return (double)(pcg_next64(state, inc) >> 11) * (1.0 / 9007199254740992.0);
}

// Full numpy PCG64 state: 128-bit state and increment plus the bit generator's
// 32-bit buffer.  Device layout (uint64[6]): state hi, state lo, inc hi, inc lo,
// has_uint32, uinteger -- the fields of bit_generator.state.
struct NpPcg64 {
  u128 state, inc;
  uint32_t has_uint32, uinteger;

  __host__ __device__ static NpPcg64 load(const uint64_t* w) {
    NpPcg64 g;
    g.state = ((u128)w[0] << 64) | (u128)w[1];
    g.inc = ((u128)w[2] << 64) | (u128)w[3];
    g.has_uint32 = (uint32_t)w[4];
    g.uinteger = (uint32_t)w[5];
    return g;
  }
  __host__ __device__ void store(uint64_t* w) const {
    w[0] = (uint64_t)(state >> 64);
    w[1] = (uint64_t)state;
    w[2] = (uint64_t)(inc >> 64);
    w[3] = (uint64_t)inc;
    w[4] = has_uint32;
    w[5] = uinteger;
  }
  __host__ __device__ uint64_t next64() { return pcg_next64(state, inc); }
  __host__ __device__ double next_double() { return pcg_next_double(state, inc); }
  __host__ __device__ uint32_t next32() {
    if (has_uint32) {
      has_uint32 = 0;
      return uinteger;
    }
    const uint64_t v = next64();
    has_uint32 = 1;
    uinteger = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // Generator.integers(0, n) for 1 <= n <= 2^32 (int64 dtype, scalar draw)
  __host__ __device__ int64_t integers(int64_t n) {
    const uint32_t rng = (uint32_t)(n - 1);
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    const uint32_t rng_excl = rng + 1u;
    uint64_t m = (uint64_t)next32() * rng_excl;
    uint32_t leftover = (uint32_t)m;
    if (leftover < rng_excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
      while (leftover < threshold) {
        m = (uint64_t)next32() * rng_excl;
        leftover = (uint32_t)m;
      }
    }
    return (int64_t)(m >> 32);
  }
};

}  // namespace apb
