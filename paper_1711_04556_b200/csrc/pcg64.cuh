// pcg64.cuh -- device replica of numpy's Generator(PCG64) draws used by the
// search: `integers(n)` (diversify, search.py:92) and `permutation`
// (initial_order, moves.py:55).  numpy 2.x algorithms: pcg64 XSL-RR 128/64
// step-then-output, bitgen next_uint32 buffering the high half
// (has_uint32/uinteger), Lemire bounded integers on next_uint32, and
// Fisher-Yates from the end with masked rejection (random_interval).
#pragma once
#include <cstdint>

namespace rt {

struct Pcg64 {
  uint64_t s_hi, s_lo, i_hi, i_lo;
  uint32_t has32, u32;

  __device__ __forceinline__ void load(const uint64_t* w) {
    s_hi = w[0]; s_lo = w[1]; i_hi = w[2]; i_lo = w[3];
    has32 = static_cast<uint32_t>(w[4]); u32 = static_cast<uint32_t>(w[5]);
  }
  __device__ __forceinline__ void store(uint64_t* w) const {
    w[0] = s_hi; w[1] = s_lo; w[2] = i_hi; w[3] = i_lo; w[4] = has32; w[5] = u32;
  }

  __device__ __forceinline__ uint64_t next64() {
    const uint64_t M_HI = 0x2360ED051FC65DA4ull, M_LO = 0x4385DF649FCCF645ull;
    // state = state * MULT + inc  (mod 2^128)
    uint64_t lo = s_lo * M_LO;
    uint64_t hi = __umul64hi(s_lo, M_LO) + s_lo * M_HI + s_hi * M_LO;
    uint64_t nlo = lo + i_lo;
    hi += i_hi + (nlo < lo ? 1ull : 0ull);
    s_lo = nlo;
    s_hi = hi;
    const unsigned rot = static_cast<unsigned>(s_hi >> 58);
    const uint64_t x = s_hi ^ s_lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  __device__ __forceinline__ uint32_t next32() {
    if (has32) {
      has32 = 0;
      return u32;
    }
    const uint64_t v = next64();
    has32 = 1;
    u32 = static_cast<uint32_t>(v >> 32);
    return static_cast<uint32_t>(v);
  }

  // Generator.integers(n), 1 <= n <= 2^32
  __device__ __forceinline__ uint32_t integers(uint32_t n) {
    const uint32_t rng = n - 1u;
    if (rng == 0) return 0;
    const uint32_t excl = rng + 1u;
    uint64_t m = static_cast<uint64_t>(next32()) * excl;
    uint32_t left = static_cast<uint32_t>(m);
    if (left < excl) {
      const uint32_t thr = (0xFFFFFFFFu - rng) % excl;
      while (left < thr) {
        m = static_cast<uint64_t>(next32()) * excl;
        left = static_cast<uint32_t>(m);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }

  // random_interval(max)
  __device__ __forceinline__ uint32_t interval(uint32_t mx) {
    if (mx == 0) return 0;
    uint32_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4; mask |= mask >> 8; mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > mx) {
    }
    return v;
  }

  // in-place permutation (Generator.shuffle order) of a[0..k)
  template <class T>
  __device__ __forceinline__ void permute(T* a, int k) {
    for (int i = k - 1; i >= 1; --i) {
      const uint32_t j = interval(static_cast<uint32_t>(i));
      T t = a[i]; a[i] = a[j]; a[j] = t;
    }
  }
};

}  // namespace rt
