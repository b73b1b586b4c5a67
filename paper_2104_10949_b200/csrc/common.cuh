// Shared definitions for the B200 RSS engine: qualifiers, status codes,
// trio (three co-resident parties) helpers.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#define DEV __device__ __forceinline__
#else
#define HD inline
#define DEV inline
#endif

#include "../../include/mpc3_b200.h"

namespace mpc3 {

// Purpose tags of the reference PRF (prf.py:24-28).
enum Purpose : uint32_t {
  ARITH_ZERO = 1,
  XOR_ZERO = 2,
  TRUNC_RHO = 3,
  TRUNC_R = 4,
  BIN_INPUT = 5,
};

// Arithmetic right shift of the two's-complement view (ring.py:75-79).
HD uint64_t sar(uint64_t v, int bits) { return (uint64_t)(((int64_t)v) >> bits); }

// Offset uniform over [-2^61, 2^61) from a uniform word (protocols.py:166-168).
HD uint64_t trunc_offset(uint64_t raw) { return (raw >> 2) - (1ull << 61); }

}  // namespace mpc3
