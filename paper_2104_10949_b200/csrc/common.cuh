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

#if defined(__CUDACC__)
// Programmatic dependent launch (sm_90+): a kernel lets the next one in the
// stream start launching CTAs (prologue: AES table expansion, barrier / TMEM
// setup) while its own last CTAs run, and waits for its predecessor's
// results only at griddep_wait().  Every thread calls griddep_wait() before
// its first global read or write of kernel-produced data.
DEV void griddep_launch() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
DEV void griddep_wait() {
#if defined(__CUDA_ARCH__)
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
#endif

HD int32_t imin32(int32_t a, int32_t b) { return a < b ? a : b; }

// Arithmetic right shift of the two's-complement view (ring.py:75-79).
HD uint64_t sar(uint64_t v, int bits) { return (uint64_t)(((int64_t)v) >> bits); }

// Offset uniform over [-2^61, 2^61) from a uniform word (protocols.py:166-168).
HD uint64_t trunc_offset(uint64_t raw) { return (raw >> 2) - (1ull << 61); }

}  // namespace mpc3
