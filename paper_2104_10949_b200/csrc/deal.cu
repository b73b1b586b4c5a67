// Input dealing on the device, bit-exact with the reference's host dealer.
//
// sharing.py:113-118 draws c0 = rng.integers(0, 2^64, n), c1 = likewise, then
// c2 = x - c0 - c1, with numpy's default Generator (PCG64).  For the full
// 64-bit range `integers` returns the raw next_uint64 outputs, i.e. PCG64
// XSL-RR steps s <- s * MULT + inc (mod 2^128), out = rotr64(hi ^ lo, hi >> 58).
// The LCG is seekable (jump-ahead in O(log n)), so each thread produces a
// run of consecutive draws from its own start state: the 2n draws of one
// sharing come out in parallel and equal numpy's sequence word for word.
// The host advances its Generator by 2n afterwards to stay in lockstep.
//
// Also: fixed-point encoding of float64 inputs (ring.py:104-115) on the
// device, so the host->device boundary carries the raw input only.
#include <math.h>

#include "launch.cuh"

namespace mpc3 {

typedef unsigned __int128 u128;
constexpr int DEAL_RUN = 32;  // consecutive draws per thread

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  unsigned rot = (unsigned)(hi >> 58);
  uint64_t v = hi ^ lo;
  return (v >> rot) | (v << ((64 - rot) & 63));
}

// state after `delta` steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 state, uint64_t delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__global__ void deal_kernel(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                            const uint64_t* __restrict__ x, uint64_t* __restrict__ out, uint64_t n) {
  const u128 MULT = mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
  const u128 inc = mk128(inc_hi, inc_lo);
  uint64_t total = 2 * n;
  uint64_t runs = (total + DEAL_RUN - 1) / DEAL_RUN;
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < runs;
       t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t i0 = t * DEAL_RUN;
    u128 s = pcg_advance(mk128(st_hi, st_lo), i0, MULT, inc);
    for (int j = 0; j < DEAL_RUN; ++j) {
      uint64_t i = i0 + j;
      if (i >= total) break;
      s = s * MULT + inc;  // step, then output of the new state
      out[i] = xsl_rr(s);  // draws [0, n) -> c0 plane, [n, 2n) -> c1 plane
    }
  }
}

__global__ void deal_finish_kernel(const uint64_t* __restrict__ x, uint64_t* __restrict__ out, uint64_t n) {
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
    out[2 * n + e] = x[e] - out[e] - out[n + e];
}

__global__ void fx_encode_kernel(const double* __restrict__ x, uint64_t* __restrict__ out, uint64_t n, int t,
                                 int* __restrict__ bad) {
  const double lim = ldexp(1.0, 63 - t), scale = ldexp(1.0, t);
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    double v = x[e];
    double a = fabs(v);
    if (!(a < lim)) {  // also catches NaN / inf
      if (bad) *bad = 1;
      out[e] = 0;
      continue;
    }
    uint64_t mag = (uint64_t)floor(__dadd_rn(__dmul_rn(a, scale), 0.5));  // no FMA contraction: numpy's rounding
    out[e] = v >= 0 ? mag : (uint64_t)0 - mag;
  }
}

}  // namespace mpc3

using namespace mpc3;

extern "C" {

int mpc3_deal_pcg64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, const uint64_t* x,
                    uint64_t* out_trio, uint64_t n, void* stream) {
  if (n == 0) return MPC3_OK;
  uint64_t runs = (2 * n + DEAL_RUN - 1) / DEAL_RUN;
  deal_kernel<<<grid_for(runs, 128), 128, 0, as_stream(stream)>>>(state_hi, state_lo, inc_hi, inc_lo, x, out_trio, n);
  int st = check_launch("deal_pcg64");
  if (st) return st;
  deal_finish_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, out_trio, n);
  return check_launch("deal_finish");
}

int mpc3_fx_encode(const double* x, uint64_t* out, uint64_t n, int t, int* bad, void* stream) {
  if (t <= 0 || t >= 32) return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  fx_encode_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, out, n, t, bad);
  return check_launch("fx_encode");
}

}  // extern "C"
