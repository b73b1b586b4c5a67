// Operand gathers for the ring GEMM: dense / im2col / weight-gradient views of
// a ring tensor (ring.py:225-256 _im2col; nn.py:435-484 conv gradients).
#pragma once
#include "common.cuh"

namespace mpc3 {

struct Operand {
  int mode;
  int64_t rows, k;
  int64_t off, s_r, t0, t1, t2, K1, K2;
  int64_t n, c, h, w, sN, sC, sH, sW;
  int64_t kh, kw, sh, sw, ph, pw, dh, dw, oh, ow;
};

// Element offset of v(r, k) in one component plane, or -1 for a structural zero.
HD int64_t gather_offset(const Operand& o, int64_t r, int64_t k) {
  if (o.mode == MPC3_GATHER_DENSE && o.K1 == 1 && o.K2 >= o.k)  // plain 2-d view: no digit split
    return o.off + r * o.s_r + k * o.t2;
  if (o.mode == MPC3_GATHER_DENSE) {
    int64_t k2 = k % o.K2;
    int64_t q = k / o.K2;
    int64_t k1 = q % o.K1;
    int64_t k0 = q / o.K1;
    return o.off + r * o.s_r + k0 * o.t0 + k1 * o.t1 + k2 * o.t2;
  }
  if (o.mode == MPC3_GATHER_IM2COL) {
    // r = (n, y, x) over (N, OH, OW); k = (c, u, v) over (C, kh, kw)
    int64_t x = r % o.ow, q = r / o.ow;
    int64_t y = q % o.oh, n = q / o.oh;
    int64_t v = k % o.kw;
    q = k / o.kw;
    int64_t u = q % o.kh, c = q / o.kh;
    int64_t iy = y * o.sh + u - o.ph, ix = x * o.sw + v - o.pw;  // dilated coordinates
    if (iy < 0 || ix < 0 || iy > (o.h - 1) * o.dh || ix > (o.w - 1) * o.dw) return -1;
    if (iy % o.dh || ix % o.dw) return -1;
    return n * o.sN + c * o.sC + (iy / o.dh) * o.sH + (ix / o.dw) * o.sW;
  }
  // WGRAD: r = (c, u, v) over (C, kh, kw); k = (n, y, x) over (N, OH, OW)
  int64_t v = r % o.kw, q = r / o.kw;
  int64_t u = q % o.kh, c = q / o.kh;
  int64_t x = k % o.ow;
  q = k / o.ow;
  int64_t y = q % o.oh, n = q / o.oh;
  int64_t iy = y * o.sh + u - o.ph, ix = x * o.sw + v - o.pw;
  if (iy < 0 || ix < 0 || iy >= o.h || ix >= o.w) return -1;
  return n * o.sN + c * o.sC + iy * o.sH + ix * o.sW;
}

// Incremental gather over consecutive k of one row: the divisions happen once
// per run (init), each next() is a digit increment with carries.
struct GatherCursor {
  int64_t base, iy0, ix0;
  int64_t d0, d1, d2;

  HD void init(const Operand& o, int64_t r, int64_t k) {
    if (o.mode == MPC3_GATHER_DENSE) {
      base = o.off + r * o.s_r;
      d2 = k % o.K2;
      int64_t q = k / o.K2;
      d1 = q % o.K1;
      d0 = q / o.K1;
      iy0 = ix0 = 0;
    } else if (o.mode == MPC3_GATHER_IM2COL) {
      int64_t x = r % o.ow, q = r / o.ow;
      int64_t y = q % o.oh, n = q / o.oh;
      base = n * o.sN;
      iy0 = y * o.sh - o.ph;
      ix0 = x * o.sw - o.pw;
      d2 = k % o.kw;
      q = k / o.kw;
      d1 = q % o.kh;
      d0 = q / o.kh;
    } else {
      int64_t v = r % o.kw, q = r / o.kw;
      int64_t u = q % o.kh, c = q / o.kh;
      base = c * o.sC;
      iy0 = u - o.ph;
      ix0 = v - o.pw;
      d2 = k % o.ow;
      q = k / o.ow;
      d1 = q % o.oh;
      d0 = q / o.oh;
    }
  }

  HD int64_t offset(const Operand& o) const {
    if (o.mode == MPC3_GATHER_DENSE) return base + d0 * o.t0 + d1 * o.t1 + d2 * o.t2;
    if (o.mode == MPC3_GATHER_IM2COL) {
      int64_t iy = iy0 + d1, ix = ix0 + d2;  // dilated coordinates
      if (iy < 0 || ix < 0 || iy > (o.h - 1) * o.dh || ix > (o.w - 1) * o.dw) return -1;
      if (o.dh == 1 && o.dw == 1) return base + d0 * o.sC + iy * o.sH + ix * o.sW;
      if (iy % o.dh || ix % o.dw) return -1;
      return base + d0 * o.sC + (iy / o.dh) * o.sH + (ix / o.dw) * o.sW;
    }
    int64_t iy = d1 * o.sh + iy0, ix = d2 * o.sw + ix0;
    if (iy < 0 || ix < 0 || iy >= o.h || ix >= o.w) return -1;
    return base + d0 * o.sN + iy * o.sH + ix * o.sW;
  }

  HD void next(const Operand& o) {
    int64_t s2 = o.mode == MPC3_GATHER_DENSE ? o.K2 : (o.mode == MPC3_GATHER_IM2COL ? o.kw : o.ow);
    int64_t s1 = o.mode == MPC3_GATHER_DENSE ? o.K1 : (o.mode == MPC3_GATHER_IM2COL ? o.kh : o.oh);
    if (++d2 == s2) {
      d2 = 0;
      if (++d1 == s1) {
        d1 = 0;
        ++d0;
      }
    }
  }
};

// __byte_perm on the device, its definition on the host (self-check build).
HD uint32_t perm32(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(a, b, sel);
#else
  uint64_t ab = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) r |= (uint32_t)((ab >> (8 * ((sel >> (4 * i)) & 7))) & 0xff) << (8 * i);
  return r;
#endif
}

// 4x4 byte transpose of four words: r[l] byte e = byte l of a[e] (8 PRMTs).
HD void byte_transpose4(const uint32_t a[4], uint32_t r[4]) {
  uint32_t t0 = perm32(a[0], a[1], 0x5140), t1 = perm32(a[0], a[1], 0x7362);
  uint32_t t2 = perm32(a[2], a[3], 0x5140), t3 = perm32(a[2], a[3], 0x7362);
  r[0] = perm32(t0, t2, 0x5410);
  r[1] = perm32(t0, t2, 0x7632);
  r[2] = perm32(t1, t3, 0x5410);
  r[3] = perm32(t1, t3, 0x7632);
}

// 8x8 byte transpose: w[l] byte e = byte l of v[e] (limb planes of 8 words).
HD void byte_transpose8(const uint64_t v[8], uint64_t w[8]) {
  uint32_t a[4], r0[4], r1[4];
  for (int half = 0; half < 2; ++half) {  // limbs 0-3 from the low words, 4-7 from the high
    for (int e = 0; e < 4; ++e) a[e] = (uint32_t)(v[e] >> (32 * half));
    byte_transpose4(a, r0);
    for (int e = 0; e < 4; ++e) a[e] = (uint32_t)(v[4 + e] >> (32 * half));
    byte_transpose4(a, r1);
    for (int l = 0; l < 4; ++l) w[4 * half + l] = (uint64_t)r0[l] | ((uint64_t)r1[l] << 32);
  }
}

// Value of the packed operand of group g (party, or 0 for a plain operand) at
// (r, kk) with kk in [0, 2K) for the cross-term roles (protocols.py:110-115).
HD uint64_t packed_value(const Operand& o, const uint64_t* src, int64_t plane, int role, int g, int64_t r,
                         int64_t kk) {
  if (role == 2) {
    if (kk >= o.k) return 0;
    int64_t off = gather_offset(o, r, kk);
    return off < 0 ? 0 : src[off];
  }
  if (kk >= 2 * o.k) return 0;
  bool first = kk < o.k;
  int64_t k = first ? kk : kk - o.k;
  int64_t off = gather_offset(o, r, k);
  if (off < 0) return 0;
  int gn = (g + 1) % 3;
  uint64_t self = src[g * plane + off], nxt = src[gn * plane + off];
  if (role == 0) return first ? self + nxt : self;  // [x_i + x_{i+1} | x_i]
  return first ? self : nxt;                        // [y_i | y_{i+1}]
}

}  // namespace mpc3
