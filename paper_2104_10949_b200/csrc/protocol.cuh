// Per-element trio protocol logic (three co-resident parties, components in
// registers).  Host+device so the CPU self-check build runs the very same code.
//
// Notation: a trio is the three additive (or XOR) components c0,c1,c2 of a
// replicated sharing; party i holds (c_i, c_{i+1}) (sharing.py:1-12).  A
// reshare keeps party i's local product z_i as its new `hi`, which makes
// z_i the new component i+1 (protocols.py:88-94, 223-230).
#pragma once
#include "aes.cuh"

namespace mpc3 {

struct Trio {
  uint64_t c[3];
};

// Three per-key words of one stream position: W[i] = F(k_i)[w].
struct KeyWords {
  uint64_t k[3];
};

// z_i = x_i*y_i + x_{i+1}*y_i + x_i*y_{i+1} + (F_i - F_{i-1}); c'_{i+1} = z_i
// (protocols.py:79-94, sharing.py:233-240).
HD Trio trio_mul(const Trio& x, const Trio& y, const KeyWords& f) {
  uint64_t z[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int n = (i + 1) % 3, p = (i + 2) % 3;
    z[i] = x.c[i] * y.c[i] + x.c[n] * y.c[i] + x.c[i] * y.c[n] + (f.k[i] - f.k[p]);
  }
  Trio o;
  o.c[1] = z[0];
  o.c[2] = z[1];
  o.c[0] = z[2];
  return o;
}

// XOR-sharing AND gate with zero share F_i ^ F_{i-1} (protocols.py:223-230).
HD Trio trio_and(const Trio& a, const Trio& b, const KeyWords& f) {
  uint64_t z[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int n = (i + 1) % 3, p = (i + 2) % 3;
    z[i] = (a.c[i] & b.c[i]) ^ (a.c[n] & b.c[i]) ^ (a.c[i] & b.c[n]) ^ f.k[i] ^ f.k[p];
  }
  Trio o;
  o.c[1] = z[0];
  o.c[2] = z[1];
  o.c[0] = z[2];
  return o;
}

// Reshare of local products z (already z_i per party) (protocols.py:88-94).
HD Trio trio_reshare(const Trio& z, const KeyWords& f) {
  Trio o;
  o.c[1] = z.c[0] + (f.k[0] - f.k[2]);
  o.c[2] = z.c[1] + (f.k[1] - f.k[0]);
  o.c[0] = z.c[2] + (f.k[2] - f.k[1]);
  return o;
}

// Truncation by `bits` with rho = offset(F(k_2, TRUNC_RHO)), r = F(k_1, TRUNC_R):
// out = (sar(rho+h), sar(c0-rho+c1+c2+h) - r, r) (protocols.py:171-216).
HD Trio trio_truncate(const Trio& x, uint64_t rho_raw, uint64_t r, int bits) {
  uint64_t half = 1ull << (bits - 1);
  uint64_t rho = trunc_offset(rho_raw);
  Trio o;
  o.c[0] = sar(rho + half, bits);
  uint64_t b = (x.c[0] - rho) + x.c[1] + x.c[2];
  o.c[1] = sar(b + half, bits) - r;
  o.c[2] = r;
  return o;
}

HD Trio trio_xor(const Trio& a, const Trio& b) {
  Trio o;
  for (int i = 0; i < 3; ++i) o.c[i] = a.c[i] ^ b.c[i];
  return o;
}
HD Trio trio_shl(const Trio& a, int d) {
  Trio o;
  for (int i = 0; i < 3; ++i) o.c[i] = a.c[i] << d;
  return o;
}

// ReLU family modes (how far the sign circuit runs).
enum SignMode : int {
  MODE_A2B = 0,    // binary sharing of x (a2b, protocols.py:266-295)
  MODE_MSB = 1,    // binary sharing of the sign bit (protocols.py:298-301)
  MODE_DRELU = 2,  // arithmetic {0,1} mask 1 - msb (protocols.py:334-337)
  MODE_RELU = 3,   // relu = x * mask, plus the mask (protocols.py:340-348)
};

// Stream heads of one sign-circuit invocation; counters are the lockstep
// per-purpose counters the host allotted (sharing.py:225-230).
struct SignStreams {
  StreamHead bin;     // BIN_INPUT, 1 counter (k_0 only)
  StreamHead x[7];    // XOR_ZERO, counters j0..j0+6
  StreamHead a[3];    // ARITH_ZERO, counters ja..ja+2 (inject, inject, mask)
  StreamHead ra, rrho, rr;  // fused layer + ReLU: the layer's reshare / truncation streams
};

// Block `blk` of one stream under the three session keys.
template <class T>
HD void prf_block3(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, Word2 w[3]) {
  for (int i = 0; i < 3; ++i) w[i] = prf_block(tab, rk3 + 44 * i, h, blk);
}
#if defined(__CUDACC__)
template <class TT>
HD void prf_block3_dev(const TT& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, Word2 w[3]) {
#if defined(__CUDA_ARCH__)
  uint32_t s[3][4];
  const uint32_t* rks[3] = {rk3, rk3 + 44, rk3 + 88};
  const uint32_t pcs[3] = {h.pc, h.pc ? h.pc + 32 : 0u, h.pc ? h.pc + 64 : 0u};
  const uint32_t s01[3][2] = {{h.s0, h.s1}, {h.s0, h.s1}, {h.s0, h.s1}};
  aes128_ctr<3>(tab, rks, pcs, s01, blk, s);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    w[i].w0 = (uint64_t)bswap32(s[i][0]) | ((uint64_t)bswap32(s[i][1]) << 32);
    w[i].w1 = (uint64_t)bswap32(s[i][2]) | ((uint64_t)bswap32(s[i][3]) << 32);
  }
#endif
}
HD void prf_block3(const SmemTables& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, Word2 w[3]) {
  prf_block3_dev(tab, rk3, h, blk, w);
}
HD void prf_block3(const SmemTables4& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, Word2 w[3]) {
  prf_block3_dev(tab, rk3, h, blk, w);
}
#endif

// Blocks ba and bb of one stream under the three session keys (on the device
// six interleaved AES chains: the Kogge-Stone level's g- and p-halves).
template <class T>
HD void prf_block3x2(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t ba, uint64_t bb, Word2 wa[3],
                     Word2 wb[3]) {
  prf_block3(tab, rk3, h, ba, wa);
  prf_block3(tab, rk3, h, bb, wb);
}
#if defined(__CUDACC__)
template <class TT>
HD void prf_block3x2_dev(const TT& tab, const uint32_t* rk3, StreamHead h, uint64_t ba, uint64_t bb, Word2 wa[3],
                         Word2 wb[3]) {
#if defined(__CUDA_ARCH__)
  uint32_t s[6][4];
  const uint32_t* rks[6] = {rk3, rk3 + 44, rk3 + 88, rk3, rk3 + 44, rk3 + 88};
  const uint32_t p1 = h.pc ? h.pc + 32 : 0u, p2 = h.pc ? h.pc + 64 : 0u;
  const uint32_t pcs[6] = {h.pc, p1, p2, h.pc, p1, p2};
  const uint32_t s01[6][2] = {{h.s0, h.s1}, {h.s0, h.s1}, {h.s0, h.s1}, {h.s0, h.s1}, {h.s0, h.s1}, {h.s0, h.s1}};
  const uint64_t blks[6] = {ba, ba, ba, bb, bb, bb};
  aes128_ctr_n<6>(tab, rks, pcs, s01, blks, s);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    Word2& w = i < 3 ? wa[i] : wb[i - 3];
    w.w0 = (uint64_t)bswap32(s[i][0]) | ((uint64_t)bswap32(s[i][1]) << 32);
    w.w1 = (uint64_t)bswap32(s[i][2]) | ((uint64_t)bswap32(s[i][3]) << 32);
  }
#endif
}
HD void prf_block3x2(const SmemTables& tab, const uint32_t* rk3, StreamHead h, uint64_t ba, uint64_t bb, Word2 wa[3],
                     Word2 wb[3]) {
  prf_block3x2_dev(tab, rk3, h, ba, bb, wa, wb);
}
HD void prf_block3x2(const SmemTables4& tab, const uint32_t* rk3, StreamHead h, uint64_t ba, uint64_t bb,
                     Word2 wa[3], Word2 wb[3]) {
  prf_block3x2_dev(tab, rk3, h, ba, bb, wa, wb);
}
#endif

// Block blk of one stream under session key k (k_0, k_1, k_2).
template <class T>
HD Word2 prf_block_k(const T& tab, const uint32_t* rk3, int k, StreamHead h, uint64_t blk) {
  return prf_block(tab, rk3 + 44 * k, h, blk);
}
#if defined(__CUDACC__)
template <class TT>
HD Word2 prf_block_k_dev(const TT& tab, const uint32_t* rk3, int k, StreamHead h, uint64_t blk) {
  Word2 w;
#if defined(__CUDA_ARCH__)
  uint32_t s[1][4];
  const uint32_t* rks[1] = {rk3 + 44 * k};
  const uint32_t pcs[1] = {h.pc ? h.pc + 32 * k : 0u};
  const uint32_t s01[1][2] = {{h.s0, h.s1}};
  aes128_ctr<1>(tab, rks, pcs, s01, blk, s);
  w.w0 = (uint64_t)bswap32(s[0][0]) | ((uint64_t)bswap32(s[0][1]) << 32);
  w.w1 = (uint64_t)bswap32(s[0][2]) | ((uint64_t)bswap32(s[0][3]) << 32);
#endif
  return w;
}
HD Word2 prf_block_k(const SmemTables& tab, const uint32_t* rk3, int k, StreamHead h, uint64_t blk) {
  return prf_block_k_dev(tab, rk3, k, h, blk);
}
HD Word2 prf_block_k(const SmemTables4& tab, const uint32_t* rk3, int k, StreamHead h, uint64_t blk) {
  return prf_block_k_dev(tab, rk3, k, h, blk);
}
#endif

#if defined(__CUDACC__)
// Keystream replay: a circuit templated on the table type runs unchanged on
// words an earlier phase computed into shared memory, one slot per AES call
// in call order (slot s of pair p at w[(s * P + p) * 3 + key]).
struct Replay {
  const Word2* w;
  int P, p;
  mutable int slot;
};
DEV Word2 prf_block(const Replay& t, const uint32_t*, StreamHead, uint64_t) {
  return t.w[((size_t)t.slot++ * t.P + t.p) * 3];
}
DEV Word2 prf_block_k(const Replay& t, const uint32_t*, int, StreamHead, uint64_t) {
  return t.w[((size_t)t.slot++ * t.P + t.p) * 3];
}
DEV void prf_block3(const Replay& t, const uint32_t*, StreamHead, uint64_t, Word2 w[3]) {
  const Word2* s = t.w + ((size_t)t.slot++ * t.P + t.p) * 3;
  w[0] = s[0];
  w[1] = s[1];
  w[2] = s[2];
}
#endif

// The truncation pair of one block position: rho from k_2 (TRUNC_RHO) and r
// from k_1 (TRUNC_R) (protocols.py:166-216), two blocks interleaved on the
// device.
template <class T>
HD void trunc_words(const T& tab, const uint32_t* rk3, StreamHead hrho, StreamHead hr, uint64_t blk, Word2& rho,
                    Word2& r) {
  rho = prf_block(tab, rk3 + 2 * 44, hrho, blk);
  r = prf_block(tab, rk3 + 1 * 44, hr, blk);
}
#if defined(__CUDACC__)
template <class TT>
HD void trunc_words_dev(const TT& tab, const uint32_t* rk3, StreamHead hrho, StreamHead hr, uint64_t blk,
                        Word2& rho, Word2& r) {
#if defined(__CUDA_ARCH__)
  uint32_t s[2][4];
  const uint32_t s01[2][2] = {{hrho.s0, hrho.s1}, {hr.s0, hr.s1}};
  const uint32_t* rks[2] = {rk3 + 2 * 44, rk3 + 1 * 44};
  const uint32_t pcs[2] = {hrho.pc ? hrho.pc + 64 : 0u, hr.pc ? hr.pc + 32 : 0u};
  aes128_ctr<2>(tab, rks, pcs, s01, blk, s);
  rho.w0 = (uint64_t)bswap32(s[0][0]) | ((uint64_t)bswap32(s[0][1]) << 32);
  rho.w1 = (uint64_t)bswap32(s[0][2]) | ((uint64_t)bswap32(s[0][3]) << 32);
  r.w0 = (uint64_t)bswap32(s[1][0]) | ((uint64_t)bswap32(s[1][1]) << 32);
  r.w1 = (uint64_t)bswap32(s[1][2]) | ((uint64_t)bswap32(s[1][3]) << 32);
#endif
}
HD void trunc_words(const SmemTables& tab, const uint32_t* rk3, StreamHead hrho, StreamHead hr, uint64_t blk,
                    Word2& rho, Word2& r) {
  trunc_words_dev(tab, rk3, hrho, hr, blk, rho, r);
}
HD void trunc_words(const SmemTables4& tab, const uint32_t* rk3, StreamHead hrho, StreamHead hr, uint64_t blk,
                    Word2& rho, Word2& r) {
  trunc_words_dev(tab, rk3, hrho, hr, blk, rho, r);
}
#endif

// The zero-share words of a pair (3 keys) and its truncation words (rho, r)
// together: on the device the five AES blocks run interleaved in one call
// (five independent T-table chains per thread instead of three then two).
template <class T>
HD void reshare_trunc_words(const T& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho, StreamHead hr,
                            uint64_t blk, Word2 w[3], Word2& rho, Word2& r) {
  prf_block3(tab, rk3, ha, blk, w);
  trunc_words(tab, rk3, hrho, hr, blk, rho, r);
}
#if defined(__CUDACC__)
template <class TT>
HD void reshare_trunc_words_dev(const TT& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho, StreamHead hr,
                                uint64_t blk, Word2 w[3], Word2& rho, Word2& r) {
#if defined(__CUDA_ARCH__)
  uint32_t s[5][4];
  const uint32_t s01[5][2] = {{ha.s0, ha.s1}, {ha.s0, ha.s1}, {ha.s0, ha.s1}, {hrho.s0, hrho.s1}, {hr.s0, hr.s1}};
  const uint32_t* rks[5] = {rk3, rk3 + 44, rk3 + 2 * 44, rk3 + 2 * 44, rk3 + 1 * 44};
  const uint32_t pcs[5] = {ha.pc, ha.pc ? ha.pc + 32 : 0u, ha.pc ? ha.pc + 64 : 0u, hrho.pc ? hrho.pc + 64 : 0u,
                           hr.pc ? hr.pc + 32 : 0u};
  aes128_ctr<5>(tab, rks, pcs, s01, blk, s);
  Word2 o[5];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    o[i].w0 = (uint64_t)bswap32(s[i][0]) | ((uint64_t)bswap32(s[i][1]) << 32);
    o[i].w1 = (uint64_t)bswap32(s[i][2]) | ((uint64_t)bswap32(s[i][3]) << 32);
  }
  w[0] = o[0];
  w[1] = o[1];
  w[2] = o[2];
  rho = o[3];
  r = o[4];
#endif
}
HD void reshare_trunc_words(const SmemTables& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho, StreamHead hr,
                            uint64_t blk, Word2 w[3], Word2& rho, Word2& r) {
  reshare_trunc_words_dev(tab, rk3, ha, hrho, hr, blk, w, rho, r);
}
HD void reshare_trunc_words(const SmemTables4& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho,
                            StreamHead hr, uint64_t blk, Word2 w[3], Word2& rho, Word2& r) {
  reshare_trunc_words_dev(tab, rk3, ha, hrho, hr, blk, w, rho, r);
}
#endif

// Key-word provider over a pair of adjacent elements (words 2b, 2b+1 of each
// stream share one AES block per key).
template <class T>
HD void key_words_pair(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, KeyWords& w0,
                       KeyWords& w1) {
  Word2 p[3];
  prf_block3(tab, rk3, h, blk, p);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    w0.k[i] = p[i].w0;
    w1.k[i] = p[i].w1;
  }
}

template <class T>
HD KeyWords key_words_one(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t w) {
  KeyWords o;
#pragma unroll
  for (int i = 0; i < 3; ++i) o.k[i] = prf_word(tab, rk3 + 44 * i, h, w);
  return o;
}

// Local products WITHOUT randomness or relabel; the zero-share words are
// folded in key by key below so only one AES block (2 words) is live at a
// time (register pressure of the fused sign kernel).
HD Trio and_local(const Trio& a, const Trio& b) {
  Trio z;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int n = (i + 1) % 3;
    z.c[i] = (a.c[i] & b.c[i]) ^ (a.c[n] & b.c[i]) ^ (a.c[i] & b.c[n]);
  }
  return z;
}
HD Trio mul_local(const Trio& x, const Trio& y) {
  Trio z;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    int n = (i + 1) % 3;
    z.c[i] = x.c[i] * y.c[i] + x.c[n] * y.c[i] + x.c[i] * y.c[n];
  }
  return z;
}
HD Trio relabel(const Trio& z) {
  Trio o;
  o.c[1] = z.c[0];
  o.c[2] = z.c[1];
  o.c[0] = z.c[2];
  return o;
}
// F(k_k) enters z_k (as +/^ F_i) and z_{k+1} (as -/^ F_{i-1}) (sharing.py:233-250)
HD void fold_word(Trio& z, int k, uint64_t w, bool xor_mode) {
  int k1 = (k + 1) % 3;
  if (xor_mode) {
    z.c[k] ^= w;
    z.c[k1] ^= w;
  } else {
    z.c[k] += w;
    z.c[k1] -= w;
  }
}
template <class T>
HD void fold_pair(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t blk, Trio z[2], bool xor_mode) {
  Word2 w[3];
  prf_block3(tab, rk3, h, blk, w);
#pragma unroll
  for (int k = 0; k < 3; ++k) {  // unrolled: k indexes registers
    fold_word(z[0], k, w[k].w0, xor_mode);
    fold_word(z[1], k, w[k].w1, xor_mode);
  }
}
// the pair's words sit at stream words w, w+1 that may straddle two blocks
template <class T>
HD void fold_words(const T& tab, const uint32_t* rk3, StreamHead h, uint64_t w, Trio z[2], bool xor_mode) {
  if ((w & 1) == 0) {
    fold_pair(tab, rk3, h, w >> 1, z, xor_mode);
    return;
  }
  Word2 a[3];
  prf_block3(tab, rk3, h, w >> 1, a);
#pragma unroll
  for (int k = 0; k < 3; ++k) fold_word(z[0], k, a[k].w1, xor_mode);
  prf_block3(tab, rk3, h, (w + 1) >> 1, a);
#pragma unroll
  for (int k = 0; k < 3; ++k) fold_word(z[1], k, a[k].w0, xor_mode);
}

// Fold the three keys' words of one AES block into a pair's local products:
// sel 0 = aligned (element 0 <- word 2b, element 1 <- word 2b+1), 1 = element
// 0 <- word 2b+1 only, 2 = element 1 <- word 2b only (a pair straddling two
// blocks, the Kogge-Stone p-half at an odd n_total).
HD void fold_sel(Trio z[2], const Word2 w[3], int sel, bool xor_mode) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (sel == 0) {
      fold_word(z[0], k, w[k].w0, xor_mode);
      fold_word(z[1], k, w[k].w1, xor_mode);
    } else if (sel == 1) {
      fold_word(z[0], k, w[k].w1, xor_mode);
    } else {
      fold_word(z[1], k, w[k].w0, xor_mode);
    }
  }
}

// Kogge-Stone level shape of sign_circuit_pair per keystream source: the
// two-phase kernel's replayed words run each level's g- and p-halves
// together (fewer, longer steps: its circuit phase 37.6 -> 33.4 us at 50 K
// elements); the persistent kernel, at its register cap, keeps one AND
// half live at a time (the merged form spills there).
template <class T>
struct MergedLevels {
  static constexpr bool value = false;
};
#if defined(__CUDACC__)
template <>
struct MergedLevels<Replay> {
  static constexpr bool value = true;
};
#endif

// The fused sign circuit for the element pair (2*blk, 2*blk+1) of a tensor of
// n_total elements (n_total sets where the Kogge-Stone p-half lives, word
// n_total + e, protocols.py:247-259).  x is read through `ld` (local element
// index e0, e0+1; second element absent => duplicate of the first, results
// discarded by the caller), twice, so the input shares need not stay live
// across the 7 AND levels.
// Outputs: out[e] (binary or arithmetic per mode) and, for MODE_RELU, mask[e].
// AES blocks per element pair: BIN 1, XOR 3 + 6*(3 + 3) - 3 (the last
// level's p-half is dead: p is never read after the loop, protocols.py:259-263),
// ARITH 3 per mul.
//
// Code shape: the 12 Kogge-Stone AND rounds are one loop of "jobs" (job 0 =
// g = a AND b; odd job 2l-1 = level l's g-half; even job 2l = level l's
// p-half) around ONE three-key AES call site, and the three arithmetic
// multiplications (2 x bit_inject, the ReLU mask) a second loop around another:
// the kernel stays small enough for the instruction cache (the fully inlined
// circuit was 5,192 instructions and stalled on instruction fetch).
template <class T, class Ld>
HD void sign_circuit_pair(const T& tab, const uint32_t* rk3, const SignStreams& st, uint64_t n_total,
                          uint64_t blk, int mode, const Ld& ld, Trio out[2], Trio mask[2]) {
  // a2b input sharing (protocols.py:278-295): w = ((c0+c1)^r, r, 0), x2 = (0,0,c2)
  const Word2 rb = prf_block_k(tab, rk3, 0, st.bin, blk);
  Trio p[2], g[2];
  if constexpr (MergedLevels<T>::value) {
    const uint64_t pw = n_total + 2 * blk;  // stream word of element 0's p-half
    const bool straddle = (pw & 1) != 0;
    {  // level 0: g = a AND b
      Trio t[2];
      for (int e = 0; e < 2; ++e) {
        Trio x = ld(e);
        uint64_t r = e ? rb.w1 : rb.w0;
        Trio a = {{(x.c[0] + x.c[1]) ^ r, r, 0}};
        Trio b = {{0, 0, x.c[2]}};
        p[e] = trio_xor(a, b);
        t[e] = and_local(a, b);
      }
      Word2 w[3];
      prf_block3(tab, rk3, st.x[0], blk, w);
      fold_sel(t, w, 0, true);
      for (int e = 0; e < 2; ++e) g[e] = relabel(t[e]);
    }
    // levels 1-6: the g-half (p AND g << d) and the p-half (p AND p << d) of a
    // level both read the level's input p, so their keystream (words 2 blk of
    // the level's XOR stream, and words n_total + 2 blk) is one six-chain AES
    // call; level 6's p-half is dead (p is not read after the loop)
  #if defined(__CUDA_ARCH__)
  #pragma unroll 1
  #endif
    for (int lvl = 1; lvl <= 6; ++lvl) {
      const int d = 1 << (lvl - 1);
      const StreamHead h = st.x[lvl];
      Trio tg[2], tp[2];
      for (int e = 0; e < 2; ++e) tg[e] = and_local(p[e], trio_shl(g[e], d));
      if (lvl < 6) {
        for (int e = 0; e < 2; ++e) tp[e] = and_local(p[e], trio_shl(p[e], d));
        Word2 wg[3], wp[3];
        prf_block3x2(tab, rk3, h, blk, pw >> 1, wg, wp);
        fold_sel(tg, wg, 0, true);
        fold_sel(tp, wp, straddle ? 1 : 0, true);
        if (straddle) {  // the pair's p-half straddles two blocks (odd n_total)
          prf_block3(tab, rk3, h, (pw >> 1) + 1, wp);
          fold_sel(tp, wp, 2, true);
        }
        for (int e = 0; e < 2; ++e) p[e] = relabel(tp[e]);
      } else {
        Word2 wg[3];
        prf_block3(tab, rk3, h, blk, wg);
        fold_sel(tg, wg, 0, true);
      }
      for (int e = 0; e < 2; ++e) g[e] = trio_xor(g[e], relabel(tg[e]));
    }
  } else {
    const uint64_t pw = n_total + 2 * blk;  // stream word of element 0's p-half
  #if defined(__CUDA_ARCH__)
  #pragma unroll 1
  #endif
    for (int job = 0; job < 12; ++job) {
      const int lvl = (job + 1) >> 1;  // 0, 1, 1, 2, 2, ..., 6
      const int d = lvl > 0 ? 1 << (lvl - 1) : 0;
      const bool phalf = job > 0 && (job & 1) == 0;
      Trio t[2];
      if (job == 0) {
        for (int e = 0; e < 2; ++e) {
          Trio x = ld(e);
          uint64_t r = e ? rb.w1 : rb.w0;
          Trio a = {{(x.c[0] + x.c[1]) ^ r, r, 0}};
          Trio b = {{0, 0, x.c[2]}};
          p[e] = trio_xor(a, b);
          t[e] = and_local(a, b);
        }
      } else {
        for (int e = 0; e < 2; ++e) t[e] = and_local(p[e], trio_shl(phalf ? p[e] : g[e], d));
      }
      const StreamHead h = st.x[lvl];
      const bool straddle = phalf && (pw & 1);
      const uint64_t b0 = phalf ? (pw >> 1) : blk;
  #if defined(__CUDA_ARCH__)
  #pragma unroll 1
  #endif
      for (int sub = 0; sub < (straddle ? 2 : 1); ++sub) {
        Word2 w[3];
        prf_block3(tab, rk3, h, b0 + sub, w);
        fold_sel(t, w, straddle ? 1 + sub : 0, true);
      }
      for (int e = 0; e < 2; ++e) {
        Trio r = relabel(t[e]);
        if (job == 0)
          g[e] = r;
        else if (phalf)
          p[e] = r;
        else
          g[e] = trio_xor(g[e], r);
      }
    }
  }
  Trio s[2];
  for (int e = 0; e < 2; ++e) {  // sum = p_leaf ^ (g << 1), p_leaf rebuilt from x and r
    Trio x = ld(e);
    uint64_t r = e ? rb.w1 : rb.w0;
    Trio pleaf = {{(x.c[0] + x.c[1]) ^ r, r, x.c[2]}};
    s[e] = trio_xor(pleaf, trio_shl(g[e], 1));
  }
  if (mode == MODE_A2B) {
    out[0] = s[0];
    out[1] = s[1];
    return;
  }
  Trio bit[2];
  for (int e = 0; e < 2; ++e)
    for (int i = 0; i < 3; ++i) bit[e].c[i] = s[e].c[i] >> 63;
  if (mode == MODE_MSB) {
    out[0] = bit[0];
    out[1] = bit[1];
    return;
  }
  // bit_inject (protocols.py:304-331): u = s0 + s1 - 2 mul(s0, s1); v = u + s2 - 2 mul(u, s2);
  // drelu = 1 - v (protocols.py:57-66, 334-337); relu = mul(x, drelu) (protocols.py:340-348)
  const int nmul = mode == MODE_DRELU ? 2 : 3;
  Trio u[2], m[2];
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
  for (int k = 0; k < nmul; ++k) {
    Trio t[2];
    for (int e = 0; e < 2; ++e) {
      if (k == 0) {
        Trio t0 = {{bit[e].c[0], 0, 0}}, t1 = {{0, bit[e].c[1], 0}};
        t[e] = mul_local(t0, t1);
      } else if (k == 1) {
        Trio t2 = {{0, 0, bit[e].c[2]}};
        t[e] = mul_local(u[e], t2);
      } else {
        t[e] = mul_local(ld(e), m[e]);
      }
    }
    Word2 w[3];
    prf_block3(tab, rk3, st.a[k], blk, w);
    fold_sel(t, w, 0, false);
    for (int e = 0; e < 2; ++e) {
      Trio pr = relabel(t[e]);
      if (k == 0) {
        u[e].c[0] = bit[e].c[0] - 2 * pr.c[0];
        u[e].c[1] = bit[e].c[1] - 2 * pr.c[1];
        u[e].c[2] = 0 - 2 * pr.c[2];
      } else if (k == 1) {
        m[e].c[0] = 1 - (u[e].c[0] - 2 * pr.c[0]);
        m[e].c[1] = 0 - (u[e].c[1] - 2 * pr.c[1]);
        m[e].c[2] = 0 - (u[e].c[2] + bit[e].c[2] - 2 * pr.c[2]);
      } else {
        out[e] = pr;
      }
    }
  }
  if (mode == MODE_DRELU) {
    out[0] = m[0];
    out[1] = m[1];
    return;
  }
  mask[0] = m[0];
  mask[1] = m[1];
}

// bit_inject alone on binary bit shares (protocols.py:304-331).
template <class T>
HD void inject_pair(const T& tab, const uint32_t* rk3, StreamHead a0, StreamHead a1, uint64_t blk,
                    const Trio bit[2], Trio out[2]) {
  KeyWords f0, f1, h0, h1;
  key_words_pair(tab, rk3, a0, blk, f0, f1);
  key_words_pair(tab, rk3, a1, blk, h0, h1);
  for (int e = 0; e < 2; ++e) {
    Trio t0 = {{bit[e].c[0], 0, 0}}, t1 = {{0, bit[e].c[1], 0}}, t2 = {{0, 0, bit[e].c[2]}};
    Trio pr = trio_mul(t0, t1, e ? f1 : f0);
    Trio u;
    for (int i = 0; i < 3; ++i) u.c[i] = t0.c[i] + t1.c[i] - 2 * pr.c[i];
    Trio pv = trio_mul(u, t2, e ? h1 : h0);
    for (int i = 0; i < 3; ++i) out[e].c[i] = u.c[i] + t2.c[i] - 2 * pv.c[i];
  }
}

#if defined(__CUDACC__)
// The two-phase kernels' circuit as a 3-lane SIMT program.  With the
// keystream replayed from shared memory, a pair's circuit is a chain of
// dependent integer steps; one thread per pair leaves 2 of 8 warps busy.
// Here lane i of a group of three holds component
// i of the pair's two elements: the AND / multiplication cross terms read
// component i+1 from the next lane and the relabel (z_i -> party i+1) takes
// component i-1 from the previous one (warp shuffles), the zero-share words
// are read straight from the slot (lane i folds F(k_i) and F(k_{i-1})), so
// the same circuit runs on three times the lanes with the same slot order
// and results bit-for-bit.  (Measured: barely faster than one thread per pair,
// 32.3 vs 32.6 us at 49 K elements: the keystream phase bounds the kernel,
// profiles/r02_sign2_lanes.txt.)
struct Lane3 {
  const Word2* w;  // keystream slots (pair p's slot s at w[(s * P + p) * 3 + key])
  int P, p;
  int i, nl, pl;  // component; lanes holding components i+1 and i-1
};
DEV uint64_t lane_nxt(const Lane3& L, uint64_t v) { return __shfl_sync(0xffffffffu, v, L.nl); }
DEV uint64_t lane_prv(const Lane3& L, uint64_t v) { return __shfl_sync(0xffffffffu, v, L.pl); }
DEV uint64_t comp(const Trio& t, int i) { return i == 0 ? t.c[0] : (i == 1 ? t.c[1] : t.c[2]); }
// (F(k_i), F(k_{i-1})) of slot s
DEV void lane_words(const Lane3& L, int s, Word2& wi, Word2& wp) {
  const Word2* b = L.w + ((size_t)s * L.P + L.p) * 3;
  wi = b[L.i];
  wp = b[L.i == 0 ? 2 : L.i - 1];
}
// z_i of a local AND / product: x_i y_i + x_{i+1} y_i + x_i y_{i+1}
DEV uint64_t lane_and(uint64_t a, uint64_t an, uint64_t b, uint64_t bn) { return (a & b) ^ (an & b) ^ (a & bn); }
DEV uint64_t lane_mul(uint64_t a, uint64_t an, uint64_t b, uint64_t bn) { return a * b + an * b + a * bn; }

// sign_circuit_pair on Lane3: x[2] the pair's input trios (every lane holds
// both full trios); out / mask: component i of the results.
DEV void sign_circuit_lane(const Lane3& L, uint64_t n_total, int mode, const Trio x[2], uint64_t out[2],
                           uint64_t mask[2]) {
  const int i = L.i;
  const bool straddle = (n_total & 1) != 0;
  const Word2 rb = L.w[(size_t)L.p * 3];  // slot 0: BIN (k_0)
  uint64_t p[2], g[2];
  {  // level 0: g = a AND b with a = ((x0+x1)^r, r, 0), b = (0, 0, x2)
    uint64_t t[2];
    const int n = i == 2 ? 0 : i + 1;
    for (int e = 0; e < 2; ++e) {
      const uint64_t r = e ? rb.w1 : rb.w0;
      const uint64_t a0 = (x[e].c[0] + x[e].c[1]) ^ r;
      const uint64_t ai = i == 0 ? a0 : (i == 1 ? r : 0), an = n == 0 ? a0 : (n == 1 ? r : 0);
      const uint64_t bi = i == 2 ? x[e].c[2] : 0, bn = n == 2 ? x[e].c[2] : 0;
      p[e] = ai ^ bi;
      t[e] = lane_and(ai, an, bi, bn);
    }
    Word2 wi, wp;
    lane_words(L, 1, wi, wp);
    t[0] ^= wi.w0 ^ wp.w0;
    t[1] ^= wi.w1 ^ wp.w1;
    for (int e = 0; e < 2; ++e) g[e] = lane_prv(L, t[e]);
  }
  int slot = 2;
#pragma unroll 1
  for (int lvl = 1; lvl <= 6; ++lvl) {
    const int d = 1 << (lvl - 1);
    uint64_t pn[2], tg[2];
    for (int e = 0; e < 2; ++e) {
      pn[e] = lane_nxt(L, p[e]);
      const uint64_t gn = lane_nxt(L, g[e]);
      tg[e] = lane_and(p[e], pn[e], g[e] << d, gn << d);
    }
    Word2 wi, wp;
    lane_words(L, slot++, wi, wp);
    tg[0] ^= wi.w0 ^ wp.w0;
    tg[1] ^= wi.w1 ^ wp.w1;
    if (lvl < 6) {  // level 6's p-half is dead
      uint64_t tp[2];
      for (int e = 0; e < 2; ++e) tp[e] = lane_and(p[e], pn[e], p[e] << d, pn[e] << d);
      lane_words(L, slot++, wi, wp);
      if (!straddle) {
        tp[0] ^= wi.w0 ^ wp.w0;
        tp[1] ^= wi.w1 ^ wp.w1;
      } else {  // element 0 <- word 2b+1 of this block, element 1 <- word 2b of the next
        tp[0] ^= wi.w1 ^ wp.w1;
        lane_words(L, slot++, wi, wp);
        tp[1] ^= wi.w0 ^ wp.w0;
      }
      for (int e = 0; e < 2; ++e) p[e] = lane_prv(L, tp[e]);
    }
    for (int e = 0; e < 2; ++e) g[e] ^= lane_prv(L, tg[e]);
  }
  uint64_t s[2], bit[2];
  for (int e = 0; e < 2; ++e) {  // sum = p_leaf ^ (g << 1), p_leaf = ((x0+x1)^r, r, x2)
    const uint64_t r = e ? rb.w1 : rb.w0;
    const uint64_t pl = i == 0 ? (x[e].c[0] + x[e].c[1]) ^ r : (i == 1 ? r : x[e].c[2]);
    s[e] = pl ^ (g[e] << 1);
    bit[e] = s[e] >> 63;
  }
  if (mode == MODE_A2B) {
    out[0] = s[0];
    out[1] = s[1];
    return;
  }
  if (mode == MODE_MSB) {
    out[0] = bit[0];
    out[1] = bit[1];
    return;
  }
  // bit_inject and the ReLU mask (the ARITH slots after level 6's g-half)
  const int sa = slot;
  uint64_t bn[2], u[2], m[2];
  for (int e = 0; e < 2; ++e) bn[e] = lane_nxt(L, bit[e]);
  {  // u = s0 + s1 - 2 mul(s0, s1): t0 = (s0, 0, 0), t1 = (0, s1, 0)
    uint64_t z[2];
    for (int e = 0; e < 2; ++e) {
      const uint64_t t0i = i == 0 ? bit[e] : 0, t1i = i == 1 ? bit[e] : 0;
      const uint64_t t0n = i == 2 ? bn[e] : 0, t1n = i == 0 ? bn[e] : 0;
      z[e] = lane_mul(t0i, t0n, t1i, t1n);
    }
    Word2 wi, wp;
    lane_words(L, sa, wi, wp);
    z[0] += wi.w0 - wp.w0;
    z[1] += wi.w1 - wp.w1;
    for (int e = 0; e < 2; ++e) u[e] = (i < 2 ? bit[e] : 0) - 2 * lane_prv(L, z[e]);
  }
  {  // v = u + s2 - 2 mul(u, s2): t2 = (0, 0, s2); drelu = 1 - v
    uint64_t z[2];
    for (int e = 0; e < 2; ++e) {
      const uint64_t t2i = i == 2 ? bit[e] : 0, t2n = i == 1 ? bn[e] : 0;
      z[e] = lane_mul(u[e], lane_nxt(L, u[e]), t2i, t2n);
    }
    Word2 wi, wp;
    lane_words(L, sa + 1, wi, wp);
    z[0] += wi.w0 - wp.w0;
    z[1] += wi.w1 - wp.w1;
    for (int e = 0; e < 2; ++e)
      m[e] = (i == 0 ? 1 : 0) - (u[e] + (i == 2 ? bit[e] : 0) - 2 * lane_prv(L, z[e]));
  }
  if (mode == MODE_DRELU) {
    out[0] = m[0];
    out[1] = m[1];
    return;
  }
  {  // relu = mul(x, drelu)
    const int n = i == 2 ? 0 : i + 1;
    uint64_t z[2];
    for (int e = 0; e < 2; ++e) z[e] = lane_mul(comp(x[e], i), comp(x[e], n), m[e], lane_nxt(L, m[e]));
    Word2 wi, wp;
    lane_words(L, sa + 2, wi, wp);
    z[0] += wi.w0 - wp.w0;
    z[1] += wi.w1 - wp.w1;
    for (int e = 0; e < 2; ++e) out[e] = lane_prv(L, z[e]);
  }
  mask[0] = m[0];
  mask[1] = m[1];
}
#endif

}  // namespace mpc3
