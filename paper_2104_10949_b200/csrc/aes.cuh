// AES-128 counter-mode keystream, bit-exact with the reference PRF
// (prf.py:31-55: cryptography's AES-128-CTR whose initial counter block is
// purpose_LE16 || index_LE48 || 0^64 and whose per-block increment runs over
// the big-endian 128-bit block).  Block b of stream (key, purpose, index) is
// AES_k(purpose_LE16 || index_LE48 || BE64(b)); it yields words 2b and 2b+1
// as the two little-endian halves of the ciphertext.
//
// T-table implementation: the four 1 KiB round tables and the S-box live in
// shared memory on the device (built once per CTA) and in static host arrays
// for the CPU self-check build (hostcheck.cpp), with one code path for both.
#pragma once
#include "common.cuh"

namespace mpc3 {

#define MPC3_SBOX_BYTES \
    0x63, 0x7c, 0x77, 0x7b, 0xf2, 0x6b, 0x6f, 0xc5, 0x30, 0x01, 0x67, 0x2b, 0xfe, 0xd7, 0xab, 0x76, \
    0xca, 0x82, 0xc9, 0x7d, 0xfa, 0x59, 0x47, 0xf0, 0xad, 0xd4, 0xa2, 0xaf, 0x9c, 0xa4, 0x72, 0xc0, \
    0xb7, 0xfd, 0x93, 0x26, 0x36, 0x3f, 0xf7, 0xcc, 0x34, 0xa5, 0xe5, 0xf1, 0x71, 0xd8, 0x31, 0x15, \
    0x04, 0xc7, 0x23, 0xc3, 0x18, 0x96, 0x05, 0x9a, 0x07, 0x12, 0x80, 0xe2, 0xeb, 0x27, 0xb2, 0x75, \
    0x09, 0x83, 0x2c, 0x1a, 0x1b, 0x6e, 0x5a, 0xa0, 0x52, 0x3b, 0xd6, 0xb3, 0x29, 0xe3, 0x2f, 0x84, \
    0x53, 0xd1, 0x00, 0xed, 0x20, 0xfc, 0xb1, 0x5b, 0x6a, 0xcb, 0xbe, 0x39, 0x4a, 0x4c, 0x58, 0xcf, \
    0xd0, 0xef, 0xaa, 0xfb, 0x43, 0x4d, 0x33, 0x85, 0x45, 0xf9, 0x02, 0x7f, 0x50, 0x3c, 0x9f, 0xa8, \
    0x51, 0xa3, 0x40, 0x8f, 0x92, 0x9d, 0x38, 0xf5, 0xbc, 0xb6, 0xda, 0x21, 0x10, 0xff, 0xf3, 0xd2, \
    0xcd, 0x0c, 0x13, 0xec, 0x5f, 0x97, 0x44, 0x17, 0xc4, 0xa7, 0x7e, 0x3d, 0x64, 0x5d, 0x19, 0x73, \
    0x60, 0x81, 0x4f, 0xdc, 0x22, 0x2a, 0x90, 0x88, 0x46, 0xee, 0xb8, 0x14, 0xde, 0x5e, 0x0b, 0xdb, \
    0xe0, 0x32, 0x3a, 0x0a, 0x49, 0x06, 0x24, 0x5c, 0xc2, 0xd3, 0xac, 0x62, 0x91, 0x95, 0xe4, 0x79, \
    0xe7, 0xc8, 0x37, 0x6d, 0x8d, 0xd5, 0x4e, 0xa9, 0x6c, 0x56, 0xf4, 0xea, 0x65, 0x7a, 0xae, 0x08, \
    0xba, 0x78, 0x25, 0x2e, 0x1c, 0xa6, 0xb4, 0xc6, 0xe8, 0xdd, 0x74, 0x1f, 0x4b, 0xbd, 0x8b, 0x8a, \
    0x70, 0x3e, 0xb5, 0x66, 0x48, 0x03, 0xf6, 0x0e, 0x61, 0x35, 0x57, 0xb9, 0x86, 0xc1, 0x1d, 0x9e, \
    0xe1, 0xf8, 0x98, 0x11, 0x69, 0xd9, 0x8e, 0x94, 0x9b, 0x1e, 0x87, 0xe9, 0xce, 0x55, 0x28, 0xdf, \
    0x8c, 0xa1, 0x89, 0x0d, 0xbf, 0xe6, 0x42, 0x68, 0x41, 0x99, 0x2d, 0x0f, 0xb0, 0x54, 0xbb, 0x16,

static const uint8_t h_sbox[256] = {MPC3_SBOX_BYTES};
#if defined(__CUDACC__)
__constant__ uint8_t d_sbox[256] = {MPC3_SBOX_BYTES};
#endif
#if defined(__CUDA_ARCH__)
#define c_sbox d_sbox
#else
#define c_sbox h_sbox
#endif


HD uint32_t ror32(uint32_t v, int r) { return (v >> r) | (v << (32 - r)); }
HD uint32_t bswap32(uint32_t v) {
  return (v >> 24) | ((v >> 8) & 0xff00u) | ((v << 8) & 0xff0000u) | (v << 24);
}
HD uint32_t xtime(uint32_t b) { return ((b << 1) ^ ((b & 0x80) ? 0x1b : 0)) & 0xff; }

// Te0[x] = (2*S[x], S[x], S[x], 3*S[x]) big-endian; Te1..3 are rotations.
HD uint32_t te0_entry(uint32_t x) {
  uint32_t s = c_sbox[x];
  uint32_t s2 = xtime(s);
  return (s2 << 24) | (s << 16) | (s << 8) | (s2 ^ s);
}

// Expanded AES-128 key: 44 big-endian round-key words (FIPS-197 5.2).
HD void aes128_expand(const uint8_t key[16], uint32_t rk[44]) {
  const uint8_t rcon[10] = {0x01, 0x02, 0x04, 0x08, 0x10, 0x20, 0x40, 0x80, 0x1b, 0x36};
  for (int i = 0; i < 4; ++i)
    rk[i] = ((uint32_t)key[4 * i] << 24) | ((uint32_t)key[4 * i + 1] << 16) |
            ((uint32_t)key[4 * i + 2] << 8) | key[4 * i + 3];
  for (int i = 4; i < 44; ++i) {
    uint32_t t = rk[i - 1];
    if (i % 4 == 0) {
      t = ((uint32_t)c_sbox[(t >> 16) & 0xff] << 24) | ((uint32_t)c_sbox[(t >> 8) & 0xff] << 16) |
          ((uint32_t)c_sbox[t & 0xff] << 8) | c_sbox[t >> 24];
      t ^= (uint32_t)rcon[i / 4 - 1] << 24;
    }
    rk[i] = rk[i - 4] ^ t;
  }
}

// Columns 0-1 of every counter block of stream (purpose, index).  pc: the
// shared-memory address of the stream's round-1/2 constants under the three
// session keys (HeadConst[3], see aes128_ctr), 0 when the launch did not
// precompute them (then every block runs all ten rounds).
struct StreamHead {
  uint32_t s0, s1;
  uint32_t pc;
};
HD StreamHead stream_head(uint32_t purpose, uint64_t index) {
  uint8_t b[8];
  b[0] = purpose & 0xff;
  b[1] = (purpose >> 8) & 0xff;
  for (int i = 0; i < 6; ++i) b[2 + i] = (index >> (8 * i)) & 0xff;
  StreamHead h;
  h.s0 = ((uint32_t)b[0] << 24) | ((uint32_t)b[1] << 16) | ((uint32_t)b[2] << 8) | b[3];
  h.s1 = ((uint32_t)b[4] << 24) | ((uint32_t)b[5] << 16) | ((uint32_t)b[6] << 8) | b[7];
  h.pc = 0;
  return h;
}

// Table access policy: T is any object exposing t0(i) and sb(i).
template <class T>
HD void aes128_block(const T& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                     uint32_t& s3) {
  s0 ^= rk[0];
  s1 ^= rk[1];
  s2 ^= rk[2];
  s3 ^= rk[3];
#if defined(__CUDA_ARCH__)
#pragma unroll 1
#endif
  for (int r = 1; r < 10; ++r) {
    const uint32_t* k = rk + 4 * r;
    uint32_t t0 = tab.t0(s0 >> 24) ^ ror32(tab.t0((s1 >> 16) & 0xff), 8) ^
                  ror32(tab.t0((s2 >> 8) & 0xff), 16) ^ ror32(tab.t0(s3 & 0xff), 24) ^ k[0];
    uint32_t t1 = tab.t0(s1 >> 24) ^ ror32(tab.t0((s2 >> 16) & 0xff), 8) ^
                  ror32(tab.t0((s3 >> 8) & 0xff), 16) ^ ror32(tab.t0(s0 & 0xff), 24) ^ k[1];
    uint32_t t2 = tab.t0(s2 >> 24) ^ ror32(tab.t0((s3 >> 16) & 0xff), 8) ^
                  ror32(tab.t0((s0 >> 8) & 0xff), 16) ^ ror32(tab.t0(s1 & 0xff), 24) ^ k[2];
    uint32_t t3 = tab.t0(s3 >> 24) ^ ror32(tab.t0((s0 >> 16) & 0xff), 8) ^
                  ror32(tab.t0((s1 >> 8) & 0xff), 16) ^ ror32(tab.t0(s2 & 0xff), 24) ^ k[3];
    s0 = t0;
    s1 = t1;
    s2 = t2;
    s3 = t3;
  }
  const uint32_t* k = rk + 40;
  uint32_t t0 = (tab.sb(s0 >> 24) << 24) | (tab.sb((s1 >> 16) & 0xff) << 16) |
                (tab.sb((s2 >> 8) & 0xff) << 8) | tab.sb(s3 & 0xff);
  uint32_t t1 = (tab.sb(s1 >> 24) << 24) | (tab.sb((s2 >> 16) & 0xff) << 16) |
                (tab.sb((s3 >> 8) & 0xff) << 8) | tab.sb(s0 & 0xff);
  uint32_t t2 = (tab.sb(s2 >> 24) << 24) | (tab.sb((s3 >> 16) & 0xff) << 16) |
                (tab.sb((s0 >> 8) & 0xff) << 8) | tab.sb(s1 & 0xff);
  uint32_t t3 = (tab.sb(s3 >> 24) << 24) | (tab.sb((s0 >> 16) & 0xff) << 16) |
                (tab.sb((s1 >> 8) & 0xff) << 8) | tab.sb(s2 & 0xff);
  s0 = t0 ^ k[0];
  s1 = t1 ^ k[1];
  s2 = t2 ^ k[2];
  s3 = t3 ^ k[3];
}

#if defined(__CUDACC__)
struct SmemTables;
struct SmemTables4;
HD void aes128_block(const SmemTables& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                     uint32_t& s3);
HD void aes128_block(const SmemTables4& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                     uint32_t& s3);
#endif

// The three session key schedules, passed to the kernels by value.
struct KeySched {
  uint32_t rk[3][44];
};

// Words 2b and 2b+1 of stream (head, key).
struct Word2 {
  uint64_t w0, w1;
};
template <class T>
HD Word2 prf_block(const T& tab, const uint32_t* rk, StreamHead h, uint64_t b) {
  uint32_t s0 = h.s0, s1 = h.s1, s2 = (uint32_t)(b >> 32), s3 = (uint32_t)b;
  aes128_block(tab, rk, s0, s1, s2, s3);
  Word2 w;
  w.w0 = (uint64_t)bswap32(s0) | ((uint64_t)bswap32(s1) << 32);
  w.w1 = (uint64_t)bswap32(s2) | ((uint64_t)bswap32(s3) << 32);
  return w;
}

// Single word w of the stream.
template <class T>
HD uint64_t prf_word(const T& tab, const uint32_t* rk, StreamHead h, uint64_t w) {
  Word2 p = prf_block(tab, rk, h, w >> 1);
  return (w & 1) ? p.w1 : p.w0;
}

#if !defined(__CUDA_ARCH__)
// Host tables for the CPU self-check build.
struct HostTables {
  uint32_t te[256];
  HostTables() {
    for (int i = 0; i < 256; ++i) te[i] = te0_entry(i);
  }
  inline uint32_t t0(uint32_t i) const { return te[i]; }
  inline uint32_t sb(uint32_t i) const { return c_sbox[i]; }
};
#endif

#if defined(__CUDACC__)
// Te0 as a compile-time constant table (1 KiB, constant bank): the source
// the per-CTA shared tables are expanded from.
struct Te0Table {
  uint32_t v[256];
};
constexpr uint8_t kSbox[256] = {MPC3_SBOX_BYTES};
constexpr uint32_t xtime_c(uint32_t b) { return ((b << 1) ^ ((b & 0x80) ? 0x1b : 0)) & 0xff; }
constexpr Te0Table make_te0() {
  Te0Table t{};
  for (int i = 0; i < 256; ++i) {
    uint32_t s = kSbox[i], s2 = xtime_c(s);
    t.v[i] = (s2 << 24) | (s << 16) | (s << 8) | (s2 ^ s);
  }
  return t;
}
__constant__ Te0Table c_te0 = make_te0();

// Shared-memory tables (64 KiB, dynamic shared memory), one per CTA.
// Entry x occupies 256 bytes: words [64x + l] = Te0[x] and [64x + 32 + l] =
// Te1[x] = ror8(Te0[x]) for lane l, i.e. lane l's copies always sit in bank l
// (a warp's 32 data-dependent lookups are one shared-memory wavefront).  The
// tables start at shared-window offset kAesTableOff (the first byte of dynamic
// shared memory after the 1 KiB the hardware reserves; checked at run time),
// so the address of lane l's Te0[x] is hi | x << 8 | 4 l, plus kAesTableOff,
// with hi = the window's CTA bits: ONE PRMT of the state word with (hi | 4 l)
// forms it, the offset is the LDS immediate, and Te1 is 128 bytes further.
// With Te0 and Te1 a column is Te0[a] ^ Te1[b] ^ ror16(Te0[c] ^ Te1[d]) ^ k
// (ror distributes over xor): 16 PRMT + 16 LDS + 16 logic ops per round.
struct SmemTables {
  uint32_t hl;  // (shared window base & 0xff000000) | 4 * lane
  static constexpr bool kFour = false;
  static constexpr int kTops = 1;  // counter top-byte values with cached round-2 constants
};
// Four-table variant (128 KiB): a second 64 KiB region holds Te2 / Te3 with
// the same entry layout, so Te2[x] and Te3[x] are the same PRMT address plus
// 0x10000 (+128): a column is Te0[a] ^ Te1[b] ^ Te2[c] ^ Te3[d] ^ k with no
// rotation — 4 fewer ALU ops per round, for the kernels that are nothing but
// AES (one 512-thread CTA per SM).
struct SmemTables4 {
  uint32_t hl;
  static constexpr bool kFour = true;
  static constexpr int kTops = 4;
};

// Counter-mode constants of one (stream, key, counter top byte v).  The
// counter blocks of a stream differ only in column 3 (the low word of the
// big-endian counter, below 2^32), so after AddRoundKey columns 0-2 are fixed
// and each column of round 1 has three fixed table terms (c[0..2], with the
// round key) and one that depends on a counter byte; for blocks whose top
// byte is v, round 1's column 3 is fixed too (c[3]), and so is one table term
// of every column of round 2 (d[j], with the round key).  Rounds 1-2 then
// take 3 + 12 lookups instead of 32 (160 -> 143 per block).  Slots are laid
// out [head][v][key]; a head's pc points at its (v = 0, key 0) constant.
struct __align__(16) HeadConst {
  uint32_t c[4], d[4];
};
constexpr int kHeadSlots = 16;   // two-table kernels (up to three CTAs per SM)
constexpr int kHeadSlots4 = 40;  // four-table kernels (one CTA per SM): the SGD launch's per-tensor heads
constexpr int kMaxTops = 4;

// (The session keys travel in the kernel parameters, not here.)
struct __align__(16) AesSmem {
  uint32_t te[256 * 64];
  uint64_t extra[24];                // per-kernel uniform data (stream heads)
  HeadConst hc[kHeadSlots * 1 * 3];  // per-launch counter-mode constants (aes128_ctr), SmemTables::kTops = 1
};
constexpr int kAesSmemBytes = (int)sizeof(AesSmem);
struct __align__(16) AesSmem4 {
  uint32_t te[2][256 * 64];
  uint64_t extra[64];
  HeadConst hc[kHeadSlots4 * kMaxTops * 3];
};
constexpr int kAesSmem4Bytes = (int)sizeof(AesSmem4);
constexpr uint32_t kAesTableOff = 1024;

// The protocol kernels' dynamic shared memory: an AesSmem at offset 0 (these
// kernels declare no static shared memory, so it starts at kAesTableOff).
extern __shared__ __align__(16) uint8_t mpc3_dsm[];

DEV uint32_t lds_te0(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+1024];" : "=r"(v) : "r"(a));
  return v;
}
DEV uint32_t lds_te1(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+1152];" : "=r"(v) : "r"(a));
  return v;
}
DEV uint32_t lds_te2(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+66560];" : "=r"(v) : "r"(a));
  return v;
}
DEV uint32_t lds_te3(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1+66688];" : "=r"(v) : "r"(a));
  return v;
}

#define MPC3_I3(x) __byte_perm((x), hl, 0x7634)
#define MPC3_I2(x) __byte_perm((x), hl, 0x7624)
#define MPC3_I1(x) __byte_perm((x), hl, 0x7614)
#define MPC3_I0(x) __byte_perm((x), hl, 0x7604)
// one output column of rounds 1-9
#define MPC3_COL(a, b, c, d, kk)                                                                     \
  (FOUR ? (lds_te0(MPC3_I3(a)) ^ lds_te1(MPC3_I2(b)) ^ lds_te2(MPC3_I1(c)) ^ lds_te3(MPC3_I0(d)) ^ (kk)) \
        : (lds_te0(MPC3_I3(a)) ^ lds_te1(MPC3_I2(b)) ^                                               \
           __byte_perm(lds_te0(MPC3_I1(c)) ^ lds_te1(MPC3_I0(d)), 0, 0x1032) ^ (kk)))
// final round column: S[x] is byte 2 (and 1) of Te0[x] = (2S, S, S, 3S)
#define MPC3_FIN(a, b, c, d, kk)                                                                     \
  (__byte_perm(__byte_perm(lds_te0(MPC3_I3(a)), lds_te0(MPC3_I2(b)), 0x2600),                        \
               __byte_perm(lds_te0(MPC3_I1(c)), lds_te0(MPC3_I0(d)), 0x0015), 0x3254) ^                \
   (kk))

template <class TT>
HD void aes128_block_dev(const TT& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                          uint32_t& s3) {
#if defined(__CUDA_ARCH__)
  constexpr bool FOUR = TT::kFour;
  const uint32_t hl = tab.hl;
  s0 ^= rk[0];
  s1 ^= rk[1];
  s2 ^= rk[2];
  s3 ^= rk[3];
#pragma unroll 1
  for (int r = 1; r < 10; ++r) {
    const uint4 k = *reinterpret_cast<const uint4*>(rk + 4 * r);
    uint32_t t0 = MPC3_COL(s0, s1, s2, s3, k.x);
    uint32_t t1 = MPC3_COL(s1, s2, s3, s0, k.y);
    uint32_t t2 = MPC3_COL(s2, s3, s0, s1, k.z);
    uint32_t t3 = MPC3_COL(s3, s0, s1, s2, k.w);
    s0 = t0;
    s1 = t1;
    s2 = t2;
    s3 = t3;
  }
  const uint4 k = *reinterpret_cast<const uint4*>(rk + 40);
  uint32_t t0 = MPC3_FIN(s0, s1, s2, s3, k.x);
  uint32_t t1 = MPC3_FIN(s1, s2, s3, s0, k.y);
  uint32_t t2 = MPC3_FIN(s2, s3, s0, s1, k.z);
  uint32_t t3 = MPC3_FIN(s3, s0, s1, s2, k.w);
  s0 = t0;
  s1 = t1;
  s2 = t2;
  s3 = t3;
#endif
}
HD void aes128_block(const SmemTables& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                     uint32_t& s3) {
  aes128_block_dev(tab, rk, s0, s1, s2, s3);
}
HD void aes128_block(const SmemTables4& tab, const uint32_t* rk, uint32_t& s0, uint32_t& s1, uint32_t& s2,
                     uint32_t& s3) {
  aes128_block_dev(tab, rk, s0, s1, s2, s3);
}

// NB independent blocks interleaved round by round (key schedule of block i
// at rks[i]): the independent dependency chains multiply the instruction-
// level parallelism of the table rounds.
template <int NB, class TT>
DEV void aes128_multi(const TT& tab, const uint32_t* const rks[NB], uint32_t s[NB][4]) {
  constexpr bool FOUR = TT::kFour;
  const uint32_t hl = tab.hl;
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s[i][j] ^= rks[i][j];
#pragma unroll 1
  for (int r = 1; r < 10; ++r) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const uint4 k = *reinterpret_cast<const uint4*>(rks[i] + 4 * r);
      uint32_t t0 = MPC3_COL(s[i][0], s[i][1], s[i][2], s[i][3], k.x);
      uint32_t t1 = MPC3_COL(s[i][1], s[i][2], s[i][3], s[i][0], k.y);
      uint32_t t2 = MPC3_COL(s[i][2], s[i][3], s[i][0], s[i][1], k.z);
      uint32_t t3 = MPC3_COL(s[i][3], s[i][0], s[i][1], s[i][2], k.w);
      s[i][0] = t0;
      s[i][1] = t1;
      s[i][2] = t2;
      s[i][3] = t3;
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint4 k = *reinterpret_cast<const uint4*>(rks[i] + 40);
    uint32_t a = s[i][0], b = s[i][1], c = s[i][2], d = s[i][3];
    s[i][0] = MPC3_FIN(a, b, c, d, k.x);
    s[i][1] = MPC3_FIN(b, c, d, a, k.y);
    s[i][2] = MPC3_FIN(c, d, a, b, k.z);
    s[i][3] = MPC3_FIN(d, a, b, c, k.w);
  }
}

// Table term k of a column (Te_k indexed by byte 3 - k of x), both layouts.
#define MPC3_TE0(x) lds_te0(MPC3_I3(x))
#define MPC3_TE1(x) lds_te1(MPC3_I2(x))
#define MPC3_TE2(x) (FOUR ? lds_te2(MPC3_I1(x)) : __byte_perm(lds_te0(MPC3_I1(x)), 0, 0x1032))
#define MPC3_TE3(x) (FOUR ? lds_te3(MPC3_I0(x)) : __byte_perm(lds_te1(MPC3_I0(x)), 0, 0x1032))

// Round-1/2 constants of stream columns (s0, s1) under the expanded key rk
// (counter word 2 = 0, top byte of word 3 = v; see HeadConst).
template <class TT>
DEV void head_const(const TT& tab, const uint32_t* rk, uint32_t s0, uint32_t s1, uint32_t v, HeadConst& o) {
  constexpr bool FOUR = TT::kFour;
  const uint32_t hl = tab.hl;
  const uint32_t x0 = s0 ^ rk[0], x1 = s1 ^ rk[1], x2 = rk[2], x3 = rk[3] ^ (v << 24);
  o.c[0] = MPC3_TE0(x0) ^ MPC3_TE1(x1) ^ MPC3_TE2(x2) ^ rk[4];
  o.c[1] = MPC3_TE0(x1) ^ MPC3_TE1(x2) ^ MPC3_TE3(x0) ^ rk[5];
  o.c[2] = MPC3_TE0(x2) ^ MPC3_TE2(x0) ^ MPC3_TE3(x1) ^ rk[6];
  const uint32_t c3 = MPC3_TE0(x3) ^ MPC3_TE1(x0) ^ MPC3_TE2(x1) ^ MPC3_TE3(x2) ^ rk[7];
  o.c[3] = c3;
  o.d[0] = MPC3_TE3(c3) ^ rk[8];
  o.d[1] = MPC3_TE2(c3) ^ rk[9];
  o.d[2] = MPC3_TE1(c3) ^ rk[10];
  o.d[3] = MPC3_TE0(c3) ^ rk[11];
}

DEV uint4 lds_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// NB blocks, block i at counter blks[i] of stream columns (s01[i][0],
// s01[i][1]) under key schedule rks[i] whose counter-mode constants (v = 0)
// sit at shared address pcs[i] (0: none).  Output: the ciphertext columns.
// Blocks whose counter top byte has constants (below kTops << 24) start at
// round 3 (rounds 1-2 from the constants, 15 lookups), other blocks below
// 2^32 at round 2 (round 1: 5 lookups); otherwise all rounds run.
template <int NB, class TT>
DEV void aes128_ctr_n(const TT& tab, const uint32_t* const rks[NB], const uint32_t pcs[NB],
                      const uint32_t s01[NB][2], const uint64_t blks[NB], uint32_t s[NB][4]) {
  constexpr bool FOUR = TT::kFour;
  const uint32_t hl = tab.hl;
  bool cached = true, top0 = true;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    cached = cached && pcs[i] != 0 && (blks[i] >> 32) == 0;
    top0 = top0 && ((uint32_t)blks[i] >> 24) < (uint32_t)TT::kTops;
  }
  int r0 = 1;
  if (cached) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const uint32_t lo = (uint32_t)blks[i];
      const uint32_t voff = top0 ? (lo >> 24) * 96u : 0u;  // [v][key] stride: 3 keys x 32 bytes
      const uint4 c = lds_v4(pcs[i] + voff);
      const uint32_t x3 = lo ^ rks[i][3];
      s[i][0] = c.x ^ MPC3_TE3(x3);
      s[i][1] = c.y ^ MPC3_TE2(x3);
      s[i][2] = c.z ^ MPC3_TE1(x3);
      s[i][3] = top0 ? c.w : c.w ^ MPC3_TE0(rks[i][3]) ^ MPC3_TE0(x3);
    }
    if (top0) {
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        const uint4 d = lds_v4(pcs[i] + ((uint32_t)blks[i] >> 24) * 96u + 16);
        const uint32_t t0 = s[i][0], t1 = s[i][1], t2 = s[i][2];
        s[i][0] = MPC3_TE0(t0) ^ MPC3_TE1(t1) ^ MPC3_TE2(t2) ^ d.x;
        s[i][1] = MPC3_TE0(t1) ^ MPC3_TE1(t2) ^ MPC3_TE3(t0) ^ d.y;
        s[i][2] = MPC3_TE0(t2) ^ MPC3_TE2(t0) ^ MPC3_TE3(t1) ^ d.z;
        s[i][3] = MPC3_TE1(t0) ^ MPC3_TE2(t1) ^ MPC3_TE3(t2) ^ d.w;
      }
      r0 = 3;
    } else {
      r0 = 2;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      s[i][0] = s01[i][0] ^ rks[i][0];
      s[i][1] = s01[i][1] ^ rks[i][1];
      s[i][2] = (uint32_t)(blks[i] >> 32) ^ rks[i][2];
      s[i][3] = (uint32_t)blks[i] ^ rks[i][3];
    }
  }
#pragma unroll 1
  for (int r = r0; r < 10; ++r) {
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      const uint4 k = *reinterpret_cast<const uint4*>(rks[i] + 4 * r);
      uint32_t t0 = MPC3_COL(s[i][0], s[i][1], s[i][2], s[i][3], k.x);
      uint32_t t1 = MPC3_COL(s[i][1], s[i][2], s[i][3], s[i][0], k.y);
      uint32_t t2 = MPC3_COL(s[i][2], s[i][3], s[i][0], s[i][1], k.z);
      uint32_t t3 = MPC3_COL(s[i][3], s[i][0], s[i][1], s[i][2], k.w);
      s[i][0] = t0;
      s[i][1] = t1;
      s[i][2] = t2;
      s[i][3] = t3;
    }
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint4 k = *reinterpret_cast<const uint4*>(rks[i] + 40);
    uint32_t a = s[i][0], b = s[i][1], c = s[i][2], d = s[i][3];
    s[i][0] = MPC3_FIN(a, b, c, d, k.x);
    s[i][1] = MPC3_FIN(b, c, d, a, k.y);
    s[i][2] = MPC3_FIN(c, d, a, b, k.z);
    s[i][3] = MPC3_FIN(d, a, b, c, k.w);
  }
}
// All NB blocks at one counter value.
template <int NB, class TT>
DEV void aes128_ctr(const TT& tab, const uint32_t* const rks[NB], const uint32_t pcs[NB], const uint32_t s01[NB][2],
                    uint64_t blk, uint32_t s[NB][4]) {
  uint64_t blks[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) blks[i] = blk;
  aes128_ctr_n<NB>(tab, rks, pcs, s01, blks, s);
}
#undef MPC3_TE0
#undef MPC3_TE1
#undef MPC3_TE2
#undef MPC3_TE3

// Three blocks with the same counter under k_0, k_1, k_2: every zero share
// needs all three keys' words at one position (sharing.py:233-250).
template <class TT>
DEV void aes128_block3(const TT& tab, const uint32_t* rk3, uint32_t s[3][4]) {
  const uint32_t* rks[3] = {rk3, rk3 + 44, rk3 + 88};
  aes128_multi<3>(tab, rks, s);
}
#undef MPC3_I3
#undef MPC3_I2
#undef MPC3_I1
#undef MPC3_I0
#undef MPC3_COL
#undef MPC3_FIN

// Expand the tables into this CTA's dynamic shared memory (16-byte stores of
// four lane copies; Te0 from the constant bank) and stage the key schedules.
// rk_dev: nkeys x 44 round-key words (k_0, k_1, k_2 of the session).
// Programmatic dependent launch: the table expansion only reads the constant
// bank and the session keys, so it runs before griddep_wait() and overlaps
// the previous kernel's tail; every protocol kernel goes through here.
__device__ inline SmemTables aes_smem_init(AesSmem& sm) {
  griddep_launch();
  uint4* dst = reinterpret_cast<uint4*>(sm.te);
  for (int i = threadIdx.x; i < 256 * 16; i += blockDim.x) {
    uint32_t v = c_te0.v[i >> 4];
    if (i & 8) v = __funnelshift_r(v, v, 8);  // words 32-63 of the entry: Te1
    dst[i] = make_uint4(v, v, v, v);
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(mpc3_dsm);
  if ((base & 0x00ffffffu) != kAesTableOff) __trap();  // the LDS immediates assume this layout
  __syncthreads();
  griddep_wait();
  SmemTables t;
  t.hl = (base & 0xff000000u) | ((threadIdx.x & 31) * 4);
  return t;
}

// Four-table expansion (Te0/Te1 in region 0, Te2/Te3 = ror16 of them in region 1).
__device__ inline SmemTables4 aes_smem_init4(AesSmem4& sm) {
  griddep_launch();
  uint4* dst = reinterpret_cast<uint4*>(&sm.te[0][0]);
  for (int i = threadIdx.x; i < 2 * 256 * 16; i += blockDim.x) {
    const int e = i & (256 * 16 - 1);
    uint32_t v = c_te0.v[e >> 4];
    const int rot = ((e & 8) ? 8 : 0) + (i >= 256 * 16 ? 16 : 0);  // Te1 / Te2 / Te3 = ror 8 / 16 / 24
    v = __funnelshift_r(v, v, rot);
    dst[i] = make_uint4(v, v, v, v);
  }
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(mpc3_dsm);
  if ((base & 0x00ffffffu) != kAesTableOff) __trap();
  __syncthreads();
  griddep_wait();
  SmemTables4 t;
  t.hl = (base & 0xff000000u) | ((threadIdx.x & 31) * 4);
  return t;
}

// Counter-mode constants of NH stream heads (aes128_ctr): every thread of the
// CTA calls this after the tables are built; thread t < 3 kTops NH computes
// (head, v, key) = (t / 3 kTops, t / 3 % kTops, t % 3), and after the barrier
// each head's pc points at its (v = 0, key 0) slot.
// (Building with -DMPC3_NO_HEAD_CACHE leaves every pc 0: the A/B baseline,
// profiles/r02_variants_aes_ctr_cache.txt.)
template <class TT, class... H>
DEV void cache_heads(const TT& tab, const uint32_t* rk3, HeadConst* slots, H&... h) {
  constexpr int KT = TT::kTops;
  static_assert(sizeof...(H) <= kHeadSlots, "head slots");
#if defined(MPC3_NO_HEAD_CACHE)
  return;
#endif
  const int t = threadIdx.x, v = t / 3 % KT, k = t % 3;
  int i = 0;
  (((t / (3 * KT) == i ? head_const(tab, rk3 + 44 * k, h.s0, h.s1, (uint32_t)v, slots[t]) : void()), ++i), ...);
  __syncthreads();
  i = 0;
  (((h.pc = (uint32_t)__cvta_generic_to_shared(&slots[i * KT * 3])), ++i), ...);
}

#define MPC3_AES_SMEM() AesSmem& sm = *reinterpret_cast<AesSmem*>(mpc3_dsm)
#define MPC3_AES_SMEM4() AesSmem4& sm = *reinterpret_cast<AesSmem4*>(mpc3_dsm)
#endif

}  // namespace mpc3
