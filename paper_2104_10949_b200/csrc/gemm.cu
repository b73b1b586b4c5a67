// Z_2^64 ring GEMM on the 5th-generation tensor cores (tcgen05 kind::i8).
//
// Replaces the reference's float-limb engine (ring.py:123-222: 4 x 16-bit
// limbs as float64, 10 dgemms, recombined with wrapping shifts).  Here each
// 64-bit operand is split into 8 unsigned byte limbs; the 36 limb pairs (i, j)
// with i + j < 8 are accumulated exactly in int32 into 8 "diagonal"
// accumulators S_d = sum_{i+j=d} A_i B_j^T held in TMEM (8 x 64 columns =
// the whole 512-column TMEM of the SM), and the epilogue forms
// sum_d S_d << 8d mod 2^64.  S_d for d >= 4 only matters mod 2^32 (the int32
// accumulator wraps); S_d for d <= 3 is exact while K <= 16512.
//
// Tile: 128 rows (M) x 64 columns (N) per CTA, K step 32 bytes.  The B tile
// of all 8 limbs is laid out as one 512-row K-major operand, so the products
// A_i x [B_0 .. B_{7-i}] are ONE MMA with N = 64 (8 - i) (split at 256)
// written at TMEM column 64 i: column block j lands on diagonal i + j.  That
// is 12 MMAs per K step instead of 36, and B is read from shared memory once
// per (i, block) instead of once per pair.
//
// Warp roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer,
// warp 2 = TMEM allocator, warps 4-7 = epilogue (TMEM lanes 0-127).
#include <cuda.h>
#include <cuda_runtime.h>
#include <string.h>

#include <mutex>
#include <set>

#include "launch.cuh"
#include "items.cuh"

namespace mpc3 {

// ---------------------------------------------------------------------------
// operand packing: u64 gather -> 8 byte-limb planes [g][limb][row][kp]

__global__ void pack_kernel(const uint64_t* __restrict__ src, int64_t plane, Operand o, int role, int groups,
                            uint8_t* __restrict__ out, int64_t kp, int64_t kh) {
  int64_t total = (int64_t)groups * o.rows * (kp / 8);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    pack_item(src, plane, o, role, out, kp, t, kh);
}

// Tiled operand packing.  One CTA packs a PT_R x PT_K tile of the packed
// operand (rows x packed columns kk of [first half | second half], 2K long for
// the cross-term roles).  The gather offset of v(r, k) splits into a row part
// and a column part (dense: off + r s_r + sum k_i t_i; im2col: n sN + c sC +
// (y sh - ph + u) sH + (x sw - pw + v) sW with bounds; wgrad: the same with the
// roles of (n, y, x) and (c, u, v) swapped), computed once per tile row and
// column into shared memory, so an element costs two adds, two multiply-adds
// and two loads.  Phase 1 walks the tile in the source's contiguous direction
// (rows for im2col and row-strided dense views, columns otherwise) so the
// loads coalesce; phase 2 reads 8 consecutive packed values of one row back
// from shared memory, byte-transposes them (PRMT) and writes one 8-byte word
// per limb plane, consecutive threads covering consecutive columns.
constexpr int PT_R = 64, PT_K = 64, PT_THREADS = 256;

struct PackTileArgs {
  int64_t rows, K, kp, lim;  // lim: packed columns with data (K or kh + K)
  int64_t kh;                // first packed column of the second half
  uint64_t* zero;            // optional: words the next GEMM accumulates into atomically,
  int64_t zero_words;        //   cleared here so it needs no memset launch of its own
  int32_t H, W, sH, sW;      // bounds / strides of the (y, x) part (dense: no bounds, 0 strides)
};

// Conflict-free shared layout of the 64 x 64 u64 tile for the three access
// patterns (phase 1 along rows, phase 1 along columns, phase 2 eight
// consecutive columns of 4 rows per warp), found by exhaustive search:
// within each 8-column chunk rotate by chunk + row, then XOR the chunk with
// row bits 3-5.
DEV int pt_swz(int i, int j) { return ((j & ~7) + (((j & 7) + (j >> 3) + (i & 7)) & 7)) ^ (((i >> 3) & 7) << 3); }

// Row / column part of the gather offset: {base, y, x, half}.  Columns past
// the data (zero padding) and rows past the end get y = -2^30, which fails
// the unsigned bounds check, so no separate flag is tested per element.
// (32-bit index arithmetic: the host only routes operands whose rows, K and
// component planes are below 2^31 here.)
DEV int4 pack_row_part(const Operand& o, int64_t r64, int64_t rows) {
  if (r64 >= rows) return make_int4(0, -(1 << 30), 0, 0);
  const uint32_t r = (uint32_t)r64;
  if (o.mode == MPC3_GATHER_DENSE) return make_int4((int32_t)(o.off + r64 * o.s_r), 0, 0, 0);
  if (o.mode == MPC3_GATHER_IM2COL) {  // r = (n, y, x)
    const uint32_t ow = (uint32_t)o.ow, oh = (uint32_t)o.oh;
    const uint32_t q = r / ow, xx = r - q * ow;
    const uint32_t n = q / oh, yy = q - n * oh;
    return make_int4((int32_t)(n * o.sN), (int32_t)(yy * o.sh - o.ph), (int32_t)(xx * o.sw - o.pw), 0);
  }
  // WGRAD: r = (c, u, v)
  const uint32_t kw = (uint32_t)o.kw, kh = (uint32_t)o.kh;
  const uint32_t q = r / kw, v = r - q * kw;
  const uint32_t c = q / kh, u = q - c * kh;
  return make_int4((int32_t)(c * o.sC), (int32_t)(u - o.ph), (int32_t)(v - o.pw), 0);
}
DEV int4 pack_col_part(const Operand& o, int64_t kk, int64_t K, int64_t lim, int64_t kh) {
  const int half = kk >= kh ? 1 : 0;
  if (kk >= lim || (!half && kk >= K)) return make_int4(0, -(1 << 30), 0, 0);
  const uint32_t k = (uint32_t)(kk - half * kh);
  if (o.mode == MPC3_GATHER_DENSE) {
    const uint32_t K2 = (uint32_t)o.K2, K1 = (uint32_t)o.K1;
    const uint32_t q = k / K2, k2 = k - q * K2;
    const uint32_t k0 = q / K1, k1 = q - k0 * K1;
    return make_int4((int32_t)(k0 * o.t0 + k1 * o.t1 + k2 * o.t2), 0, 0, half);
  }
  if (o.mode == MPC3_GATHER_IM2COL) {  // k = (c, u, v)
    const uint32_t kw = (uint32_t)o.kw, kh = (uint32_t)o.kh;
    const uint32_t q = k / kw, v = k - q * kw;
    const uint32_t c = q / kh, u = q - c * kh;
    return make_int4((int32_t)(c * o.sC), (int32_t)u, (int32_t)v, half);
  }
  // WGRAD: k = (n, y, x)
  const uint32_t ow = (uint32_t)o.ow, oh = (uint32_t)o.oh;
  const uint32_t q = k / ow, xx = k - q * ow;
  const uint32_t n = q / oh, yy = q - n * oh;
  return make_int4((int32_t)(n * o.sN), (int32_t)(yy * o.sh), (int32_t)(xx * o.sw), half);
}

template <bool R_FAST, int ROLE>
__global__ void __launch_bounds__(PT_THREADS) pack_tile_kernel(const uint64_t* __restrict__ src, int64_t plane,
                                                               Operand o, PackTileArgs a,
                                                               uint8_t* __restrict__ out) {
  __shared__ uint64_t tile[PT_R * PT_K];
  __shared__ int4 rpart[PT_R], cpart[PT_K];
  griddep_launch();
  const int g = blockIdx.z;
  const int64_t r0 = (int64_t)blockIdx.y * PT_R, c0 = (int64_t)blockIdx.x * PT_K;
  const int t = threadIdx.x;
  if (t < PT_R)
    rpart[t] = pack_row_part(o, r0 + t, a.rows);
  else if (t < PT_R + PT_K)
    cpart[t - PT_R] = pack_col_part(o, c0 + (t - PT_R), a.K, a.lim, a.kh);
  __syncthreads();
  griddep_wait();  // the source tensor is the previous kernel's output
  if (a.zero) {
    const int64_t nblk = (int64_t)gridDim.x * gridDim.y * gridDim.z;
    const int64_t bid = blockIdx.x + (int64_t)gridDim.x * (blockIdx.y + (int64_t)gridDim.y * blockIdx.z);
    for (int64_t i = bid * PT_THREADS + t; i < a.zero_words; i += nblk * PT_THREADS) a.zero[i] = 0;
  }
  // phase 1: gather the packed values of the tile.  Each thread keeps one
  // row (R_FAST) or one column fixed in registers; a warp's 32 lanes walk
  // the source's contiguous direction.  All loads first (16 in flight).
  const uint64_t* sg = src + (ROLE == 2 ? 0 : (int64_t)g * plane);
  const uint64_t* sn = src + (int64_t)((g + 1) % 3) * plane;
  const int fixed = R_FAST ? (t % PT_R) : (t % PT_K);
  const int4 fp = R_FAST ? rpart[fixed] : cpart[fixed];
  constexpr int PER = (PT_R * PT_K) / PT_THREADS;
  constexpr int STEP = PT_THREADS / (R_FAST ? PT_R : PT_K);
  const int var0 = t / (R_FAST ? PT_R : PT_K);
  const uint32_t H = (uint32_t)a.H, W = (uint32_t)a.W;
  uint64_t vs[PER], vn[PER > 0 && ROLE == 0 ? PER : 1];
  // only the components a half needs are loaded: role 1 reads x_i (first
  // half) or x_{i+1} (second), role 0 reads x_{i+1} for the first half only
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int4 vp = R_FAST ? cpart[var0 + it * STEP] : rpart[var0 + it * STEP];
    const int half = R_FAST ? vp.w : fp.w;
    const int32_t yy = fp.y + vp.y, xx = fp.z + vp.z;
    const bool ok = (uint32_t)yy < H && (uint32_t)xx < W;
    const uint32_t off = ok ? (uint32_t)(fp.x + vp.x + yy * a.sH + xx * a.sW) : 0u;
    vs[it] = ok ? __ldg((ROLE == 1 && half ? sn : sg) + off) : 0ull;  // (ROLE 3: plane g only, no halves)
    if (ROLE == 0) vn[it] = ok && !half ? __ldg(sn + off) : 0ull;
  }
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int var = var0 + it * STEP;
    const int i = R_FAST ? fixed : var, j = R_FAST ? var : fixed;
    // [x_i + x_{i+1} | x_i] (role 0) / [y_i | y_{i+1}] (role 1)  (protocols.py:110-115)
    const uint64_t v = ROLE == 0 ? vs[it] + vn[it] : vs[it];
    tile[i * PT_K + pt_swz(i, j)] = v;
  }
  __syncthreads();
  // phase 2: 8 consecutive columns of one row -> one u64 per limb plane
  const int64_t pstride = a.rows * a.kp;
#pragma unroll 1
  for (int e = t; e < PT_R * (PT_K / 8); e += PT_THREADS) {
    const int i = e / (PT_K / 8), ch = e % (PT_K / 8);
    const int64_t r = r0 + i, kk = c0 + ch * 8;
    if (r >= a.rows || kk >= a.kp) continue;
    const int cb = (ch * 8) ^ (((i >> 3) & 7) << 3), rot = (ch + i) & 7;
    uint64_t v[8], w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = tile[i * PT_K + cb + ((q + rot) & 7)];
    byte_transpose8(v, w);
    uint64_t* dst = reinterpret_cast<uint64_t*>(out + ((int64_t)g * 8 * a.rows + r) * a.kp + kk);
#pragma unroll
    for (int l = 0; l < 8; ++l) dst[l * (pstride >> 3)] = w[l];
  }
}

// ---------------------------------------------------------------------------
// SIMT reference kernel (64-bit IMAD on CUDA cores)

constexpr int ST = 32;
__global__ void __launch_bounds__(256) gemm_simt_kernel(const uint64_t* __restrict__ A,
                                                       const uint64_t* __restrict__ B, uint64_t* __restrict__ C,
                                                       int64_t M, int64_t N, int64_t K, int64_t sam, int64_t sak,
                                                       int64_t sbk, int64_t sbn, int64_t ldc) {
  __shared__ uint64_t sa[16][ST + 1];
  __shared__ uint64_t sb[16][ST + 1];
  int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8 threads, 4 rows each
  int64_t m0 = blockIdx.y * (int64_t)ST, n0 = blockIdx.x * (int64_t)ST;
  uint64_t acc[4] = {0, 0, 0, 0};
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * ST; i += 256) {
      int kk = i % 16, mm = i / 16;
      int64_t m = m0 + mm, k = k0 + kk;
      sa[kk][mm] = (m < M && k < K) ? A[m * sam + k * sak] : 0;
      int nn = i % ST, kb = i / ST;
      int64_t n = n0 + nn, k2 = k0 + kb;
      sb[kb][nn] = (n < N && k2 < K) ? B[k2 * sbk + n * sbn] : 0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      uint64_t b = sb[kk][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] += sa[kk][ty * 4 + r] * b;
    }
    __syncthreads();
  }
  for (int r = 0; r < 4; ++r) {
    int64_t m = m0 + ty * 4 + r, n = n0 + tx;
    if (m < M && n < N) C[m * ldc + n] = acc[r];
  }
}

// ---------------------------------------------------------------------------
// tcgen05 kernel

constexpr int BM = 128;            // rows per CTA (TMEM lanes)
constexpr int BN = 64;             // output columns per CTA (per limb block)
constexpr int BK = 32;             // K bytes per stage (one kind::i8 MMA K)
#ifndef MPC3_GEMM_STAGES
#define MPC3_GEMM_STAGES 4
#endif
constexpr int STAGES = MPC3_GEMM_STAGES;
constexpr int A_STAGE = 8 * BM * BK;  // 32 KiB
constexpr int B_STAGE = 8 * BN * BK;  // 16 KiB
constexpr int SMEM_BYTES = STAGES * (A_STAGE + B_STAGE) + 1024 /*align*/ + 256 /*barriers*/;
constexpr int MAX_SPLIT_K = 16384;   // exactness: S_3 <= 4 K 255^2 < 2^32

DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
DEV void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// K-major, 32-byte-swizzled UMMA shared-memory descriptor (atom 8 rows x 32 B).
DEV uint64_t umma_desc_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);      // start address
  d |= (uint64_t)0 << 16;                       // LBO (unused: one atom along K)
  d |= (uint64_t)((256 >> 4) & 0x3fff) << 32;  // SBO: 8 rows x 32 B
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;                       // SWIZZLE_32B
  return d;
}

// Instruction descriptor: u8 x u8 -> s32, K-major A and B, M = 128.
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

DEV void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Operands read in place from another GEMM's packed buffer ("MN-major"): the
// contraction index is the SOURCE's row index and this GEMM's rows / columns
// are a source column range, so a weight gradient consumes the forward pass's
// packed activations and the input-gradient pass's packed gradient directly
// (transposed views, no repack).  Per half h of the cross-term concatenation
// the contraction runs over source rows [0, kc_half) (zero-filled past the
// source's rows) at source columns h * half + tile offset.  tcgen05 reads
// such tiles MN-major (instruction-descriptor bits 15 / 16): A as 128-byte
// SWIZZLE_128B rows (8-row atoms, SBO 1 KiB), B limb tiles as 64-byte
// SWIZZLE_64B rows (SBO 512 B, the next limb tile = the next 64-wide MN atom,
// LBO 2 KiB).
struct MnArgs {
  int a_mn, b_mn;
  int a_half, b_half;  // source column of half 1 (a_rh: A's source row of half 1)
  int nkb_half;        // contraction K-blocks per half
  int a_cs;            // A's halves are component planes g and g + 1 (role-3 pack of a role-1 operand)
  int a_rh;            // MN-read A whose second half is further source rows (a plain transposed pack)
  int b_cs;            // K-major B whose halves are component planes g and g + 1 (role-3 pack)
};

DEV uint64_t umma_desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// A operand: mode 0 = K-major SWIZZLE_32B limb tiles [limb][row][32 B];
// mode 1 = MN-major SWIZZLE_128B (transposed read, see MnArgs).  The 128-byte
// rows of mode 1 spread the tensor core's shared-memory reads over every bank
// group; the 32-byte rows of mode 0 meet 2-way conflicts (1.17x slower at
// M=N=K=4096, profiles/README.md).  (A K-major 4-limb interleave through a 4-D
// box with a 32-byte inner extent does not work: TMA pads each 32-byte box row
// to the 128-byte swizzle span.)
DEV uint64_t desc_a(uint32_t addr, int mode) {
  return mode ? umma_desc_mn(addr, 0, 1024, 2) : umma_desc_sw32(addr);
}
DEV uint64_t desc_b(uint32_t addr, bool mn) {
  return mn ? umma_desc_mn(addr, BN * BK, 8 * BN, 4) : umma_desc_sw32(addr);
}

// One pipeline stage: the A and B limb tiles of K-block kb of tile (m0, n0),
// group g (MN operands: source rows / half of the transposed read).
DEV void load_stage(const CUtensorMap* tmA, const CUtensorMap* tmB, uint64_t* bar, uint8_t* sa, uint8_t* sb, int kb,
                    int m0, int n0, int g, const MnArgs& mn) {
  mbar_expect_tx(bar, A_STAGE + B_STAGE);
  const int kc = kb * BK;
  const int h = kb >= mn.nkb_half ? 1 : 0, r = (kb - h * mn.nkb_half) * BK;
  if (mn.a_cs) {  // half h of [x_g | x_{g+1}] is component plane g + h
    const int ap = ((g + h) % 3) * 8;
    if (mn.a_mn)
      tma_load_3d(tmA, bar, sa, m0, r, ap);
    else
      tma_load_3d(tmA, bar, sa, r, m0, ap);
  } else if (mn.a_mn) {
    if (mn.a_rh)
      tma_load_3d(tmA, bar, sa, m0, r + h * mn.a_half, g * 8);
    else
      tma_load_3d(tmA, bar, sa, h * mn.a_half + m0, r, g * 8);
  } else {
    tma_load_3d(tmA, bar, sa, kc, m0, g * 8);
  }
  if (mn.b_mn)
    tma_load_3d(tmB, bar, sb, h * mn.b_half + n0, r, g * 8);
  else if (mn.b_cs)
    tma_load_3d(tmB, bar, sb, r, n0, ((g + h) % 3) * 8);
  else
    tma_load_3d(tmB, bar, sb, kc, n0, g * 8);
}

// The 36 limb-pair products of one stage as 12 MMAs into the 8 diagonal
// accumulators (diagonal d = li + lj at TMEM columns d * BN).
DEV void mma_stage(uint32_t tmem, uint32_t a_base, uint32_t b_base, bool first, const MnArgs& mn) {
  const uint32_t idesc_mn = ((uint32_t)(mn.a_mn != 0) << 15) | ((uint32_t)(mn.b_mn != 0) << 16);
#pragma unroll
  for (int li = 0; li < 8; ++li) {
    const uint64_t da = desc_a(a_base + li * (BM * BK), mn.a_mn);
    const int nblk = 8 - li;  // limb blocks j = 0 .. 7 - li  ->  diagonals li .. 7
    const int nfirst = nblk > 4 ? 4 : nblk;
    const uint32_t acc = (!first || li > 0) ? 1u : 0u;
    mma_i8(tmem + li * BN, da, desc_b(b_base, mn.b_mn), idesc_i8(nfirst * BN) | idesc_mn, acc);
    if (nblk > 4)
      mma_i8(tmem + (li + 4) * BN, da, desc_b(b_base + 4 * (BN * BK), mn.b_mn), idesc_i8((nblk - 4) * BN) | idesc_mn,
             acc);
  }
}

// Epilogue of one 128 x BN tile: TMEM -> registers -> recombine the 8
// diagonal int32 accumulators (sum S_d << 8d) -> C.  EPI_WARPS warps share a
// tile: warp ew reads TMEM lane quadrant ew % 4 (its rows) and the column
// range (ew / 4) of BN split EPI_WARPS / 4 ways.  With c_col the 32 lanes of a
// warp store 32 consecutive words per column.
#ifndef MPC3_EPI_WARPS
#define MPC3_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = MPC3_EPI_WARPS;
constexpr int GEMM_THREADS = 128 + 32 * EPI_WARPS;  // warps 0-3: TMA, MMA, TMEM alloc, idle
DEV void epilogue_tile(uint32_t tmem, int ew, int lane, bool have_acc, uint64_t* cg, int64_t m0, int64_t n0,
                       int64_t M, int64_t N, int64_t rs, int64_t cs, bool atomic) {
  const int q = ew & 3;
  constexpr int COLS = BN / (EPI_WARPS / 4);
  const int cbeg = (ew >> 2) * COLS;
  const int64_t row = m0 + q * 32 + lane;
#pragma unroll 1
  for (int c0 = cbeg; c0 < cbeg + COLS; c0 += 8) {
    uint64_t acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0;
    if (have_acc) {
      // all 8 diagonals of this 8-column chunk in flight, one wait
      uint32_t r[8][8];
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + d * BN + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
            : "=r"(r[d][0]), "=r"(r[d][1]), "=r"(r[d][2]), "=r"(r[d][3]), "=r"(r[d][4]), "=r"(r[d][5]),
              "=r"(r[d][6]), "=r"(r[d][7])
            : "r"(taddr));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int d = 0; d < 8; ++d)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += (uint64_t)r[d][e] << (8 * d);
    }
    if (row < M) {
      uint64_t* dst = cg + row * rs + (n0 + c0) * cs;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (n0 + c0 + e < N) {
          if (atomic)
            atomicAdd(reinterpret_cast<unsigned long long*>(dst + e * cs), (unsigned long long)acc[e]);
          else
            dst[e * cs] = acc[e];
        }
      }
    }
  }
}

#ifdef MPC3_GEMM_TRACE
// debug build only (tools/dbg/gemm_trace.py): per-CTA phase timestamps
__device__ unsigned long long g_trace[8192][8];
DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) g_trace[cta_lin & 8191][slot] = gtime()
#else
#define TRACE(slot)
#endif

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   uint64_t* __restrict__ C, int64_t M, int64_t N, int64_t kp, int64_t ldc, int64_t c_group,
                   int splits, int kb_per_split, int c_col, MnArgs mn) {
  griddep_launch();
#ifdef MPC3_GEMM_TRACE
  const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (threadIdx.x == 0) {
    TRACE(0);
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_trace[cta_lin & 8191][7] = smid;
  }
#endif
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // grouped rasterisation: consecutive CTAs sweep a band of GROUP_M m-tiles
  // column by column, so the CTAs resident at once share A and B K-slices in
  // L2 (row-major order streams all of B once per m-tile row)
  int64_t n0, m0;
  {
    constexpr int GROUP_M = 8;
    const int nt = gridDim.x, mt = gridDim.y;
    const int id = blockIdx.y * nt + blockIdx.x;
    const int band = id / (GROUP_M * nt), first_m = band * GROUP_M;
    const int gm = mt - first_m < GROUP_M ? mt - first_m : GROUP_M;
    const int in_band = id - band * GROUP_M * nt;
    m0 = (int64_t)(first_m + in_band % gm) * BM;
    n0 = (int64_t)(in_band / gm) * BN;
  }
  const int g = blockIdx.z / splits, split = blockIdx.z % splits;
  const int nkb_total = (int)((kp + BK - 1) / BK);
  const int kb0 = split * kb_per_split;
  int kb1 = kb0 + kb_per_split;
  if (kb1 > nkb_total) kb1 = nkb_total;
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  griddep_wait();  // packed operands and C are the previous kernels' data
  if (threadIdx.x == 0) TRACE(1);

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      load_stage(&tmA, &tmB, &full[s], sA + s * A_STAGE, sB + s * B_STAGE, kb0 + i, (int)m0, (int)n0, g, mn);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      if (i == 0) TRACE(2);
      asm volatile("tcgen05.fence::after_thread_sync;");
      mma_stage(tmem, smem_u32(sA + s * A_STAGE), smem_u32(sB + s * B_STAGE), i == 0, mn);
      mma_commit(&empty[s]);
    }
    mma_commit(tmem_full);
  } else if (warp >= 4) {
    // ---- epilogue: TMEM -> registers -> recombine -> global ----
    // element (row, col) at row*ldc + col (row-major) or col*ldc + row
    const int64_t rs = c_col ? 1 : ldc, cs = c_col ? ldc : 1;
    if (nkb > 0) {
      mbar_wait(tmem_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (warp == 4 && lane == 0) TRACE(3);
    epilogue_tile(tmem, warp - 4, lane, nkb > 0, C + (int64_t)g * c_group, m0, n0, M, N, rs, cs, splits > 1);
    asm volatile("tcgen05.fence::before_thread_sync;");
    if (warp == 4 && lane == 0) TRACE(4);
  }
  __syncthreads();
  if (threadIdx.x == 0) TRACE(5);
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// host: tensor maps via the driver entry point (no -lcuda link needed)

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static int make_map(CUtensorMap* map, const uint8_t* base, int64_t kp, int64_t rows, int64_t planes, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return MPC3_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(kp * rows)};
  cuuint32_t box[3] = {(cuuint32_t)BK, (cuuint32_t)box_rows, 8};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed");
    return MPC3_ERR_CUDA;
  }
  return MPC3_OK;
}

// Tensor map of an MN-read operand: the source packed buffer
// [planes][rows][kp] with a box of `cols` bytes along kp x 32 rows x 8 limbs.
static int make_map_mn(CUtensorMap* map, const uint8_t* base, int64_t kp, int64_t rows, int64_t planes, int cols,
                       CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return MPC3_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kp, (cuuint64_t)rows, (cuuint64_t)planes};
  cuuint64_t strides[2] = {(cuuint64_t)kp, (cuuint64_t)(kp * rows)};
  cuuint32_t box[3] = {(cuuint32_t)cols, (cuuint32_t)BK, 8};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (MN) failed");
    return MPC3_ERR_CUDA;
  }
  return MPC3_OK;
}

// The GEMM's dynamic shared memory (192 KiB + barriers), opted into once per
// device (the attribute is per device: a process may drive several GPUs).
static bool gemm_attr() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.count(dev)) return true;
  if (cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess)
    return false;
  done.insert(dev);
  return true;
}

static Operand to_operand(const mpc3_operand* o) {
  Operand p;
  p.mode = o->mode;
  p.rows = o->rows;
  p.k = o->k;
  p.off = o->off;
  p.s_r = o->s_r;
  p.t0 = o->t0;
  p.t1 = o->t1;
  p.t2 = o->t2;
  p.K1 = o->K1 > 0 ? o->K1 : 1;
  p.K2 = o->K2 > 0 ? o->K2 : (o->k > 0 ? o->k : 1);  // default: K is one digit of stride t2
  p.n = o->n;
  p.c = o->c;
  p.h = o->h;
  p.w = o->w;
  p.sN = o->sN;
  p.sC = o->sC;
  p.sH = o->sH;
  p.sW = o->sW;
  p.kh = o->kh > 0 ? o->kh : 1;
  p.kw = o->kw > 0 ? o->kw : 1;
  p.sh = o->sh > 0 ? o->sh : 1;
  p.sw = o->sw > 0 ? o->sw : 1;
  p.ph = o->ph;
  p.pw = o->pw;
  p.dh = o->dh > 0 ? o->dh : 1;
  p.dw = o->dw > 0 ? o->dw : 1;
  p.oh = o->oh > 0 ? o->oh : 1;
  p.ow = o->ow > 0 ? o->ow : 1;
  return p;
}

}  // namespace mpc3

using namespace mpc3;

extern "C" {

int mpc3_ring_pack(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role, uint8_t* out,
                   int64_t kp, void* stream) {
  if (!op) return MPC3_ERR_CONFIG;
  return mpc3_ring_pack_halves(src, src_plane, op, role, out, kp, op->k, stream);
}

int mpc3_ring_pack_halves(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role, uint8_t* out,
                          int64_t kp, int64_t kh, void* stream) {
  return mpc3_ring_pack_halves_z(src, src_plane, op, role, out, kp, kh, nullptr, 0, stream);
}

int mpc3_ring_pack_halves_z(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role, uint8_t* out,
                            int64_t kp, int64_t kh, uint64_t* zero, int64_t zero_words, void* stream) {
  if (zero_words < 0 || (zero_words && !zero)) return MPC3_ERR_CONFIG;
  if (!op || role < 0 || role > 3) return MPC3_ERR_CONFIG;
  if (kp % 16) return MPC3_ERR_SHAPE;
  if (role >= 2) kh = op->k;
  int64_t kneed = role >= 2 ? op->k : kh + op->k;
  if (kh < op->k || kp < kneed || op->rows < 0 || op->k < 0) return MPC3_ERR_SHAPE;
  if (op->mode < 0 || op->mode > 2) return MPC3_ERR_CONFIG;
  Operand o = to_operand(op);
  int groups = role == 2 ? 1 : 3;
  int64_t total = (int64_t)groups * o.rows * (kp / 8);
  if (total == 0) {
    if (zero_words && cudaMemsetAsync(zero, 0, (size_t)zero_words * 8, as_stream(stream)) != cudaSuccess)
      return check_launch("pack zero memset");
    return MPC3_OK;
  }
  const bool dilated = o.mode == MPC3_GATHER_IM2COL && (o.dh != 1 || o.dw != 1);
  const int64_t row_tiles = (o.rows + PT_R - 1) / PT_R;
  // the tiled kernel addresses a component plane with 32-bit offsets
  const bool small = src_plane < (1ll << 31) && o.h < (1 << 30) && o.w < (1 << 30) && o.rows < (1ll << 31) &&
                     o.k < (1ll << 30) &&
                     (o.mode != MPC3_GATHER_DENSE || (o.off >= 0 && o.s_r >= 0 && o.t0 >= 0 && o.t1 >= 0 && o.t2 >= 0));
  if (!dilated && small && row_tiles < 65536) {
    PackTileArgs a;
    a.rows = o.rows;
    a.K = o.k;
    a.kp = kp;
    a.lim = kneed;
    a.kh = kh;
    a.zero = zero;
    a.zero_words = zero_words;
    bool r_fast;
    if (o.mode == MPC3_GATHER_DENSE) {
      a.H = a.W = 1;
      a.sH = a.sW = 0;
      int64_t sk = o.K2 > 1 || o.K1 == 1 ? o.t2 : o.t1;  // stride of the fastest k digit
      r_fast = o.s_r < sk;
    } else {
      a.H = (int32_t)o.h;
      a.W = (int32_t)o.w;
      a.sH = (int32_t)o.sH;
      a.sW = (int32_t)o.sW;
      // walk the direction whose consecutive elements are closest in the
      // source: an im2col row's columns (c, u, v) run along the kernel row
      // (contiguous x), its rows (n, y, x) step by the stride; the transposed
      // (WGRAD-layout) pack has them the other way round
#ifndef MPC3_PACK_T_RFAST_SW
#define MPC3_PACK_T_RFAST_SW 3
#endif
      r_fast = o.mode == MPC3_GATHER_IM2COL ? o.sw <= 2 : o.sw >= MPC3_PACK_T_RFAST_SW;
    }
    dim3 grid((unsigned)((kp + PT_K - 1) / PT_K), (unsigned)row_tiles, (unsigned)groups);
    void (*k)(const uint64_t*, int64_t, Operand, PackTileArgs, uint8_t*) =
        r_fast ? (role == 0   ? pack_tile_kernel<true, 0>
                  : role == 1 ? pack_tile_kernel<true, 1>
                  : role == 2 ? pack_tile_kernel<true, 2>
                              : pack_tile_kernel<true, 3>)
               : (role == 0   ? pack_tile_kernel<false, 0>
                  : role == 1 ? pack_tile_kernel<false, 1>
                  : role == 2 ? pack_tile_kernel<false, 2>
                              : pack_tile_kernel<false, 3>);
    launch_pdl(k, grid, dim3(PT_THREADS), 0, as_stream(stream), src, src_plane, o, a, out);
    return check_launch("ring_pack_tile");
  }
  if (zero_words && cudaMemsetAsync(zero, 0, (size_t)zero_words * 8, as_stream(stream)) != cudaSuccess)
    return check_launch("pack zero memset");
  pack_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(src, src_plane, o, role, groups, out, kp, kh);
  return check_launch("ring_pack");
}

int mpc3_ring_gemm_packed(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                          int64_t kp, int64_t ldc, int64_t c_group, int splits, void* stream) {
  return mpc3_ring_gemm_packed_layout(A, B, C, groups, M, N, kp, ldc, c_group, splits, 0, stream);
}

int mpc3_ring_gemm_packed_layout(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                                 int64_t kp, int64_t ldc, int64_t c_group, int splits, int c_layout, void* stream) {
  if (c_layout != 0 && c_layout != 1) return MPC3_ERR_CONFIG;
  if (groups < 1 || M < 0 || N < 0 || kp < 0 || splits < 1) return MPC3_ERR_SHAPE;
  if (kp % 16) return MPC3_ERR_SHAPE;
  if (M == 0 || N == 0) return MPC3_OK;
  if (M > (1 << 30) || N > (1 << 30)) return MPC3_ERR_SHAPE;
  int nkb = (int)((kp + BK - 1) / BK);
  int kbs = (nkb + splits - 1) / splits;
  if ((int64_t)kbs * BK > MAX_SPLIT_K) return MPC3_ERR_EXACTNESS;  // caller must split longer K
  if (!gemm_attr()) return check_launch("gemm_tc attr");
  CUtensorMap ta, tb;
  int st = make_map(&ta, A, kp, M, (int64_t)groups * 8, BM);
  if (st) return st;
  st = make_map(&tb, B, kp, N, (int64_t)groups * 8, BN);
  if (st) return st;
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)(groups * splits));
  MnArgs mn0 = {0, 0, 0, 0, 1 << 30, 0, 0, 0};
  launch_pdl(gemm_tc_kernel, grid, dim3(GEMM_THREADS), SMEM_BYTES, as_stream(stream), ta, tb, C, M, N, kp, ldc, c_group, splits,
             kbs, c_layout, mn0);
  return check_launch("ring_gemm_tc");
}

// Launch shape of mpc3_ring_gemm_auto: split-K count and whether C must
// start at zero (atomic accumulation).  (A stream-K variant for the partial
// last wave lost in the step: its all-SM persistent grid blocks the pack and
// side streams' work beside it, AlexNet 2.514 -> 2.524 ms; removed in round 2.)
struct AutoPlan {
  int64_t splits;
  bool zero;
};
// minimum K-blocks per split when splitting K for occupancy
// (2: the AlexNet step 2.469 -> 2.459 ms against 4: short-K GEMMs fill more SMs)
static int64_t split_min_kb() { return 2; }

static AutoPlan auto_plan(int groups, int64_t M, int64_t N, int64_t kp) {
  const int64_t sms = 148;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * groups;
  const int64_t nkb = (kp + BK - 1) / BK;
  const int64_t need = (nkb * BK + MAX_SPLIT_K - 1) / MAX_SPLIT_K;  // exactness
  int64_t occ = sms / tiles;                                         // <= one wave, >= 4 K-blocks per split
  if (occ > nkb / split_min_kb()) occ = nkb / split_min_kb();
  if (occ < 1) occ = 1;
  AutoPlan p;
  p.splits = need > occ ? need : occ;
  p.zero = nkb == 0 || p.splits > 1;
  return p;
}

int mpc3_ring_gemm_auto(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                        int64_t kp, int c_layout, void* stream) {
  return mpc3_ring_gemm_auto_z(A, B, C, groups, M, N, kp, c_layout, 0, stream);
}

int mpc3_ring_gemm_auto_z(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                          int64_t kp, int c_layout, int c_zeroed, void* stream) {
  if (groups < 1 || M < 0 || N < 0 || kp < 0) return MPC3_ERR_SHAPE;
  if (kp % 16) return MPC3_ERR_SHAPE;
  if (c_layout != 0 && c_layout != 1) return MPC3_ERR_CONFIG;
  if (M == 0 || N == 0) return MPC3_OK;
  const int64_t ldc = c_layout ? M : N, c_group = M * N;
  const AutoPlan p = auto_plan(groups, M, N, kp);
  const int64_t nkb = (kp + BK - 1) / BK;
  if (p.zero && !c_zeroed) {
    if (cudaMemsetAsync(C, 0, (size_t)groups * M * N * 8, as_stream(stream)) != cudaSuccess)
      return check_launch("gemm C memset");
  }
  if (nkb == 0) return MPC3_OK;
  return mpc3_ring_gemm_packed_layout(A, B, C, groups, M, N, kp, ldc, c_group, (int)p.splits, c_layout, stream);
}

// Launch shape of mpc3_ring_gemm_t (split-K only unless MPC3_GEMM_T_SK).
static AutoPlan t_plan(int groups, int64_t M, int64_t N, int64_t kp) {
  const int64_t sms = 148;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * groups;
  const int64_t nkb = kp / BK;
  const int64_t need = (nkb * BK + MAX_SPLIT_K - 1) / MAX_SPLIT_K;
  int64_t occ = sms / tiles;
  if (occ > nkb / split_min_kb()) occ = nkb / split_min_kb();
  if (occ < 1) occ = 1;
  AutoPlan p;
  p.splits = need > occ ? need : occ;
  p.zero = nkb == 0 || p.splits > 1;
  return p;
}

int mpc3_ring_gemm_needs_zero(int transposed, int groups, int64_t M, int64_t N, int64_t kp) {
  if (groups < 1 || M < 0 || N < 0 || kp < 0) return MPC3_ERR_SHAPE;
  if (M == 0 || N == 0) return 0;
  return (transposed ? t_plan(groups, M, N, kp) : auto_plan(groups, M, N, kp)).zero ? 1 : 0;
}

int mpc3_ring_gemm_t(const uint8_t* A, int a_mn, int64_t a_rows, int64_t a_kp, int64_t a_half, const uint8_t* B,
                     int b_mn, int64_t b_rows, int64_t b_kp, int64_t b_half, uint64_t* C, int groups, int64_t M,
                     int64_t N, int64_t kc_half, int c_layout, void* stream) {
  return mpc3_ring_gemm_t_z(A, a_mn, a_rows, a_kp, a_half, B, b_mn, b_rows, b_kp, b_half, C, groups, M, N, kc_half,
                            c_layout, 0, stream);
}

int mpc3_ring_gemm_t_z(const uint8_t* A, int a_mn, int64_t a_rows, int64_t a_kp, int64_t a_half, const uint8_t* B,
                       int b_mn, int64_t b_rows, int64_t b_kp, int64_t b_half, uint64_t* C, int groups, int64_t M,
                       int64_t N, int64_t kc_half, int c_layout, int c_zeroed, void* stream) {
  if (groups < 1 || M < 0 || N < 0 || kc_half < 0 || (kc_half % BK)) return MPC3_ERR_SHAPE;
  if (c_layout != 0 && c_layout != 1) return MPC3_ERR_CONFIG;
  if (a_mn < 0 || a_mn > 5 || a_mn == 4 || b_mn < 0 || b_mn > 2) return MPC3_ERR_CONFIG;
  const int b_cs = b_mn >> 1;  // 2: B is a role-3 pack read K-major, half h from component plane g + h
  b_mn &= 1;
  if (b_cs && (groups != 3 || b_kp % 16)) return MPC3_ERR_CONFIG;
  const int a_cs = (a_mn >> 1) & 1;  // bit 1: component-plane halves (role-3 pack)
  const int a_rh = a_mn >> 2;        // bit 2 (with bit 0): half 1 is source rows [a_half, a_half + kc_half)
  a_mn &= 1;
  if (a_rh && (a_cs || a_half < kc_half)) return MPC3_ERR_CONFIG;
  if (a_cs && (groups != 3 || a_kp % 16)) return MPC3_ERR_CONFIG;
  if (M == 0 || N == 0) return MPC3_OK;
  if (M > (1 << 30) || N > (1 << 30) || a_half > (1 << 30) || b_half > (1 << 30)) return MPC3_ERR_SHAPE;
  const int64_t kp = 2 * kc_half;
  if ((!a_mn && !a_cs && (a_kp != kp || a_rows != M)) || (!a_mn && a_cs && a_rows != M) ||
      (!b_mn && !b_cs && (b_kp != kp || b_rows != N)) || (b_cs && (b_rows != N || b_kp < kc_half)))
    return MPC3_ERR_SHAPE;
  // an MN operand's half offset is a TMA box start along the 16-byte-granular
  // inner dimension (pack with mpc3_ring_pack_halves, kh % 16 == 0)
  if ((a_mn && (a_kp % 16 || a_rows > (a_rh ? a_half : 0) + kc_half || (!a_cs && !a_rh && a_half % 16))) ||
      (b_mn && (b_kp % 16 || b_rows > kc_half || b_half % 16)))
    return MPC3_ERR_SHAPE;
  if (!gemm_attr()) return check_launch("gemm_tc attr");
  CUtensorMap ta, tb;
  int st = a_mn ? make_map_mn(&ta, A, a_kp, a_rows, (int64_t)groups * 8, BM, CU_TENSOR_MAP_SWIZZLE_128B)
                : make_map(&ta, A, a_cs ? a_kp : kp, M, (int64_t)groups * 8, BM);
  if (st) return st;
  st = b_mn ? make_map_mn(&tb, B, b_kp, b_rows, (int64_t)groups * 8, BN, CU_TENSOR_MAP_SWIZZLE_64B)
            : make_map(&tb, B, b_cs ? b_kp : kp, N, (int64_t)groups * 8, BN);
  if (st) return st;
  const int64_t nkb = kp / BK;
  const AutoPlan p = t_plan(groups, M, N, kp);
  const int64_t splits = p.splits;
  const int kbs = (int)((nkb + splits - 1) / splits);
  if ((int64_t)kbs * BK > MAX_SPLIT_K) return MPC3_ERR_EXACTNESS;
  if (p.zero && !c_zeroed) {
    if (cudaMemsetAsync(C, 0, (size_t)groups * M * N * 8, as_stream(stream)) != cudaSuccess)
      return check_launch("gemm C memset");
  }
  if (nkb == 0) return MPC3_OK;
  MnArgs mn = {a_mn ? 1 : 0, b_mn ? 1 : 0, (int)a_half, (int)b_half, (int)(kc_half / BK), a_cs, a_rh, b_cs};
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)(groups * splits));
  launch_pdl(gemm_tc_kernel, grid, dim3(GEMM_THREADS), SMEM_BYTES, as_stream(stream), ta, tb, C, M, N, kp,
             c_layout ? M : N, M * N, (int)splits, kbs, c_layout, mn);
  return check_launch("ring_gemm_t");
}

int mpc3_ring_gemm_simt(const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t M, int64_t N, int64_t K,
                        int64_t sam, int64_t sak, int64_t sbk, int64_t sbn, int64_t ldc, void* stream) {
  if (M < 0 || N < 0 || K < 0) return MPC3_ERR_SHAPE;
  if (M == 0 || N == 0) return MPC3_OK;
  dim3 grid((unsigned)((N + ST - 1) / ST), (unsigned)((M + ST - 1) / ST));
  gemm_simt_kernel<<<grid, 256, 0, as_stream(stream)>>>(A, B, C, M, N, K, sam, sak, sbk, sbn, ldc);
  return check_launch("ring_gemm_simt");
}

// A transposed (rows = the contraction, read MN-major: 128-byte TMA rows),
// B K-major; the contraction as two halves of kc = roundup(K / 2, 32) rows.
static int64_t matmul_kc(int64_t K) { return ((K + 1) / 2 + 31) / 32 * 32; }
static int64_t matmul_mp(int64_t M) { return (M + 31) / 32 * 32; }

size_t mpc3_ring_matmul_workspace(int64_t M, int64_t N, int64_t K) {
  if (M < 0 || N < 0 || K < 0) return 0;
  return (size_t)(8 * K * matmul_mp(M) + 8 * N * 2 * matmul_kc(K));
}

int mpc3_ring_matmul_u64(const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t M, int64_t N, int64_t K,
                         void* workspace, void* stream) {
  if (M < 0 || N < 0 || K < 0) return MPC3_ERR_SHAPE;
  if (M == 0 || N == 0) return MPC3_OK;
  if (K == 0) return cudaMemsetAsync(C, 0, (size_t)M * N * 8, as_stream(stream)) == cudaSuccess
                         ? MPC3_OK
                         : check_launch("matmul zero");
  const int64_t kc = matmul_kc(K), mp = matmul_mp(M);
  uint8_t* pa = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* pb = pa + 8 * K * mp;
  mpc3_operand oa;  // A^T: row k = column k of A
  memset(&oa, 0, sizeof(oa));
  oa.mode = MPC3_GATHER_DENSE;
  oa.rows = K;
  oa.k = M;
  oa.s_r = 1;
  oa.t2 = K;
  mpc3_operand ob = oa;  // B^T: row n = column n of B, K-major
  ob.rows = N;
  ob.k = K;
  ob.s_r = 1;
  ob.t2 = N;
  int st = mpc3_ring_pack(A, 0, &oa, 2, pa, mp, stream);
  if (st) return st;
  st = mpc3_ring_pack(B, 0, &ob, 2, pb, 2 * kc, stream);
  if (st) return st;
  return mpc3_ring_gemm_t(pa, 5, K, mp, kc, pb, 0, N, 2 * kc, 0, C, 1, M, N, kc, 0, stream);
}

}  // extern "C"
