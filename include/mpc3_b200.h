/*
 * mpc3_b200.h — C ABI of the B200-native 3-party replicated-secret-sharing
 * engine over Z_2^64 (CryptGPU, arXiv 2104.10949).
 *
 * The reference (`mpc3`, pure Python) has no FFI; its drop-in boundary is the
 * Python protocol API and the duck-typed nn engine seam.
 * Every entry point below is the native body of one reference function; the
 * comment on each cites the reference file:line it replaces
 * (paths relative to /root/reference/pkg/src/mpc3/).
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers (cudaMalloc / torch storage) to
 *    little-endian uint64 ring words, except where stated.  The library never
 *    retains caller buffers and never allocates on the hot path; the caller
 *    owns outputs and workspaces.
 *  - A "trio" tensor of n elements is the three additive (or XOR) share
 *    components stored as 3 planes: component c at ptr[c * n + e].  Party i's
 *    replicated share (lo, hi) is (plane i, plane (i+1)%3) (sharing.py:37-49).
 *  - rk3 points to 3 x 44 uint32 AES-128 round-key words (keys k_0, k_1, k_2
 *    of the session, as produced by mpc3_aes128_expand).
 *  - Counters j_* are the per-purpose lockstep stream counters that
 *    PartyContext.take (sharing.py:225-230) would hand out; the host keeps
 *    them and checks freshness before launch (sharing.py:190-204).
 *  - ctr (nullable) is a DEVICE pointer to uint64[8] indexed by purpose tag;
 *    the effective counter is j + ctr[purpose].  A CUDA graph captured with a
 *    ctr buffer advances its PRF counters on every replay by bumping ctr,
 *    reproducing the sequential counter schedule of the reference.
 *  - `stream` is a cudaStream_t passed as void*.  Calls are asynchronous on
 *    it and reentrant.  Return value: MPC3_OK or an error status; statuses
 *    map 1:1 onto the reference's exception taxonomy (errors.py:4-53).
 */
#ifndef MPC3_B200_H
#define MPC3_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-53) ---- */
#define MPC3_OK 0
#define MPC3_ERR_RANGE 1      /* RangeError      */
#define MPC3_ERR_SHAPE 2      /* ShapeError      */
#define MPC3_ERR_EXACTNESS 3  /* ExactnessError  */
#define MPC3_ERR_CONFIG 4     /* ConfigError     */
#define MPC3_ERR_FRESHNESS 5  /* FreshnessError  */
#define MPC3_ERR_TOPOLOGY 6   /* TopologyError   */
#define MPC3_ERR_INTEGRITY 7  /* IntegrityError  */
#define MPC3_ERR_CUDA 100     /* CUDA runtime / launch failure */
#define MPC3_ERR_UNSUPPORTED 101 /* device is not sm_100 */

#define MPC3_ABI_VERSION 1

int mpc3_abi_version(void);
const char* mpc3_status_name(int status);
/* Last CUDA error string seen by the library on this thread (diagnostics). */
const char* mpc3_last_error(void);

/* ---- PRF (prf.py:31-61) ---- */

/* Host function: AES-128 key expansion of one 16-byte key (prf.py:36-38,
 * the key schedule behind cryptography's AES). */
int mpc3_aes128_expand(const uint8_t key[16], uint32_t round_keys[44]);

/* words[i] = word (word_off + i) of stream (key, purpose, index); the stream
 * is PrfKey.words(purpose, index, .) of prf.py:40-49, seekable by word.
 * rk = one key's 44 round-key words (device). */
int mpc3_prf_words(const uint32_t* rk, uint32_t purpose, uint64_t index, uint64_t word_off,
                   uint64_t count, uint64_t* words, void* stream);

/* Arithmetic (xor_mode=0) or XOR (xor_mode=1) zero sharing of n words,
 * trio output z_i = F(k_i) -/^ F(k_{i-1}) (sharing.py:233-250). */
int mpc3_rss_zero_share(const uint32_t* rk3, const uint64_t* ctr, uint32_t purpose, uint64_t index, int xor_mode,
                        uint64_t n, uint64_t* out_trio, void* stream);

/* ---- host->device boundary: encoding and dealing (ring.py:104-115,
 *      sharing.py:113-118, session.py:62-91) ---- */

/* Fixed-point encoding of float64 inputs: round-half-away-from-zero of
 * x * 2^t, two's complement; *bad (device int, nullable) is set to 1 when
 * some |x| >= 2^(63-t) or is not finite (the reference's RangeError). */
int mpc3_fx_encode(const double* x, uint64_t* out, uint64_t n, int t, int* bad, void* stream);

/* Dealer on the device, bit-exact with numpy's PCG64 Generator:
 * c0 = the next n draws of rng.integers(0, 2^64), c1 = the following n,
 * c2 = x - c0 - c1, written as trio planes.  (state, inc) is the 128-bit
 * PCG64 state of the host Generator (bit_generator.state); the caller then
 * advances the host Generator by 2n (bit_generator.advance). */
int mpc3_deal_pcg64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, const uint64_t* x,
                    uint64_t* out_trio, uint64_t n, void* stream);

/* ---- local ring ops (ring.py:50-79, protocols.py:57-72, sharing.py:54-67) ---- */
#define MPC3_EW_ADD 0      /* out = a + b          */
#define MPC3_EW_SUB 1      /* out = a - b          */
#define MPC3_EW_NEG 2      /* out = -a             */
#define MPC3_EW_MULC 3     /* out = a * c          */
#define MPC3_EW_ADDC 4     /* out = a + c          */
#define MPC3_EW_XOR 5      /* out = a ^ b          */
#define MPC3_EW_SHL 6      /* out = a << c         */
#define MPC3_EW_SHR 7      /* out = a >> c (logical) */
#define MPC3_EW_SAR 8      /* out = sar(a, c)      */
#define MPC3_EW_AXPY 9     /* out = a + c * b      */
/* Elementwise over n words; b may be NULL for unary ops. */
int mpc3_ring_ew(int op, const uint64_t* a, const uint64_t* b, uint64_t c, uint64_t* out, uint64_t n,
                 void* stream);

/* Broadcast-add along a trailing axis: out[r, j] = a[r, j] op b[r] (max_tree /
 * softmax centring, protocols.py:463-466).  op: ADD or SUB.  rows x cols. */
int mpc3_ring_rowop(int op, const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t rows,
                    uint64_t cols, void* stream);

/* Row sums of the last axis: out[r] = sum_j a[r, j] (protocols.py:466). */
int mpc3_ring_rowsum(const uint64_t* a, uint64_t* out, uint64_t rows, uint64_t cols, void* stream);

/* ---- elementwise protocols on trio tensors ----
 * elem_off (even): global stream-word index of the call's element 0, i.e. the
 * offset of a batch shard inside the reference's flat tensor (0 when the call
 * covers the whole tensor); PRF words are drawn at elem_off + local index. */

/* mul (protocols.py:79-94): out = reshare(x*y), 1 ARITH_ZERO counter. */
int mpc3_rss_mul(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, const uint64_t* x, const uint64_t* y,
                 uint64_t* out, uint64_t n, uint64_t elem_off, void* stream);

/* truncate (protocols.py:171-216): bits in [1,61]; TRUNC_RHO and TRUNC_R counters. */
int mpc3_rss_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, const uint64_t* x,
                      uint64_t* out, uint64_t n, uint64_t elem_off, void* stream);

/* mul + truncate fused (protocols.py:79-94 then 171-216; the `truncate(mul())`
 * pairs of exp_approx / reciprocal / division / softmax, 414-468). */
int mpc3_rss_mul_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r, int bits,
                          const uint64_t* x, const uint64_t* y, uint64_t* out, uint64_t n, uint64_t elem_off,
                          void* stream);

/* SGD update of every parameter in one launch (nn.py:539-543):
 * param_i <- param_i - truncate(c * grad_i, bits), in place, tensor i's
 * truncation words from TRUNC_RHO j_rho and TRUNC_R j_r (the counters its
 * own truncate call would take).  Trio tensors: 3 planes of n words. */
#define MPC3_SGD_MAX_TENSORS 64
typedef struct {
  uint64_t* param;
  const uint64_t* grad;
  uint64_t n, j_rho, j_r;
} MPC3SgdTensor;
int mpc3_rss_sgd_multi(const uint32_t* rk3, const uint64_t* ctr, const MPC3SgdTensor* ts, int nt, int bits,
                       uint64_t c, void* stream);

/* One level of max_tree (protocols.py:356-380) on a (rows, m) trio tensor v
 * (3 planes of rows*m words): out[r, j] = v[r, 2j+1] + relu(v[r, 2j] -
 * v[r, 2j+1]) for j < m/2, and out[r, m/2] = v[r, m-1] when m is odd; out is
 * (rows, m/2 + m%2).  The relu draws its words as mpc3_rss_sign mode 3 on the
 * (rows, m/2) difference tensor (counters j_bin, j_xor..+6, j_arith..+2;
 * elem_off / n_total for batch shards).  One launch instead of the
 * slice / sub / relu / add / concat sequence. */
int mpc3_rss_max_level(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                       const uint64_t* v, uint64_t* out, uint64_t rows, uint64_t m, uint64_t elem_off,
                       uint64_t n_total, void* stream);

/* The whole max_tree (protocols.py:356-380) of rows x m in ONE launch:
 * `levels` = the number of halvings of m down to 1; level l uses BIN
 * j_bin[l], XOR_ZERO j_xor[l]..+6 and ARITH_ZERO j_arith[l]..+2 (host
 * arrays), exactly the counters of mpc3_rss_max_level per level.  scratch:
 * 2 * 3 * rows * ceil(m/2) words; out: (rows, 1).  row_off / rows_total: a
 * batch shard of the rows (row_off even). */
int mpc3_rss_max_tree(const uint32_t* rk3, const uint64_t* ctr, int levels, const uint64_t* j_bin,
                      const uint64_t* j_xor, const uint64_t* j_arith, const uint64_t* v, uint64_t* scratch,
                      uint64_t* out, uint64_t rows, uint64_t m, uint64_t row_off, uint64_t rows_total, void* stream);

/* Fused elementwise chain over a per-element trio z (starts as x), the chain
 * input x and a temporary t; replaces the launch-per-call sequences of
 * exp_approx (add_const + squarings, protocols.py:414-424) and reciprocal
 * (Newton iterations, protocols.py:427-440).  The k-th SQ/SQT/MULX step uses
 * counters j_arith + k, j_rho + k, j_r + k (the counters the unfused
 * mul_truncate calls take).  Output: z. */
#define MPC3_CHAIN_MAX_STEPS 48
#define MPC3_CHAIN_ADDC 0   /* z.c0 += c (public constant into component 0, protocols.py:57-62) */
#define MPC3_CHAIN_SETC 1   /* z = (c, 0, 0) (const_share, sharing.py:184-187) */
#define MPC3_CHAIN_SQ 2     /* z = truncate(mul(z, z), bits) */
#define MPC3_CHAIN_MULX 3   /* t = truncate(mul(x, t), bits) */
#define MPC3_CHAIN_NEWTON 4 /* z = 2 z - t */
#define MPC3_CHAIN_SQT 5    /* t = truncate(mul(z, z), bits) */
typedef struct {
  int op, bits;
  uint64_t c;
} MPC3ChainStep;
int mpc3_rss_chain(const uint32_t* rk3, const uint64_t* ctr, const MPC3ChainStep* steps, int nsteps, uint64_t j_arith,
                   uint64_t j_rho, uint64_t j_r, const uint64_t* x, uint64_t* out, uint64_t n, uint64_t elem_off,
                   void* stream);

/* Sign circuit (protocols.py:266-348): a2b + 64-bit Kogge-Stone + msb +
 * bit_inject + relu, fused, all 11 rounds in registers.
 * mode 0 = a2b (out: XOR trio of x), 1 = msb (XOR trio of the sign bit),
 * 2 = drelu (arithmetic {0,1} trio), 3 = relu (out = relu, mask = drelu).
 * Counters: BIN_INPUT j_bin; XOR_ZERO j_xor..j_xor+6; ARITH_ZERO j_arith..+2
 * (modes 2/3 use 2/3 of them).  n_total/elem_off allow a shard of a larger
 * tensor (the Kogge-Stone p-half lives at word n_total + e). */
int mpc3_rss_sign(const uint32_t* rk3, const uint64_t* ctr, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                  const uint64_t* x, uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total,
                  uint64_t elem_off, void* stream);


/* bit_inject of XOR-shared bits (protocols.py:304-331), 2 ARITH counters;
 * elem_off (even) = the global flat index of bits[0] (batch shard). */
int mpc3_rss_bit_inject(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, const uint64_t* bits, uint64_t* out,
                        uint64_t n, uint64_t elem_off, void* stream);

/* Output view of a bilinear result: the logical ("full") output is a 4-d
 * C-order tensor of sizes full[4]; PRF word index = its flat index.  Only the
 * sub-box [origin, origin + crop) is produced (the reference's crop /
 * embed of conv gradients, nn.py:456, 478-482).  Element (i0..i3) reads z at
 * z + sum i_k*z_stride[k] (plane stride z_plane) and writes
 * out + sum (i_k - origin_k)*out_stride[k] (plane stride out_plane). */
typedef struct {
  int64_t full[4];
  int64_t origin[4];
  int64_t crop[4];
  int64_t z_stride[4];
  int64_t out_stride[4];
  int64_t z_plane;
  int64_t out_plane;
} mpc3_view4;

/* Reshare of per-party local products z (z_i in plane i) followed by
 * truncation (protocols.py:110-117 / 129-136: _reshare then truncate).
 * bits = 0 skips truncation (bare reshare). */
int mpc3_rss_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r,
                              int bits, const uint64_t* z, const mpc3_view4* view, uint64_t* out,
                              uint64_t elem_off, void* stream);
/* Same, then a shared bias added component-wise (the inference extension's
 * folded-BN / FC bias: out = truncate(reshare(z)) + bias, a local add):
 * element i of the view gets bias[k * bias_plane + i_{bias_dim}] in
 * component k.  bias = NULL: no bias. */
int mpc3_rss_reshare_truncate_bias(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                   uint64_t j_r, int bits, const uint64_t* z, const mpc3_view4* view,
                                   const uint64_t* bias, int64_t bias_plane, int bias_dim, uint64_t* out,
                                   uint64_t elem_off, void* stream);

/* A secure layer's epilogue fused with the sign circuit after it
 * (conv2d_shares / matmul_shares then relu, protocols.py:97-136, 334-353):
 * the ReLU input is the layer's cross terms z (view: no crop / origin; bias
 * optional, as mpc3_rss_reshare_truncate_bias) reshared with ARITH_ZERO j_ra
 * and truncated by `bits` with TRUNC_RHO j_rho / TRUNC_R j_r in registers,
 * then the circuit as mpc3_rss_sign (mode, j_bin, j_xor, j_arith).  Shares
 * and PRF words are exactly those of the two separate calls; the reshared
 * tensor itself is never written.  out / mask: the view's full size n. */
int mpc3_rss_layer_sign(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_ra, uint64_t j_rho, uint64_t j_r,
                        int bits, const uint64_t* z, const mpc3_view4* view, const uint64_t* bias, int64_t bias_plane,
                        int bias_dim, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith, uint64_t* out,
                        uint64_t* mask, uint64_t elem_off, uint64_t n_total, void* stream);
/* Same with a residual block's shortcut added after the bias (the local add
 * of the inference extension's residual layer before its ReLU): element f of
 * the view gets res[k * res_plane + f] in component k (res_plane >= n).  The
 * caller takes the counters in the unfused order (the layer's reshare and
 * truncation before the shortcut branch, the ReLU's after). */
int mpc3_rss_layer_sign_residual(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_ra, uint64_t j_rho,
                                 uint64_t j_r, int bits, const uint64_t* z, const mpc3_view4* view,
                                 const uint64_t* bias, int64_t bias_plane, int bias_dim, const uint64_t* res,
                                 int64_t res_plane, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                                 uint64_t* out, uint64_t* mask, uint64_t elem_off, uint64_t n_total, void* stream);

/* Input gradient epilogue (nn.py:460-484): z holds per-party cross terms
 * cols[(n,y,x), (c,a,b)] = sum_o g[n,o,y,x] k[o,c,a,b] (a GEMM with inner
 * length O, instead of the reference's correlation of the dilated, padded
 * gradient with the flipped kernel).  Each element of the reference's full
 * output (N, C, hf, wf), hf = (OH-1)*sh + kh, is the col2im sum of its
 * contributions, reshared and truncated with PRF words at its flat index,
 * and written at (y'-ph, x'-pw) of out (N, C, H, W) when inside (out must be
 * zero-initialised; uncovered positions stay 0 as in the reference's embed). */
int mpc3_rss_col2im_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                     uint64_t j_r, int bits, const uint64_t* z, int64_t N, int64_t C, int64_t OH,
                                     int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw, int64_t H,
                                     int64_t W, uint64_t* out, uint64_t elem_off, void* stream);
/* Same with z's layout chosen: z_layout 1 = column-major cols (element
 * ((n,y,x), (c,a,b)) at ((c*kh+a)*kw+b) * N*OH*OW + (n*OH+y)*OW + x, the
 * GEMM's c_layout 1), so a warp's gathers for consecutive x coalesce. */
int mpc3_rss_col2im_reshare_truncate_layout(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith,
                                            uint64_t j_rho, uint64_t j_r, int bits, const uint64_t* z, int z_layout,
                                            int64_t N, int64_t C, int64_t OH, int64_t OW, int kh, int kw, int sh,
                                            int sw, int ph, int pw, int64_t H, int64_t W, uint64_t* out,
                                            uint64_t elem_off, void* stream);

/* avgpool (protocols.py:139-159): window sums, then truncate(log2 area) when
 * the area is a power of two, else mul_const(mulc) + truncate(t).  x/out are
 * trio NCHW; bits/mulc chosen by the caller (mulc = 1 for power-of-two).
 * ph/pw: zero padding with the full window area as divisor (the reference
 * has no padded pooling; used by ResNet's stem, composed as pad + avgpool). */
int mpc3_rss_avgpool(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, uint64_t mulc,
                     const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W,
                     int kh, int kw, int sh, int sw, int ph, int pw, uint64_t elem_off, void* stream);

/* avgpool backward (nn.py:487-499): scatter-add of g into the windows, then
 * div_area (truncate / mul_const+truncate) — fused. g: (N,C,OH,OW) trio;
 * out: (N,C,H,W) trio. */
int mpc3_rss_avgpool_backward(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, uint64_t mulc,
                              const uint64_t* g, uint64_t* out, int64_t N, int64_t C, int64_t H,
                              int64_t W, int64_t OH, int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw,
                              uint64_t elem_off, void* stream);

/* _avgpool_backward then the mask multiply of the ReLU before the pool
 * (nn.py:487-499, 515-517) in one pass: out = reshare(truncate(pool_bwd(g))
 * * mask) with TRUNC_RHO j_rho / TRUNC_R j_r then ARITH_ZERO j_arith, the
 * counters and shares of the two separate calls. */
int mpc3_rss_avgpool_backward_mask(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits,
                                   uint64_t mulc, const uint64_t* g, const uint64_t* mask, uint64_t j_arith,
                                   uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int64_t OH, int64_t OW,
                                   int kh, int kw, int sh, int sw, int ph, int pw, uint64_t elem_off, void* stream);

/* Max-pool windows of a trio tensor x (3, N, C, H, W) -> out (3, N*C*OH*OW,
 * kh*kw), (kh, kw) row-major; positions in the padding hold the public
 * constant `pad` in component 0 (sharing.py:184-187 const placement).  The
 * max-pool extension (absent from the reference) is then
 * max_tree (protocols.py:356-380) over each window row: the reference's
 * composition, bit for bit (tests/golden/make_golden_configs.py maxpool). */
int mpc3_rss_window_gather(const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W,
                           int kh, int kw, int sh, int sw, int ph, int pw, uint64_t pad, void* stream);

/* Plain sum-pool of one ring tensor (ring.py:259-268). */
int mpc3_ring_sumpool(const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W,
                      int kh, int kw, int sh, int sw, void* stream);

/* ---- ring GEMM (ring.py:144-256 bilinear_exact; protocols.py:97-136) ----
 *
 * Operands are packed into u8 limb planes: packed[g][limb][row][kp] with
 * limb l = byte l of the 64-bit word, kp = roundup(K, 16) (zero padded).
 * The tcgen05 kernel computes, per group g, C[g] = A[g] . B[g]^T over Z_2^64
 * with A (M rows) and B (N rows) both K-contiguous: 36 u8 x u8 limb-pair MMAs
 * accumulate 8 diagonal int32 sums S_d in TMEM; the epilogue recombines
 * sum_d S_d << 8d mod 2^64.  Exact for K <= 16512 per split (S_3 < 2^32);
 * longer K is split and the splits are added with 64-bit atomics. */

/* Operand gather descriptor for packing. */
#define MPC3_GATHER_DENSE 0   /* v(r,k) = src[off + r*s_r + k0*t0 + k1*t1 + k2*t2], k=(k0,k1,k2) */
#define MPC3_GATHER_IM2COL 1  /* r=(n,y,x), k=(c,u,v): in[n,c,(y*sh+u-ph)/dh,(x*sw+v-pw)/dw] */
#define MPC3_GATHER_WGRAD 2   /* r=(c,u,v), k=(n,y,x): in[n,c,y*sh+u-ph,x*sw+v-pw]           */
typedef struct {
  int mode;
  int64_t rows, k;         /* logical operand rows and inner length K */
  /* DENSE */
  int64_t off, s_r, t0, t1, t2, K1, K2;
  /* IM2COL / WGRAD geometry: input (N,C,H,W) with element strides */
  int64_t n, c, h, w, sN, sC, sH, sW;
  int64_t kh, kw, sh, sw, ph, pw, dh, dw, oh, ow;
} mpc3_operand;

/* Cross-term packing for the secure bilinear op (protocols.py:110-115):
 * for each party i, K' = 2K and
 *   role 0 (left operand):  row r of party i = [x_i + x_{i+1} | x_i]
 *   role 1 (right operand): row r of party i = [y_i | y_{i+1}]
 * so that z_i = x_i y_i + x_{i+1} y_i + x_i y_{i+1} is ONE ring GEMM with
 * inner length 2K.  role 2 packs a single plain operand (group count 1);
 * role 3 packs the three components as planes of their own ([3][8][rows][kp],
 * plane g = x_g, K columns): a role-1 operand stored once per component. 
 * src: trio planes (plane stride src_plane) or one plane for role 2.
 * out: [3 or 1][8][rows][kp], kp = roundup(K', 16). */
int mpc3_ring_pack(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role,
                   uint8_t* out, int64_t kp, void* stream);

/* mpc3_ring_pack with the second half at packed column kh >= K (zeros in
 * [K, kh)), kp >= kh + K: a 16-aligned kh lets another GEMM read the halves
 * in place as MN operands (mpc3_ring_gemm_t); kh = K is mpc3_ring_pack. */
int mpc3_ring_pack_halves(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role,
                          uint8_t* out, int64_t kp, int64_t kh, void* stream);

/* mpc3_ring_pack_halves that also clears zero[0 .. zero_words) (after the
 * previous kernel has finished): the C of the GEMM that follows, when that
 * GEMM accumulates atomically (mpc3_ring_gemm_needs_zero), so it needs no
 * memset launch of its own.  zero may be NULL (zero_words 0). */
int mpc3_ring_pack_halves_z(const uint64_t* src, int64_t src_plane, const mpc3_operand* op, int role,
                            uint8_t* out, int64_t kp, int64_t kh, uint64_t* zero, int64_t zero_words,
                            void* stream);

/* 1 if mpc3_ring_gemm_auto (transposed 0, kp = packed inner length) or
 * mpc3_ring_gemm_t (transposed 1, kp = 2 * kc_half) accumulates into C
 * atomically for this shape (so C must start at zero), else 0. */
int mpc3_ring_gemm_needs_zero(int transposed, int groups, int64_t M, int64_t N, int64_t kp);

/* C[g] (+)= A[g] . B[g]^T over Z_2^64 (tcgen05 kind::i8, TMA-fed).
 * A: [groups][8][M][kp] u8, B: [groups][8][N][kp] u8, C: rows M, cols N,
 * leading dim ldc, group stride c_group.  splits > 1 requires C zeroed (the
 * splits add with u64 atomics).  kp % 16 == 0. */
int mpc3_ring_gemm_packed(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M,
                          int64_t N, int64_t kp, int64_t ldc, int64_t c_group, int splits, void* stream);

/* Same with the C layout chosen: c_layout 0 = C[g][m][ldc] (as above),
 * 1 = C[g][n][ldc] (column-major: element (m, n) at n*ldc + m).  The
 * column-major form makes an NCHW conv output's (y, x) runs contiguous in C,
 * so the following reshare/truncate reads coalesce, and the epilogue's
 * stores coalesce across a warp's 32 rows. */
int mpc3_ring_gemm_packed_layout(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M,
                                 int64_t N, int64_t kp, int64_t ldc, int64_t c_group, int splits, int c_layout,
                                 void* stream);

/* C[g] = A[g] . B[g]^T with the launch shape chosen for the size: split-K
 * (exactness above 16384 K, occupancy for few tiles, <= one wave).  C is dense ([g][M][N], or
 * [g][N][M] for c_layout 1) and is zeroed here when partial sums are
 * accumulated atomically. */
int mpc3_ring_gemm_auto(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                        int64_t kp, int c_layout, void* stream);
/* Same; c_zeroed = 1 promises C is already zero where the launch needs it
 * (no memset issued). */
int mpc3_ring_gemm_auto_z(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N,
                          int64_t kp, int c_layout, int c_zeroed, void* stream);

/* C[g] = A[g] . B[g]^T where either operand may be read in place from
 * another GEMM's packed buffer, transposed ("MN" operand): the weight
 * gradient dW = g^T x of a layer consumes the input-gradient pass's role-0
 * pack of g and the forward pass's role-1 pack of x directly (nn.py:435-484).
 * The contraction runs over two halves of kc_half (a multiple of 32) each:
 *   MN operand  (x_mn = 1): source [groups][8][x_rows][x_kp] (x_rows <=
 *     kc_half, the rest zero), output row/column j of half h reads source
 *     column h * x_half + j; x_half % 16 == 0 (mpc3_ring_pack_halves);
 *   K-major     (x_mn = 0): a normal pack with x_rows = M (or N) and
 *     x_kp = 2 * kc_half, half h at columns [h * kc_half, (h+1) * kc_half).
 * a_mn bit 1 (values 2 / 3: K-major / MN): A is a role-3 pack (component
 *   planes, mpc3_ring_pack_halves role 3) of a role-1 operand [x_g | x_{g+1}]:
 *   half h of group g is read from component plane (g + h) % 3, at no column
 *   offset (a_half unused; K-major: a_kp = the component pack's kp, the
 *   contraction per half kc_half); groups must be 3.
 * b_mn = 2: B is a role-3 pack (component planes) read K-major, half h of
 *   group g from component plane (g + h) % 3 at no column offset (b_rows = N,
 *   b_kp >= kc_half, groups 3) — the weight gradient g^T x with x's
 *   transposed forward pack as B.
 * a_mn = 5 (bit 2 with MN): A is a plain transposed pack (rows = the
 *   contraction) whose second half is source ROWS [a_half, a_half +
 *   kc_half), a_half >= kc_half, a_rows <= a_half + kc_half (the rest zero).
 * C dense [g][M][N] (c_layout 0) or [g][N][M] (1); zeroed here when the
 * split-K partials add atomically. */
int mpc3_ring_gemm_t(const uint8_t* A, int a_mn, int64_t a_rows, int64_t a_kp, int64_t a_half, const uint8_t* B,
                     int b_mn, int64_t b_rows, int64_t b_kp, int64_t b_half, uint64_t* C, int groups, int64_t M,
                     int64_t N, int64_t kc_half, int c_layout, void* stream);
int mpc3_ring_gemm_t_z(const uint8_t* A, int a_mn, int64_t a_rows, int64_t a_kp, int64_t a_half, const uint8_t* B,
                       int b_mn, int64_t b_rows, int64_t b_kp, int64_t b_half, uint64_t* C, int groups, int64_t M,
                       int64_t N, int64_t kc_half, int c_layout, int c_zeroed, void* stream);

/* Reference GPU path (CUDA cores, 64-bit IMAD): C = A . B mod 2^64 with
 * arbitrary strides; used as an on-device cross-check and for tiny shapes. */
int mpc3_ring_gemm_simt(const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t M, int64_t N, int64_t K,
                        int64_t sam, int64_t sak, int64_t sbk, int64_t sbn, int64_t ldc, void* stream);

/* Convenience: plain ring matmul C (M,N) = A (M,K) . B (K,N), row-major,
 * exactly `bilinear_exact(a, b, matmul_spec(m,k,n))` (ring.py:183-222) minus
 * its 2^20 limit.  workspace >= mpc3_ring_matmul_workspace(M,N,K) bytes
 * (A packed transposed and read MN-major, B K-major: mpc3_ring_gemm_t with
 * a_mn = 5). */
size_t mpc3_ring_matmul_workspace(int64_t M, int64_t N, int64_t K);
int mpc3_ring_matmul_u64(const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t M, int64_t N,
                         int64_t K, void* workspace, void* stream);

/* The training step's loss gradient softmax(z) - y (nn.py:561-568;
 * protocols.py:453-468: max_tree, z - max, exp_approx, row sum, reciprocal,
 * mul + truncate) of a (rows, d) trio z against labels y, in ONE launch;
 * every step draws its unfused launch's counters and PRF words: max_tree
 * level counters as mpc3_rss_max_tree, the exp / reciprocal chain programs
 * and counters as mpc3_rss_chain, the final mul_truncate's (fin_j).
 * scratch: mpc3_rss_softmax_loss_scratch(rows, d) bytes. */
typedef struct {
  int levels;
  uint64_t j_bin[16], j_xor[16], j_arith[16];
  uint64_t exp_j[3];  /* ARITH_ZERO, TRUNC_RHO, TRUNC_R of the exp chain's first multiply */
  const MPC3ChainStep* exp_steps;
  int exp_count;
  uint64_t rec_j[3];
  const MPC3ChainStep* rec_steps;
  int rec_count;
  uint64_t fin_j[3];
  int bits;           /* the final truncation (t) */
  uint64_t row_off, rows_total;  /* batch shard (row_off even) */
} mpc3_softmax_loss_args;
size_t mpc3_rss_softmax_loss_scratch(uint64_t rows, uint64_t d);
int mpc3_rss_softmax_loss(const uint32_t* rk3, const uint64_t* ctr, const mpc3_softmax_loss_args* a, const uint64_t* z,
                          const uint64_t* y, uint64_t* scratch, uint64_t* out, uint64_t rows, uint64_t d,
                          void* stream);

/* ---- single-call layers (csrc/layers.cu; SURVEY.md §8(b) minimum list) ----
 * Each is the composition of the calls above (limb packs, tcgen05 ring GEMM,
 * fused reshare + truncate) behind one entry; workspace >= the matching
 * *_workspace() bytes, caller-owned (the library keeps no buffer). */

/* Plain ring conv2d, NCHW cross-correlation (ring.py:225-256 _conv2d_exact /
 * bilinear_exact with conv2d_spec): y (N, O, OH, OW) = x (N, C, H, W) * w
 * (O, C, kh, kw) mod 2^64; ExactnessError past C*kh*kw = 2^20 (ring.py:191). */
size_t mpc3_ring_conv2d_workspace(int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw,
                                  int sh, int sw, int ph, int pw);
int mpc3_ring_conv2d_u64(const uint64_t* x, const uint64_t* w, uint64_t* y, int64_t N, int64_t C, int64_t H,
                         int64_t W, int64_t O, int kh, int kw, int sh, int sw, int ph, int pw, void* workspace,
                         void* stream);

/* matmul_shares (protocols.py:97-117) of trio tensors x (3, M, K) and y
 * (3, K, N) into out (3, M, N): the three cross-term GEMMs, the ARITH_ZERO
 * reshare (j_arith) and the truncation by bits (j_rho, j_r). */
size_t mpc3_rss_matmul_workspace(int64_t M, int64_t K, int64_t N);
int mpc3_rss_matmul_reshare_trunc(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                  uint64_t j_r, int bits, const uint64_t* x, const uint64_t* y, uint64_t* out,
                                  int64_t M, int64_t K, int64_t N, void* workspace, void* stream);

/* conv2d_shares (protocols.py:120-136) of trio tensors x (3, N, C, H, W) and
 * w (3, O, C, kh, kw) into out (3, N, O, OH, OW). */
size_t mpc3_rss_conv2d_workspace(int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw,
                                 int sh, int sw, int ph, int pw);
int mpc3_rss_conv2d_reshare_trunc(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                  uint64_t j_r, int bits, const uint64_t* x, const uint64_t* w, uint64_t* out,
                                  int64_t N, int64_t C, int64_t H, int64_t W, int64_t O, int kh, int kw, int sh,
                                  int sw, int ph, int pw, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MPC3_B200_H */
