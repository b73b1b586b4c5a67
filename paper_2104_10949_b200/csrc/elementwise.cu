// Elementwise protocol kernels on trio tensors (three co-resident parties).
//
// Every kernel walks PRF *blocks*: thread item b owns the element pair
// (2b, 2b+1), because one AES block yields two adjacent stream words
// (prf.py:40-49).  Randomness is generated inline and never touches HBM.
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <set>
#include <utility>

#include "launch.cuh"
#include "items.cuh"

namespace mpc3 {

static thread_local char g_last_error[256] = "";
void set_last_error(const char* msg) {
  strncpy(g_last_error, msg, sizeof(g_last_error) - 1);
  g_last_error[sizeof(g_last_error) - 1] = 0;
}

// Two-phase circuit phase on three lanes per pair (Lane3, items.cuh); 0
// builds the one-thread-per-pair form for A/B.
#ifndef MPC3_SIGN2_LANES
#define MPC3_SIGN2_LANES 1
#endif
#ifndef MPC3_SIGN2_WAVES  // two-phase grids: at most this many waves of CTAs (the rest loop over chunks)
#define MPC3_SIGN2_WAVES 8
#endif
#ifndef MPC3_DBG_S2PHASE  // timing builds: 1 = sign2's keystream phase only, 2 = its circuit phase only
#define MPC3_DBG_S2PHASE 0
#endif
constexpr int kThreads = 256;
constexpr int kSignThreads = 384;  // four-table AES kernels: one CTA per SM
// The protocol kernels (everything but the sign / sign2 / chain kernels) come
// in two AES table layouts, chosen per launch by size:
//  * four-table (128 KiB, no rotations), one 384-thread CTA per SM on a
//    persistent grid: the throughput layout (reshare+truncate at 1.2 M
//    elements 73 -> 65 us, 42 -> 47 G AES blocks/s; AlexNet step 2.68 ->
//    2.60 ms when every launch used it);
//  * two-table (64 KiB), 256-thread CTAs, up to 3 per SM: ~2 us less fixed
//    cost per launch standalone (half the table to expand; reshare at 32 K
//    elements 8.6 -> 6.9 us), kept for the tiny tensors only: in the AlexNet
//    step a crossover at 65 K / 262 K pairs measured 2.68 / 2.67 ms against
//    2.59 ms at 16 K pairs or with every launch four-table, and 2.71 ms with
//    every launch two-table (tools/dbg/run_variants.sh).
constexpr int kProto4Threads = kSignThreads, kProto2Threads = kThreads, kProto2CtasPerSm = 8;
#ifndef MPC3_FOUR_MIN_PAIRS
#define MPC3_FOUR_MIN_PAIRS 16384
#endif
constexpr uint64_t kFourMinPairs = MPC3_FOUR_MIN_PAIRS;
template <bool F>
struct Proto;
template <>
struct Proto<true> {
  using TT = SmemTables4;
  static constexpr int threads = kProto4Threads, min_ctas = 1;
  DEV static TT init() { return aes_smem_init4(*reinterpret_cast<AesSmem4*>(mpc3_dsm)); }
  DEV static HeadConst* slots() { return reinterpret_cast<AesSmem4*>(mpc3_dsm)->hc; }
};
template <>
struct Proto<false> {
  using TT = SmemTables;
  static constexpr int threads = kProto2Threads, min_ctas = 3;  // 3 x 64 KiB tables per SM
  DEV static TT init() { return aes_smem_init(*reinterpret_cast<AesSmem*>(mpc3_dsm)); }
  DEV static HeadConst* slots() { return reinterpret_cast<AesSmem*>(mpc3_dsm)->hc; }
};
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MPC3_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// MPC3_SIGN_FUSED=1 selects the single-phase sign kernel (AES inline in the circuit)
static const bool g_sign_fused = [] {
  const char* e = getenv("MPC3_SIGN_FUSED");
  return e && e[0] == '1';
}();

// Protocol kernels take 64 KiB+ of dynamic shared memory (the AES tables):
// opt in once per (device, kernel).
static bool aes_attr(const void* fn, int bytes = kAesSmemBytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (done.count({dev, fn})) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  done.insert({dev, fn});
  return true;
}
// Session keys travel in the kernel parameters (KeySched, 528 bytes): the
// round keys are then constant-bank operands (LDC / LDCU) instead of
// shared-memory loads competing with the T-table lookups (+10 % AES rate on
// the LSU-bound sign kernel).  The engine keeps its key schedule in pinned
// host memory, read here directly; a device buffer is copied back once
// (not allowed while a graph is being captured).
static int load_keys(const uint32_t* rk, int nkeys, void* stream, KeySched* ks) {
  if (!rk) {
    set_last_error("null key schedule");
    return MPC3_ERR_CONFIG;
  }
  memset(ks, 0, sizeof(*ks));
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, rk) != cudaSuccess) {
    cudaGetLastError();
    at.type = cudaMemoryTypeUnregistered;
  }
  const size_t bytes = (size_t)nkeys * 44 * sizeof(uint32_t);
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(as_stream(stream), &cs);
    if (cs != cudaStreamCaptureStatusNone) {
      set_last_error("device-resident key schedule cannot be read during graph capture (use pinned host memory)");
      return MPC3_ERR_CONFIG;
    }
    if (cudaMemcpy(&ks->rk[0][0], rk, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return check_launch("key copy");
  } else {
    memcpy(&ks->rk[0][0], rk, bytes);
  }
  return MPC3_OK;
}

#define AES_LAUNCH(kern, pairs, stream, ...)                                                              \
  do {                                                                                                     \
    const uint64_t pairs_ = (pairs);                                                                       \
    if (pairs_ >= kFourMinPairs) {                                                                         \
      if (!aes_attr((const void*)kern<true>, kAesSmem4Bytes)) return check_launch(#kern " smem attribute"); \
      if (launch_pdl(kern<true>, dim3(grid_for(pairs_, kProto4Threads, 1)), dim3(kProto4Threads),          \
                     kAesSmem4Bytes, (stream), __VA_ARGS__) != cudaSuccess)                                \
        return check_launch(#kern);                                                                        \
    } else {                                                                                               \
      if (!aes_attr((const void*)kern<false>, kAesSmemBytes)) return check_launch(#kern " smem attribute"); \
      if (launch_pdl(kern<false>, dim3(grid_for(pairs_, kProto2Threads, kProto2CtasPerSm)),               \
                     dim3(kProto2Threads), kAesSmemBytes, (stream), __VA_ARGS__) != cudaSuccess)          \
        return check_launch(#kern);                                                                        \
    }                                                                                                      \
  } while (0)

// Stream counters may be offset by a device-resident per-purpose base
// (ctr[purpose], nullable) so a captured CUDA graph advances its PRF counters
// on every replay exactly as the sequential schedule would.
struct StreamRef {
  uint32_t purpose;
  uint64_t j;
};
DEV StreamHead resolve(StreamRef r, const uint64_t* __restrict__ ctr) {
  return stream_head(r.purpose, r.j + (ctr ? ctr[r.purpose] : 0));
}
HD StreamRef sref(uint32_t purpose, uint64_t j) {
  StreamRef r;
  r.purpose = purpose;
  r.j = j;
  return r;
}

#define GRID_LOOP(var, count) \
  for (uint64_t var = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; var < (count); \
       var += (uint64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// PRF streams

__global__ void __launch_bounds__(kSignThreads, 1) prf_words_kernel(const __grid_constant__ KeySched ks,
                                                                   StreamHead h, uint64_t word_off,
                                                                   uint64_t count, uint64_t* __restrict__ out) {
  MPC3_AES_SMEM4();
  SmemTables4 tab = aes_smem_init4(sm);
  StreamHead hc = h;
  cache_heads(tab, &ks.rk[0][0], sm.hc, hc);  // (keys 1-2 of ks are zero here: their slots go unused)
  uint64_t nblk = ((word_off + count - 1) >> 1) - (word_off >> 1) + 1;
  GRID_LOOP(t, nblk) prf_words_item(tab, &ks.rk[0][0], hc, word_off, count, out, t);
}

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) zero_share_kernel(const __grid_constant__ KeySched ks,
                                                             const uint64_t* __restrict__ ctr, StreamRef rh,
                                                             int xor_mode, uint64_t n, uint64_t* __restrict__ out) {
  StreamHead h = resolve(rh, ctr);
  auto tab = Proto<F>::init();
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), h);
  GRID_LOOP(b, (n + 1) >> 1) zero_share_item(tab, &ks.rk[0][0], h, xor_mode, n, out, b);
}

// ---------------------------------------------------------------------------
// local ring ops

__global__ void ring_ew_kernel(int op, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                               uint64_t c, uint64_t* __restrict__ out, uint64_t n) {
  griddep_launch();
  griddep_wait();
  GRID_LOOP(i, n) {
    uint64_t x = a[i], r;
    switch (op) {
      case MPC3_EW_ADD: r = x + b[i]; break;
      case MPC3_EW_SUB: r = x - b[i]; break;
      case MPC3_EW_NEG: r = 0 - x; break;
      case MPC3_EW_MULC: r = x * c; break;
      case MPC3_EW_ADDC: r = x + c; break;
      case MPC3_EW_XOR: r = x ^ b[i]; break;
      case MPC3_EW_SHL: r = x << c; break;
      case MPC3_EW_SHR: r = x >> c; break;
      case MPC3_EW_SAR: r = sar(x, (int)c); break;
      default: r = x + c * b[i]; break;  // AXPY
    }
    out[i] = r;
  }
}

__global__ void ring_rowop_kernel(int op, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                                  uint64_t* __restrict__ out, uint64_t rows, uint64_t cols) {
  griddep_launch();
  griddep_wait();
  GRID_LOOP(i, rows * cols) {
    uint64_t v = b[i / cols];
    out[i] = op == MPC3_EW_SUB ? a[i] - v : a[i] + v;
  }
}

__global__ void ring_rowsum_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                   uint64_t rows, uint64_t cols) {
  griddep_launch();
  griddep_wait();
  GRID_LOOP(r, rows) {
    uint64_t s = 0;
    for (uint64_t j = 0; j < cols; ++j) s += a[r * cols + j];
    out[r] = s;
  }
}

// ---------------------------------------------------------------------------
// protocols

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) arith_kernel(int kind, const __grid_constant__ KeySched ks,
                                                        const uint64_t* __restrict__ ctr, StreamRef ra,
                                                        StreamRef rrho, StreamRef rr, int bits, const uint64_t* __restrict__ x,
                                                        const uint64_t* __restrict__ y,
                                                        uint64_t* __restrict__ out, uint64_t n, uint64_t pb0) {
  auto tab = Proto<F>::init();
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), ha, hrho, hr);
  GRID_LOOP(b, (n + 1) >> 1) arith_item(tab, &ks.rk[0][0], kind, ha, hrho, hr, bits, x, y, out, n, b, pb0);
}

struct SignArgs {
  uint64_t jbin, jxor, ja;
  uint64_t jra, jrho, jr;  // fused layer + ReLU: the layer's ARITH_ZERO / TRUNC_RHO / TRUNC_R counters
};

// Counter-mode constants of a launch's SignStreams (all threads, after the
// tables are built; heads in declaration order -> slots; two barriers).
template <class TT>
DEV void cache_sign_streams(const TT& tab, const uint32_t* rk3, SignStreams& st, HeadConst* slots, bool rs) {
  static_assert(sizeof(SignStreams) == 14 * sizeof(StreamHead), "SignStreams is an array of heads");
#if defined(MPC3_NO_HEAD_CACHE)
  return;
#endif
  constexpr int KT = TT::kTops;
  StreamHead* hs = reinterpret_cast<StreamHead*>(&st);
  const int nh = rs ? 14 : 11;
  for (int t = threadIdx.x; t < 3 * KT * nh; t += blockDim.x) {
    const StreamHead h = hs[t / (3 * KT)];
    head_const(tab, rk3 + 44 * (t % 3), h.s0, h.s1, (uint32_t)(t / 3 % KT), slots[t]);
  }
  __syncthreads();
  if (threadIdx.x < nh) hs[threadIdx.x].pc = (uint32_t)__cvta_generic_to_shared(&slots[threadIdx.x * KT * 3]);
  __syncthreads();
}

// the stream heads a sign launch needs, resolved by one thread into shared memory
DEV void sign_streams(SignStreams& st, const SignArgs& args, const uint64_t* ctr, bool rs) {
  st.bin = resolve(sref(BIN_INPUT, args.jbin), ctr);
  for (int l = 0; l < 7; ++l) st.x[l] = resolve(sref(XOR_ZERO, args.jxor + l), ctr);
  for (int l = 0; l < 3; ++l) st.a[l] = resolve(sref(ARITH_ZERO, args.ja + l), ctr);
  if (rs) {
    st.ra = resolve(sref(ARITH_ZERO, args.jra), ctr);
    st.rrho = resolve(sref(TRUNC_RHO, args.jrho), ctr);
    st.rr = resolve(sref(TRUNC_R, args.jr), ctr);
  }
}

// Large tensors: one 512-thread CTA per SM with the four-table AES layout
// (128 KiB) — the kernel is nothing but AES rounds.
// RS: the input is a secure layer's cross terms (RsIn), reshared and
// truncated in registers (fused layer + ReLU); otherwise the trio x.
template <bool RS>
__global__ void __launch_bounds__(kSignThreads, 1) sign_kernel(const __grid_constant__ KeySched ks,
                                                          const uint64_t* __restrict__ ctr, SignArgs args,
                                                          int mode, const uint64_t* __restrict__ x,
                                                          uint64_t* __restrict__ out,
                                                          uint64_t* __restrict__ mask, uint64_t n,
                                                          uint64_t n_total, uint64_t elem_off, uint64_t plane,
                                                          const __grid_constant__ RsIn rin) {
  MPC3_AES_SMEM4();
  static_assert(sizeof(SignStreams) <= sizeof(sm.extra), "stream heads fit the AesSmem extra area");
  SignStreams& st = *reinterpret_cast<SignStreams*>(sm.extra);  // uniform stream heads, indexed by level
  if (threadIdx.x == 0) sign_streams(st, args, ctr, RS);
  SmemTables4 tab = aes_smem_init4(sm);  // includes the barrier
  cache_sign_streams(tab, &ks.rk[0][0], st, sm.hc, RS);
  if constexpr (RS) {
    GRID_LOOP(b, (n + 1) >> 1) {
      Word2 w3[3], rho, r;
      reshare_trunc_words(tab, &ks.rk[0][0], st.ra, st.rrho, st.rr, (elem_off >> 1) + b, w3, rho, r);
      sign_item_rs(tab, &ks.rk[0][0], st, mode, rin, w3, rho, r, out, mask, n, n_total, elem_off, b, plane);
    }
  } else {
    GRID_LOOP(b, (n + 1) >> 1) sign_item(tab, &ks.rk[0][0], st, mode, x, out, mask, n, n_total, elem_off, b, plane);
  }
}

// Two-phase sign circuit.  The 46 AES blocks an element pair consumes do not
// depend on the data, so phase 1 computes them for P pairs with all 256
// threads in parallel (one three-key block per (slot, pair) item, a warp per
// 32 pairs of one slot) into shared memory, and phase 2 runs the circuit of
// each pair (three lanes per pair, Lane3 in protocol.cuh; one thread per pair
// with -DMPC3_SIGN2_LANES=0) replaying those words.  A pair's latency
// is then ~1/4 of its AES work instead of all 16 dependent AES groups, which
// is what bounds the many small ReLU / max_tree launches of a training step;
// at large n it is throughput-bound like sign_kernel.
// Slots, in the circuit's call order: 0 = BIN (k_0 only); 1 = XOR level 0;
// then per level l = 1..5: g-half, p-half (two slots when n_total is odd: the
// pair straddles two blocks); then level 6's g-half; then the 3 ARITH muls.
constexpr int SW_SLOT_BYTES = 3 * (int)sizeof(Word2);
HD int sign_slots(bool straddle) { return straddle ? 21 : 16; }

// F: four-table AES (one 384-thread CTA per SM, up to 128 pairs per chunk)
// or two-table (two 256-thread CTAs per SM, up to 64 pairs each).
// Keystream slot s (circuit call order, see above) of the pair at PRF block
// blk: one three-key block, or BIN's single block.
template <class TT>
DEV void sign_slot_fill(const TT& tab, const uint32_t* rk, const SignStreams& st, int s, uint64_t blk,
                        uint64_t n_total, int L, Word2* dst) {
  if (s == 0) {
    dst[0] = prf_block_k(tab, rk, 0, st.bin, blk);
    return;
  }
  StreamHead h;
  uint64_t b = blk;
  if (s == 1) {
    h = st.x[0];
  } else if (s < 2 + 5 * L) {
    const int lvl = (s - 2) / L + 1, r = (s - 2) % L;
    h = st.x[lvl];
    if (r > 0) b = ((n_total + 2 * blk) >> 1) + (r - 1);  // p-half words n_total + 2 blk (+1)
  } else if (s == 2 + 5 * L) {
    h = st.x[6];
  } else {
    h = st.a[s - 3 - 5 * L];
  }
  Word2 w[3];
  prf_block3(tab, rk, h, b, w);
  dst[0] = w[0];
  dst[1] = w[1];
  dst[2] = w[2];
}

// KIND: 0 sign / ReLU of x; 1 one max_tree level; 2 fused layer + ReLU (two
// leading slots hold the pair's reshare words (3 keys) and truncation words
// (rho, r); the circuit's slots follow).
constexpr int S2_SIGN = 0, S2_MAXL = 1, S2_RS = 2;
template <int KIND, bool F>
__global__ void __launch_bounds__(F ? kSignThreads : kThreads, F ? 1 : 2)
    sign2_kernel(const __grid_constant__ KeySched ks, const uint64_t* __restrict__ ctr, SignArgs args, int mode,
                 const uint64_t* __restrict__ x, uint64_t* __restrict__ out, uint64_t* __restrict__ mask, uint64_t n,
                 uint64_t n_total, uint64_t elem_off, int P, uint64_t plane, MaxGeom mg,
                 const __grid_constant__ RsIn rin) {
  constexpr bool MAXL = KIND == S2_MAXL;
  constexpr int PRE = KIND == S2_RS ? 2 : 0;
  SignStreams& st = *reinterpret_cast<SignStreams*>(F ? reinterpret_cast<AesSmem4*>(mpc3_dsm)->extra
                                                      : reinterpret_cast<AesSmem*>(mpc3_dsm)->extra);
  if (threadIdx.x == 0) sign_streams(st, args, ctr, KIND == S2_RS);
  auto tab = Proto<F>::init();  // (its __syncthreads publishes st)
  cache_sign_streams(tab, &ks.rk[0][0], st, Proto<F>::slots(), KIND == S2_RS);
  Word2* pre = reinterpret_cast<Word2*>(mpc3_dsm + (F ? sizeof(AesSmem4) : sizeof(AesSmem)));
  Word2* slots = pre + (size_t)PRE * P * 3;
  const bool straddle = (n_total & 1) != 0;
  const int L = straddle ? 3 : 2;  // slots per level 1..5
  const int nslots = sign_slots(straddle);
  const int used = mode <= MODE_MSB ? nslots - 3 : (mode == MODE_DRELU ? nslots - 1 : nslots);
  const uint64_t npairs = (n + 1) >> 1;
  for (uint64_t c0 = (uint64_t)blockIdx.x * P; c0 < npairs; c0 += (uint64_t)gridDim.x * P) {
    for (int q = threadIdx.x; q < (MPC3_DBG_S2PHASE == 2 ? 0 : (used + PRE) * P); q += blockDim.x) {
      const int sa = q / P, p = q % P;
      if (c0 + p >= npairs) continue;
      const uint64_t blk = (elem_off >> 1) + c0 + p;
      if (PRE && sa < PRE) {  // the fused layer's reshare / truncation words
        Word2* dst = pre + ((size_t)sa * P + p) * 3;
        if (sa == 0) {
          prf_block3(tab, &ks.rk[0][0], st.ra, blk, dst);
        } else {
          dst[0] = prf_block_k(tab, &ks.rk[0][0], 2, st.rrho, blk);  // protocols.py:166-216
          dst[1] = prf_block_k(tab, &ks.rk[0][0], 1, st.rr, blk);
        }
        continue;
      }
      const int s = sa - PRE;
      sign_slot_fill(tab, &ks.rk[0][0], st, s, blk, n_total, L, slots + ((size_t)s * P + p) * 3);
    }
    __syncthreads();
#if MPC3_SIGN2_LANES
    if (MPC3_DBG_S2PHASE != 1) {  // the circuit, three lanes per pair (Lane3)
      const LaneGroup G = lane_group();
      const int nw = blockDim.x >> 5;
      for (int base = (threadIdx.x >> 5) * 10; base < P; base += nw * 10) {
        const int pp = base + G.gi;
        const bool live = G.gi < 10 && pp < P && c0 + pp < npairs;
        const Lane3 L = {slots, P, live ? pp : 0, G.ci, G.nl, G.pl};  // pair 0 of a chunk always exists
        if constexpr (MAXL) {
          maxlevel_item_lane(L, x, out, mg, n, n_total, c0 + L.p, live);
        } else if constexpr (KIND == S2_RS) {
          const Word2* w3 = pre + (size_t)L.p * 3;
          const Word2* tr = pre + ((size_t)P + L.p) * 3;
          sign_item_rs_lane(L, mode, rin, w3, tr[0], tr[1], out, mask, n, n_total, c0 + L.p, plane, live);
        } else {
          sign_item_lane(L, mode, x, out, mask, n, n_total, c0 + L.p, plane, live);
        }
      }
    }
#else
    if (MPC3_DBG_S2PHASE != 1 && threadIdx.x < P && c0 + threadIdx.x < npairs) {
      Replay rp;
      rp.w = slots;
      rp.P = P;
      rp.p = threadIdx.x;
      rp.slot = 0;
      if constexpr (MAXL) {
        maxlevel_item(rp, &ks.rk[0][0], st, x, out, mg, n, n_total, elem_off, c0 + threadIdx.x);
      } else if constexpr (KIND == S2_RS) {
        const Word2* w3 = pre + (size_t)threadIdx.x * 3;
        const Word2* tr = pre + ((size_t)P + threadIdx.x) * 3;
        sign_item_rs(rp, &ks.rk[0][0], st, mode, rin, w3, tr[0], tr[1], out, mask, n, n_total, elem_off,
                     c0 + threadIdx.x, plane);
      } else {
        sign_item(rp, &ks.rk[0][0], st, mode, x, out, mask, n, n_total, elem_off, c0 + threadIdx.x, plane);
      }
    }
#endif
    __syncthreads();
  }
  if constexpr (MAXL) {  // odd m: the last column passes through to the last output column
    if (mg.m & 1) {
      const uint64_t pv = mg.rows * mg.m, mo = mg.k + 1, po = mg.rows * mo;
      for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < mg.rows;
           r += (uint64_t)gridDim.x * blockDim.x)
        store_trio(out, po, r * mo + mg.k, load_trio(x, pv, r * mg.m + mg.m - 1));
    }
  }
}

// The whole max_tree (protocols.py:356-380) in one launch.  Rows are
// independent, so each CTA takes R rows (R even: the rows' level tensors then
// start on AES-block boundaries) through every level, two-phase per level as
// sign2_kernel (keystream slots, then three lanes per pair run the circuit),
// with __syncthreads between levels; the level outputs ping-pong through
// global scratch.  Counters per level as the per-level launches.
constexpr int MT_MAX_LEVELS = 16, MT_PMAX = 64;
struct MaxTreeArgs {
  int levels;
  uint64_t jbin[MT_MAX_LEVELS], jxor[MT_MAX_LEVELS], ja[MT_MAX_LEVELS];
  uint64_t rows_total, row_off;  // batch shard of the rows
};
__global__ void __launch_bounds__(kThreads, 1) maxtree_kernel(const __grid_constant__ KeySched ks,
                                                            const uint64_t* __restrict__ ctr,
                                                            const __grid_constant__ MaxTreeArgs ta,
                                                            const uint64_t* __restrict__ v, uint64_t* s0, uint64_t* s1,
                                                            uint64_t* __restrict__ out, uint64_t rows, uint64_t m0,
                                                            int R) {
  SignStreams& st = *reinterpret_cast<SignStreams*>(reinterpret_cast<AesSmem*>(mpc3_dsm)->extra);
  auto tab = Proto<false>::init();
  Word2* slots = reinterpret_cast<Word2*>(mpc3_dsm + sizeof(AesSmem));
  const uint64_t r0 = (uint64_t)blockIdx.x * R;
  const uint64_t rn = rows - r0 < (uint64_t)R ? rows - r0 : (uint64_t)R;
  const uint64_t* in = v;
  uint64_t m = m0;
  for (int l = 0; l < ta.levels; ++l) {
    const uint64_t k = m / 2, mo = k + (m & 1);
    uint64_t* o = l == ta.levels - 1 ? out : ((l & 1) ? s1 : s0);
    if (threadIdx.x == 0) {
      const SignArgs a = {ta.jbin[l], ta.jxor[l], ta.ja[l], 0, 0, 0};
      sign_streams(st, a, ctr, false);
    }
    __syncthreads();
    cache_sign_streams(tab, &ks.rk[0][0], st, reinterpret_cast<AesSmem*>(mpc3_dsm)->hc, false);
    const uint64_t n = rows * k, n_total = ta.rows_total * k, elem_off = ta.row_off * k;
    const bool straddle = (n_total & 1) != 0;
    const int L = straddle ? 3 : 2, used = sign_slots(straddle);
    const uint64_t p0 = r0 * k / 2, P = (rn * k + 1) / 2;  // this CTA's pairs
    const MaxGeom g = {rows, m, k};
    for (uint64_t c = 0; c < P; c += MT_PMAX) {
      const int Pc = (int)(P - c < (uint64_t)MT_PMAX ? P - c : (uint64_t)MT_PMAX);
      for (int q = threadIdx.x; q < used * Pc; q += blockDim.x) {
        const int s = q / Pc, p = q % Pc;
        sign_slot_fill(tab, &ks.rk[0][0], st, s, (elem_off >> 1) + p0 + c + p, n_total, L,
                       slots + ((size_t)s * Pc + p) * 3);
      }
      __syncthreads();
#if MPC3_SIGN2_LANES
      {
        const LaneGroup G = lane_group();
        const int nw = blockDim.x >> 5;
        for (int base = (threadIdx.x >> 5) * 10; base < Pc; base += nw * 10) {
          const int pp = base + G.gi;
          const bool live = G.gi < 10 && pp < Pc;
          const Lane3 L = {slots, Pc, live ? pp : 0, G.ci, G.nl, G.pl};
          maxlevel_item_lane(L, in, o, g, n, n_total, p0 + c + L.p, live);
        }
      }
#else
      if (threadIdx.x < Pc) {
        Replay rp;
        rp.w = slots;
        rp.P = Pc;
        rp.p = threadIdx.x;
        rp.slot = 0;
        maxlevel_item(rp, &ks.rk[0][0], st, in, o, g, n, n_total, elem_off, p0 + c + threadIdx.x);
      }
#endif
      __syncthreads();
    }
    if (m & 1)  // odd m: the last column passes through to the last output column
      for (uint64_t r = threadIdx.x; r < rn; r += blockDim.x)
        store_trio(o, rows * mo, (r0 + r) * mo + k, load_trio(in, rows * m, (r0 + r) * m + m - 1));
    __syncthreads();
    in = o;
    m = mo;
  }
}

// Fused elementwise chain (exp_approx's squarings, reciprocal's Newton
// iterations, protocols.py:414-440): a short program over a per-element
// register trio z, the chain input x and a temporary t, whose k-th mul+truncate
// uses ARITH_ZERO j_a + k, TRUNC_RHO j_rho + k and TRUNC_R j_r + k, exactly the
// counters the unfused sequence of mul_truncate calls takes.  Two phases as in
// sign2_kernel: the 5 AES blocks per (mul, pair) are computed by all threads
// into shared memory, then one thread per pair runs the program.
struct ChainProgram {
  int nsteps, nmul;
  MPC3ChainStep s[MPC3_CHAIN_MAX_STEPS];
};
constexpr int CH_SLOT_WORDS = 5;  // ARITH k0..k2, RHO (k2), R (k1)

__global__ void __launch_bounds__(kThreads, 1) chain_kernel(const __grid_constant__ KeySched ks,
                                                           const uint64_t* __restrict__ ctr, ChainProgram prog,
                                                           uint64_t ja, uint64_t jrho, uint64_t jr,
                                                           const uint64_t* __restrict__ x, uint64_t* __restrict__ out,
                                                           uint64_t n, uint64_t pb0, int P) {
  MPC3_AES_SMEM();
  SmemTables tab = aes_smem_init(sm);
  Word2* slots = reinterpret_cast<Word2*>(mpc3_dsm + sizeof(AesSmem));
  const uint64_t npairs = (n + 1) >> 1;
  const uint32_t* rk = &ks.rk[0][0];
  for (uint64_t c0 = (uint64_t)blockIdx.x * P; c0 < npairs; c0 += (uint64_t)gridDim.x * P) {
    for (int q = threadIdx.x; q < prog.nmul * P; q += blockDim.x) {
      const int k = q / P, p = q % P;
      if (c0 + p >= npairs) continue;
      const uint64_t blk = pb0 + c0 + p;
      Word2* dst = slots + ((size_t)k * P + p) * CH_SLOT_WORDS;
      Word2 w[3];
      prf_block3(tab, rk, resolve(sref(ARITH_ZERO, ja + k), ctr), blk, w);
      dst[0] = w[0];
      dst[1] = w[1];
      dst[2] = w[2];
      trunc_words(tab, rk, resolve(sref(TRUNC_RHO, jrho + k), ctr), resolve(sref(TRUNC_R, jr + k), ctr), blk, dst[3],
                  dst[4]);
    }
    __syncthreads();
    const int p = threadIdx.x;
    const uint64_t b = c0 + p;
    if (p < P && b < npairs) {
      const bool two = 2 * b + 1 < n;
      Trio xv[2], z[2], t[2];
      xv[0] = load_trio(x, n, 2 * b);
      xv[1] = two ? load_trio(x, n, 2 * b + 1) : xv[0];
      z[0] = xv[0];
      z[1] = xv[1];
      t[0] = t[1] = z[0];
      int k = 0;
      for (int i = 0; i < prog.nsteps; ++i) {
        const MPC3ChainStep st = prog.s[i];
        if (st.op == MPC3_CHAIN_ADDC) {
          z[0].c[0] += st.c;
          z[1].c[0] += st.c;
        } else if (st.op == MPC3_CHAIN_SETC) {
          for (int e = 0; e < 2; ++e) z[e] = Trio{{st.c, 0, 0}};
        } else if (st.op == MPC3_CHAIN_NEWTON) {
          for (int e = 0; e < 2; ++e)
            for (int c = 0; c < 3; ++c) z[e].c[c] = 2 * z[e].c[c] - t[e].c[c];
        } else {  // SQ: z = trunc(z * z); SQT: t = trunc(z * z); MULX: t = trunc(x * t)
          const Word2* sl = slots + ((size_t)k * P + p) * CH_SLOT_WORDS;
          KeyWords f0, f1;
          for (int c = 0; c < 3; ++c) {
            f0.k[c] = sl[c].w0;
            f1.k[c] = sl[c].w1;
          }
          const Word2 rho = sl[3], r = sl[4];
          for (int e = 0; e < 2; ++e) {
            Trio v = st.op == MPC3_CHAIN_MULX ? trio_mul(xv[e], t[e], e ? f1 : f0) : trio_mul(z[e], z[e], e ? f1 : f0);
            v = trio_truncate(v, e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, st.bits);
            if (st.op == MPC3_CHAIN_SQ)
              z[e] = v;
            else
              t[e] = v;
          }
          ++k;
        }
      }
      store_trio(out, n, 2 * b, z[0]);
      if (two) store_trio(out, n, 2 * b + 1, z[1]);
    }
    __syncthreads();
  }
}

// The training step's loss gradient softmax(z) - y (nn.py:561-568 via
// protocols.py:453-468) in ONE launch.  Rows are independent, so each CTA
// takes R rows (R even: every per-op tensor range then starts on an AES-block
// boundary) through the whole chain, with __syncthreads between the steps
// and the intermediate tensors in global scratch (this CTA's rows only):
//   max_tree over the row (levels as maxtree_kernel), x = z - max,
//   e = exp_approx(x) (chain program, two-phase as chain_kernel),
//   s = sum_j e, r = reciprocal(s) (chain program), out = truncate(e * r) - y.
// Every step uses the counters and PRF word indices of its unfused launch
// (each op's own flat tensor index at the batch shard's global offset), so
// the shares are those of the separate max_tree / chain / mul_truncate calls.
struct LossArgs {
  int levels;
  uint64_t jbin[MT_MAX_LEVELS], jxor[MT_MAX_LEVELS], ja[MT_MAX_LEVELS];
  uint64_t ej[3], rj[3], fj[3];  // exp / reciprocal / final mul: ARITH, TRUNC_RHO, TRUNC_R
  int bits;                       // final truncation (t)
  uint64_t rows_total, row_off;   // batch shard (row_off even)
  ChainProgram ep, rp;
};
constexpr int LOSS_SLOT_BYTES = 64 * 1024;

// one chain program over pairs [lo, hi) of an n-element trio tensor x -> out
// The chain's keystream item (mul k, pair p): the three ARITH words, then
// TRUNC_RHO / TRUNC_R, at PRF block blk.
DEV void chain_slot_fill(const SmemTables& tab, const uint32_t* rk, const uint64_t* ctr, uint64_t ja, uint64_t jrho,
                         uint64_t jr, int k, uint64_t blk, Word2* dst) {
  Word2 w[3], rho, r;  // the five AES blocks interleaved in one call (one chain's latency)
  reshare_trunc_words(tab, rk, resolve(sref(ARITH_ZERO, ja + k), ctr), resolve(sref(TRUNC_RHO, jrho + k), ctr),
                      resolve(sref(TRUNC_R, jr + k), ctr), blk, w, rho, r);
  dst[0] = w[0];
  dst[1] = w[1];
  dst[2] = w[2];
  dst[3] = rho;
  dst[4] = r;
}

// pre: the whole range's keystream already in shared memory ((k * (hi - lo)
// + p) * CH_SLOT_WORDS, one chunk), else filled chunk by chunk into `slots`
DEV void chain_pairs(const SmemTables& tab, const uint32_t* rk, const uint64_t* ctr, const ChainProgram& prog,
                     uint64_t ja, uint64_t jrho, uint64_t jr, const uint64_t* x, uint64_t* out, uint64_t n,
                     uint64_t pb0, uint64_t lo, uint64_t hi, Word2* slots, const Word2* pre = nullptr) {
  int P = 64;
  while (P > 1 && P * prog.nmul * CH_SLOT_WORDS * (int)sizeof(Word2) > LOSS_SLOT_BYTES) P >>= 1;
  if (pre) {
    P = (int)(hi - lo);
    slots = const_cast<Word2*>(pre);
  }
  for (uint64_t c0 = lo; c0 < hi; c0 += P) {
    const int Pc = (int)(hi - c0 < (uint64_t)P ? hi - c0 : (uint64_t)P);
    for (int q = threadIdx.x; q < (pre ? 0 : prog.nmul * Pc); q += blockDim.x) {
      const int k = q / Pc, p = q % Pc;
      chain_slot_fill(tab, rk, ctr, ja, jrho, jr, k, pb0 + c0 + p, slots + ((size_t)k * Pc + p) * CH_SLOT_WORDS);
    }
    __syncthreads();
    const int p = threadIdx.x;
    if (p < Pc) {
      const uint64_t b = c0 + p;
      const bool two = 2 * b + 1 < n;
      Trio xv[2], z[2], t[2];
      xv[0] = load_trio(x, n, 2 * b);
      xv[1] = two ? load_trio(x, n, 2 * b + 1) : xv[0];
      z[0] = xv[0];
      z[1] = xv[1];
      t[0] = t[1] = z[0];
      int k = 0;
      for (int i = 0; i < prog.nsteps; ++i) {
        const MPC3ChainStep st = prog.s[i];
        if (st.op == MPC3_CHAIN_ADDC) {
          z[0].c[0] += st.c;
          z[1].c[0] += st.c;
        } else if (st.op == MPC3_CHAIN_SETC) {
          for (int e = 0; e < 2; ++e) z[e] = Trio{{st.c, 0, 0}};
        } else if (st.op == MPC3_CHAIN_NEWTON) {
          for (int e = 0; e < 2; ++e)
            for (int c = 0; c < 3; ++c) z[e].c[c] = 2 * z[e].c[c] - t[e].c[c];
        } else {
          const Word2* sl = slots + ((size_t)k * Pc + p) * CH_SLOT_WORDS;
          KeyWords f0, f1;
          for (int c = 0; c < 3; ++c) {
            f0.k[c] = sl[c].w0;
            f1.k[c] = sl[c].w1;
          }
          const Word2 rho = sl[3], r = sl[4];
          for (int e = 0; e < 2; ++e) {
            Trio v = st.op == MPC3_CHAIN_MULX ? trio_mul(xv[e], t[e], e ? f1 : f0) : trio_mul(z[e], z[e], e ? f1 : f0);
            v = trio_truncate(v, e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, st.bits);
            if (st.op == MPC3_CHAIN_SQ)
              z[e] = v;
            else
              t[e] = v;
          }
          ++k;
        }
      }
      store_trio(out, n, 2 * b, z[0]);
      if (two) store_trio(out, n, 2 * b + 1, z[1]);
    }
    __syncthreads();
  }
}

#ifdef MPC3_LOSS_TRACE
// debug build only (tools/dbg/loss_trace.py): phase timestamps of CTA 0
__device__ unsigned long long g_loss_trace[16];
#define LOSS_TRACE(k)                                                                          \
  do {                                                                                         \
    __syncthreads();                                                                           \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                                                 \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_));                                    \
      g_loss_trace[k] = t_;                                                                    \
    }                                                                                          \
  } while (0)
extern "C" int mpc3_dbg_loss_trace(unsigned long long* host8) {
  return cudaMemcpyFromSymbol(host8, g_loss_trace, sizeof(g_loss_trace)) == cudaSuccess ? 0 : 1;
}
#else
#define LOSS_TRACE(k)
#endif
__global__ void __launch_bounds__(kThreads, 1) softmax_loss_kernel(
    const __grid_constant__ KeySched ks, const uint64_t* __restrict__ ctr, const __grid_constant__ LossArgs la,
    const uint64_t* __restrict__ z, const uint64_t* __restrict__ y, uint64_t* scratch, uint64_t* __restrict__ out,
    uint64_t rows, uint64_t d, int R) {
  SignStreams& st = *reinterpret_cast<SignStreams*>(reinterpret_cast<AesSmem*>(mpc3_dsm)->extra);
  LOSS_TRACE(0);
  auto tab = Proto<false>::init();
  Word2* slots = reinterpret_cast<Word2*>(mpc3_dsm + sizeof(AesSmem));
  const uint32_t* rk = &ks.rk[0][0];
  const uint64_t r0 = (uint64_t)blockIdx.x * R;
  const uint64_t rn = rows - r0 < (uint64_t)R ? rows - r0 : (uint64_t)R;
  const uint64_t half = rows * ((d + 1) / 2) * 3;
  uint64_t* s0 = scratch;          // max_tree ping-pong
  uint64_t* s1 = s0 + half;
  uint64_t* mx = s1 + half;        // (rows) max
  uint64_t* X = mx + 3 * rows;     // (rows, d) z - max, then e
  uint64_t* E = X + 3 * rows * d;
  uint64_t* T = E + 3 * rows * d;  // (rows) sum, then reciprocal
  uint64_t* RR = T + 3 * rows;
  const uint64_t n = rows * d;

  // Small problems (AlexNet's 128 x 10): every phase's keystream — each
  // max_tree level's slots, the exp and reciprocal chains', the final
  // mul + truncate's — in ONE parallel fill up front (full AES rounds, no
  // counter-mode constants), so the phases after it are circuits only: the
  // per-phase fills were serial latency (profiles/r02_loss_phases.txt).
  // Sized with R rows (every CTA takes the same decision); regions are laid
  // out with this CTA's own pair counts.
  const uint64_t plo = r0 * d / 2, phi = ((r0 + rn) * d + 1) / 2;
  const uint64_t rlo = r0 / 2, rhi = (r0 + rn + 1) / 2;
  bool prefill = MPC3_SIGN2_LANES && la.levels <= MT_MAX_LEVELS;
  {
    uint64_t words = 0, mm = d;
    for (int l = 0; l < la.levels; ++l) {
      const uint64_t kk = mm / 2;
      words += (uint64_t)sign_slots((la.rows_total * kk) & 1) * (((uint64_t)R * kk + 1) / 2) * 3;
      mm = kk + (mm & 1);
    }
    const uint64_t pe = ((uint64_t)R * d + 1) / 2 + 1, pr = (uint64_t)R / 2 + 1;
    words += (uint64_t)(la.ep.nmul + 1) * pe * CH_SLOT_WORDS + (uint64_t)la.rp.nmul * pr * CH_SLOT_WORDS;
    prefill = prefill && words * sizeof(Word2) + MT_MAX_LEVELS * sizeof(SignStreams) <= (uint64_t)LOSS_SLOT_BYTES;
  }
  Word2 *pre_l[MT_MAX_LEVELS], *pre_e = nullptr, *pre_r = nullptr, *pre_f = nullptr;
  if (prefill) {
    uint64_t cnt[MT_MAX_LEVELS + 3], kl[MT_MAX_LEVELS];
    Word2* at = slots;
    uint64_t mm = d;
    for (int l = 0; l < la.levels; ++l) {
      kl[l] = mm / 2;
      const uint64_t Pl = (rn * kl[l] + 1) / 2;
      cnt[l] = (uint64_t)sign_slots((la.rows_total * kl[l]) & 1) * Pl;
      pre_l[l] = at;
      at += cnt[l] * 3;
      mm = kl[l] + (mm & 1);
    }
    const uint64_t Pe = phi - plo, Pr = rhi - rlo;
    cnt[la.levels] = (uint64_t)la.ep.nmul * Pe;
    pre_e = at;
    at += cnt[la.levels] * CH_SLOT_WORDS;
    cnt[la.levels + 1] = (uint64_t)la.rp.nmul * Pr;
    pre_r = at;
    at += cnt[la.levels + 1] * CH_SLOT_WORDS;
    cnt[la.levels + 2] = Pe;
    pre_f = at;
    at += Pe * CH_SLOT_WORDS;
    SignStreams* sts = reinterpret_cast<SignStreams*>(at);
    if (threadIdx.x < (unsigned)la.levels) {
      const SignArgs a = {la.jbin[threadIdx.x], la.jxor[threadIdx.x], la.ja[threadIdx.x], 0, 0, 0};
      sign_streams(sts[threadIdx.x], a, ctr, false);
    }
    __syncthreads();
    uint64_t total = 0;
    for (int sg = 0; sg < la.levels + 3; ++sg) total += cnt[sg];
    // item order: the chains' five-block items first, then the max_tree
    // levels' slots (a partial last round then holds the cheaper items)
    for (uint64_t q0 = threadIdx.x; q0 < total; q0 += blockDim.x) {
      uint64_t q = q0;
      int sg = la.levels;
      while (q >= cnt[sg]) {
        q -= cnt[sg];
        sg = sg == la.levels + 2 ? 0 : sg + 1;
      }
      if (sg < la.levels) {  // a max_tree level's slot (s, p)
        const uint64_t Pl = (rn * kl[sg] + 1) / 2, nt = la.rows_total * kl[sg];
        const int sidx = (int)(q / Pl), pp = (int)(q % Pl);
        sign_slot_fill(tab, rk, sts[sg], sidx, ((la.row_off * kl[sg]) >> 1) + r0 * kl[sg] / 2 + pp, nt,
                       (nt & 1) ? 3 : 2, pre_l[sg] + ((size_t)sidx * Pl + pp) * 3);
      } else if (sg == la.levels) {  // exp chain: mul k, pair p
        const uint64_t Pe = phi - plo;
        chain_slot_fill(tab, rk, ctr, la.ej[0], la.ej[1], la.ej[2], (int)(q / Pe),
                        la.row_off * d / 2 + plo + q % Pe, pre_e + q * CH_SLOT_WORDS);
      } else if (sg == la.levels + 1) {  // reciprocal chain
        const uint64_t Pr = rhi - rlo;
        chain_slot_fill(tab, rk, ctr, la.rj[0], la.rj[1], la.rj[2], (int)(q / Pr), la.row_off / 2 + rlo + q % Pr,
                        pre_r + q * CH_SLOT_WORDS);
      } else {  // the final mul + truncate of pair plo + q
        chain_slot_fill(tab, rk, ctr, la.fj[0], la.fj[1], la.fj[2], 0, la.row_off * d / 2 + plo + q,
                        pre_f + q * CH_SLOT_WORDS);
      }
    }
    __syncthreads();
  }

  LOSS_TRACE(1);
  // 1. max_tree (protocols.py:356-380): level by level, as maxtree_kernel
  const uint64_t* in = z;
  uint64_t m = d;
  for (int l = 0; l < la.levels; ++l) {
    const uint64_t k = m / 2, mo = k + (m & 1);
    uint64_t* o = l == la.levels - 1 ? mx : ((l & 1) ? s1 : s0);
    if (prefill) {  // slots filled up front: the circuit only
      const uint64_t nl = rows * k, n_total = la.rows_total * k;
      const int Pl = (int)((rn * k + 1) / 2);
      const MaxGeom g = {rows, m, k};
      const LaneGroup G = lane_group();
      const int nw = blockDim.x >> 5;
      for (int base = (threadIdx.x >> 5) * 10; base < Pl; base += nw * 10) {
        const int pp = base + G.gi;
        const bool live = G.gi < 10 && pp < Pl;
        const Lane3 L = {pre_l[l], Pl, live ? pp : 0, G.ci, G.nl, G.pl};
        maxlevel_item_lane(L, in, o, g, nl, n_total, r0 * k / 2 + L.p, live);
      }
      __syncthreads();
      if (m & 1)
        for (uint64_t r = threadIdx.x; r < rn; r += blockDim.x)
          store_trio(o, rows * mo, (r0 + r) * mo + k, load_trio(in, rows * m, (r0 + r) * m + m - 1));
      __syncthreads();
      in = o;
      m = mo;
      continue;
    }
    if (threadIdx.x == 0) {
      const SignArgs a = {la.jbin[l], la.jxor[l], la.ja[l], 0, 0, 0};
      sign_streams(st, a, ctr, false);
    }
    __syncthreads();
    cache_sign_streams(tab, &ks.rk[0][0], st, reinterpret_cast<AesSmem*>(mpc3_dsm)->hc, false);
    if (l == 0) LOSS_TRACE(8);
    const uint64_t nl = rows * k, n_total = la.rows_total * k, elem_off = la.row_off * k;
    const bool straddle = (n_total & 1) != 0;
    const int L = straddle ? 3 : 2, used = sign_slots(straddle);
    const uint64_t p0 = r0 * k / 2, P = (rn * k + 1) / 2;
    const MaxGeom g = {rows, m, k};
    for (uint64_t c = 0; c < P; c += MT_PMAX) {
      const int Pc = (int)(P - c < (uint64_t)MT_PMAX ? P - c : (uint64_t)MT_PMAX);
      for (int q = threadIdx.x; q < used * Pc; q += blockDim.x) {
        const int sidx = q / Pc, p = q % Pc;
        sign_slot_fill(tab, rk, st, sidx, (elem_off >> 1) + p0 + c + p, n_total, L, slots + ((size_t)sidx * Pc + p) * 3);
      }
      __syncthreads();
      if (l == 0 && c == 0) LOSS_TRACE(9);
#if MPC3_SIGN2_LANES
      {
        const LaneGroup G = lane_group();
        const int nw = blockDim.x >> 5;
        for (int base = (threadIdx.x >> 5) * 10; base < Pc; base += nw * 10) {
          const int pp = base + G.gi;
          const bool live = G.gi < 10 && pp < Pc;
          const Lane3 L = {slots, Pc, live ? pp : 0, G.ci, G.nl, G.pl};
          maxlevel_item_lane(L, in, o, g, nl, n_total, p0 + c + L.p, live);
        }
      }
#else
      if (threadIdx.x < Pc) {
        Replay rp;
        rp.w = slots;
        rp.P = Pc;
        rp.p = threadIdx.x;
        rp.slot = 0;
        maxlevel_item(rp, rk, st, in, o, g, nl, n_total, elem_off, p0 + c + threadIdx.x);
      }
#endif
      __syncthreads();
      if (l == 0 && c == 0) LOSS_TRACE(10);
    }
    if (m & 1)
      for (uint64_t r = threadIdx.x; r < rn; r += blockDim.x)
        store_trio(o, rows * mo, (r0 + r) * mo + k, load_trio(in, rows * m, (r0 + r) * m + m - 1));
    __syncthreads();
    if (l == 0) LOSS_TRACE(11);
    in = o;
    m = mo;
  }
  LOSS_TRACE(2);
  // 2. x = z - max (a local op)
  for (uint64_t i = threadIdx.x; i < rn * d; i += blockDim.x) {
    const uint64_t f = r0 * d + i, row = f / d;
    const Trio a = load_trio(z, n, f), b = load_trio(mx, rows, row);
    Trio v;
    for (int c = 0; c < 3; ++c) v.c[c] = a.c[c] - b.c[c];
    store_trio(X, n, f, v);
  }
  __syncthreads();
  LOSS_TRACE(3);
  // 3. e = exp_approx(x) over this CTA's pairs of the (rows, d) tensor
  chain_pairs(tab, rk, ctr, la.ep, la.ej[0], la.ej[1], la.ej[2], X, E, n, la.row_off * d / 2, plo, phi, slots, pre_e);
  LOSS_TRACE(4);
  // 4. s = sum_j e (a local op)
  for (uint64_t r = threadIdx.x; r < rn; r += blockDim.x) {
    Trio acc{{0, 0, 0}};
    for (uint64_t j = 0; j < d; ++j) {
      const Trio v = load_trio(E, n, (r0 + r) * d + j);
      for (int c = 0; c < 3; ++c) acc.c[c] += v.c[c];
    }
    store_trio(T, rows, r0 + r, acc);
  }
  __syncthreads();
  LOSS_TRACE(5);
  // 5. 1/s (reciprocal's Newton chain) over this CTA's rows
  chain_pairs(tab, rk, ctr, la.rp, la.rj[0], la.rj[1], la.rj[2], T, RR, rows, la.row_off / 2, rlo, rhi, slots, pre_r);
  LOSS_TRACE(6);
  // 6. out = truncate(e * (1/s)) - y (mul_truncate, then the loss gradient's local sub)
  const StreamHead ha = resolve(sref(ARITH_ZERO, la.fj[0]), ctr), hrho = resolve(sref(TRUNC_RHO, la.fj[1]), ctr),
                   hr = resolve(sref(TRUNC_R, la.fj[2]), ctr);
  for (uint64_t b = plo + threadIdx.x; b < phi; b += blockDim.x) {
    const uint64_t blk = la.row_off * d / 2 + b;
    Word2 w[3], rho, r;
    if (pre_f) {
      const Word2* sl = pre_f + (b - plo) * CH_SLOT_WORDS;
      w[0] = sl[0];
      w[1] = sl[1];
      w[2] = sl[2];
      rho = sl[3];
      r = sl[4];
    } else {
      prf_block3(tab, rk, ha, blk, w);
      trunc_words(tab, rk, hrho, hr, blk, rho, r);
    }
    for (int e = 0; e < 2; ++e) {
      const uint64_t f = 2 * b + e;
      if (f >= n || f >= (r0 + rn) * d) break;
      KeyWords kw;
      for (int c = 0; c < 3; ++c) kw.k[c] = e ? w[c].w1 : w[c].w0;
      Trio v = trio_mul(load_trio(E, n, f), load_trio(RR, rows, f / d), kw);
      v = trio_truncate(v, e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, la.bits);
      const Trio yy = load_trio(y, n, f);
      for (int c = 0; c < 3; ++c) v.c[c] -= yy.c[c];
      store_trio(out, n, f, v);
    }
  }
  LOSS_TRACE(7);
}

// SGD on every parameter in one launch (nn.py:539-543, the reference's
// W <- W - truncate(c * grad) per parameter): tensor i's elements use its own
// TRUNC_RHO / TRUNC_R counters; the pair space of all tensors is one
// grid-stride range (prefix sums in the launch parameters).
struct SgdTable {
  int nt;
  MPC3SgdTensor t[MPC3_SGD_MAX_TENSORS];
  uint64_t pair0[MPC3_SGD_MAX_TENSORS + 1];  // first pair of tensor i in the flattened range
};

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) sgd_kernel(const __grid_constant__ KeySched ks,
                                                      const uint64_t* __restrict__ ctr, SgdTable tb, int bits,
                                                      uint64_t c) {
  auto tab = Proto<F>::init();
  const uint64_t total = tb.pair0[tb.nt];
  // the first kHeadSlots4 / 2 tensors' (rho, r) heads with counter-mode
  // constants in shared memory (four-table launches: one CTA per SM); the
  // rest resolved per pair
  constexpr int KT = Proto<F>::TT::kTops;
  const int nc = F ? imin32(tb.nt, kHeadSlots4 / 2) : 0;
  StreamHead* hs = reinterpret_cast<StreamHead*>(reinterpret_cast<AesSmem4*>(mpc3_dsm)->extra);
  static_assert(sizeof(StreamHead) * kHeadSlots4 <= sizeof(AesSmem4::extra), "SGD heads fit the extra area");
  if constexpr (F) {
    HeadConst* slots = Proto<F>::slots();
    if (threadIdx.x < 2 * nc) {
      const MPC3SgdTensor& T = tb.t[threadIdx.x >> 1];
      hs[threadIdx.x] = (threadIdx.x & 1) ? resolve(sref(TRUNC_R, T.j_r), ctr) : resolve(sref(TRUNC_RHO, T.j_rho), ctr);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * nc * KT * 3; t += blockDim.x) {
      const StreamHead h = hs[t / (3 * KT)];
      head_const(tab, &ks.rk[0][0] + 44 * (t % 3), h.s0, h.s1, (uint32_t)(t / 3 % KT), slots[t]);
    }
    __syncthreads();
    if (threadIdx.x < 2 * nc) hs[threadIdx.x].pc = (uint32_t)__cvta_generic_to_shared(&slots[threadIdx.x * KT * 3]);
    __syncthreads();
  }
  GRID_LOOP(q, total) {
    int i = 0;
    while (q >= tb.pair0[i + 1]) ++i;  // few tensors: linear scan
    const MPC3SgdTensor& T = tb.t[i];
    const uint64_t b = q - tb.pair0[i], n = T.n;
    // the pair's gradient and parameter loads are issued before its AES
    // blocks, whose latency then covers them (ncu: long-scoreboard stalls
    // were a quarter of the warp samples with the loads after)
    Trio g[2], w[2];
    const bool two = 2 * b + 1 < n;
    g[0] = load_trio(T.grad, n, 2 * b);
    w[0] = load_trio(T.param, n, 2 * b);
    if (two) {
      g[1] = load_trio(T.grad, n, 2 * b + 1);
      w[1] = load_trio(T.param, n, 2 * b + 1);
    }
    Word2 rho, r;
    if (i < nc)
      trunc_words(tab, &ks.rk[0][0], hs[2 * i], hs[2 * i + 1], b, rho, r);
    else
      trunc_words(tab, &ks.rk[0][0], resolve(sref(TRUNC_RHO, T.j_rho), ctr), resolve(sref(TRUNC_R, T.j_r), ctr), b,
                  rho, r);
    for (int e = 0; e < (two ? 2 : 1); ++e) {
      for (int k = 0; k < 3; ++k) g[e].c[k] *= c;
      const Trio v = trio_truncate(g[e], e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, bits);
      for (int k = 0; k < 3; ++k) w[e].c[k] -= v.c[k];
      store_trio(T.param, n, 2 * b + e, w[e]);
    }
  }
}

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) inject_kernel(const __grid_constant__ KeySched ks,
                                                         const uint64_t* __restrict__ ctr, StreamRef r0,
                                                         StreamRef r1, const uint64_t* __restrict__ bits,
                                                         uint64_t* __restrict__ out, uint64_t n, uint64_t pb0) {
  auto tab = Proto<F>::init();
  StreamHead a0 = resolve(r0, ctr), a1 = resolve(r1, ctr);
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), a0, a1);
  GRID_LOOP(b, (n + 1) >> 1) inject_item(tab, &ks.rk[0][0], a0, a1, bits, out, n, b, pb0);
}

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) reshare_trunc_kernel(const __grid_constant__ KeySched ks,
                                                                const uint64_t* __restrict__ ctr, StreamRef ra,
                                                                StreamRef rrho, StreamRef rr, int bits,
                                                                const uint64_t* __restrict__ z, View4 v,
                                                                uint64_t* __restrict__ out, uint64_t n,
                                                                uint64_t pb0) {
  auto tab = Proto<F>::init();
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), ha, hrho, hr);
  if (n < (1ull << 32))
    GRID_LOOP(b, (n + 1) >> 1) reshare_trunc_item<typename Proto<F>::TT, uint32_t>(tab, &ks.rk[0][0], ha, hrho, hr, bits, z, v, out,
                                                                         n, b, pb0);
  else
    GRID_LOOP(b, (n + 1) >> 1) reshare_trunc_item(tab, &ks.rk[0][0], ha, hrho, hr, bits, z, v, out, n, b, pb0);
}

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) pool_kernel(const __grid_constant__ KeySched ks,
                                                       const uint64_t* __restrict__ ctr, int backward,
                                                       StreamRef rrho, StreamRef rr, int bits, uint64_t mulc,
                                                       const uint64_t* __restrict__ x,
                                                       uint64_t* __restrict__ out, PoolGeom p, uint64_t n,
                                                       uint64_t pb0, const uint64_t* __restrict__ mask,
                                                       StreamRef ra) {
  auto tab = Proto<F>::init();
  StreamHead hrho = resolve(rrho, ctr), hr = resolve(rr, ctr), ha = mask ? resolve(ra, ctr) : StreamHead{0, 0, 0};
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), hrho, hr, ha);
  if (2 * n < (1ull << 32) && (uint64_t)p.N * p.C * p.H * p.W < (1ull << 32))
    GRID_LOOP(b, (n + 1) >> 1) pool_item<typename Proto<F>::TT, uint32_t>(tab, &ks.rk[0][0], backward != 0, hrho, hr, bits, mulc, x,
                                                                out, p, b, pb0, mask, ha);
  else
    GRID_LOOP(b, (n + 1) >> 1) pool_item(tab, &ks.rk[0][0], backward != 0, hrho, hr, bits, mulc, x, out, p, b, pb0,
                                         mask, ha);
}

template <bool F>
__global__ void __launch_bounds__(Proto<F>::threads, Proto<F>::min_ctas) col2im_kernel(const __grid_constant__ KeySched ks,
                                                         const uint64_t* __restrict__ ctr, StreamRef ra,
                                                         StreamRef rrho, StreamRef rr, int bits,
                                                         const uint64_t* __restrict__ z, Col2Im g,
                                                         uint64_t* __restrict__ out, uint64_t n, uint64_t pb0) {
  auto tab = Proto<F>::init();
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  cache_heads(tab, &ks.rk[0][0], Proto<F>::slots(), ha, hrho, hr);
  if (2 * n < (1ull << 32))
    GRID_LOOP(b, (n + 1) >> 1) col2im_item<typename Proto<F>::TT, uint32_t>(tab, &ks.rk[0][0], ha, hrho, hr, bits, z, g, out, b,
                                                                  pb0);
  else
    GRID_LOOP(b, (n + 1) >> 1) col2im_item(tab, &ks.rk[0][0], ha, hrho, hr, bits, z, g, out, b, pb0);
}

__global__ void sumpool_kernel(const uint64_t* __restrict__ x, uint64_t* __restrict__ out, PoolGeom p) {
  uint64_t n = (uint64_t)p.N * p.C * p.OH * p.OW;
  GRID_LOOP(f, n) {
    int64_t ox = f % p.OW, oy = (f / p.OW) % p.OH, nc = f / (p.OW * p.OH);
    const uint64_t* base = x + nc * p.H * p.W + (oy * p.sh) * p.W + ox * p.sw;
    uint64_t s = 0;
    for (int u = 0; u < p.kh; ++u)
      for (int q = 0; q < p.kw; ++q) s += base[u * p.W + q];
    out[f] = s;
  }
}


// Max-pool windows (nn.MaxPool extension): out[(n, c, oy, ox), (u, v)] =
// x[n, c, oy*sh - ph + u, ox*sw - pw + v] for the three components, (u, v)
// row-major; a window position in the zero padding holds the public
// constant pad in component 0 and 0 in components 1, 2 (sharing.py:184-187),
// so max_tree over the window row is the composed reference max-pool.
__global__ void window_gather_kernel(const uint64_t* __restrict__ x, uint64_t* __restrict__ out, PoolGeom p,
                                     int ph, int pw, uint64_t pad) {
  griddep_launch();
  griddep_wait();
  const uint64_t kk = (uint64_t)p.kh * p.kw;
  const uint64_t n = (uint64_t)p.N * p.C * p.OH * p.OW * kk;
  const uint64_t plane_in = (uint64_t)p.N * p.C * p.H * p.W;
  GRID_LOOP(f, 3 * n) {
    const uint64_t comp = f / n, e = f - comp * n;
    const uint64_t w = e / kk, uv = e - w * kk;
    const int64_t u = (int64_t)(uv / p.kw), v = (int64_t)(uv % p.kw);
    const int64_t ox = w % p.OW, oy = (w / p.OW) % p.OH, nc = w / ((uint64_t)p.OW * p.OH);
    const int64_t yy = oy * p.sh - ph + u, xx = ox * p.sw - pw + v;
    uint64_t r;
    if (yy < 0 || yy >= p.H || xx < 0 || xx >= p.W)
      r = comp == 0 ? pad : 0;
    else
      r = x[comp * plane_in + (nc * p.H + yy) * p.W + xx];
    out[f] = r;
  }
}

}  // namespace mpc3

using namespace mpc3;

extern "C" {

int mpc3_abi_version(void) { return MPC3_ABI_VERSION; }

const char* mpc3_status_name(int s) {
  switch (s) {
    case MPC3_OK: return "OK";
    case MPC3_ERR_RANGE: return "RangeError";
    case MPC3_ERR_SHAPE: return "ShapeError";
    case MPC3_ERR_EXACTNESS: return "ExactnessError";
    case MPC3_ERR_CONFIG: return "ConfigError";
    case MPC3_ERR_FRESHNESS: return "FreshnessError";
    case MPC3_ERR_TOPOLOGY: return "TopologyError";
    case MPC3_ERR_INTEGRITY: return "IntegrityError";
    case MPC3_ERR_CUDA: return "CudaError";
    case MPC3_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "Unknown";
}

const char* mpc3_last_error(void) { return g_last_error; }

int mpc3_aes128_expand(const uint8_t key[16], uint32_t rk[44]) {
  if (!key || !rk) return MPC3_ERR_CONFIG;
  aes128_expand(key, rk);
  return MPC3_OK;
}

static int check_stream_args(uint32_t purpose, uint64_t index) {
  if (purpose >= (1u << 16)) return MPC3_ERR_RANGE;  // prf.py:42-43
  if (index >= (1ull << 48)) return MPC3_ERR_RANGE;  // prf.py:44-45
  return MPC3_OK;
}

int mpc3_prf_words(const uint32_t* rk, uint32_t purpose, uint64_t index, uint64_t word_off, uint64_t count,
                   uint64_t* words, void* stream) {
  int st = check_stream_args(purpose, index);
  if (st) return st;
  if (count == 0) return MPC3_OK;
  uint64_t nblk = ((word_off + count - 1) >> 1) - (word_off >> 1) + 1;
  KeySched ks;
  if (int e = load_keys(rk, 1, stream, &ks)) return e;
  if (!aes_attr((const void*)prf_words_kernel, kAesSmem4Bytes)) return check_launch("prf smem attribute");
  launch_pdl(prf_words_kernel, dim3(grid_for(nblk, kSignThreads, 8)), dim3(kSignThreads), kAesSmem4Bytes,
             as_stream(stream), ks, stream_head(purpose, index), word_off, count, words);
  return check_launch("prf_words");
}

int mpc3_rss_zero_share(const uint32_t* rk3, const uint64_t* ctr, uint32_t purpose, uint64_t index, int xor_mode, uint64_t n,
                        uint64_t* out, void* stream) {
  int st = check_stream_args(purpose, index);
  if (st) return st;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(zero_share_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, sref(purpose, index), xor_mode, n, out);
  return check_launch("zero_share");
}

int mpc3_ring_ew(int op, const uint64_t* a, const uint64_t* b, uint64_t c, uint64_t* out, uint64_t n,
                 void* stream) {
  if (op < 0 || op > MPC3_EW_AXPY) return MPC3_ERR_CONFIG;
  if ((op == MPC3_EW_SHL || op == MPC3_EW_SHR || op == MPC3_EW_SAR) && c >= 64) return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  launch_pdl(ring_ew_kernel, dim3(grid_for(n, 256)), dim3(256), 0, as_stream(stream), op, a, b, c, out, n);
  return check_launch("ring_ew");
}

int mpc3_ring_rowop(int op, const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t rows, uint64_t cols,
                    void* stream) {
  if (rows * cols == 0) return MPC3_OK;
  launch_pdl(ring_rowop_kernel, dim3(grid_for(rows * cols, 256)), dim3(256), 0, as_stream(stream), op, a, b, out, rows,
             cols);
  return check_launch("ring_rowop");
}

int mpc3_ring_rowsum(const uint64_t* a, uint64_t* out, uint64_t rows, uint64_t cols, void* stream) {
  if (rows == 0) return MPC3_OK;
  launch_pdl(ring_rowsum_kernel, dim3(grid_for(rows, 128)), dim3(128), 0, as_stream(stream), a, out, rows, cols);
  return check_launch("ring_rowsum");
}

static int arith_launch(int kind, const uint32_t* rk3, const uint64_t* ctr, uint64_t ja, uint64_t jrho, uint64_t jr, int bits,
                        const uint64_t* x, const uint64_t* y, uint64_t* out, uint64_t n, uint64_t elem_off,
                        void* stream) {
  if (kind != 0 && (bits < 1 || bits > 61)) return MPC3_ERR_RANGE;  // protocols.py:185-186
  if (ja >= (1ull << 48) || jrho >= (1ull << 48) || jr >= (1ull << 48)) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(arith_kernel, (n + 1) / 2, as_stream(stream), 
      kind, ks, ctr, sref(ARITH_ZERO, ja), sref(TRUNC_RHO, jrho), sref(TRUNC_R, jr), bits, x, y, out, n,
      elem_off >> 1);
  return check_launch("rss_arith");
}

int mpc3_rss_mul(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, const uint64_t* x, const uint64_t* y, uint64_t* out,
                 uint64_t n, uint64_t elem_off, void* stream) {
  return arith_launch(0, rk3, ctr, j_arith, 0, 0, 0, x, y, out, n, elem_off, stream);
}

int mpc3_rss_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, const uint64_t* x,
                      uint64_t* out, uint64_t n, uint64_t elem_off, void* stream) {
  return arith_launch(1, rk3, ctr, 0, j_rho, j_r, bits, x, nullptr, out, n, elem_off, stream);
}

int mpc3_rss_mul_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r, int bits,
                          const uint64_t* x, const uint64_t* y, uint64_t* out, uint64_t n, uint64_t elem_off,
                          void* stream) {
  return arith_launch(2, rk3, ctr, j_arith, j_rho, j_r, bits, x, y, out, n, elem_off, stream);
}

int mpc3_rss_sgd_multi(const uint32_t* rk3, const uint64_t* ctr, const MPC3SgdTensor* ts, int nt, int bits,
                       uint64_t c, void* stream) {
  if (!ts || nt < 0 || nt > MPC3_SGD_MAX_TENSORS) return MPC3_ERR_CONFIG;
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  SgdTable tb;
  tb.nt = nt;
  tb.pair0[0] = 0;
  for (int i = 0; i < nt; ++i) {
    if (ts[i].j_rho >= (1ull << 48) || ts[i].j_r >= (1ull << 48)) return MPC3_ERR_RANGE;
    tb.t[i] = ts[i];
    tb.pair0[i + 1] = tb.pair0[i] + (ts[i].n + 1) / 2;
  }
  if (tb.pair0[nt] == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(sgd_kernel, tb.pair0[nt], as_stream(stream), ks, ctr, tb, bits, c);
  return check_launch("rss_sgd_multi");
}

int mpc3_rss_chain(const uint32_t* rk3, const uint64_t* ctr, const MPC3ChainStep* steps, int nsteps, uint64_t j_arith,
                   uint64_t j_rho, uint64_t j_r, const uint64_t* x, uint64_t* out, uint64_t n, uint64_t elem_off,
                   void* stream) {
  if (!steps || nsteps < 0 || nsteps > MPC3_CHAIN_MAX_STEPS) return MPC3_ERR_CONFIG;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  ChainProgram prog;
  prog.nsteps = nsteps;
  prog.nmul = 0;
  for (int i = 0; i < nsteps; ++i) {
    prog.s[i] = steps[i];
    const int op = steps[i].op;
    if (op < MPC3_CHAIN_ADDC || op > MPC3_CHAIN_SQT) return MPC3_ERR_CONFIG;
    if (op == MPC3_CHAIN_SQ || op == MPC3_CHAIN_MULX || op == MPC3_CHAIN_SQT) {
      if (steps[i].bits < 1 || steps[i].bits > 61) return MPC3_ERR_RANGE;  // protocols.py:185-186
      ++prog.nmul;
    }
  }
  if (j_arith + prog.nmul >= (1ull << 48) || j_rho + prog.nmul >= (1ull << 48) || j_r + prog.nmul >= (1ull << 48))
    return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  int P = 64;
  while (P > 8 && P * prog.nmul * CH_SLOT_WORDS * (int)sizeof(Word2) > 96 * 1024) P >>= 1;
  if (P * (prog.nmul > 0 ? prog.nmul : 1) * CH_SLOT_WORDS * (int)sizeof(Word2) > 96 * 1024) return MPC3_ERR_CONFIG;
  const int smem = kAesSmemBytes + P * prog.nmul * CH_SLOT_WORDS * (int)sizeof(Word2);
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  if (!aes_attr((const void*)chain_kernel, kAesSmemBytes + 96 * 1024)) return check_launch("chain smem attribute");
  uint64_t chunks = ((n + 1) / 2 + P - 1) / P;
  unsigned grid = (unsigned)(chunks < 148 * 8 ? chunks : 148 * 8);
  launch_pdl(chain_kernel, dim3(grid), dim3(kThreads), smem, as_stream(stream), ks, ctr, prog, j_arith, j_rho, j_r,
             x, out, n, elem_off >> 1, P);
  return check_launch("rss_chain");
}

// Two-phase chunk size: at most 64 pairs (32 when the p-half straddles
// blocks: more keystream slots), and just enough that the CTA count fills
// whole waves of the 2 x 148 resident CTAs (a 1.3-wave grid would leave most
// SMs idle for the second wave).
// sign2 with the four-table layout (one 384-thread CTA per SM, 128-pair
// chunks) measured the same as two-table in the AlexNet step (2.597 vs 2.593
// ms): the two-phase kernel is latency-bound, not lookup-bound
#ifndef MPC3_SIGN2_FOUR
#define MPC3_SIGN2_FOUR 0
#endif
constexpr bool kSign2Four = MPC3_SIGN2_FOUR;
static int sign2_pmax(bool straddle, bool rs) {
  if (rs) return straddle ? 32 : 48;  // two more slots per pair (the layer's reshare / truncation words)
  // 60, not 64: two two-table CTAs (AES tables + counter-mode constants + 16
  // slots x 48 B per pair) must fit one SM's 228 KiB
  return (straddle ? 32 : 60) * (kSign2Four ? 2 : 1);
}
static_assert(kSign2Four || 2 * (kAesSmemBytes + 60 * 16 * 3 * (int)sizeof(Word2) + 1024) <= 228 * 1024,
              "two sign2 CTAs per SM");
static int sign2_chunk(uint64_t pairs, bool straddle, bool rs = false) {
  const uint64_t pmax = sign2_pmax(straddle, rs), slots = (kSign2Four ? 1 : 2) * 148;
  const uint64_t waves = (pairs + slots * pmax - 1) / (slots * pmax);
  uint64_t P = (pairs + waves * slots - 1) / (waves * slots);
  if (P < 8) P = 8;
  return (int)(P > pmax ? pmax : P);
}

static int sign2_smem(int P, bool straddle, bool rs = false) {
  return (kSign2Four ? kAesSmem4Bytes : kAesSmemBytes) + P * (sign_slots(straddle) + (rs ? 2 : 0)) * SW_SLOT_BYTES;
}
static int sign2_smem_max(bool rs = false) {  // the largest chunk a launch uses
  const int a = sign2_smem(sign2_pmax(false, rs), false, rs), b = sign2_smem(sign2_pmax(true, rs), true, rs);
  return a > b ? a : b;
}

// The sign circuit over n elements (x, or a fused layer's cross terms rin):
// whole rounds of the persistent single-phase kernel, the rest two-phase.
#ifndef MPC3_SIGN_ROUND_PCT
#define MPC3_SIGN_ROUND_PCT 72
#endif
#ifndef MPC3_SIGN_ROUND_RS_PCT
#define MPC3_SIGN_ROUND_RS_PCT 55
#endif
static int sign_launch(const KeySched& ks, const uint64_t* ctr, const SignArgs& a, int mode, const uint64_t* x,
                       const RsIn* rin, uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total,
                       uint64_t elem_off, void* stream) {
  const bool rs = rin != nullptr;
  RsIn ri = rs ? *rin : RsIn{};
  // large tensors: the single-phase kernel (throughput-bound, all threads in
  // the circuit) on a persistent grid, one 384-thread CTA per SM, every
  // thread exactly k pairs (no partial wave, no CTA-boundary bubbles); the
  // remainder and small tensors: the two-phase kernel (latency-bound work)
  const uint64_t pairs = (n + 1) / 2;
  const uint64_t persist = 148ull * kSignThreads;
  uint64_t main_pairs = 0;
  if (!g_sign_fused) {
    // whole rounds of the persistent grid (one pair per thread per round,
    // ~50 us a round full or not), the remainder in the two-phase kernel
    // (~8 us + 57 us x the fraction of a round; 85 us with the fused layer
    // epilogue) — unless the remainder is large enough that one more
    // persistent round is cheaper (tools/dbg/sign_sizes.py), also for
    // tensors below one round
    main_pairs = pairs / persist * persist;
    const uint64_t rem = pairs - main_pairs;
    if (rem * 100 >= persist * (rs ? MPC3_SIGN_ROUND_RS_PCT : MPC3_SIGN_ROUND_PCT)) main_pairs = pairs;
  }
  if (g_sign_fused) main_pairs = pairs;
  if (main_pairs) {
    const uint64_t nm = main_pairs == pairs ? n : 2 * main_pairs;
    const unsigned grid = g_sign_fused ? grid_for(pairs, kSignThreads, 8) : grid_for(main_pairs, kSignThreads, 1);
    auto kern = rs ? sign_kernel<true> : sign_kernel<false>;
    if (!aes_attr((const void*)kern, kAesSmem4Bytes)) return check_launch("sign smem attribute");
    launch_pdl(kern, dim3(grid), dim3(kSignThreads), kAesSmem4Bytes, as_stream(stream), ks, ctr, a, mode, x, out,
               mask, nm, n_total, elem_off, n, ri);
    if (check_launch("rss_sign")) return MPC3_ERR_CUDA;
  }
  if (main_pairs < pairs) {
    // two-phase kernel: P pairs per chunk, tables + keystream slots in
    // dynamic shared memory
    const uint64_t e0 = 2 * main_pairs, nr = n - e0;
    const bool straddle = (n_total & 1) != 0;
    const int P = sign2_chunk((nr + 1) / 2, straddle, rs);
    const int smem = sign2_smem(P, straddle, rs);
    auto kern = rs ? (kSign2Four ? sign2_kernel<S2_RS, true> : sign2_kernel<S2_RS, false>)
                   : (kSign2Four ? sign2_kernel<S2_SIGN, true> : sign2_kernel<S2_SIGN, false>);
    if (!aes_attr((const void*)kern, sign2_smem_max(rs))) return check_launch("sign2 smem attribute");
    uint64_t chunks = ((nr + 1) / 2 + P - 1) / P;
    unsigned grid = (unsigned)(chunks < 148 * 2 * MPC3_SIGN2_WAVES ? chunks : 148 * 2 * MPC3_SIGN2_WAVES);
    ri.f0 += e0;
    launch_pdl(kern, dim3(grid), dim3(kSign2Four ? kSignThreads : kThreads), smem, as_stream(stream), ks, ctr, a, mode,
               rs ? x : x + e0, out + e0, mask ? mask + e0 : mask, nr, n_total, elem_off + e0, P, n,
               MaxGeom{0, 0, 1}, ri);
    return check_launch("rss_sign2");
  }
  return MPC3_OK;
}

int mpc3_rss_sign(const uint32_t* rk3, const uint64_t* ctr, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                  const uint64_t* x, uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total,
                  uint64_t elem_off, void* stream) {
  if (mode < MODE_A2B || mode > MODE_RELU) return MPC3_ERR_CONFIG;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (elem_off + n > n_total) return MPC3_ERR_SHAPE;
  if (j_bin >= (1ull << 48) || j_xor + 6 >= (1ull << 48) || j_arith + 2 >= (1ull << 48))
    return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  SignArgs a = {j_bin, j_xor, j_arith, 0, 0, 0};
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  return sign_launch(ks, ctr, a, mode, x, nullptr, out, mask, n, n_total, elem_off, stream);
}

int mpc3_rss_layer_sign(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_ra, uint64_t j_rho, uint64_t j_r,
                        int bits, const uint64_t* z, const mpc3_view4* view, const uint64_t* bias, int64_t bias_plane,
                        int bias_dim, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith, uint64_t* out,
                        uint64_t* mask, uint64_t elem_off, uint64_t n_total, void* stream) {
  return mpc3_rss_layer_sign_residual(rk3, ctr, j_ra, j_rho, j_r, bits, z, view, bias, bias_plane, bias_dim, nullptr, 0,
                                      mode, j_bin, j_xor, j_arith, out, mask, elem_off, n_total, stream);
}

int mpc3_rss_layer_sign_residual(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_ra, uint64_t j_rho,
                                 uint64_t j_r, int bits, const uint64_t* z, const mpc3_view4* view,
                                 const uint64_t* bias, int64_t bias_plane, int bias_dim, const uint64_t* res,
                                 int64_t res_plane, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                                 uint64_t* out, uint64_t* mask, uint64_t elem_off, uint64_t n_total, void* stream) {
  if (mode < MODE_A2B || mode > MODE_RELU) return MPC3_ERR_CONFIG;
  if (res && res_plane < 0) return MPC3_ERR_CONFIG;
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (bias && (bias_dim < 0 || bias_dim > 3 || bias_plane < 0)) return MPC3_ERR_CONFIG;
  if (!view || !z || (elem_off & 1)) return MPC3_ERR_CONFIG;
  RsIn ri;
  ri.z = z;
  ri.bits = bits;
  ri.f0 = 0;
  uint64_t n = 1;
  for (int k = 0; k < 4; ++k) {
    ri.v.full[k] = view->full[k];
    ri.v.org[k] = view->origin[k];
    ri.v.crop[k] = view->crop[k];
    ri.v.zs[k] = view->z_stride[k];
    ri.v.os[k] = view->out_stride[k];
    if (ri.v.full[k] < 0 || ri.v.org[k] != 0 || ri.v.crop[k] != ri.v.full[k]) return MPC3_ERR_SHAPE;  // no crop
    n *= (uint64_t)ri.v.full[k];
  }
  ri.v.zp = view->z_plane;
  ri.v.op = view->out_plane;
  ri.v.bias = bias;
  ri.v.bias_plane = bias_plane;
  ri.v.bias_dim = bias_dim;
  ri.small = n < (1ull << 32) ? 1 : 0;
  ri.res = res;
  ri.res_plane = (uint64_t)res_plane;
  if (res && (uint64_t)res_plane < n) return MPC3_ERR_SHAPE;
  if (elem_off + n > n_total) return MPC3_ERR_SHAPE;
  if (j_bin >= (1ull << 48) || j_xor + 6 >= (1ull << 48) || j_arith + 2 >= (1ull << 48) || j_ra >= (1ull << 48) ||
      j_rho >= (1ull << 48) || j_r >= (1ull << 48))
    return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  SignArgs a = {j_bin, j_xor, j_arith, j_ra, j_rho, j_r};
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  return sign_launch(ks, ctr, a, mode, nullptr, &ri, out, mask, n, n_total, elem_off, stream);
}

int mpc3_rss_max_level(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                       const uint64_t* v, uint64_t* out, uint64_t rows, uint64_t m, uint64_t elem_off,
                       uint64_t n_total, void* stream) {
  if (m < 2) return MPC3_ERR_SHAPE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  const uint64_t k = m / 2, n = rows * k;
  if (elem_off + n > n_total) return MPC3_ERR_SHAPE;
  if (j_bin >= (1ull << 48) || j_xor + 6 >= (1ull << 48) || j_arith + 2 >= (1ull << 48)) return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  SignArgs a = {j_bin, j_xor, j_arith, 0, 0, 0};
  const bool straddle = (n_total & 1) != 0;
  const int P = sign2_chunk((n + 1) / 2, straddle);
  const int smem = sign2_smem(P, straddle);
  auto kern = kSign2Four ? sign2_kernel<S2_MAXL, true> : sign2_kernel<S2_MAXL, false>;
  if (!aes_attr((const void*)kern, sign2_smem_max())) return check_launch("max_level smem attribute");
  uint64_t chunks = ((n + 1) / 2 + P - 1) / P;
  unsigned grid = (unsigned)(chunks < 148 * 2 * MPC3_SIGN2_WAVES ? chunks : 148 * 2 * MPC3_SIGN2_WAVES);
  launch_pdl(kern, dim3(grid), dim3(kSign2Four ? kSignThreads : kThreads), smem, as_stream(stream), ks, ctr, a,
             (int)MODE_RELU, v, out, (uint64_t*)nullptr, n, n_total, elem_off, P, (uint64_t)0, MaxGeom{rows, m, k},
             RsIn{});
  return check_launch("rss_max_level");
}

int mpc3_rss_max_tree(const uint32_t* rk3, const uint64_t* ctr, int levels, const uint64_t* j_bin,
                      const uint64_t* j_xor, const uint64_t* j_arith, const uint64_t* v, uint64_t* scratch,
                      uint64_t* out, uint64_t rows, uint64_t m, uint64_t row_off, uint64_t rows_total, void* stream) {
  if (!j_bin || !j_xor || !j_arith || !v || !out) return MPC3_ERR_CONFIG;
  int lv = 0;
  for (uint64_t mm = m; mm > 1; mm = mm / 2 + mm % 2) ++lv;
  if (m < 2 || levels != lv || levels > MT_MAX_LEVELS) return MPC3_ERR_SHAPE;
  if (row_off + rows > rows_total || (row_off & 1)) return MPC3_ERR_SHAPE;
  if (rows == 0) return MPC3_OK;
  MaxTreeArgs ta;
  ta.levels = levels;
  for (int l = 0; l < levels; ++l) {
    if (j_bin[l] >= (1ull << 48) || j_xor[l] + 6 >= (1ull << 48) || j_arith[l] + 2 >= (1ull << 48))
      return MPC3_ERR_RANGE;
    ta.jbin[l] = j_bin[l];
    ta.jxor[l] = j_xor[l];
    ta.ja[l] = j_arith[l];
  }
  ta.rows_total = rows_total;
  ta.row_off = row_off;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  const int R = 2;
  const uint64_t half = rows * ((m + 1) / 2) * 3;  // one level output, three components
  const int smem = kAesSmemBytes + MT_PMAX * sign_slots(true) * SW_SLOT_BYTES;
  if (!aes_attr((const void*)maxtree_kernel, smem)) return check_launch("max_tree smem attribute");
  launch_pdl(maxtree_kernel, dim3((unsigned)((rows + R - 1) / R)), dim3(kThreads), smem, as_stream(stream), ks, ctr,
             ta, v, scratch, scratch + half, out, rows, m, R);
  return check_launch("rss_max_tree");
}

int mpc3_rss_bit_inject(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, const uint64_t* bits, uint64_t* out,
                        uint64_t n, uint64_t elem_off, void* stream) {
  if (j_arith + 1 >= (1ull << 48)) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(inject_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, sref(ARITH_ZERO, j_arith), sref(ARITH_ZERO, j_arith + 1), bits, out, n, elem_off >> 1);
  return check_launch("rss_bit_inject");
}

int mpc3_rss_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r, int bits,
                              const uint64_t* z, const mpc3_view4* view, uint64_t* out, uint64_t elem_off,
                              void* stream) {
  return mpc3_rss_reshare_truncate_bias(rk3, ctr, j_arith, j_rho, j_r, bits, z, view, nullptr, 0, 0, out, elem_off,
                                        stream);
}

int mpc3_rss_reshare_truncate_bias(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                   uint64_t j_r, int bits, const uint64_t* z, const mpc3_view4* view,
                                   const uint64_t* bias, int64_t bias_plane, int bias_dim, uint64_t* out,
                                   uint64_t elem_off, void* stream) {
  if (bits != 0 && (bits < 1 || bits > 61)) return MPC3_ERR_RANGE;
  if (bias && (bias_dim < 0 || bias_dim > 3 || bias_plane < 0)) return MPC3_ERR_CONFIG;
  if (!view || (elem_off & 1)) return MPC3_ERR_CONFIG;
  View4 v;
  uint64_t n = 1;
  for (int k = 0; k < 4; ++k) {
    v.full[k] = view->full[k];
    v.org[k] = view->origin[k];
    v.crop[k] = view->crop[k];
    v.zs[k] = view->z_stride[k];
    v.os[k] = view->out_stride[k];
    if (v.org[k] < 0 || v.full[k] < 0 || v.crop[k] < 0) return MPC3_ERR_SHAPE;
    n *= (uint64_t)v.full[k];
  }
  v.zp = view->z_plane;
  v.op = view->out_plane;
  v.bias = bias;
  v.bias_plane = bias_plane;
  v.bias_dim = bias_dim;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(reshare_trunc_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, sref(ARITH_ZERO, j_arith), sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, z, v, out, n,
      elem_off >> 1);
  return check_launch("rss_reshare_truncate");
}

static PoolGeom pool_geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t OH, int64_t OW, int kh, int kw,
                          int sh, int sw, int ph = 0, int pw = 0) {
  PoolGeom p;
  p.N = N; p.C = C; p.H = H; p.W = W; p.OH = OH; p.OW = OW;
  p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw; p.ph = ph; p.pw = pw;
  return p;
}

int mpc3_rss_avgpool(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, uint64_t mulc,
                     const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int kh,
                     int kw, int sh, int sw, int ph, int pw, uint64_t elem_off, void* stream) {
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0 || H + 2 * ph < kh || W + 2 * pw < kw)
    return MPC3_ERR_SHAPE;
  int64_t OH = (H + 2 * ph - kh) / sh + 1, OW = (W + 2 * pw - kw) / sw + 1;
  uint64_t n = (uint64_t)N * C * OH * OW;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(pool_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, 0, sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, mulc, x, out,
      pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw, ph, pw), n, elem_off >> 1, (const uint64_t*)nullptr,
      sref(ARITH_ZERO, 0));
  return check_launch("rss_avgpool");
}

int mpc3_rss_avgpool_backward(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits, uint64_t mulc,
                              const uint64_t* g, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W,
                              int64_t OH, int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw,
                              uint64_t elem_off, void* stream) {
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0) return MPC3_ERR_SHAPE;
  uint64_t n = (uint64_t)N * C * H * W;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(pool_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, 1, sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, mulc, g, out,
      pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw, ph, pw), n, elem_off >> 1, (const uint64_t*)nullptr,
      sref(ARITH_ZERO, 0));
  return check_launch("rss_avgpool_backward");
}

int mpc3_rss_avgpool_backward_mask(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_rho, uint64_t j_r, int bits,
                                   uint64_t mulc, const uint64_t* g, const uint64_t* mask, uint64_t j_arith,
                                   uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int64_t OH, int64_t OW,
                                   int kh, int kw, int sh, int sw, int ph, int pw, uint64_t elem_off, void* stream) {
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (!mask || (elem_off & 1)) return MPC3_ERR_CONFIG;
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0) return MPC3_ERR_SHAPE;
  if (j_arith >= (1ull << 48)) return MPC3_ERR_RANGE;
  uint64_t n = (uint64_t)N * C * H * W;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(pool_kernel, (n + 1) / 2, as_stream(stream),
      ks, ctr, 1, sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, mulc, g, out,
      pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw, ph, pw), n, elem_off >> 1, mask, sref(ARITH_ZERO, j_arith));
  return check_launch("rss_avgpool_backward_mask");
}

int mpc3_rss_col2im_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                     uint64_t j_r, int bits, const uint64_t* z, int64_t N, int64_t C, int64_t OH,
                                     int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw, int64_t H,
                                     int64_t W, uint64_t* out, uint64_t elem_off, void* stream) {
  return mpc3_rss_col2im_reshare_truncate_layout(rk3, ctr, j_arith, j_rho, j_r, bits, z, 0, N, C, OH, OW, kh, kw, sh,
                                                 sw, ph, pw, H, W, out, elem_off, stream);
}

int mpc3_rss_col2im_reshare_truncate_layout(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith,
                                            uint64_t j_rho, uint64_t j_r, int bits, const uint64_t* z, int z_layout,
                                            int64_t N, int64_t C, int64_t OH, int64_t OW, int kh, int kw, int sh,
                                            int sw, int ph, int pw, int64_t H, int64_t W, uint64_t* out,
                                            uint64_t elem_off, void* stream) {
  if (z_layout != 0 && z_layout != 1) return MPC3_ERR_CONFIG;
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0) return MPC3_ERR_SHAPE;
  Col2Im g;
  g.N = N; g.C = C; g.OH = OH; g.OW = OW; g.H = H; g.W = W;
  g.kh = kh; g.kw = kw; g.sh = sh; g.sw = sw; g.ph = ph; g.pw = pw;
  g.zcol = z_layout;
  g.hf = (OH - 1) * sh + kh;
  g.wf = (OW - 1) * sw + kw;
  uint64_t n = (uint64_t)N * C * g.hf * g.wf;
  if (n == 0) return MPC3_OK;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  AES_LAUNCH(col2im_kernel, (n + 1) / 2, as_stream(stream), 
      ks, ctr, sref(ARITH_ZERO, j_arith), sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, z, g, out, n,
      elem_off >> 1);
  return check_launch("rss_col2im_reshare_truncate");
}

int mpc3_ring_sumpool(const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int kh,
                      int kw, int sh, int sw, void* stream) {
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || H < kh || W < kw) return MPC3_ERR_SHAPE;
  int64_t OH = (H - kh) / sh + 1, OW = (W - kw) / sw + 1;
  uint64_t n = (uint64_t)N * C * OH * OW;
  if (n == 0) return MPC3_OK;
  sumpool_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, out,
                                                                pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw));
  return check_launch("ring_sumpool");
}

int mpc3_rss_window_gather(const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int kh,
                           int kw, int sh, int sw, int ph, int pw, uint64_t pad, void* stream) {
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0 || 2 * ph >= kh + 1 || 2 * pw >= kw + 1 ||
      H + 2 * ph < kh || W + 2 * pw < kw)
    return MPC3_ERR_SHAPE;
  int64_t OH = (H + 2 * ph - kh) / sh + 1, OW = (W + 2 * pw - kw) / sw + 1;
  uint64_t n = 3ull * N * C * OH * OW * kh * kw;
  if (n == 0) return MPC3_OK;
  launch_pdl(window_gather_kernel, dim3(grid_for(n, 256)), dim3(256), 0, as_stream(stream), x, out,
             pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw), ph, pw, pad);
  return check_launch("rss_window_gather");
}

size_t mpc3_rss_softmax_loss_scratch(uint64_t rows, uint64_t d) {
  return (size_t)(2 * rows * ((d + 1) / 2) * 3 + 3 * rows + 2 * 3 * rows * d + 2 * 3 * rows) * sizeof(uint64_t);
}

int mpc3_rss_softmax_loss(const uint32_t* rk3, const uint64_t* ctr, const mpc3_softmax_loss_args* a, const uint64_t* z,
                          const uint64_t* y, uint64_t* scratch, uint64_t* out, uint64_t rows, uint64_t d,
                          void* stream) {
  if (!a || !z || !y || !scratch || !out) return MPC3_ERR_CONFIG;
  int lv = 0;
  for (uint64_t mm = d; mm > 1; mm = mm / 2 + mm % 2) ++lv;
  if (d < 2 || a->levels != lv || lv > MT_MAX_LEVELS) return MPC3_ERR_SHAPE;
  if (a->row_off + rows > a->rows_total || (a->row_off & 1)) return MPC3_ERR_SHAPE;
  if (a->bits < 1 || a->bits > 61) return MPC3_ERR_RANGE;
  if (rows == 0) return MPC3_OK;
  LossArgs la;
  la.levels = lv;
  for (int l = 0; l < lv; ++l) {
    if (a->j_bin[l] >= (1ull << 48) || a->j_xor[l] + 6 >= (1ull << 48) || a->j_arith[l] + 2 >= (1ull << 48))
      return MPC3_ERR_RANGE;
    la.jbin[l] = a->j_bin[l];
    la.jxor[l] = a->j_xor[l];
    la.ja[l] = a->j_arith[l];
  }
  const MPC3ChainStep* progs[2] = {a->exp_steps, a->rec_steps};
  const int counts[2] = {a->exp_count, a->rec_count};
  ChainProgram* dst[2] = {&la.ep, &la.rp};
  for (int q = 0; q < 2; ++q) {
    if (counts[q] < 0 || counts[q] > MPC3_CHAIN_MAX_STEPS || (counts[q] && !progs[q])) return MPC3_ERR_CONFIG;
    dst[q]->nsteps = counts[q];
    dst[q]->nmul = 0;
    for (int i = 0; i < counts[q]; ++i) {
      dst[q]->s[i] = progs[q][i];
      const int op = progs[q][i].op;
      if (op < MPC3_CHAIN_ADDC || op > MPC3_CHAIN_SQT) return MPC3_ERR_CONFIG;
      if (op == MPC3_CHAIN_SQ || op == MPC3_CHAIN_MULX || op == MPC3_CHAIN_SQT) {
        if (progs[q][i].bits < 1 || progs[q][i].bits > 61) return MPC3_ERR_RANGE;
        ++dst[q]->nmul;
      }
    }
  }
  for (int i = 0; i < 3; ++i) {
    la.ej[i] = a->exp_j[i];
    la.rj[i] = a->rec_j[i];
    la.fj[i] = a->fin_j[i];
    if (la.ej[i] + la.ep.nmul >= (1ull << 48) || la.rj[i] + la.rp.nmul >= (1ull << 48) || la.fj[i] >= (1ull << 48))
      return MPC3_ERR_RANGE;
  }
  la.bits = a->bits;
  la.rows_total = a->rows_total;
  la.row_off = a->row_off;
  KeySched ks;
  if (int e = load_keys(rk3, 3, stream, &ks)) return e;
  const int R = 2;
  const int smem = kAesSmemBytes + (MT_PMAX * sign_slots(true) * SW_SLOT_BYTES > LOSS_SLOT_BYTES
                                        ? MT_PMAX * sign_slots(true) * SW_SLOT_BYTES
                                        : LOSS_SLOT_BYTES);
  if (!aes_attr((const void*)softmax_loss_kernel, smem)) return check_launch("softmax_loss smem attribute");
  launch_pdl(softmax_loss_kernel, dim3((unsigned)((rows + R - 1) / R)), dim3(kThreads), smem, as_stream(stream), ks,
             ctr, la, z, y, scratch, out, rows, d, R);
  return check_launch("rss_softmax_loss");
}

}  // extern "C"
