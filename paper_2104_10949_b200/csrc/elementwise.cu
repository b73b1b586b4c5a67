// Elementwise protocol kernels on trio tensors (three co-resident parties).
//
// Every kernel walks PRF *blocks*: thread item b owns the element pair
// (2b, 2b+1), because one AES block yields two adjacent stream words
// (prf.py:40-49).  Randomness is generated inline and never touches HBM.
#include <string.h>

#include "launch.cuh"
#include "items.cuh"

namespace mpc3 {

static thread_local char g_last_error[256] = "";
void set_last_error(const char* msg) {
  strncpy(g_last_error, msg, sizeof(g_last_error) - 1);
  g_last_error[sizeof(g_last_error) - 1] = 0;
}

constexpr int kThreads = 256;

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

__global__ void __launch_bounds__(kThreads) prf_words_kernel(const uint32_t* __restrict__ rk_dev,
                                                            StreamHead h, uint64_t word_off,
                                                            uint64_t count, uint64_t* __restrict__ out) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk_dev, 1);
  uint64_t nblk = ((word_off + count - 1) >> 1) - (word_off >> 1) + 1;
  GRID_LOOP(t, nblk) prf_words_item(tab, sm.rk[0], h, word_off, count, out, t);
}

__global__ void __launch_bounds__(kThreads) zero_share_kernel(const uint32_t* __restrict__ rk3,
                                                             const uint64_t* __restrict__ ctr, StreamRef rh,
                                                             int xor_mode, uint64_t n, uint64_t* __restrict__ out) {
  __shared__ AesSmem sm;
  StreamHead h = resolve(rh, ctr);
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  GRID_LOOP(b, (n + 1) >> 1) zero_share_item(tab, &sm.rk[0][0], h, xor_mode, n, out, b);
}

// ---------------------------------------------------------------------------
// local ring ops

__global__ void ring_ew_kernel(int op, const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                               uint64_t c, uint64_t* __restrict__ out, uint64_t n) {
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
  GRID_LOOP(i, rows * cols) {
    uint64_t v = b[i / cols];
    out[i] = op == MPC3_EW_SUB ? a[i] - v : a[i] + v;
  }
}

__global__ void ring_rowsum_kernel(const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                   uint64_t rows, uint64_t cols) {
  GRID_LOOP(r, rows) {
    uint64_t s = 0;
    for (uint64_t j = 0; j < cols; ++j) s += a[r * cols + j];
    out[r] = s;
  }
}

// ---------------------------------------------------------------------------
// protocols

__global__ void __launch_bounds__(kThreads) arith_kernel(int kind, const uint32_t* __restrict__ rk3,
                                                        const uint64_t* __restrict__ ctr, StreamRef ra,
                                                        StreamRef rrho, StreamRef rr, int bits, const uint64_t* __restrict__ x,
                                                        const uint64_t* __restrict__ y,
                                                        uint64_t* __restrict__ out, uint64_t n, uint64_t pb0) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  GRID_LOOP(b, (n + 1) >> 1) arith_item(tab, &sm.rk[0][0], kind, ha, hrho, hr, bits, x, y, out, n, b, pb0);
}

struct SignArgs {
  uint64_t jbin, jxor, ja;
};

__global__ void __launch_bounds__(kThreads, 3) sign_kernel(const uint32_t* __restrict__ rk3,
                                                          const uint64_t* __restrict__ ctr, SignArgs args,
                                                          int mode, const uint64_t* __restrict__ x,
                                                          uint64_t* __restrict__ out,
                                                          uint64_t* __restrict__ mask, uint64_t n,
                                                          uint64_t n_total, uint64_t elem_off) {
  __shared__ AesSmem sm;
  __shared__ SignStreams st;  // uniform stream heads, indexed by level from shared memory
  if (threadIdx.x == 0) {
    st.bin = resolve(sref(BIN_INPUT, args.jbin), ctr);
    for (int l = 0; l < 7; ++l) st.x[l] = resolve(sref(XOR_ZERO, args.jxor + l), ctr);
    for (int l = 0; l < 3; ++l) st.a[l] = resolve(sref(ARITH_ZERO, args.ja + l), ctr);
  }
  SmemTables tab = aes_smem_init(sm, rk3, 3);  // includes the barrier
  GRID_LOOP(b, (n + 1) >> 1) sign_item(tab, &sm.rk[0][0], st, mode, x, out, mask, n, n_total, elem_off, b);
}

__global__ void __launch_bounds__(kThreads) inject_kernel(const uint32_t* __restrict__ rk3,
                                                         const uint64_t* __restrict__ ctr, StreamRef r0,
                                                         StreamRef r1, const uint64_t* __restrict__ bits,
                                                         uint64_t* __restrict__ out, uint64_t n) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  StreamHead a0 = resolve(r0, ctr), a1 = resolve(r1, ctr);
  GRID_LOOP(b, (n + 1) >> 1) inject_item(tab, &sm.rk[0][0], a0, a1, bits, out, n, b);
}

__global__ void __launch_bounds__(kThreads) reshare_trunc_kernel(const uint32_t* __restrict__ rk3,
                                                                const uint64_t* __restrict__ ctr, StreamRef ra,
                                                                StreamRef rrho, StreamRef rr, int bits,
                                                                const uint64_t* __restrict__ z, View4 v,
                                                                uint64_t* __restrict__ out, uint64_t n,
                                                                uint64_t pb0) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  GRID_LOOP(b, (n + 1) >> 1) reshare_trunc_item(tab, &sm.rk[0][0], ha, hrho, hr, bits, z, v, out, n, b, pb0);
}

__global__ void __launch_bounds__(kThreads) pool_kernel(const uint32_t* __restrict__ rk3,
                                                       const uint64_t* __restrict__ ctr, int backward,
                                                       StreamRef rrho, StreamRef rr, int bits, uint64_t mulc,
                                                       const uint64_t* __restrict__ x,
                                                       uint64_t* __restrict__ out, PoolGeom p, uint64_t n,
                                                       uint64_t pb0) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  StreamHead hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  GRID_LOOP(b, (n + 1) >> 1) pool_item(tab, &sm.rk[0][0], backward != 0, hrho, hr, bits, mulc, x, out, p, b, pb0);
}

__global__ void __launch_bounds__(kThreads) col2im_kernel(const uint32_t* __restrict__ rk3,
                                                         const uint64_t* __restrict__ ctr, StreamRef ra,
                                                         StreamRef rrho, StreamRef rr, int bits,
                                                         const uint64_t* __restrict__ z, Col2Im g,
                                                         uint64_t* __restrict__ out, uint64_t n, uint64_t pb0) {
  __shared__ AesSmem sm;
  SmemTables tab = aes_smem_init(sm, rk3, 3);
  StreamHead ha = resolve(ra, ctr), hrho = resolve(rrho, ctr), hr = resolve(rr, ctr);
  GRID_LOOP(b, (n + 1) >> 1) col2im_item(tab, &sm.rk[0][0], ha, hrho, hr, bits, z, g, out, b, pb0);
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
  prf_words_kernel<<<grid_for(nblk, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk, stream_head(purpose, index), word_off, count, words);
  return check_launch("prf_words");
}

int mpc3_rss_zero_share(const uint32_t* rk3, const uint64_t* ctr, uint32_t purpose, uint64_t index, int xor_mode, uint64_t n,
                        uint64_t* out, void* stream) {
  int st = check_stream_args(purpose, index);
  if (st) return st;
  if (n == 0) return MPC3_OK;
  zero_share_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, sref(purpose, index), xor_mode, n, out);
  return check_launch("zero_share");
}

int mpc3_ring_ew(int op, const uint64_t* a, const uint64_t* b, uint64_t c, uint64_t* out, uint64_t n,
                 void* stream) {
  if (op < 0 || op > MPC3_EW_AXPY) return MPC3_ERR_CONFIG;
  if ((op == MPC3_EW_SHL || op == MPC3_EW_SHR || op == MPC3_EW_SAR) && c >= 64) return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  ring_ew_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(op, a, b, c, out, n);
  return check_launch("ring_ew");
}

int mpc3_ring_rowop(int op, const uint64_t* a, const uint64_t* b, uint64_t* out, uint64_t rows, uint64_t cols,
                    void* stream) {
  if (rows * cols == 0) return MPC3_OK;
  ring_rowop_kernel<<<grid_for(rows * cols, 256), 256, 0, as_stream(stream)>>>(op, a, b, out, rows, cols);
  return check_launch("ring_rowop");
}

int mpc3_ring_rowsum(const uint64_t* a, uint64_t* out, uint64_t rows, uint64_t cols, void* stream) {
  if (rows == 0) return MPC3_OK;
  ring_rowsum_kernel<<<grid_for(rows, 128), 128, 0, as_stream(stream)>>>(a, out, rows, cols);
  return check_launch("ring_rowsum");
}

static int arith_launch(int kind, const uint32_t* rk3, const uint64_t* ctr, uint64_t ja, uint64_t jrho, uint64_t jr, int bits,
                        const uint64_t* x, const uint64_t* y, uint64_t* out, uint64_t n, uint64_t elem_off,
                        void* stream) {
  if (kind != 0 && (bits < 1 || bits > 61)) return MPC3_ERR_RANGE;  // protocols.py:185-186
  if (ja >= (1ull << 48) || jrho >= (1ull << 48) || jr >= (1ull << 48)) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (n == 0) return MPC3_OK;
  arith_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      kind, rk3, ctr, sref(ARITH_ZERO, ja), sref(TRUNC_RHO, jrho), sref(TRUNC_R, jr), bits, x, y, out, n,
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

int mpc3_rss_sign(const uint32_t* rk3, const uint64_t* ctr, int mode, uint64_t j_bin, uint64_t j_xor, uint64_t j_arith,
                  const uint64_t* x, uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total,
                  uint64_t elem_off, void* stream) {
  if (mode < MODE_A2B || mode > MODE_RELU) return MPC3_ERR_CONFIG;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (elem_off + n > n_total) return MPC3_ERR_SHAPE;
  if (j_bin >= (1ull << 48) || j_xor + 6 >= (1ull << 48) || j_arith + 2 >= (1ull << 48))
    return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  SignArgs a;
  a.jbin = j_bin;
  a.jxor = j_xor;
  a.ja = j_arith;
  sign_kernel<<<grid_for((n + 1) / 2, kThreads, 16), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, a, mode, x, out, mask, n, n_total, elem_off);
  return check_launch("rss_sign");
}

int mpc3_rss_bit_inject(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, const uint64_t* bits, uint64_t* out,
                        uint64_t n, void* stream) {
  if (j_arith + 1 >= (1ull << 48)) return MPC3_ERR_RANGE;
  if (n == 0) return MPC3_OK;
  inject_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, sref(ARITH_ZERO, j_arith), sref(ARITH_ZERO, j_arith + 1), bits, out, n);
  return check_launch("rss_bit_inject");
}

int mpc3_rss_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho, uint64_t j_r, int bits,
                              const uint64_t* z, const mpc3_view4* view, uint64_t* out, uint64_t elem_off,
                              void* stream) {
  if (bits != 0 && (bits < 1 || bits > 61)) return MPC3_ERR_RANGE;
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
  if (n == 0) return MPC3_OK;
  reshare_trunc_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, sref(ARITH_ZERO, j_arith), sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, z, v, out, n,
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
  pool_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, 0, sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, mulc, x, out,
      pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw, ph, pw), n, elem_off >> 1);
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
  pool_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, 1, sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, mulc, g, out,
      pool_geom(N, C, H, W, OH, OW, kh, kw, sh, sw, ph, pw), n, elem_off >> 1);
  return check_launch("rss_avgpool_backward");
}

int mpc3_rss_col2im_reshare_truncate(const uint32_t* rk3, const uint64_t* ctr, uint64_t j_arith, uint64_t j_rho,
                                     uint64_t j_r, int bits, const uint64_t* z, int64_t N, int64_t C, int64_t OH,
                                     int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw, int64_t H,
                                     int64_t W, uint64_t* out, uint64_t elem_off, void* stream) {
  if (bits < 1 || bits > 61) return MPC3_ERR_RANGE;
  if (elem_off & 1) return MPC3_ERR_CONFIG;
  if (kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0) return MPC3_ERR_SHAPE;
  Col2Im g;
  g.N = N; g.C = C; g.OH = OH; g.OW = OW; g.H = H; g.W = W;
  g.kh = kh; g.kw = kw; g.sh = sh; g.sw = sw; g.ph = ph; g.pw = pw;
  g.hf = (OH - 1) * sh + kh;
  g.wf = (OW - 1) * sw + kw;
  uint64_t n = (uint64_t)N * C * g.hf * g.wf;
  if (n == 0) return MPC3_OK;
  col2im_kernel<<<grid_for((n + 1) / 2, kThreads), kThreads, 0, as_stream(stream)>>>(
      rk3, ctr, sref(ARITH_ZERO, j_arith), sref(TRUNC_RHO, j_rho), sref(TRUNC_R, j_r), bits, z, g, out, n,
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

}  // extern "C"
