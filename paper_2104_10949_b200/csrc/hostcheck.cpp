// CPU self-check build of the device protocol logic (TEST INFRASTRUCTURE).
//
// Compiles items.cuh / protocol.cuh / aes.cuh with g++ and runs every work
// item in a plain loop, so `tests/test_hostcheck.py` can compare the exact
// code the kernels execute against the oracle on a machine without a GPU.
// Not used by the product path.
#include <stdlib.h>
#include <string.h>

#include "items.cuh"

using namespace mpc3;

static const HostTables& tabs() {
  static HostTables t;
  return t;
}

static void expand3(const uint8_t* keys48, uint32_t* rk3) {
  for (int i = 0; i < 3; ++i) aes128_expand(keys48 + 16 * i, rk3 + 44 * i);
}

extern "C" {

void hc_prf_words(const uint8_t* key16, uint32_t purpose, uint64_t index, uint64_t word_off, uint64_t count,
                  uint64_t* out) {
  uint32_t rk[44];
  aes128_expand(key16, rk);
  if (!count) return;
  uint64_t nblk = ((word_off + count - 1) >> 1) - (word_off >> 1) + 1;
  for (uint64_t t = 0; t < nblk; ++t) prf_words_item(tabs(), rk, stream_head(purpose, index), word_off, count, out, t);
}

void hc_zero_share(const uint8_t* keys48, uint32_t purpose, uint64_t index, int xor_mode, uint64_t n, uint64_t* out) {
  uint32_t rk[132];
  expand3(keys48, rk);
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    zero_share_item(tabs(), rk, stream_head(purpose, index), xor_mode, n, out, b);
}

void hc_arith(const uint8_t* keys48, int kind, uint64_t ja, uint64_t jrho, uint64_t jr, int bits, const uint64_t* x,
              const uint64_t* y, uint64_t* out, uint64_t n) {
  uint32_t rk[132];
  expand3(keys48, rk);
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    arith_item(tabs(), rk, kind, stream_head(ARITH_ZERO, ja), stream_head(TRUNC_RHO, jrho), stream_head(TRUNC_R, jr),
               bits, x, y, out, n, b);
}

void hc_sign(const uint8_t* keys48, int mode, uint64_t jbin, uint64_t jxor, uint64_t ja, const uint64_t* x,
             uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total, uint64_t off) {
  uint32_t rk[132];
  expand3(keys48, rk);
  SignStreams st;
  st.bin = stream_head(BIN_INPUT, jbin);
  for (int l = 0; l < 7; ++l) st.x[l] = stream_head(XOR_ZERO, jxor + l);
  for (int l = 0; l < 3; ++l) st.a[l] = stream_head(ARITH_ZERO, ja + l);
  for (uint64_t b = 0; b < (n + 1) / 2; ++b) sign_item(tabs(), rk, st, mode, x, out, mask, n, n_total, off, b);
}

void hc_inject(const uint8_t* keys48, uint64_t ja, const uint64_t* bits, uint64_t* out, uint64_t n) {
  uint32_t rk[132];
  expand3(keys48, rk);
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    inject_item(tabs(), rk, stream_head(ARITH_ZERO, ja), stream_head(ARITH_ZERO, ja + 1), bits, out, n, b);
}

void hc_reshare_truncate(const uint8_t* keys48, uint64_t ja, uint64_t jrho, uint64_t jr, int bits, const uint64_t* z,
                         const mpc3_view4* view, uint64_t* out) {
  uint32_t rk[132];
  expand3(keys48, rk);
  View4 v;
  uint64_t n = 1;
  for (int k = 0; k < 4; ++k) {
    v.full[k] = view->full[k];
    v.org[k] = view->origin[k];
    v.crop[k] = view->crop[k];
    v.zs[k] = view->z_stride[k];
    v.os[k] = view->out_stride[k];
    n *= (uint64_t)v.full[k];
  }
  v.zp = view->z_plane;
  v.op = view->out_plane;
  v.bias = nullptr;
  v.bias_plane = 0;
  v.bias_dim = 0;
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    reshare_trunc_item(tabs(), rk, stream_head(ARITH_ZERO, ja), stream_head(TRUNC_RHO, jrho), stream_head(TRUNC_R, jr),
                       bits, z, v, out, n, b);
}

void hc_pool(const uint8_t* keys48, int backward, uint64_t jrho, uint64_t jr, int bits, uint64_t mulc,
             const uint64_t* x, uint64_t* out, int64_t N, int64_t C, int64_t H, int64_t W, int64_t OH, int64_t OW,
             int kh, int kw, int sh, int sw, int ph, int pw) {
  uint32_t rk[132];
  expand3(keys48, rk);
  PoolGeom p;
  p.N = N; p.C = C; p.H = H; p.W = W; p.OH = OH; p.OW = OW;
  p.kh = kh; p.kw = kw; p.sh = sh; p.sw = sw; p.ph = ph; p.pw = pw;
  uint64_t n = backward ? (uint64_t)N * C * H * W : (uint64_t)N * C * OH * OW;
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    pool_item(tabs(), rk, backward != 0, stream_head(TRUNC_RHO, jrho), stream_head(TRUNC_R, jr), bits, mulc, x, out,
              p, b);
}

void hc_col2im(const uint8_t* keys48, uint64_t ja, uint64_t jrho, uint64_t jr, int bits, const uint64_t* z,
               int64_t N, int64_t C, int64_t OH, int64_t OW, int kh, int kw, int sh, int sw, int ph, int pw,
               int64_t H, int64_t W, uint64_t* out) {
  uint32_t rk[132];
  expand3(keys48, rk);
  Col2Im g;
  g.zcol = 0;
  g.N = N; g.C = C; g.OH = OH; g.OW = OW; g.H = H; g.W = W;
  g.kh = kh; g.kw = kw; g.sh = sh; g.sw = sw; g.ph = ph; g.pw = pw;
  g.hf = (OH - 1) * sh + kh;
  g.wf = (OW - 1) * sw + kw;
  uint64_t n = (uint64_t)N * C * g.hf * g.wf;
  for (uint64_t b = 0; b < (n + 1) / 2; ++b)
    col2im_item(tabs(), rk, stream_head(ARITH_ZERO, ja), stream_head(TRUNC_RHO, jrho), stream_head(TRUNC_R, jr), bits,
                z, g, out, b);
}

void hc_pack(const uint64_t* src, int64_t plane, const mpc3_operand* op, int role, uint8_t* out, int64_t kp,
             int64_t kh) {
  Operand o;
  memset(&o, 0, sizeof(o));
  o.mode = op->mode; o.rows = op->rows; o.k = op->k; o.off = op->off; o.s_r = op->s_r;
  o.t0 = op->t0; o.t1 = op->t1; o.t2 = op->t2; o.K1 = op->K1 > 0 ? op->K1 : 1; o.K2 = op->K2 > 0 ? op->K2 : (op->k > 0 ? op->k : 1);
  o.n = op->n; o.c = op->c; o.h = op->h; o.w = op->w; o.sN = op->sN; o.sC = op->sC; o.sH = op->sH; o.sW = op->sW;
  o.kh = op->kh > 0 ? op->kh : 1; o.kw = op->kw > 0 ? op->kw : 1; o.sh = op->sh > 0 ? op->sh : 1;
  o.sw = op->sw > 0 ? op->sw : 1; o.ph = op->ph; o.pw = op->pw; o.dh = op->dh > 0 ? op->dh : 1;
  o.dw = op->dw > 0 ? op->dw : 1; o.oh = op->oh > 0 ? op->oh : 1; o.ow = op->ow > 0 ? op->ow : 1;
  int groups = role == 2 ? 1 : 3;
  int64_t total = (int64_t)groups * o.rows * (kp / 8);
  for (int64_t t = 0; t < total; ++t) pack_item(src, plane, o, role, out, kp, t, kh < 0 ? o.k : kh);
}

// Emulates the tensor-core GEMM on packed limbs: 8 int32 (wrapping) diagonal
// accumulators per output, recombined sum S_d << 8d (the epilogue's math).
void hc_gemm_packed(const uint8_t* A, const uint8_t* B, uint64_t* C, int groups, int64_t M, int64_t N, int64_t kp,
                    int64_t ldc, int64_t c_group, int64_t split_k) {
  for (int g = 0; g < groups; ++g)
    for (int64_t m = 0; m < M; ++m)
      for (int64_t n = 0; n < N; ++n) {
        uint64_t out = 0;
        for (int64_t k0 = 0; k0 < kp; k0 += split_k) {
          int64_t k1 = k0 + split_k < kp ? k0 + split_k : kp;
          uint32_t S[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          for (int i = 0; i < 8; ++i)
            for (int j = 0; i + j < 8; ++j) {
              const uint8_t* a = A + (((int64_t)g * 8 + i) * M + m) * kp;
              const uint8_t* b = B + (((int64_t)g * 8 + j) * N + n) * kp;
              uint32_t s = 0;
              for (int64_t k = k0; k < k1; ++k) s += (uint32_t)a[k] * b[k];
              S[i + j] += s;
            }
          for (int d = 0; d < 8; ++d) out += (uint64_t)S[d] << (8 * d);
        }
        C[g * c_group + m * ldc + n] = out;
      }
}

}  // extern "C"
