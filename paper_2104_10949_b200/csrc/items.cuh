// Per-work-item bodies of the elementwise protocol kernels.  Each kernel in
// elementwise.cu is a grid-stride loop over these; hostcheck.cpp runs the same
// functions in a plain loop on the CPU so the oracle can check the device
// logic bit-for-bit without a GPU.
#pragma once
#include "pack.cuh"
#include "protocol.cuh"

namespace mpc3 {

HD Trio load_trio(const uint64_t* p, uint64_t plane, uint64_t e) {
  Trio t;
  t.c[0] = p[e];
  t.c[1] = p[plane + e];
  t.c[2] = p[2 * plane + e];
  return t;
}
HD void store_trio(uint64_t* p, uint64_t plane, uint64_t e, const Trio& t) {
  p[e] = t.c[0];
  p[plane + e] = t.c[1];
  p[2 * plane + e] = t.c[2];
}

// words [word_off, word_off+count) of one stream; item t = stream block first_blk + t
template <class T>
HD void prf_words_item(const T& tab, const uint32_t* rk, StreamHead h, uint64_t word_off, uint64_t count,
                       uint64_t* out, uint64_t t) {
  uint64_t blk = (word_off >> 1) + t;
  Word2 w = prf_block_k(tab, rk, 0, h, blk);
  uint64_t w0 = 2 * blk;
  if (w0 >= word_off && w0 < word_off + count) out[w0 - word_off] = w.w0;
  if (w0 + 1 >= word_off && w0 + 1 < word_off + count) out[w0 + 1 - word_off] = w.w1;
}

template <class T>
HD void zero_share_item(const T& tab, const uint32_t* rk3, StreamHead h, int xor_mode, uint64_t n,
                        uint64_t* out, uint64_t b) {
  KeyWords f[2];
  key_words_pair(tab, rk3, h, b, f[0], f[1]);
  for (int e = 0; e < 2; ++e) {
    uint64_t idx = 2 * b + e;
    if (idx >= n) break;
    for (int i = 0; i < 3; ++i) {
      uint64_t a = f[e].k[i], p = f[e].k[(i + 2) % 3];
      out[i * n + idx] = xor_mode ? (a ^ p) : (a - p);
    }
  }
}

// kind: 0 = mul, 1 = truncate, 2 = mul then truncate
template <class T>
HD void arith_item(const T& tab, const uint32_t* rk3, int kind, StreamHead ha, StreamHead hrho, StreamHead hr,
                   int bits, const uint64_t* x, const uint64_t* y, uint64_t* out, uint64_t n, uint64_t b,
                   uint64_t pb0 = 0) {
  // pb0: PRF block of local element 0 (a batch shard starts at an even global word)
  const uint64_t pb = pb0 + b;
  bool two = 2 * b + 1 < n;
  Trio v[2];
  v[0] = load_trio(x, n, 2 * b);
  v[1] = two ? load_trio(x, n, 2 * b + 1) : v[0];
  if (kind != 1) {
    Trio w[2];
    w[0] = load_trio(y, n, 2 * b);
    w[1] = two ? load_trio(y, n, 2 * b + 1) : w[0];
    KeyWords f0, f1;
    key_words_pair(tab, rk3, ha, pb, f0, f1);
    v[0] = trio_mul(v[0], w[0], f0);
    v[1] = trio_mul(v[1], w[1], f1);
  }
  if (kind != 0) {
    Word2 rho, r;
    trunc_words(tab, rk3, hrho, hr, pb, rho, r);
    v[0] = trio_truncate(v[0], rho.w0, r.w0, bits);
    v[1] = trio_truncate(v[1], rho.w1, r.w1, bits);
  }
  store_trio(out, n, 2 * b, v[0]);
  if (two) store_trio(out, n, 2 * b + 1, v[1]);
}

// plane: component stride of x / out / mask (0: n, the tensor is the whole
// range; a launch over a sub-range of a larger tensor passes the full plane).
template <class T>
HD void sign_item(const T& tab, const uint32_t* rk3, const SignStreams& st, int mode, const uint64_t* x,
                  uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total, uint64_t elem_off, uint64_t b,
                  uint64_t plane = 0) {
  const uint64_t pl = plane ? plane : n;
  bool two = 2 * b + 1 < n;
  Trio o[2], m[2];
  struct Loader {
    const uint64_t* x;
    uint64_t pl, e0;
    bool two;
    HD Trio operator()(int e) const { return load_trio(x, pl, (e && two) ? e0 + 1 : e0); }
  } ld{x, pl, 2 * b, two};
  sign_circuit_pair(tab, rk3, st, n_total, (elem_off >> 1) + b, mode, ld, o, m);
  store_trio(out, pl, 2 * b, o[0]);
  if (two) store_trio(out, pl, 2 * b + 1, o[1]);
  if (mode == MODE_RELU && mask) {
    store_trio(mask, pl, 2 * b, m[0]);
    if (two) store_trio(mask, pl, 2 * b + 1, m[1]);
  }
}

// One max_tree level (protocols.py:356-380) on rows of a (rows, m) trio
// tensor v: element f = (row, j), j < k = m / 2, is relu(v[row, 2j] -
// v[row, 2j+1]) with the relu's PRF words at flat index f of the (rows, k)
// difference tensor; the output max is v[row, 2j+1] + that relu, written to
// out[row, j] of the (rows, k + m % 2) result.
struct MaxGeom {
  uint64_t rows, m, k;
};
template <class T>
HD void maxlevel_item(const T& tab, const uint32_t* rk3, const SignStreams& st, const uint64_t* v, uint64_t* out,
                      const MaxGeom& g, uint64_t n, uint64_t n_total, uint64_t elem_off, uint64_t b) {
  const bool two = 2 * b + 1 < n;
  const uint64_t pv = g.rows * g.m, mo = g.k + (g.m & 1), po = g.rows * mo;
  struct Loader {
    const uint64_t* v;
    uint64_t pv, m, k, e0;
    bool two;
    HD Trio operator()(int e) const {
      const uint64_t f = (e && two) ? e0 + 1 : e0;
      const uint64_t row = f / k, j = f - row * k;
      const Trio a = load_trio(v, pv, row * m + 2 * j), c = load_trio(v, pv, row * m + 2 * j + 1);
      Trio d;
      for (int i = 0; i < 3; ++i) d.c[i] = a.c[i] - c.c[i];
      return d;
    }
  } ld{v, pv, g.m, g.k, 2 * b, two};
  Trio o[2], mk[2];
  sign_circuit_pair(tab, rk3, st, n_total, (elem_off >> 1) + b, MODE_RELU, ld, o, mk);
  for (int e = 0; e < (two ? 2 : 1); ++e) {
    const uint64_t f = 2 * b + e, row = f / g.k, j = f - row * g.k;
    const Trio c = load_trio(v, pv, row * g.m + 2 * j + 1);
    Trio r;
    for (int i = 0; i < 3; ++i) r.c[i] = c.c[i] + o[e].c[i];
    store_trio(out, po, row * mo + j, r);
  }
}

template <class T>
HD void inject_item(const T& tab, const uint32_t* rk3, StreamHead a0, StreamHead a1, const uint64_t* bits,
                    uint64_t* out, uint64_t n, uint64_t b, uint64_t pb0 = 0) {
  bool two = 2 * b + 1 < n;
  Trio v[2], o[2];
  v[0] = load_trio(bits, n, 2 * b);
  v[1] = two ? load_trio(bits, n, 2 * b + 1) : v[0];
  inject_pair(tab, rk3, a0, a1, pb0 + b, v, o);  // PRF block of the pair: shard offset + local pair
  store_trio(out, n, 2 * b, o[0]);
  if (two) store_trio(out, n, 2 * b + 1, o[1]);
}

struct View4 {
  int64_t full[4], org[4], crop[4], zs[4], os[4], zp, op;
  const uint64_t* bias;  // optional shared bias added after the truncation: bias[k * bias_plane + i_{bias_dim}]
  int64_t bias_plane;
  int bias_dim;
};

// A secure layer fused with the ReLU after it (protocols.py:120-136 then
// 334-353): the ReLU input x is the layer's cross terms z (View4 layout, no
// crop) reshared, truncated and biased in registers exactly as
// reshare_trunc_item does, from the pair's zero-share words kw (3 keys) and
// truncation words rho, r — so x never goes through HBM.
struct RsIn {
  const uint64_t* z;
  View4 v;
  int bits;
  uint64_t f0;  // flat index (in v) of the launch's element 0
  int small;    // the view's element count fits 32 bits
  const uint64_t* res;  // optional residual trio added after the bias (element f at res[k * res_plane + f])
  uint64_t res_plane;
};
template <class I>
HD void view_index(const View4& v, uint64_t f, int64_t& i0, int64_t& i1, int64_t& i2, int64_t& i3) {
  I q = (I)f;
  const I f3 = (I)v.full[3], f2 = (I)v.full[2], f1 = (I)v.full[1];
  i3 = (int64_t)(q % f3);
  q /= f3;
  i2 = (int64_t)(q % f2);
  q /= f2;
  i1 = (int64_t)(q % f1);
  i0 = (int64_t)(q / f1);
}
HD Trio reshare_input(const RsIn& in, uint64_t f, const uint64_t kw[3], uint64_t rho, uint64_t r) {
  const View4& v = in.v;
  int64_t i0, i1, i2, i3;
  if (in.small)  // every extent below 2^32: 32-bit divisions (short inline sequences)
    view_index<uint32_t>(v, f, i0, i1, i2, i3);
  else
    view_index<uint64_t>(v, f, i0, i1, i2, i3);
  Trio t = load_trio(in.z + i0 * v.zs[0] + i1 * v.zs[1] + i2 * v.zs[2] + i3 * v.zs[3], v.zp, 0);
  KeyWords w;
  for (int k = 0; k < 3; ++k) w.k[k] = kw[k];
  t = trio_reshare(t, w);
  if (in.bits) t = trio_truncate(t, rho, r, in.bits);
  if (v.bias) {
    const int64_t bi = v.bias_dim == 0 ? i0 : v.bias_dim == 1 ? i1 : v.bias_dim == 2 ? i2 : i3;
    for (int k = 0; k < 3; ++k) t.c[k] += v.bias[k * v.bias_plane + bi];
  }
  if (in.res)  // a residual block's shortcut, a local add before its ReLU
    for (int k = 0; k < 3; ++k) t.c[k] += in.res[k * in.res_plane + f];
  return t;
}

// sign_item on a fused layer output: w3 / rho / r are the pair's reshare and
// truncation words (block elem_off / 2 + b of each stream).
template <class T>
HD void sign_item_rs(const T& tab, const uint32_t* rk3, const SignStreams& st, int mode, const RsIn& in,
                     const Word2 w3[3], Word2 rho, Word2 r, uint64_t* out, uint64_t* mask, uint64_t n,
                     uint64_t n_total, uint64_t elem_off, uint64_t b, uint64_t plane) {
  const bool two = 2 * b + 1 < n;
  const uint64_t pl = plane ? plane : n;
  Trio xin[2];
  {
    const uint64_t k0[3] = {w3[0].w0, w3[1].w0, w3[2].w0}, k1[3] = {w3[0].w1, w3[1].w1, w3[2].w1};
    xin[0] = reshare_input(in, in.f0 + 2 * b, k0, rho.w0, r.w0);
    xin[1] = two ? reshare_input(in, in.f0 + 2 * b + 1, k1, rho.w1, r.w1) : xin[0];
  }
  struct Loader {
    const Trio* x;
    HD Trio operator()(int e) const { return x[e]; }
  } ld{xin};
  Trio o[2], m[2];
  sign_circuit_pair(tab, rk3, st, n_total, (elem_off >> 1) + b, mode, ld, o, m);
  store_trio(out, pl, 2 * b, o[0]);
  if (two) store_trio(out, pl, 2 * b + 1, o[1]);
  if (mode == MODE_RELU && mask) {
    store_trio(mask, pl, 2 * b, m[0]);
    if (two) store_trio(mask, pl, 2 * b + 1, m[1]);
  }
}

// I: index arithmetic type (uint32_t when every extent fits: the kernels pick
// it on the host, which turns the 64-bit division calls into short inline
// sequences).
template <class T, class I = uint64_t>
HD void reshare_trunc_item(const T& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho, StreamHead hr,
                           int bits, const uint64_t* z, const View4& v, uint64_t* out, uint64_t n, uint64_t b,
                           uint64_t pb0 = 0) {
  const uint64_t pb = pb0 + b;
  int64_t zoff[2] = {0, 0}, ooff[2] = {0, 0}, bidx[2] = {0, 0};
  bool ok[2];
  for (int e = 0; e < 2; ++e) {
    uint64_t f = 2 * b + e;
    ok[e] = f < n;
    I r = (I)f;
    const I f3 = (I)v.full[3], f2 = (I)v.full[2], f1 = (I)v.full[1];
    int64_t i3 = (int64_t)(r % f3);
    r /= f3;
    int64_t i2 = (int64_t)(r % f2);
    r /= f2;
    int64_t i1 = (int64_t)(r % f1);
    int64_t i0 = (int64_t)(r / f1);
    zoff[e] = i0 * v.zs[0] + i1 * v.zs[1] + i2 * v.zs[2] + i3 * v.zs[3];
    bidx[e] = v.bias_dim == 0 ? i0 : v.bias_dim == 1 ? i1 : v.bias_dim == 2 ? i2 : i3;
    i0 -= v.org[0];
    i1 -= v.org[1];
    i2 -= v.org[2];
    i3 -= v.org[3];
    ok[e] = ok[e] && i0 >= 0 && i1 >= 0 && i2 >= 0 && i3 >= 0 && i0 < v.crop[0] && i1 < v.crop[1] &&
            i2 < v.crop[2] && i3 < v.crop[3];
    ooff[e] = i0 * v.os[0] + i1 * v.os[1] + i2 * v.os[2] + i3 * v.os[3];
  }
  if (!ok[0] && !ok[1]) return;
  // the cross terms are loaded before the pair's AES blocks (their latency
  // hides the loads)
  Trio zt[2];
  for (int e = 0; e < 2; ++e)
    if (ok[e]) zt[e] = load_trio(z + zoff[e], v.zp, 0);
  KeyWords f0, f1;
  Word2 rho = {0, 0}, r = {0, 0};
  if (bits) {
    Word2 w[3];
    reshare_trunc_words(tab, rk3, ha, hrho, hr, pb, w, rho, r);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      f0.k[i] = w[i].w0;
      f1.k[i] = w[i].w1;
    }
  } else {
    key_words_pair(tab, rk3, ha, pb, f0, f1);
  }
  for (int e = 0; e < 2; ++e) {
    if (!ok[e]) continue;
    Trio t = trio_reshare(zt[e], e ? f1 : f0);
    if (bits) t = trio_truncate(t, e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, bits);
    if (v.bias) {  // local add of the bias shares (component-wise), as a separate add would
      for (int k = 0; k < 3; ++k) t.c[k] += v.bias[k * v.bias_plane + bidx[e]];
    }
    store_trio(out + ooff[e], v.op, 0, t);
  }
}

// Input gradient as GEMM + col2im (nn.py:460-484).  z holds, per party, the
// cross terms cols[(n,y,x), (c,a,b)] = sum_o g[n,o,y,x] k[o,c,a,b]; element
// (n, c, y', x') of the reference's full correlation output (N,C,hf,wf) is the
// sum of cols over the (a, b) with y' = y*sh + a, x' = x*sw + b (the
// transposed convolution), then reshared and truncated with PRF words at its
// flat index, and embedded at (y'-ph, x'-pw) if inside (H, W).
struct Col2Im {
  int64_t N, C, OH, OW, hf, wf, H, W;
  int kh, kw, sh, sw, ph, pw;
  int zcol;  // z column-major: cols[(n,y,x), (c,a,b)] at ((c*kh+a)*kw+b) * N*OH*OW + (n*OH+y)*OW + x
};

template <class T, class I = uint64_t>
HD void col2im_item(const T& tab, const uint32_t* rk3, StreamHead ha, StreamHead hrho, StreamHead hr, int bits,
                    const uint64_t* z, const Col2Im& g, uint64_t* out, uint64_t b, uint64_t pb0 = 0) {
  const uint64_t pb = pb0 + b;
  const uint64_t n_full = (uint64_t)g.N * g.C * g.hf * g.wf;
  const int64_t ncols = (int64_t)g.C * g.kh * g.kw;
  const int64_t zplane = (int64_t)g.N * g.OH * g.OW * ncols;
  const int64_t oplane = g.N * g.C * g.H * g.W;
  Trio s[2];
  int64_t ooff[2] = {-1, -1};
  for (int e = 0; e < 2; ++e) {
    uint64_t f = 2 * b + e;
    s[e].c[0] = s[e].c[1] = s[e].c[2] = 0;
    if (f >= n_full) continue;
    const I fi = (I)f, wf = (I)g.wf, hf = (I)g.hf, Cc = (I)g.C;
    const I q1 = fi / wf, q2 = q1 / hf;
    int64_t xq = (int64_t)(fi - q1 * wf), yq = (int64_t)(q1 - q2 * hf);
    int64_t c = (int64_t)(q2 % Cc), n = (int64_t)(q2 / Cc);
    int64_t yo = yq - g.ph, xo = xq - g.pw;
    if (yo < 0 || xo < 0 || yo >= g.H || xo >= g.W) continue;
    ooff[e] = ((n * g.C + c) * g.H + yo) * g.W + xo;
    // the (y, x) of the gradient whose window covers (yq, xq): yq = y*sh + a,
    // 0 <= a < kh, 0 <= y < OH (same for x); walked directly, no modulo tests
    const int32_t yqi = (int32_t)yq, xqi = (int32_t)xq, sh = g.sh, sw = g.sw;
    const int32_t y_hi = imin32(yqi / sh, (int32_t)g.OH - 1), x_hi = imin32(xqi / sw, (int32_t)g.OW - 1);
    const int32_t y_lo = yqi >= g.kh ? (yqi - g.kh + sh) / sh : 0, x_lo = xqi >= g.kw ? (xqi - g.kw + sw) / sw : 0;
    const int64_t mrows = g.N * g.OH * g.OW;
    for (int32_t y = y_lo; y <= y_hi; ++y) {
      const int32_t a = yqi - y * sh;
      for (int32_t x = x_lo; x <= x_hi; ++x) {
        const int32_t bb = xqi - x * sw;
        const int64_t zr = (n * g.OH + y) * g.OW + x, zc = (c * g.kh + a) * g.kw + bb;
        const int64_t zi = g.zcol ? zc * mrows + zr : zr * ncols + zc;
        for (int i = 0; i < 3; ++i) s[e].c[i] += z[i * zplane + zi];
      }
    }
  }
  if (ooff[0] < 0 && ooff[1] < 0) return;
  KeyWords f0, f1;
  Word2 rho, r, w[3];
  reshare_trunc_words(tab, rk3, ha, hrho, hr, pb, w, rho, r);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    f0.k[i] = w[i].w0;
    f1.k[i] = w[i].w1;
  }
  for (int e = 0; e < 2; ++e) {
    if (ooff[e] < 0) continue;
    Trio t = trio_reshare(s[e], e ? f1 : f0);
    t = trio_truncate(t, e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, bits);
    store_trio(out + ooff[e], oplane, 0, t);
  }
}

struct PoolGeom {
  int64_t N, C, H, W, OH, OW;
  int kh, kw, sh, sw;
  int ph, pw;  // zero padding (count_include_pad): the window area stays kh*kw
};

// fused window sum (x mulc) + truncate; backward = scatter-add then the same
template <class T, class I = uint64_t>
HD void pool_item(const T& tab, const uint32_t* rk3, bool backward, StreamHead hrho, StreamHead hr, int bits,
                  uint64_t mulc, const uint64_t* x, uint64_t* out, const PoolGeom& p, uint64_t b, uint64_t pb0 = 0,
                  const uint64_t* mask = nullptr, StreamHead ha = StreamHead{0, 0}) {
  const uint64_t pb = pb0 + b;
  uint64_t n = backward ? (uint64_t)p.N * p.C * p.H * p.W : (uint64_t)p.N * p.C * p.OH * p.OW;
  uint64_t nin = backward ? (uint64_t)p.N * p.C * p.OH * p.OW : (uint64_t)p.N * p.C * p.H * p.W;
  Trio s[2];
  for (int e = 0; e < 2; ++e) {
    uint64_t f = 2 * b + e;
    s[e].c[0] = s[e].c[1] = s[e].c[2] = 0;
    if (f >= n) continue;
    if (!backward) {
      const I fi = (I)f, q1 = fi / (I)p.OW;
      int64_t ox = (int64_t)(fi - q1 * (I)p.OW), oy = (int64_t)(q1 % (I)p.OH), nc = (int64_t)(q1 / (I)p.OH);
      const int32_t y0 = (int32_t)(oy * p.sh - p.ph), x0 = (int32_t)(ox * p.sw - p.pw);
      const int32_t H = (int32_t)p.H, W = (int32_t)p.W;
      const uint64_t* base = x + nc * p.H * p.W;
      for (int u = 0; u < p.kh; ++u) {
        const int32_t iy = y0 + u;
        if (iy < 0 || iy >= H) continue;
        for (int q = 0; q < p.kw; ++q) {
          const int32_t ix = x0 + q;
          if (ix < 0 || ix >= W) continue;
          for (int i = 0; i < 3; ++i) s[e].c[i] += base[i * nin + (uint64_t)(iy * W + ix)];
        }
      }
    } else {
      // windows (oy, ox) with oy*sh - ph <= iy < oy*sh - ph + kh, oy < OH (nn.py:487-499)
      const I fi = (I)f, q1 = fi / (I)p.W;
      int64_t ix = (int64_t)(fi - q1 * (I)p.W) + p.pw, iy = (int64_t)(q1 % (I)p.H) + p.ph,
              nc = (int64_t)(q1 / (I)p.H);
      const int32_t iyi = (int32_t)iy, ixi = (int32_t)ix, sh = p.sh, sw = p.sw;
      const uint64_t gbase = (uint64_t)nc * p.OH * p.OW;
      for (int32_t oy = iyi / sh; oy >= 0 && oy * sh + p.kh > iyi; --oy) {
        if (oy >= p.OH) continue;
        for (int32_t ox = ixi / sw; ox >= 0 && ox * sw + p.kw > ixi; --ox) {
          if (ox >= p.OW) continue;
          const uint64_t gi = gbase + (uint64_t)oy * p.OW + ox;
          for (int i = 0; i < 3; ++i) s[e].c[i] += x[i * nin + gi];
        }
      }
    }
    for (int i = 0; i < 3; ++i) s[e].c[i] *= mulc;
  }
  Word2 rho, r;
  if (!mask) {
    trunc_words(tab, rk3, hrho, hr, pb, rho, r);
    for (int e = 0; e < 2; ++e) {
      uint64_t f = 2 * b + e;
      if (f >= n) break;
      store_trio(out, n, f, trio_truncate(s[e], e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, bits));
    }
    return;
  }
  // backward through the ReLU before the pool in the same pass: the truncated
  // gradient times the ReLU's mask, reshared with ARITH_ZERO words (the
  // "mul.mask" of nn.py:515-517) — five AES blocks per pair in one call
  Word2 w[3];
  reshare_trunc_words(tab, rk3, ha, hrho, hr, pb, w, rho, r);
  for (int e = 0; e < 2; ++e) {
    uint64_t f = 2 * b + e;
    if (f >= n) break;
    const Trio t = trio_truncate(s[e], e ? rho.w1 : rho.w0, e ? r.w1 : r.w0, bits);
    KeyWords kw;
    for (int i = 0; i < 3; ++i) kw.k[i] = e ? w[i].w1 : w[i].w0;
    store_trio(out, n, f, trio_mul(t, load_trio(mask, n, f), kw));
  }
}

// packing item: 8 consecutive kk of one (g, r) -> one u64 per limb plane
// kh: packed column of the second half's first element (K for the adjacent
// [first | second] layout; larger leaves zero columns [K, kh) between them).
HD void pack_item(const uint64_t* src, int64_t plane, const Operand& o, int role, uint8_t* out, int64_t kp,
                  int64_t t, int64_t kh) {
  int64_t chunks = kp / 8;
  int64_t ch = t % chunks;
  int64_t q = t / chunks;
  int64_t r = q % o.rows;
  int g = (int)(q / o.rows);
  uint64_t v[8];
  // role 3: component planes (plane g = x_g, no halves) — the role-1 operand
  // [x_g | x_{g+1}] stored once per component, its halves read from planes g, g+1
  const int64_t K = o.k, lim = role >= 2 ? K : kh + K;
  const int gn = (g + 1) % 3;
  GatherCursor cur;
  int half = -1;
  for (int e = 0; e < 8; ++e) {
    int64_t kk = ch * 8 + e;
    if (kk >= lim) {
      v[e] = 0;
      continue;
    }
    int h = (role < 2 && kk >= kh) ? 1 : 0;
    if (h == 0 && kk >= K) {  // gap between the halves
      v[e] = 0;
      continue;
    }
    if (h != half) {  // (re)start the cursor at this half's first k
      cur.init(o, r, h ? kk - kh : kk);
      half = h;
    }
    int64_t off = cur.offset(o);
    uint64_t val = 0;
    if (off >= 0) {
      if (role == 2) {
        val = src[off];
      } else if (role == 3) {
        val = src[g * plane + off];
      } else {
        uint64_t self = src[g * plane + off], nxt = src[gn * plane + off];
        val = role == 0 ? (h == 0 ? self + nxt : self) : (h == 0 ? self : nxt);  // protocols.py:110-115
      }
    }
    v[e] = val;
    cur.next(o);
  }
  uint8_t* base = out + ((int64_t)g * 8 * o.rows + r) * kp + ch * 8;
  uint64_t w[8];
  byte_transpose8(v, w);  // w[l] byte e = byte l of v[e]
  for (int l = 0; l < 8; ++l) *reinterpret_cast<uint64_t*>(base + (int64_t)l * o.rows * kp) = w[l];
}

#if defined(__CUDACC__)
// Lane3 forms of sign_item / sign_item_rs / maxlevel_item for the two-phase
// kernels' circuit phase: every lane of a group builds the pair's input
// trios, lane i stores component i; `live` false (padding lanes, pairs past
// the chunk) runs the circuit (the shuffles need every lane) without stores.
DEV void store_lane(uint64_t* p, uint64_t plane, uint64_t e, int i, uint64_t v) { p[i * plane + e] = v; }

DEV void sign_item_lane(const Lane3& L, int mode, const uint64_t* x, uint64_t* out, uint64_t* mask, uint64_t n,
                        uint64_t n_total, uint64_t b, uint64_t plane, bool live) {
  const uint64_t pl = plane ? plane : n;
  const bool two = 2 * b + 1 < n;
  Trio xin[2];
  xin[0] = load_trio(x, pl, 2 * b);
  xin[1] = two ? load_trio(x, pl, 2 * b + 1) : xin[0];
  uint64_t o[2], m[2];
  sign_circuit_lane(L, n_total, mode, xin, o, m);
  if (!live) return;
  store_lane(out, pl, 2 * b, L.i, o[0]);
  if (two) store_lane(out, pl, 2 * b + 1, L.i, o[1]);
  if (mode == MODE_RELU && mask) {
    store_lane(mask, pl, 2 * b, L.i, m[0]);
    if (two) store_lane(mask, pl, 2 * b + 1, L.i, m[1]);
  }
}

DEV void sign_item_rs_lane(const Lane3& L, int mode, const RsIn& in, const Word2 w3[3], Word2 rho, Word2 r,
                           uint64_t* out, uint64_t* mask, uint64_t n, uint64_t n_total, uint64_t b, uint64_t plane,
                           bool live) {
  const bool two = 2 * b + 1 < n;
  const uint64_t pl = plane ? plane : n;
  Trio xin[2];
  {
    const uint64_t k0[3] = {w3[0].w0, w3[1].w0, w3[2].w0}, k1[3] = {w3[0].w1, w3[1].w1, w3[2].w1};
    xin[0] = reshare_input(in, in.f0 + 2 * b, k0, rho.w0, r.w0);
    xin[1] = two ? reshare_input(in, in.f0 + 2 * b + 1, k1, rho.w1, r.w1) : xin[0];
  }
  uint64_t o[2], m[2];
  sign_circuit_lane(L, n_total, mode, xin, o, m);
  if (!live) return;
  store_lane(out, pl, 2 * b, L.i, o[0]);
  if (two) store_lane(out, pl, 2 * b + 1, L.i, o[1]);
  if (mode == MODE_RELU && mask) {
    store_lane(mask, pl, 2 * b, L.i, m[0]);
    if (two) store_lane(mask, pl, 2 * b + 1, L.i, m[1]);
  }
}

DEV void maxlevel_item_lane(const Lane3& L, const uint64_t* v, uint64_t* out, const MaxGeom& g, uint64_t n,
                            uint64_t n_total, uint64_t b, bool live) {
  const bool two = 2 * b + 1 < n;
  const uint64_t pv = g.rows * g.m, mo = g.k + (g.m & 1), po = g.rows * mo;
  Trio d[2];
  uint64_t c[2];  // component i of the odd column (the max = it + relu(difference))
  for (int e = 0; e < 2; ++e) {
    const uint64_t f = (e && two) ? 2 * b + 1 : 2 * b, row = f / g.k, j = f - row * g.k;
    const Trio a = load_trio(v, pv, row * g.m + 2 * j), cc = load_trio(v, pv, row * g.m + 2 * j + 1);
    for (int k = 0; k < 3; ++k) d[e].c[k] = a.c[k] - cc.c[k];
    c[e] = comp(cc, L.i);
  }
  uint64_t o[2], mk[2];
  sign_circuit_lane(L, n_total, MODE_RELU, d, o, mk);
  if (!live) return;
  for (int e = 0; e < (two ? 2 : 1); ++e) {
    const uint64_t f = 2 * b + e, row = f / g.k, j = f - row * g.k;
    store_lane(out, po, row * mo + j, L.i, c[e] + o[e]);
  }
}

// The group geometry of a lane in a CTA of whole warps: 10 groups of three
// lanes per warp (lanes 30 and 31 pad); group q of warp w handles the
// chunk's pairs w * 10 + q, + 10 * warps, ...
struct LaneGroup {
  int gi, ci, nl, pl;
};
DEV LaneGroup lane_group() {
  const int lane = threadIdx.x & 31;
  LaneGroup G;
  G.gi = lane < 30 ? lane / 3 : 10;
  G.ci = lane < 30 ? lane % 3 : lane - 30;
  const int base = lane - G.ci;
  G.nl = (base + (G.ci == 2 ? 0 : G.ci + 1)) & 31;
  G.pl = (base + (G.ci == 0 ? 2 : G.ci - 1)) & 31;
  return G;
}
#endif

}  // namespace mpc3
