"""CPU build of the device logic (items.cuh / protocol.cuh / aes.cuh) against the oracle.

The exact per-element code the CUDA kernels run is compiled with g++ into
libmpc3hostcheck.so (test infrastructure) and compared bit-for-bit with the
oracle, which is itself pinned to the reference (test_oracle.py).
"""

import os

import numpy as np
import pytest

import hostcheck as H
from oracle import nnmirror as N
from oracle import rss as R
from paper_2104_10949_b200 import _capi

pytestmark = pytest.mark.skipif(not os.path.exists(H.PATH), reason="hostcheck library not built")
U64 = np.uint64


def rnd(rng, shape):
    return rng.integers(0, 1 << 64, size=shape, dtype=U64)


@pytest.mark.parametrize("purpose,index,off,count", [(1, 0, 0, 4), (2, 5, 3, 17), (5, (1 << 48) - 1, 1, 1),
                                                     (4, 123456, 0, 33), (3, 7, 10, 0)])
def test_prf_words(purpose, index, off, count):
    key = R.party_keys(3)[1]
    ref = R.prf_words(key, purpose, index, off + count)[off:]
    assert np.array_equal(H.prf_words(key, purpose, index, off, count), ref)


def test_prf_kat():
    got = H.prf_words(bytes(range(16)), 1, 0, 0, 4)
    assert [hex(int(v)) for v in got] == ["0xa0877cdd63d37ce3", "0x829ce0603e0eff9a",
                                          "0x19ff076bfae7e67f", "0x62f3c9d7c774a10d"]


@pytest.mark.parametrize("xor_mode", [0, 1])
@pytest.mark.parametrize("n", [1, 8, 9])
def test_zero_share(xor_mode, n):
    s = R.Session(2)
    s.seq[2 if xor_mode else 1] = 4
    ref = R.zero_share(s, 2 if xor_mode else 1, (n,), xor=bool(xor_mode))
    assert np.array_equal(H.zero_share(s.keys, 2 if xor_mode else 1, 4, xor_mode, n), ref)


@pytest.mark.parametrize("n", [1, 2, 7, 64])
def test_mul_truncate(n):
    rng = np.random.default_rng(n)
    x, y = rnd(rng, (3, n)), rnd(rng, (3, n))
    s = R.Session(5)
    assert np.array_equal(H.arith(s.keys, 0, 0, 0, 0, 0, x, y), R.mul(s, x, y))
    v = rng.integers(-(1 << 61), 1 << 61, n, dtype=np.int64).view(U64)
    xs = R.share(v, rng)
    for bits in (1, 20, 61):
        s = R.Session(5)
        assert np.array_equal(H.arith(s.keys, 1, 0, 0, 0, bits, xs), R.truncate(s, xs, bits))
    a = R.share(R.fx_encode(rng.uniform(-4, 4, n)), rng)
    b = R.share(R.fx_encode(rng.uniform(-4, 4, n)), rng)
    s = R.Session(6)
    ref = R.truncate(s, R.mul(s, a, b))
    assert np.array_equal(H.arith(s.keys, 2, 0, 0, 0, 20, a, b), ref)


@pytest.mark.parametrize("n", [1, 2, 5, 64, 101])
def test_sign_circuit_modes(n):
    rng = np.random.default_rng(100 + n)
    edges = np.array([0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1], U64)
    x = np.concatenate([edges, rnd(rng, n)])[:n]
    xs = R.share(x, rng)
    keys = R.Session(9).keys
    s = R.Session(9)
    assert np.array_equal(H.sign(keys, 0, 0, 0, 0, xs)[0], R.a2b(s, xs))
    s = R.Session(9)
    assert np.array_equal(H.sign(keys, 1, 0, 0, 0, xs)[0], R.msb(s, xs))
    s = R.Session(9)
    assert np.array_equal(H.sign(keys, 2, 0, 0, 0, xs)[0], R.drelu(s, xs))
    s = R.Session(9)
    out, mask = H.sign(keys, 3, 0, 0, 0, xs)
    ro, rm = R.relu_with_mask(s, xs)
    assert np.array_equal(out, ro) and np.array_equal(mask, rm)


@pytest.mark.parametrize("n,cut", [(10, 4), (11, 6), (64, 32)])
def test_sign_circuit_shards_match_whole(n, cut):
    rng = np.random.default_rng(n)
    xs = R.share(rnd(rng, n), rng)
    keys = R.Session(1).keys
    whole, wm = H.sign(keys, 3, 2, 3, 4, xs)
    a, am = H.sign(keys, 3, 2, 3, 4, xs[:, :cut], n_total=n, off=0)
    b, bm = H.sign(keys, 3, 2, 3, 4, xs[:, cut:], n_total=n, off=cut)
    assert np.array_equal(np.concatenate([a, b], axis=1), whole)
    assert np.array_equal(np.concatenate([am, bm], axis=1), wm)


def test_bit_inject():
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, (3, 33), dtype=U64)
    s = R.Session(4)
    assert np.array_equal(H.inject(s.keys, 0, bits), R.bit_inject(s, bits))


def _cross(x, y):
    return np.stack([x[i] @ y[i] for i in range(3)])


def test_pack_gemm_matmul_reshare_truncate():
    rng = np.random.default_rng(11)
    M, K, Nn = 9, 33, 7
    x = R.share(R.fx_encode(rng.uniform(-4, 4, (M, K))), rng)
    y = R.share(R.fx_encode(rng.uniform(-4, 4, (K, Nn))), rng)
    kp = (2 * K + 15) // 16 * 16
    A = H.pack(x, M * K, _capi.dense_operand(M, K, s_r=K, t2=1), 0, kp)
    B = H.pack(y, K * Nn, _capi.dense_operand(Nn, K, s_r=1, t2=Nn), 1, kp)
    z = H.gemm_packed(A, B)
    ref_z = R._bilinear3(R.wrap_matmul, x, y)
    assert np.array_equal(z, ref_z)
    s = R.Session(7)
    ref = R.truncate(s, R.reshare(s, ref_z))
    view = _capi.make_view((1, 1, M, Nn))
    got = H.reshare_truncate(s.keys, 0, 0, 0, 20, z, view, (3, M, Nn))
    assert np.array_equal(got, ref)
    # split-K emulation equals the single-pass result
    assert np.array_equal(H.gemm_packed(A, B, split_k=32), z)


def test_plain_matmul_pack_extremes():
    rng = np.random.default_rng(12)
    a = np.full((5, 300), (1 << 64) - 1, U64)
    b = rnd(rng, (300, 4))
    kp = (300 + 15) // 16 * 16
    A = H.pack(a, 0, _capi.dense_operand(5, 300, s_r=300, t2=1), 2, kp)
    B = H.pack(b, 0, _capi.dense_operand(4, 300, s_r=1, t2=4), 2, kp)
    assert np.array_equal(H.gemm_packed(A, B)[0], R.wrap_matmul(a, b))


@pytest.mark.parametrize("geom", [((2, 3, 10, 10), (4, 3, 3, 3), (2, 2), (1, 1)),
                                  ((1, 3, 16, 16), (8, 3, 11, 11), (4, 4), (0, 0)),
                                  ((2, 2, 9, 7), (3, 2, 5, 2), (1, 2), (2, 0))])
def test_conv_fwd_wgrad_dgrad_products(geom):
    xs_, ks_, st, pd = geom
    rng = np.random.default_rng(sum(xs_))
    n, c, h, w = xs_
    o, _, kh, kw = ks_
    oh, ow = R.conv_out_hw(h, w, kh, kw, st, pd)
    x = rnd(rng, (3,) + xs_)
    k = rnd(rng, (3,) + ks_)
    # forward: A = im2col(x) rows (n,y,x) k (c,u,v); B = k rows o
    K = c * kh * kw
    kp = (2 * K + 15) // 16 * 16
    A = H.pack(x, x[0].size, _capi.conv_operand(_capi.GATHER_IM2COL, n * oh * ow, K, n, c, h, w,
                                                (c * h * w, h * w, w, 1), kh, kw, st[0], st[1], pd[0], pd[1], oh, ow), 0, kp)
    B = H.pack(k, k[0].size, _capi.dense_operand(o, K, s_r=K, t2=1), 1, kp)
    z = H.gemm_packed(A, B).reshape(3, n, oh, ow, o).transpose(0, 1, 4, 2, 3)
    ref = R._bilinear3(lambda a, b: R.wrap_conv2d(a, b, st, pd), x, k)
    assert np.array_equal(z, ref)
    # weight gradient: rows (c,u,v), k (n,y,x), against the reference's dilated form
    g = rnd(rng, (3, n, o, oh, ow))
    Kw = n * oh * ow
    kp = (2 * Kw + 15) // 16 * 16
    A = H.pack(x, x[0].size, _capi.conv_operand(_capi.GATHER_WGRAD, c * kh * kw, Kw, n, c, h, w,
                                                (c * h * w, h * w, w, 1), kh, kw, st[0], st[1], pd[0], pd[1], oh, ow), 0, kp)
    B = H.pack(g, g[0].size, _capi.dense_operand(o, Kw, s_r=oh * ow, t0=o * oh * ow, t1=ow, t2=1, K1=oh, K2=ow), 1, kp)
    zw = H.gemm_packed(A, B).reshape(3, c, kh, kw, o).transpose(0, 4, 1, 2, 3)

    class Raw:
        t = 20

        def shape(self, v):
            return v.shape[1:]

        def map_structural(self, v, f):
            return np.stack([f(v[i]) for i in range(3)])

        def conv2d(self, a, b, stride, padding, bits=None):
            return R._bilinear3(lambda p, q: R.wrap_conv2d(p, q, stride, padding), a, b)

    L = N.conv(o, (kh, kw), st, pd)
    assert np.array_equal(zw, N.conv_grad_kernel(Raw(), x, g, L, 20))
    # input gradient: dilated/padded g correlated with the flipped kernel
    hf, wf = (oh - 1) * st[0] + kh, (ow - 1) * st[1] + kw
    Kd = o * kh * kw
    kp = (2 * Kd + 15) // 16 * 16
    A = H.pack(g, g[0].size, _capi.conv_operand(_capi.GATHER_IM2COL, n * hf * wf, Kd, n, o, oh, ow,
                                                (o * oh * ow, oh * ow, ow, 1), kh, kw, 1, 1, kh - 1, kw - 1, hf, wf,
                                                dh=st[0], dw=st[1]), 0, kp)
    B = H.pack(k, k[0].size, _capi.dense_operand(c, Kd, s_r=kh * kw, off=(kh - 1) * kw + kw - 1, t0=c * kh * kw,
                                                 t1=-kw, t2=-1, K1=kh, K2=kw), 1, kp)
    zd = H.gemm_packed(A, B).reshape(3, n, hf, wf, c).transpose(0, 1, 4, 2, 3)
    gp = np.stack([np.pad(N.dilate(g[i], st), ((0, 0), (0, 0), (kh - 1, kh - 1), (kw - 1, kw - 1))) for i in range(3)])
    kf = np.stack([k[i].transpose(1, 0, 2, 3)[:, :, ::-1, ::-1] for i in range(3)])
    assert np.array_equal(zd, R._bilinear3(lambda p, q: R.wrap_conv2d(p, q), gp, kf))


@pytest.mark.parametrize("win,stride,shape", [((2, 2), (2, 2), (1, 2, 6, 6)), ((3, 3), (2, 2), (2, 3, 9, 8)),
                                              ((2, 2), (1, 1), (1, 2, 5, 5)), ((3, 3), (3, 3), (1, 1, 9, 9))])
def test_avgpool_forward_backward(win, stride, shape):
    rng = np.random.default_rng(21)
    x = R.share(R.fx_encode(rng.uniform(-4, 4, shape)), rng)
    nb, c, h, w = shape
    oh, ow = (h - win[0]) // stride[0] + 1, (w - win[1]) // stride[1] + 1
    area = win[0] * win[1]
    pow2 = area & (area - 1) == 0
    bits = area.bit_length() - 1 if pow2 else 20
    mulc = 1 if pow2 else int(R.fx_encode(1.0 / area))
    s = R.Session(3)
    ref = R.avgpool_shares(s, x, win, stride)
    got = H.pool(s.keys, 0, 0, 0, bits, mulc, x, nb, c, h, w, oh, ow, win[0], win[1], stride[0], stride[1])
    assert np.array_equal(got.reshape(ref.shape), ref)
    g = R.share(R.fx_encode(rng.uniform(-1, 1, (nb, c, oh, ow))), rng)
    s = R.Session(3)
    ref = N.avgpool_backward(N.TrioEngine(s), g, win, stride, shape)
    got = H.pool(s.keys, 1, 0, 0, bits, mulc, g, nb, c, h, w, oh, ow, win[0], win[1], stride[0], stride[1])
    assert np.array_equal(got.reshape(ref.shape), ref)


@pytest.mark.parametrize("geom", [((2, 3, 10, 10), (4, 3, 3, 3), (2, 2), (1, 1)),
                                  ((2, 4, 4, 4), (6, 4, 5, 5), (1, 1), (1, 1)),
                                  ((1, 3, 32, 32), (8, 3, 11, 11), (4, 4), (9, 9)),
                                  ((2, 2, 9, 7), (3, 2, 5, 2), (1, 2), (2, 0))])
def test_dgrad_gemm_col2im_matches_reference_schedule(geom):
    """Input gradient via cols = g-rows x k (inner length O) + col2im equals the
    reference's correlation of the dilated/padded gradient with the flipped
    kernel, including reshare + truncate words and the embed."""
    xs_, ks_, st, pd = geom
    rng = np.random.default_rng(sum(xs_) + 1)
    n, c, h, w = xs_
    o, _, kh, kw = ks_
    oh, ow = R.conv_out_hw(h, w, kh, kw, st, pd)
    g = R.share(R.fx_encode(rng.uniform(-1, 1, (n, o, oh, ow))), rng)
    k = R.share(R.fx_encode(rng.uniform(-0.5, 0.5, ks_)), rng)
    s = R.Session(4)
    ref = N.conv_grad_input(N.TrioEngine(s), g, k, N.conv(o, (kh, kw), st, pd), (n, c, h, w), 20)
    ncols = c * kh * kw
    kp = (2 * o + 15) // 16 * 16
    A = H.pack(g, g[0].size, _capi.conv_operand(_capi.GATHER_IM2COL, n * oh * ow, o, n, o, oh, ow,
                                                (o * oh * ow, oh * ow, ow, 1), 1, 1, 1, 1, 0, 0, oh, ow), 0, kp)
    B = H.pack(k, k[0].size, _capi.dense_operand(ncols, o, s_r=1, t2=ncols), 1, kp)
    z = H.gemm_packed(A, B)
    got = H.col2im(R.Session(4).keys, 0, 0, 0, 20, z, n, c, oh, ow, kh, kw, st[0], st[1], pd[0], pd[1], h, w)
    assert np.array_equal(got, ref)


def _mn_to_kmajor(src, half, n, kc_half):
    """K-major packed operand equivalent to reading the packed buffer `src`
    ([g][8][rows][kp]) transposed, as mpc3_ring_gemm_t's MN operands do:
    element (j, h * kc_half + r) = src[..., r, h * half + j]."""
    g, _, rows, kp = src.shape
    out = np.zeros((g, 8, n, 2 * kc_half), np.uint8)
    for h in range(2):
        cols = np.arange(n) + h * half
        ok = cols < kp
        blk = np.zeros((g, 8, rows, n), np.uint8)
        blk[..., ok] = src[..., cols[ok]]
        out[..., h * kc_half:h * kc_half + rows] = blk.transpose(0, 1, 3, 2)
    return out


@pytest.mark.parametrize("Rn,O,Kc", [(50, 7, 20), (64, 16, 33)])
def test_pack_halves_and_transposed_gemm_semantics(Rn, O, Kc):
    """Packs with the second half at a 16-aligned column (zero gap) give the
    same cross terms, and reading the role-0 pack of g and the role-1 pack of
    x transposed (the weight-gradient GEMM mpc3_ring_gemm_t) gives
    dW[g] = (g_g + g_{g+1})^T x_g + g_g^T x_{g+1}."""
    rng = np.random.default_rng(Rn * O)
    gt = rng.integers(0, 1 << 64, size=(3, Rn, O), dtype=np.uint64)
    xt = rng.integers(0, 1 << 64, size=(3, Rn, Kc), dtype=np.uint64)
    kha, khb = (O + 15) // 16 * 16, (Kc + 15) // 16 * 16
    kpa, kpb = (kha + O + 15) // 16 * 16, (khb + Kc + 15) // 16 * 16
    A = H.pack(gt, Rn * O, _capi.dense_operand(Rn, O, s_r=O, t2=1), 0, kpa, kha)
    B = H.pack(xt, Rn * Kc, _capi.dense_operand(Rn, Kc, s_r=Kc, t2=1), 1, kpb, khb)
    assert not A[..., O:kha].any() and not B[..., Kc:khb].any()
    Aadj = H.pack(gt, Rn * O, _capi.dense_operand(Rn, O, s_r=O, t2=1), 0, (2 * O + 15) // 16 * 16)
    assert np.array_equal(A[..., kha:kha + O], Aadj[..., O:2 * O]) and np.array_equal(A[..., :O], Aadj[..., :O])
    kc_half = (Rn + 31) // 32 * 32
    z = H.gemm_packed(_mn_to_kmajor(A, kha, O, kc_half), _mn_to_kmajor(B, khb, Kc, kc_half))
    for g in range(3):
        h = (g + 1) % 3
        want = R.wrap_matmul(gt[g].T + gt[h].T, xt[g]) + R.wrap_matmul(gt[g].T, xt[h])
        assert np.array_equal(z[g], want)


def test_gemm_t_rejects_unaligned_half():
    import ctypes as C

    lib = _capi.lib()
    nul = C.c_void_p(0)
    # MN operand whose half offset is not a 16-byte TMA granule
    assert lib.mpc3_ring_gemm_t(nul, 1, 64, 160, 70, nul, 1, 64, 160, 64, nul, 3, 70, 64, 64, 0, nul) == \
        2  # MPC3_ERR_SHAPE
    # K-major partner must hold the halves at kc_half
    assert lib.mpc3_ring_gemm_t(nul, 1, 64, 160, 80, nul, 0, 64, 96, 0, nul, 3, 70, 64, 64, 0, nul) == \
        2  # MPC3_ERR_SHAPE


def test_gemm_needs_zero_plan():
    """mpc3_ring_gemm_needs_zero (host-only planner): C must be zeroed exactly
    when the launch accumulates atomically — split-K beyond the 16384-K
    exactness bound, or a contraction short enough to split for occupancy."""
    lib = _capi.lib()
    assert lib.mpc3_ring_gemm_needs_zero(0, 3, 4096, 4096, 1024) == 0  # many tiles, one split
    assert lib.mpc3_ring_gemm_needs_zero(0, 1, 128, 64, 40000) == 1   # exactness split
    assert lib.mpc3_ring_gemm_needs_zero(1, 3, 256, 256, 2 * 4096) == 1  # few tiles, long K: occupancy split
    assert lib.mpc3_ring_gemm_needs_zero(1, 3, 0, 256, 64) == 0
    assert lib.mpc3_ring_gemm_needs_zero(0, 0, 1, 1, 16) == 2  # MPC3_ERR_SHAPE
