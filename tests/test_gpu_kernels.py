"""Device kernels through the C ABI vs the oracle (needs a B200)."""

import ctypes as C

import numpy as np
import pytest

from oracle import nnmirror as N
from oracle import rss as R

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2104_10949_b200 import _capi  # noqa: E402

U64 = np.uint64


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, U64).view(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(U64)


_PINNED = []


def p(t):
    # keep temporaries alive: a freed block could be handed to the next
    # argument's allocation before the launch reads it
    _PINNED.append(t)
    if len(_PINNED) > 64:
        del _PINNED[:32]
    return C.c_void_p(t.data_ptr())


def rk3(keys):
    rk = np.zeros((3, 44), np.uint32)
    for i, k in enumerate(keys):
        _capi.check(_capi.lib().mpc3_aes128_expand(C.c_char_p(k), rk[i].ctypes.data_as(C.c_void_p)))
    return torch.from_numpy(rk.view(np.int32)).cuda()


S = None


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def rnd(rng, shape):
    return rng.integers(0, 1 << 64, size=shape, dtype=U64)


def test_library_loads_and_abi():
    assert _capi.lib().mpc3_abi_version() == 1
    cap = torch.cuda.get_device_capability()
    assert cap[0] == 10, cap


@pytest.mark.parametrize("purpose,index,off,count", [(1, 0, 0, 4), (2, 5, 3, 17), (5, (1 << 48) - 1, 1, 1),
                                                     (4, 123456, 0, 100001)])
def test_prf_words(purpose, index, off, count):
    keys = R.party_keys(3)
    rk = rk3(keys)
    out = torch.zeros(count, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_prf_words", C.c_void_p(rk.data_ptr() + 44 * 4), purpose, index, off, count, p(out), stream())
    ref = R.prf_words(keys[1], purpose, index, off + count)[off:]
    assert np.array_equal(host(out), ref)


# counter-mode constants (aes.cuh aes128_ctr): blocks below 4 x 2^24 start
# at round 3 (per-top-byte constants), other blocks below 2^32 at round 2,
# the rest run all rounds; these offsets straddle every boundary (words
# 2^25, 2^27 and 2^33)
@pytest.mark.parametrize("purpose,index,off,count", [(1, 3, (1 << 25) - 37, 80), (4, 1, (1 << 27) - 37, 80),
                                                     (2, 9, (1 << 33) - 37, 80),
                                                     (5, 77, (1 << 40) + 1, 33), (3, 0, (1 << 24) + 5, 4099)])
def test_prf_words_far_offsets(purpose, index, off, count):
    keys = R.party_keys(4)
    rk = rk3(keys)
    out = torch.zeros(count, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_prf_words", C.c_void_p(rk.data_ptr() + 44 * 8), purpose, index, off, count, p(out), stream())
    ref = R.prf_words_at(keys[2], purpose, index, off, count)
    assert np.array_equal(host(out), ref)


def test_prf_range_errors():
    rk = rk3(R.party_keys(0))
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    with pytest.raises(_capi.E.RangeError):
        _capi.call("mpc3_prf_words", p(rk), 1 << 16, 0, 0, 4, p(out), stream())
    with pytest.raises(_capi.E.RangeError):
        _capi.call("mpc3_prf_words", p(rk), 1, 1 << 48, 0, 4, p(out), stream())


@pytest.mark.parametrize("n", [1, 2, 7, 1 << 16, (1 << 16) + 3])
def test_mul_truncate(n):
    rng = np.random.default_rng(n)
    x, y = R.share(rnd(rng, n), rng), R.share(rnd(rng, n), rng)
    s = R.Session(5)
    rk = rk3(s.keys)
    out = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_mul", p(rk), None, 0, p(dev(x)), p(dev(y)), p(out), n, 0, stream())
    assert np.array_equal(host(out).reshape(3, n), R.mul(s, x, y))
    v = R.share(rng.integers(-(1 << 61), 1 << 61, n, dtype=np.int64).view(U64), rng)
    for bits in (1, 20, 61):
        s = R.Session(5)
        _capi.call("mpc3_rss_truncate", p(rk), None, 0, 0, bits, p(dev(v)), p(out), n, 0, stream())
        assert np.array_equal(host(out).reshape(3, n), R.truncate(s, v, bits))
    with pytest.raises(_capi.E.RangeError):
        _capi.call("mpc3_rss_truncate", p(rk), None, 0, 0, 62, p(dev(v)), p(out), n, 0, stream())


@pytest.mark.parametrize("n", [5, 101, 4096, 100003])
def test_sign_modes(n):
    rng = np.random.default_rng(n)
    edges = np.array([0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1], U64)
    x = np.concatenate([edges, rnd(rng, n)])[:n]
    xs = R.share(x, rng)
    keys = R.Session(9).keys
    rk = rk3(keys)
    xd = dev(xs)
    out = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    mask = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    for mode, fn in [(0, R.a2b), (1, R.msb), (2, R.drelu)]:
        _capi.call("mpc3_rss_sign", p(rk), None, mode, 0, 0, 0, p(xd), p(out), p(mask), n, n, 0, stream())
        assert np.array_equal(host(out).reshape(3, n), fn(R.Session(9), xs)), mode
    _capi.call("mpc3_rss_sign", p(rk), None, 3, 0, 0, 0, p(xd), p(out), p(mask), n, n, 0, stream())
    ro, rm = R.relu_with_mask(R.Session(9), xs)
    assert np.array_equal(host(out).reshape(3, n), ro)
    assert np.array_equal(host(mask).reshape(3, n), rm)


# one persistent round = 148 x 384 pairs; a remainder of >= 72 % of a round
# takes one more persistent round, below that the two-phase kernel
# (elementwise.cu sign_launch): sizes either side of both policies' edges
@pytest.mark.parametrize("n", [81836, 81841, 113664 + 81836, 113664 + 81843])
def test_relu_partial_round_edges_vs_oracle(n):
    rng = np.random.default_rng(n)
    xs = R.share(rnd(rng, n), rng)
    rk = rk3(R.Session(10).keys)
    out = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    mask = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_sign", p(rk), None, 3, 0, 0, 0, p(dev(xs)), p(out), p(mask), n, n, 0, stream())
    ro, rm = R.relu_with_mask(R.Session(10), xs)
    assert np.array_equal(host(out).reshape(3, n), ro)
    assert np.array_equal(host(mask).reshape(3, n), rm)


@pytest.mark.parametrize("n", [600000, 600001])
def test_sign_single_phase_equals_two_phase_shards(n):
    """Large tensors run the single-phase sign kernel, small ones the two-phase
    (keystream-then-circuit) kernel: the full call and its batch shards
    (elem_off / n_total, 3 shards below the crossover) agree share for share,
    odd n_total included (Kogge-Stone p-half straddling AES blocks)."""
    rng = np.random.default_rng(n)
    xs = rng.integers(0, 1 << 64, size=(3, n), dtype=U64)
    rk = rk3(R.Session(4).keys)
    xd = dev(xs)
    full, fmask = torch.empty(3 * n, dtype=torch.int64, device="cuda"), torch.empty(3 * n, dtype=torch.int64,
                                                                                   device="cuda")
    _capi.call("mpc3_rss_sign", p(rk), None, 3, 2, 5, 7, p(xd), p(full), p(fmask), n, n, 0, stream())
    bounds = [0, 200000, 400000, n]
    for a, b in zip(bounds[:-1], bounds[1:]):
        m = b - a
        xsh = dev(np.ascontiguousarray(xs[:, a:b]))
        o, mk = torch.empty(3 * m, dtype=torch.int64, device="cuda"), torch.empty(3 * m, dtype=torch.int64,
                                                                                   device="cuda")
        _capi.call("mpc3_rss_sign", p(rk), None, 3, 2, 5, 7, p(xsh), p(o), p(mk), m, n, a, stream())
        assert np.array_equal(host(o).reshape(3, m), host(full).reshape(3, n)[:, a:b])
        assert np.array_equal(host(mk).reshape(3, m), host(fmask).reshape(3, n)[:, a:b])


@pytest.mark.parametrize("shape", [(2, 64, 7, 7), (1, 256, 14, 14), (3, 5, 7, 9)])
def test_layer_sign_residual_equals_reshare_add_sign(shape):
    """mpc3_rss_layer_sign_residual = reshare/truncate + bias, the shortcut's
    local add, then the ReLU, share for share (a residual block's tail)."""
    rng = np.random.default_rng(7 + sum(shape))
    nb, o, oh, ow = shape
    n = nb * o * oh * ow
    M = nb * oh * ow
    z = dev(rnd(rng, (3, n)))
    view = _capi.make_view(shape, z_stride=(oh * ow, M, ow, 1))
    bv = dev(rnd(rng, (3, o)))
    res = dev(rnd(rng, (3, n)))
    rk = rk3(R.Session(8).keys)
    x = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_reshare_truncate_bias", p(rk), None, 11, 12, 13, 20, p(z), C.byref(view), p(bv), o, 1, p(x),
               0, stream())
    x += res.reshape(-1)
    out1, m1 = torch.empty_like(x), torch.empty_like(x)
    _capi.call("mpc3_rss_sign", p(rk), None, 3, 4, 5, 6, p(x), p(out1), p(m1), n, n, 0, stream())
    out2, m2 = torch.full_like(x, -1), torch.full_like(x, -1)
    _capi.call("mpc3_rss_layer_sign_residual", p(rk), None, 11, 12, 13, 20, p(z), C.byref(view), p(bv), o, 1, p(res),
               n, 3, 4, 5, 6, p(out2), p(m2), 0, n, stream())
    assert np.array_equal(host(out2), host(out1))
    assert np.array_equal(host(m2), host(m1))


@pytest.mark.parametrize("shape,bias,shard", [((128, 96, 10, 10), False, None), ((128, 96, 10, 10), True, None),
                                              ((3, 5, 7, 9), True, None), ((64, 256, 1, 1), False, None),
                                              ((1, 1, 128, 257), True, None), ((40, 7, 33, 33), False, (2, 3))])
def test_layer_sign_equals_reshare_then_sign(shape, bias, shard):
    """mpc3_rss_layer_sign (a layer's reshare + truncate + bias fused into the
    ReLU) = mpc3_rss_reshare_truncate_bias then mpc3_rss_sign, share for
    share, over a column-major conv z view: persistent and two-phase paths,
    odd sizes (Kogge-Stone p-half straddling AES blocks), and a batch shard
    (elem_off / n_total) of a larger tensor."""
    rng = np.random.default_rng(sum(shape))
    nb, o, oh, ow = shape
    n = nb * o * oh * ow
    M = nb * oh * ow
    z = dev(rnd(rng, (3, n)))  # column-major cross terms: (m, o) at o * M + m
    view = _capi.make_view(shape, z_stride=(oh * ow, M, ow, 1))
    bv = dev(rnd(rng, (3, o))) if bias else None
    rk = rk3(R.Session(6).keys)
    elem_off, n_total = (0, n) if shard is None else (n * shard[0] // shard[1] // 2 * 2, 2 * n + 1)
    x = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_reshare_truncate_bias", p(rk), None, 11, 12, 13, 20, p(z), C.byref(view),
               p(bv) if bias else None, o if bias else 0, 1, p(x), elem_off, stream())
    out1, m1 = torch.empty_like(x), torch.empty_like(x)
    _capi.call("mpc3_rss_sign", p(rk), None, 3, 4, 5, 6, p(x), p(out1), p(m1), n, n_total, elem_off, stream())
    out2, m2 = torch.full_like(x, -1), torch.full_like(x, -1)
    _capi.call("mpc3_rss_layer_sign", p(rk), None, 11, 12, 13, 20, p(z), C.byref(view), p(bv) if bias else None,
               o if bias else 0, 1, 3, 4, 5, 6, p(out2), p(m2), elem_off, n_total, stream())
    assert np.array_equal(host(out2), host(out1))
    assert np.array_equal(host(m2), host(m1))


@pytest.mark.parametrize("rows,m,shard", [(128, 10, None), (7, 5, None), (32, 200, None), (3, 2, None),
                                          (64, 37, (2, 6)), (1, 3, None)])
def test_max_tree_one_launch_equals_levels(rows, m, shard):
    """mpc3_rss_max_tree (every level in one launch, R rows per CTA) = one
    mpc3_rss_max_level per level, share for share (odd m, odd rows, a batch
    shard of the rows)."""
    rng = np.random.default_rng(rows * m)
    v = dev(rnd(rng, (3, rows, m)) >> U64(8))
    rk = rk3(R.Session(8).keys)
    row_off, rows_total = (0, rows) if shard is None else (shard[0] * rows // 2 * 2, shard[1] * rows)
    levels, mm = [], m
    while mm > 1:
        levels.append(mm)
        mm = mm // 2 + mm % 2
    jb = np.array([3 + 11 * i for i in range(len(levels))], U64)
    jx = jb + U64(1)
    ja = jb + U64(8)
    cur, cm = v, m
    for i, ml in enumerate(levels):
        k, mo = ml // 2, ml // 2 + ml % 2
        o = torch.empty(3 * rows * mo, dtype=torch.int64, device="cuda")
        _capi.call("mpc3_rss_max_level", p(rk), None, int(jb[i]), int(jx[i]), int(ja[i]), p(cur), p(o), rows, ml,
                   row_off * k, rows_total * k, stream())
        cur, cm = o, mo
    scratch = torch.empty(2 * 3 * rows * ((m + 1) // 2), dtype=torch.int64, device="cuda")
    out = torch.full((3 * rows,), -1, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_max_tree", p(rk), None, len(levels), jb.ctypes.data, jx.ctypes.data, ja.ctypes.data,
               p(v), p(scratch), p(out), rows, m, row_off, rows_total, stream())
    assert np.array_equal(host(out), host(cur))


@pytest.mark.parametrize("geom", [(128, 96, 10, 10, 3, 2, 0), (128, 256, 2, 2, 2, 1, 0), (3, 5, 7, 9, 2, 2, 1),
                                  (2, 3, 6, 6, 3, 3, 0)])
def test_avgpool_backward_mask_equals_two_calls(geom):
    """The pool's backward with the ReLU-mask multiply in the same pass equals
    mpc3_rss_avgpool_backward then mpc3_rss_mul, share for share (power-of-two
    and general windows, padding)."""
    nb, c, h, w, k, st, pd = geom
    oh, ow = (h + 2 * pd - k) // st + 1, (w + 2 * pd - k) // st + 1
    rng = np.random.default_rng(nb * c * h)
    g = dev(rnd(rng, (3, nb * c * oh * ow)) >> U64(3))
    mask = dev(rnd(rng, (3, nb * c * h * w)))
    rk = rk3(R.Session(5).keys)
    area = k * k
    bits, mulc = (area.bit_length() - 1, 1) if area & (area - 1) == 0 else (20, round((1 << 20) / area))
    n = nb * c * h * w
    t = torch.empty(3 * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_avgpool_backward", p(rk), None, 3, 4, bits, mulc, p(g), p(t), nb, c, h, w, oh, ow, k, k, st,
               st, pd, pd, 0, stream())
    want = torch.empty_like(t)
    _capi.call("mpc3_rss_mul", p(rk), None, 9, p(t), p(mask), p(want), n, 0, stream())
    got = torch.full_like(t, -1)
    _capi.call("mpc3_rss_avgpool_backward_mask", p(rk), None, 3, 4, bits, mulc, p(g), p(mask), 9, p(got), nb, c, h, w,
               oh, ow, k, k, st, st, pd, pd, 0, stream())
    assert np.array_equal(host(got), host(want))


def _gemm_packed(A, B, groups, M, Nn, kp, splits):
    Cm = torch.zeros(groups * M * Nn, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_packed", p(A), p(B), p(Cm), groups, M, Nn, kp, Nn, M * Nn, splits, stream())
    return host(Cm).reshape(groups, M, Nn)


def _pack(src, plane, op, role, kp):
    groups = 1 if role == 2 else 3
    out = torch.empty(groups * 8 * op.rows * kp, dtype=torch.uint8, device="cuda")
    _capi.call("mpc3_ring_pack", p(src), plane, C.byref(op), role, p(out), kp, stream())
    return out


@pytest.mark.parametrize("M,K,Nn", [(1, 1, 1), (9, 33, 7), (128, 64, 64), (130, 100, 70), (300, 257, 129),
                                    (64, 16384, 40), (200, 4608, 512)])
def test_ring_matmul_tcgen05_exact(M, K, Nn):
    rng = np.random.default_rng(M * 7 + K)
    a = rnd(rng, (M, K))
    b = rnd(rng, (K, Nn))
    ref = R.wrap_matmul(a, b) if M * K * Nn <= 50_000_000 else None
    kp = (K + 15) // 16 * 16
    A = _pack(dev(a), 0, _capi.dense_operand(M, K, s_r=K, t2=1), 2, kp)
    B = _pack(dev(b), 0, _capi.dense_operand(Nn, K, s_r=1, t2=Nn), 2, kp)
    got = _gemm_packed(A, B, 1, M, Nn, kp, 1)[0]
    simt = torch.empty(M * Nn, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_simt", p(dev(a)), p(dev(b)), p(simt), M, Nn, K, K, 1, Nn, 1, Nn, stream())
    simt = host(simt).reshape(M, Nn)
    assert np.array_equal(got, simt)
    if ref is not None:
        assert np.array_equal(got, ref)


def test_ring_matmul_all_ones_worst_case_and_split():
    # adversarial all-0xFF limbs at the exactness edge, and split-K beyond it
    for K, splits in [(16384, 1), (16384 * 2 + 48, 3)]:
        a = np.full((128, K), (1 << 64) - 1, U64)
        b = np.full((K, 64), (1 << 64) - 1, U64)
        kp = (K + 15) // 16 * 16
        A = _pack(dev(a), 0, _capi.dense_operand(128, K, s_r=K, t2=1), 2, kp)
        B = _pack(dev(b), 0, _capi.dense_operand(64, K, s_r=1, t2=64), 2, kp)
        got = _gemm_packed(A, B, 1, 128, 64, kp, splits)[0]
        assert np.all(got == U64(K % (1 << 64)))  # (-1)(-1) K = K


@pytest.mark.parametrize("splits", [1, 3])
def test_ring_gemm_column_major_output(splits):
    """c_layout 1 writes element (m, n) at n*ldc + m: the transpose of the
    row-major result, split-K included."""
    rng = np.random.default_rng(11 + splits)
    M, K, Nn = 300, 1000, 96
    a, b = rnd(rng, (M, K)), rnd(rng, (K, Nn))
    kp = (K + 15) // 16 * 16
    A = _pack(dev(a), 0, _capi.dense_operand(M, K, s_r=K, t2=1), 2, kp)
    B = _pack(dev(b), 0, _capi.dense_operand(Nn, K, s_r=1, t2=Nn), 2, kp)
    Cm = torch.zeros(M * Nn, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_packed_layout", p(A), p(B), p(Cm), 1, M, Nn, kp, M, M * Nn, splits, 1, stream())
    assert np.array_equal(host(Cm).reshape(Nn, M).T, R.wrap_matmul(a, b))


def _pack_halves(src, plane, op, role, kp, kh):
    out = torch.empty(3 * 8 * op.rows * kp, dtype=torch.uint8, device="cuda")
    _capi.call("mpc3_ring_pack_halves", p(src), plane, C.byref(op), role, p(out), kp, kh, stream())
    return out


@pytest.mark.parametrize("Rn,O,Kc,a_mn,b_mn,layout", [(300, 70, 150, 1, 1, 0), (4096, 200, 100, 1, 1, 1),
                                                      (20000, 64, 96, 1, 1, 0), (250, 130, 70, 1, 0, 0),
                                                      (96, 40, 300, 0, 1, 1), (1, 3, 5, 1, 1, 0),
                                                      (1000, 256, 4608, 1, 1, 1)])
def test_ring_gemm_transposed_operands(Rn, O, Kc, a_mn, b_mn, layout):
    """mpc3_ring_gemm_t reads operands in place from other GEMMs' packed
    buffers (MN-major tiles): the weight-gradient cross terms
      dW[g] = (g_g + g_{g+1})^T x_g + g_g^T x_{g+1}
    from the role-0 pack of g (rows R, K = O) and the role-1 pack of x (rows R,
    K = Kc), halves at 16-aligned columns, contraction over R zero-filled to a
    multiple of 32; K-major partners hold their halves at kc_half."""
    rng = np.random.default_rng(Rn + O + Kc + 2 * a_mn + b_mn)
    gt, xt = rnd(rng, (3, Rn, O)), rnd(rng, (3, Rn, Kc))
    kc_half = (Rn + 31) // 32 * 32
    r16 = lambda v: (v + 15) // 16 * 16  # noqa: E731
    if a_mn:
        A = _pack_halves(dev(gt), Rn * O, _capi.dense_operand(Rn, O, s_r=O, t2=1), 0, r16(r16(O) + O), r16(O))
        a_args = (1, Rn, r16(r16(O) + O), r16(O))
    else:
        A = _pack_halves(dev(gt), Rn * O, _capi.dense_operand(O, Rn, s_r=1, t2=O), 0, 2 * kc_half, kc_half)
        a_args = (0, O, 2 * kc_half, 0)
    if b_mn:
        B = _pack_halves(dev(xt), Rn * Kc, _capi.dense_operand(Rn, Kc, s_r=Kc, t2=1), 1, r16(r16(Kc) + Kc), r16(Kc))
        b_args = (1, Rn, r16(r16(Kc) + Kc), r16(Kc))
    else:
        B = _pack_halves(dev(xt), Rn * Kc, _capi.dense_operand(Kc, Rn, s_r=1, t2=Kc), 1, 2 * kc_half, kc_half)
        b_args = (0, Kc, 2 * kc_half, 0)
    Cm = torch.full((3 * O * Kc,), -1, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_t", p(A), *a_args, p(B), *b_args, p(Cm), 3, O, Kc, kc_half, layout, stream())
    got = host(Cm).reshape(3, Kc, O).transpose(0, 2, 1) if layout else host(Cm).reshape(3, O, Kc)
    for g in range(3):
        h = (g + 1) % 3
        want = R.wrap_matmul(gt[g].T + gt[h].T, xt[g]) + R.wrap_matmul(gt[g].T, xt[h])
        assert np.array_equal(got[g], want), g


@pytest.mark.parametrize("Mm,K,Nn,layout", [(300, 70, 150, 0), (12800, 363, 96, 1), (5, 3, 7, 1), (128, 2304, 384, 1)])
def test_gemm_component_plane_operand_kmajor(Mm, K, Nn, layout):
    """A role-1 operand [x_g | x_{g+1}] stored once per component (role-3
    pack) and read K-major with its second half from plane g + 1
    (mpc3_ring_gemm_t a_mn = 2): C[g] = x_g (W_g + W_{g+1})^T + x_{g+1} W_g^T."""
    rng = np.random.default_rng(Mm + K + Nn)
    xt, wt = rnd(rng, (3, Mm, K)), rnd(rng, (3, Nn, K))
    kc = (K + 31) // 32 * 32
    kpc = (K + 15) // 16 * 16
    A = torch.empty(3 * 8 * Mm * kpc, dtype=torch.uint8, device="cuda")
    _capi.call("mpc3_ring_pack_halves", p(dev(xt)), Mm * K, C.byref(_capi.dense_operand(Mm, K, s_r=K, t2=1)), 3,
               p(A), kpc, K, stream())
    B = _pack_halves(dev(wt), Nn * K, _capi.dense_operand(Nn, K, s_r=K, t2=1), 0, 2 * kc, kc)
    Cm = torch.full((3 * Mm * Nn,), -1, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_t", p(A), 2, Mm, kpc, 0, p(B), 0, Nn, 2 * kc, 0, p(Cm), 3, Mm, Nn, kc, layout, stream())
    got = host(Cm).reshape(3, Nn, Mm).transpose(0, 2, 1) if layout else host(Cm).reshape(3, Mm, Nn)
    for g in range(3):
        h = (g + 1) % 3
        want = R.wrap_matmul(xt[g], (wt[g] + wt[h]).T) + R.wrap_matmul(xt[h], wt[g].T)
        assert np.array_equal(got[g], want), g


@pytest.mark.parametrize("Rn,Kc,O", [(300, 150, 70), (12800, 363, 96), (1, 5, 3)])
def test_gemm_component_plane_operand_mn(Rn, Kc, O):
    """The same role-3 pack read MN-major (a_mn = 3, the weight gradient):
    C[g] = x_g^T (g_g + g_{g+1}) + x_{g+1}^T g_g, column-major."""
    rng = np.random.default_rng(Rn + Kc + O)
    xt, gt = rnd(rng, (3, Rn, Kc)), rnd(rng, (3, Rn, O))
    kc = (Rn + 31) // 32 * 32
    kpc = (Kc + 15) // 16 * 16
    A = torch.empty(3 * 8 * Rn * kpc, dtype=torch.uint8, device="cuda")
    _capi.call("mpc3_ring_pack_halves", p(dev(xt)), Rn * Kc, C.byref(_capi.dense_operand(Rn, Kc, s_r=Kc, t2=1)), 3,
               p(A), kpc, Kc, stream())
    kh = (O + 15) // 16 * 16
    B = _pack_halves(dev(gt), Rn * O, _capi.dense_operand(Rn, O, s_r=O, t2=1), 0, (kh + O + 15) // 16 * 16, kh)
    Cm = torch.full((3 * Kc * O,), -1, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_t", p(A), 3, Rn, kpc, 0, p(B), 1, Rn, (kh + O + 15) // 16 * 16, kh, p(Cm), 3, Kc, O,
               kc, 1, stream())
    got = host(Cm).reshape(3, O, Kc).transpose(0, 2, 1)
    for g in range(3):
        h = (g + 1) % 3
        want = R.wrap_matmul(xt[g].T, gt[g] + gt[h]) + R.wrap_matmul(xt[h].T, gt[g])
        assert np.array_equal(got[g], want), g


def test_pack_halves_z_clears_the_next_gemm_output():
    """The pack's zero region (the following atomic GEMM's C) is cleared and
    the pack itself is unchanged."""
    rng = np.random.default_rng(3)
    xt = rnd(rng, (3, 300, 70))
    op = _capi.dense_operand(300, 70, s_r=70, t2=1)
    ref = _pack_halves(dev(xt), 300 * 70, op, 1, 160, 80)
    out = torch.empty_like(ref)
    z = torch.full((12345,), -1, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_pack_halves_z", p(dev(xt)), 300 * 70, C.byref(op), 1, p(out), 160, 80, p(z), z.numel(),
               stream())
    assert torch.equal(out, ref)
    assert int(torch.count_nonzero(z)) == 0


@pytest.mark.parametrize("M,K,Nn", [(77, 20000, 33), (1, 1, 1), (9, 33, 7), (130, 100, 70), (300, 257, 129),
                                    (200, 4608, 512), (64, 63, 65)])
def test_ring_matmul_u64_convenience(M, K, Nn):
    """The single-call ring matmul (A packed transposed and read MN-major
    with its halves along the source rows, a_mn = 5) vs the oracle."""
    rng = np.random.default_rng(3 + M + K)
    a, b = rnd(rng, (M, K)), rnd(rng, (K, Nn))
    ws = torch.empty(_capi.lib().mpc3_ring_matmul_workspace(M, Nn, K), dtype=torch.uint8, device="cuda")
    out = torch.empty(M * Nn, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_matmul_u64", p(dev(a)), p(dev(b)), p(out), M, Nn, K, p(ws), stream())
    assert np.array_equal(host(out).reshape(M, Nn), R.wrap_matmul(a, b))


def test_ring_matmul_u64_all_ones_exactness_edge():
    """All-0xFF limbs through the single-call path at and past the per-split
    exactness edge (K = 16384 and 3 x 16384 + 48: exactness splits)."""
    for K in (16384, 3 * 16384 + 48):
        a = np.full((128, K), (1 << 64) - 1, U64)
        b = np.full((K, 64), (1 << 64) - 1, U64)
        ws = torch.empty(_capi.lib().mpc3_ring_matmul_workspace(128, 64, K), dtype=torch.uint8, device="cuda")
        out = torch.empty(128 * 64, dtype=torch.int64, device="cuda")
        _capi.call("mpc3_ring_matmul_u64", p(dev(a)), p(dev(b)), p(out), 128, 64, K, p(ws), stream())
        assert np.all(host(out) == U64(K))


def test_ring_gemm_t_row_halves_config_errors():
    z = torch.zeros(64, dtype=torch.int64, device="cuda")
    buf = torch.zeros(8 * 64 * 64, dtype=torch.uint8, device="cuda")
    with pytest.raises(_capi.E.ConfigError):  # row halves need a_half >= kc_half
        _capi.call("mpc3_ring_gemm_t", p(buf), 5, 32, 64, 16, p(buf), 0, 8, 64, 0, p(z), 1, 8, 8, 32, 0, stream())
    with pytest.raises(_capi.E.ConfigError):  # not with component-plane halves
        _capi.call("mpc3_ring_gemm_t", p(buf), 7, 32, 64, 32, p(buf), 0, 8, 64, 0, p(z), 3, 8, 8, 32, 0, stream())


def test_secure_matmul_cross_terms_reshare_truncate():
    rng = np.random.default_rng(11)
    M, K, Nn = 37, 200, 19
    x = R.share(R.fx_encode(rng.uniform(-4, 4, (M, K))), rng)
    y = R.share(R.fx_encode(rng.uniform(-4, 4, (K, Nn))), rng)
    kp = (2 * K + 15) // 16 * 16
    A = _pack(dev(x), M * K, _capi.dense_operand(M, K, s_r=K, t2=1), 0, kp)
    B = _pack(dev(y), K * Nn, _capi.dense_operand(Nn, K, s_r=1, t2=Nn), 1, kp)
    Cm = torch.zeros(3 * M * Nn, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_gemm_packed", p(A), p(B), p(Cm), 3, M, Nn, kp, Nn, M * Nn, 1, stream())
    s = R.Session(7)
    ref = R.matmul_shares(s, x, y)
    out = torch.empty(3 * M * Nn, dtype=torch.int64, device="cuda")
    v = _capi.make_view((1, 1, M, Nn))
    _capi.call("mpc3_rss_reshare_truncate", p(rk3(s.keys)), None, 0, 0, 0, 20, p(Cm), C.byref(v), p(out), 0,
               stream())
    assert np.array_equal(host(out).reshape(3, M, Nn), ref)


def test_avgpool_kernels():
    rng = np.random.default_rng(21)
    shape, win, stride = (2, 3, 9, 8), (3, 3), (2, 2)
    x = R.share(R.fx_encode(rng.uniform(-4, 4, shape)), rng)
    s = R.Session(3)
    ref = R.avgpool_shares(s, x, win, stride)
    rk = rk3(s.keys)
    out = torch.empty(ref.size, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_avgpool", p(rk), None, 0, 0, 20, int(R.fx_encode(1.0 / 9)), p(dev(x)), p(out), *shape, 3, 3, 2, 2, 0, 0, 0,
               stream())
    assert np.array_equal(host(out).reshape(ref.shape), ref)
    g = R.share(R.fx_encode(rng.uniform(-1, 1, ref.shape[1:])), rng)
    s = R.Session(3)
    refb = N.avgpool_backward(N.TrioEngine(s), g, win, stride, shape)
    outb = torch.empty(refb.size, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_avgpool_backward", p(rk), None, 0, 0, 20, int(R.fx_encode(1.0 / 9)), p(dev(g)), p(outb), *shape,
               ref.shape[3], ref.shape[4], 3, 3, 2, 2, 0, 0, 0, stream())
    assert np.array_equal(host(outb).reshape(refb.shape), refb)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 100003])
def test_device_dealer_matches_numpy_pcg64(n):
    from paper_2104_10949_b200.engine import TrioSession

    rng = np.random.default_rng(5 + n)
    x = rnd(rng, n)
    s = TrioSession(0)
    r_host, r_dev = np.random.default_rng(99), np.random.default_rng(99)
    r_host.integers(0, 10, 7)  # arbitrary prior use of the generator
    r_dev.integers(0, 10, 7)
    ref = R.share(x, r_host)
    got = s.share_device(dev(x), r_dev)
    assert np.array_equal(got.data.cpu().numpy().view(U64), ref)
    # the host generator stays in lockstep afterwards
    assert np.array_equal(r_host.integers(0, 1 << 64, 5, dtype=U64), r_dev.integers(0, 1 << 64, 5, dtype=U64))


def test_device_fx_encode_matches_reference():
    from paper_2104_10949_b200.engine import TrioSession

    rng = np.random.default_rng(1)
    x = np.concatenate([rng.uniform(-1e6, 1e6, 10000), [0.0, -0.0, 0.5 / (1 << 20), -0.5 / (1 << 20), 3.5, -3.5]])
    s = TrioSession(0)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    got = s.fx_encode_device(torch.from_numpy(x).cuda(), bad)
    assert np.array_equal(got.cpu().numpy().view(U64), R.fx_encode(x))
    assert int(bad.item()) == 0
    s.fx_encode_device(torch.tensor([float(1 << 43)], dtype=torch.float64, device="cuda"), bad)
    assert int(bad.item()) == 1


# ---------------------------------------------------------------------------
# single-call layers (csrc/layers.cu): one C-ABI entry per reference function


@pytest.mark.parametrize("shape", [(2, 3, 10, 10, 4, 3, 3, 2, 2, 1, 1), (3, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1),
                                   (1, 3, 32, 32, 8, 11, 11, 4, 4, 2, 2)])
def test_ring_conv2d_u64_single_call(shape):
    nb, c, h, w, o, kh, kw, sh, sw, ph, pw = shape
    rng = np.random.default_rng(sum(shape))
    x, k = rnd(rng, (nb, c, h, w)), rnd(rng, (o, c, kh, kw))
    oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
    ws = torch.empty(_capi.lib().mpc3_ring_conv2d_workspace(nb, c, h, w, o, kh, kw, sh, sw, ph, pw),
                     dtype=torch.uint8, device="cuda")
    y = torch.empty(nb * o * oh * ow, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_ring_conv2d_u64", p(dev(x)), p(dev(k)), p(y), nb, c, h, w, o, kh, kw, sh, sw, ph, pw, p(ws),
               stream())
    assert np.array_equal(host(y).reshape(nb, o, oh, ow), R.wrap_conv2d(x, k, (sh, sw), (ph, pw)))


@pytest.mark.parametrize("m,k,n,bits", [(12, 32, 9, 20), (64, 300, 80, 23), (1, 5, 1, 1), (130, 1000, 70, 40)])
def test_rss_matmul_reshare_trunc_single_call(m, k, n, bits):
    rng = np.random.default_rng(m * k + n)
    x = R.share(R.fx_encode(rng.uniform(-2, 2, (m, k))), rng)
    y = R.share(R.fx_encode(rng.uniform(-2, 2, (k, n))), rng)
    s = R.Session(3)
    ref = R.matmul_shares(s, x, y, bits)  # counters ARITH 0, TRUNC_RHO 0, TRUNC_R 0
    ws = torch.empty(_capi.lib().mpc3_rss_matmul_workspace(m, k, n), dtype=torch.uint8, device="cuda")
    out = torch.empty(3 * m * n, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_matmul_reshare_trunc", p(rk3(s.keys)), None, 0, 0, 0, bits, p(dev(x)), p(dev(y)), p(out), m,
               k, n, p(ws), stream())
    assert np.array_equal(host(out).reshape(3, m, n), ref)
    with pytest.raises(_capi.E.RangeError):
        _capi.call("mpc3_rss_matmul_reshare_trunc", p(rk3(s.keys)), None, 0, 0, 0, 62, p(dev(x)), p(dev(y)), p(out),
                   m, k, n, p(ws), stream())


@pytest.mark.parametrize("shape", [(2, 3, 10, 10, 4, 3, 3, 2, 2, 1, 1), (4, 16, 12, 12, 32, 3, 3, 1, 1, 1, 1),
                                   (2, 3, 32, 32, 96, 11, 11, 4, 4, 9, 9)])
def test_rss_conv2d_reshare_trunc_single_call(shape):
    nb, c, h, w, o, kh, kw, sh, sw, ph, pw = shape
    rng = np.random.default_rng(sum(shape) + 1)
    x = R.share(R.fx_encode(rng.uniform(-2, 2, (nb, c, h, w))), rng)
    k = R.share(R.fx_encode(rng.uniform(-0.3, 0.3, (o, c, kh, kw))), rng)
    s = R.Session(5)
    ref = R.conv2d_shares(s, x, k, (sh, sw), (ph, pw))
    ws = torch.empty(_capi.lib().mpc3_rss_conv2d_workspace(nb, c, h, w, o, kh, kw, sh, sw, ph, pw),
                     dtype=torch.uint8, device="cuda")
    out = torch.empty(ref.size, dtype=torch.int64, device="cuda")
    _capi.call("mpc3_rss_conv2d_reshare_trunc", p(rk3(s.keys)), None, 0, 0, 0, 20, p(dev(x)), p(dev(k)), p(out), nb,
               c, h, w, o, kh, kw, sh, sw, ph, pw, p(ws), stream())
    assert np.array_equal(host(out).reshape(ref.shape), ref)
