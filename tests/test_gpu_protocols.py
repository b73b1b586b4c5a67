"""Protocol guarantees of the reference test-suite, on the B200 engine.

Ports of the reference's property/acceptance checks (tests/test_protocols.py,
tests/test_acceptance.py) through the drop-in API, with the tolerances the
reference pins, plus oracle bit-exactness at larger sizes.
"""

import numpy as np
import pytest

from b200_helpers import agree, private_eval, run3
from oracle import nnmirror as N
from oracle import rss as R

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import protocols as P  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402

U64 = np.uint64
FP = M.DEFAULT_FP
ULP = 2.0 ** -20


def rand_u64(rng, shape):
    return rng.integers(0, 1 << 64, size=shape, dtype=U64)


def test_local_ops():
    assert private_eval(lambda ctx, x: P.add_const(x, M.fx_encode(2.25, FP)), np.array([1.5, -3.0])).tolist() == [3.75, -0.75]
    assert private_eval(lambda ctx, x: P.sub_from_const(M.fx_encode(5.0, FP), x), np.array([1.5])).tolist() == [3.5]
    assert private_eval(lambda ctx, x: P.mul_const(x, 3), np.array([1.25, -2.0])).tolist() == [3.75, -6.0]


def test_mul_exact_and_one_round():
    rng = np.random.default_rng(0)
    x, y = rand_u64(rng, (1000,)), rand_u64(rng, (1000,))

    def job(ctx):
        rin = np.random.default_rng(7)
        xs = M.distribute_input(ctx, x if ctx.party == 0 else None, rin, shape=x.shape)
        ys = M.distribute_input(ctx, y if ctx.party == 0 else None, rin, shape=y.shape)
        base = ctx.transport.stats.copy()
        z = P.mul(ctx, xs, ys)
        d = ctx.transport.stats.since(base)
        return M.open_share(ctx, z), d.payload_bytes_sent(), d.rounds, d.round_labels

    for opened, payload, rounds, labels in run3(job):
        assert np.array_equal(opened, x * y)
        assert payload == 8 * 1000 and rounds == 1 and labels == ["mul.reshare"]


def test_truncate_within_one_ulp_all_bits():
    rng = np.random.default_rng(4)
    vals = rng.integers(-(1 << 61), 1 << 61, size=20000, dtype=np.int64)
    for bits in (1, 20, 40, 61):
        out = private_eval(P.truncate, vals.view(U64), encode=False, decode=False, bits=bits)
        d = out.view(np.int64).astype(object) - np.array([v >> bits for v in vals.astype(object)], dtype=object)
        assert set(np.unique(d)) <= {0, 1}


def test_truncate_range_errors():
    def job(ctx):
        rin = np.random.default_rng(7)
        xs = M.distribute_input(ctx, np.zeros(2, U64) if ctx.party == 0 else None, rin, shape=(2,))
        with pytest.raises(M.RangeError):
            P.truncate(ctx, xs, bits=0)
        with pytest.raises(M.RangeError):
            P.truncate(ctx, xs, bits=62)
        return True

    assert all(run3(job))


def test_relu_exact_on_1e6_values_and_round_structure():
    # acceptance criterion 5 (tests/test_acceptance.py:138-152) at full size
    rng = np.random.default_rng(105)
    signed = rng.integers(-(1 << 40) + 1, 1 << 40, size=10 ** 6, dtype=np.int64)
    out = private_eval(P.relu, signed.view(U64), encode=False, decode=False)
    assert np.array_equal(out.view(np.int64), np.maximum(signed, 0))

    def job(ctx):
        rin = np.random.default_rng(7)
        xs = M.distribute_input(ctx, M.fx_encode(np.ones(16), FP) if ctx.party == 0 else None, rin, shape=(16,))
        base = ctx.transport.stats.copy()
        P.relu(ctx, xs)
        return ctx.transport.stats.since(base)

    for d in run3(job):
        assert d.and_rounds() == 7 and d.rounds == 11
        assert d.round_labels == ["share.a2b", "and.ks.g", "and.ks.1", "and.ks.2", "and.ks.4", "and.ks.8",
                                  "and.ks.16", "and.ks.32", "mul.inject", "mul.inject", "mul.mask"]


def test_truncation_unit_error_1e6():
    rng = np.random.default_rng(104)
    a, b = rng.uniform(-16, 16, 10 ** 6), rng.uniform(-16, 16, 10 ** 6)
    prod = M.fx_encode(a, FP) * M.fx_encode(b, FP)
    got = private_eval(P.truncate, prod, encode=False, decode=False).view(np.int64)
    floor = prod.view(np.int64) >> np.int64(FP.t)
    assert np.all((got == floor) | (got == floor + 1))


def test_exp_and_reciprocal_tolerances():
    xs = np.linspace(-45.0, 0.0, 4501)
    assert np.max(np.abs(private_eval(P.exp_approx, xs) - np.exp(xs))) <= 6e-4
    ys = np.linspace(1.0, 200.0, 1991)
    assert np.max(np.abs(private_eval(P.reciprocal, ys) - 1.0 / ys)) <= 2e-4


def test_softmax_matches_offset_replay_mirror():
    rng = np.random.default_rng(18)
    x = rng.uniform(-5, 5, (6, 10))
    out = private_eval(P.softmax, x, seed=44, decode=False)
    ref = N.FixedEngine(20, R.TruncationRandomness(44)).softmax(R.fx_encode(x))
    assert np.array_equal(out, ref)


def test_max_tree_examples_and_empty():
    assert private_eval(P.max_tree, np.array([[1.0, 2.0, 3.0, 4.0]])).tolist() == [4.0]
    assert private_eval(P.max_tree, np.array([[2.0, -1.0, 2.0]])).tolist() == [2.0]

    def job(ctx):
        rin = np.random.default_rng(7)
        xs = M.distribute_input(ctx, np.zeros((1, 0), U64) if ctx.party == 0 else None, rin, shape=(1, 0))
        with pytest.raises(M.ShapeError):
            P.max_tree(ctx, xs)
        return True

    assert all(run3(job))


def test_large_trio_ops_match_oracle():
    """Trio API vs oracle at sizes beyond the golden fixtures."""
    rng = np.random.default_rng(5)
    s, o = TrioSession(12), R.Session(12)
    x = R.share(R.fx_encode(rng.uniform(-3, 3, (64, 300))), rng)
    y = R.share(R.fx_encode(rng.uniform(-3, 3, (300, 80))), rng)
    xd, yd = s.from_components(x), s.from_components(y)
    assert np.array_equal(s.matmul(xd, yd).data.cpu().numpy().view(U64), R.matmul_shares(o, x, y))
    v = R.share(R.fx_encode(rng.uniform(-8, 8, 50001)), rng)
    vd = s.from_components(v)
    r1, m1 = s.relu_with_mask(vd)
    r2, m2 = R.relu_with_mask(o, v)
    assert np.array_equal(r1.data.cpu().numpy().view(U64), r2)
    assert np.array_equal(m1.data.cpu().numpy().view(U64), m2)
    c = R.share(R.fx_encode(rng.uniform(-1, 1, (4, 16, 12, 12))), rng)
    k = R.share(R.fx_encode(rng.uniform(-0.2, 0.2, (32, 16, 3, 3))), rng)
    got = s.conv2d(s.from_components(c), s.from_components(k), (1, 1), (1, 1))
    assert np.array_equal(got.data.cpu().numpy().view(U64), R.conv2d_shares(o, c, k, (1, 1), (1, 1)))


@pytest.mark.parametrize("swap", [False, True])
def test_tiny_model_backward_bit_exact_vs_oracle(swap, monkeypatch):
    """Forward + backward of a small conv net vs the oracle; `swap` runs every
    weight gradient as g^T x (x's transposed pack as B, b_mn = 2)."""
    from paper_2104_10949_b200 import engine as E

    if swap:
        monkeypatch.setattr(E, "WGRAD_SWAP_MIN_KC", 0)
    layers = (N.conv(4, 3, 2, 1), N.relu(), N.pool(2), N.flat(), N.fc(5))
    ishape = (3, 8, 8)
    rng = np.random.default_rng(31)
    x = rng.uniform(-1, 1, (2,) + ishape)
    g = rng.uniform(-0.5, 0.5, (2, 5))
    w = N.init_params(layers, ishape, 20, 31)
    o = R.Session(17)
    rin = np.random.default_rng(1)
    P_o = [R.share(t, rin) for t in w]
    xs = R.share(R.fx_encode(x), rin)
    gs = R.share(R.fx_encode(g), rin)
    lo, acts = N.forward(N.TrioEngine(o), layers, P_o, xs, True)
    ref = N.backward(N.TrioEngine(o), layers, acts, gs, 1)

    m = M.ModelGraph([M.conv2d(4, 3, 2, 1), M.nn.relu(), M.avgpool(2), M.flatten(), M.fully_connected(5)], ishape)
    s = TrioSession(17)
    net = M.TrioNet(s)
    Pd = [s.from_components(t) for t in P_o]
    ld, actsd = net.forward(m, Pd, s.from_components(xs), True)
    assert np.array_equal(ld.data.cpu().numpy().view(U64), lo)
    gd = net.backward(m, actsd, s.from_components(gs), 1)
    for a, b in zip(gd, ref):
        assert np.array_equal(a.data.cpu().numpy().view(U64), b)


@pytest.mark.parametrize("batch", [1, 3])
def test_tiny_resnet_inference_bit_exact_vs_composed_oracle(batch):
    """Bottleneck blocks, folded-BN biases, padded avg-pool stem, residual adds."""
    from paper_2104_10949_b200.models import tiny_resnet

    model = tiny_resnet()
    layers = tuple(N.from_spec(sp) for sp in model.layers)
    rng = np.random.default_rng(40 + batch)
    w = M.init_params(model, seed=3)
    x = rng.uniform(0, 1, (batch, 3, 16, 16))
    rin = np.random.default_rng(2)
    P_o = [R.share(t, rin) for t in w]
    xs = R.share(R.fx_encode(x), rin)
    ref = N.forward_ext(R.Session(8), layers, iter(P_o), xs)
    s = TrioSession(8)
    got = M.infer_trio(s, model, [s.from_components(t) for t in P_o], s.from_components(xs))
    assert np.array_equal(got.data.cpu().numpy().view(U64), ref)
    # and the decoded logits track a float64 evaluation of the same network
    assert got.shape == (batch, 10)


@pytest.mark.parametrize("nb,o,oh,ow,c,kh,kw,ph", [(2, 8, 5, 6, 3, 3, 3, 1), (3, 4, 4, 4, 5, 5, 5, 2),
                                                  (1, 16, 7, 3, 8, 3, 2, 0), (4, 2, 6, 6, 2, 1, 1, 0),
                                                  (2, 4, 7, 8, 3, 3, 3, 3),  # padding > k-1: full grid
                                                  (8, 24, 20, 20, 40, 3, 3, 1)])  # 3200 rows, 40 columns
def test_dgrad_formulations_share_for_share(nb, o, oh, ow, c, kh, kw, ph):
    """The transposed-convolution (col2im) and padded-correlation (im2col)
    input gradients are the same ring values with the same PRF words: every
    party's share equal, same counters consumed (stride 1)."""
    import torch

    from paper_2104_10949_b200.engine import RssTensor, TrioSession

    rng = np.random.default_rng(nb * 100 + o)
    h, w = oh + kh - 1 - 2 * ph, ow + kw - 1 - 2 * ph
    g = rng.integers(0, 1 << 64, size=(3, nb, o, oh, ow), dtype=np.uint64)
    k = rng.integers(0, 1 << 64, size=(3, o, c, kh, kw), dtype=np.uint64)
    outs = []
    for path in ("conv2d_dgrad_col2im", "conv2d_dgrad_im2col"):
        s = TrioSession(8)
        gd = RssTensor(torch.from_numpy(g.view(np.int64)).cuda())
        kd = RssTensor(torch.from_numpy(k.view(np.int64)).cuda())
        y = getattr(s, path)(gd, kd, (1, 1), (ph, ph), (nb, c, h, w), 20)
        outs.append((y.data.cpu().numpy().view(np.uint64), dict(s.seq)))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]


@pytest.mark.parametrize("rows,d,shard", [(128, 10, None), (7, 10, None), (32, 200, None), (3, 2, None),
                                          (5, 3, None), (64, 37, (2, 4)), (1, 10, None),
                                          (64, 10, (1, 4)), (10, 10, (1, 2))])
def test_fused_softmax_loss_equals_separate_launches_and_oracle(rows, d, shard):
    """mpc3_rss_softmax_loss (max_tree, exp, row sum, reciprocal, mul +
    truncate and the label sub in ONE launch) = softmax() then sub(): every
    share, the counters consumed and the CommStats; and = the oracle's
    softmax(z) - y (protocols.py:453-468)."""
    from paper_2104_10949_b200.nn import DataParallel

    rng = np.random.default_rng(rows * 1000 + d)
    z = R.share(R.fx_encode(rng.uniform(-6, 6, (rows, d))), rng)
    y = R.share(R.fx_encode(np.eye(d)[rng.integers(0, d, rows)]), rng)
    outs = []
    for fused in (True, False):
        s = TrioSession(12)
        if shard is not None:
            s.dp = DataParallel(shard[0], shard[1], None)
        base = [t.stats.copy() for t in s.ledger.parties]
        zs, ys = s.from_components(z), s.from_components(y)
        g = s.softmax_loss(zs, ys) if fused else s.sub(s.softmax(zs), ys)
        acct = [t.stats.since(b) for t, b in zip(s.ledger.parties, base)]
        outs.append((g.data.cpu().numpy().view(U64), dict(s.seq), [(a.round_labels, a.payload_bytes_sent())
                                                                   for a in acct]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
    assert outs[0][2] == outs[1][2]
    if shard is None:
        assert np.array_equal(outs[0][0], R.softmax(R.Session(12), z) - y)
