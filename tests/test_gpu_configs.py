"""Bit-exact parity at the BASELINE.json configurations (needs a B200).

The fixtures come from the REAL reference run at the benchmarked sizes
(tests/golden/make_golden_configs.py): AlexNet-CIFAR `train_private` at batch
128 (the headline bench step), LeNet b64 / VGG-16-TI b32 `infer_private`,
one VGG-16-TI b32 training step, ResNet-50 224x224 b1 composed from the
reference's per-party protocols, and the max-pool composition.  Both the
eager engine and the CUDA-graph replays the bench times are checked, and
the sign circuit is checked against the CPU oracle at the sizes where its
persistent single-phase kernel runs (>= 113,664 elements, many rounds).
"""

import numpy as np
import pytest

from golden_configs import alexnet_b128_data, available, cfg, digest, vgg16ti_train_data
from oracle import rss as R

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import engine as E  # noqa: E402
from paper_2104_10949_b200 import nn  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402

U64 = np.uint64


def host(t):
    return t.data.detach().cpu().numpy().view(U64)


def need(name):
    if not available(name):
        pytest.skip(f"fixture cfg_{name}.npz not generated")
    return cfg(name)


# ---------------------------------------------------------------------------
# AlexNet-CIFAR private training step, batch 128 (the bench's headline step)


def _alexnet_state():
    s = TrioSession(0)
    st = nn.TrainState(s, M.alexnet_cifar(), M.TrainConfig(0.01, 128, 2, seed=0))
    imgs, labels = alexnet_b128_data()
    xe, ye = M.fx_encode(imgs), M.fx_encode(nn.one_hot(labels, 10))
    return s, st, [st.deal_batch(xe, ye) for _ in range(2)]


def test_alexnet_b128_eager_steps_match_reference_digest():
    _, meta = need("alexnet_b128")
    s, st, batches = _alexnet_state()
    for it, (xs, ys) in enumerate(batches, start=1):
        logits = st.step(xs, ys)
        ce = nn.cross_entropy(M.fx_decode(s.reveal(logits)), alexnet_b128_data()[1])
        assert abs(ce - meta[f"ce_{it}"][it - 1]) < 1e-12
        assert digest([s.reveal(p) for p in st.params]) == meta[f"digest_{it}"], f"iteration {it}"


def test_alexnet_b128_graph_replays_match_reference_digest():
    """The CUDA-graph step bench.py times: captured on fresh state, replayed
    twice (device counter base advancing), weights opened after each."""
    _, meta = need("alexnet_b128")
    s, st, batches = _alexnet_state()
    xs = E.RssTensor(batches[0][0].data.clone())
    ys = E.RssTensor(batches[0][1].data.clone())
    g = st.capture(xs, ys)
    for it, (xb, yb) in enumerate(batches, start=1):
        xs.data.copy_(xb.data)
        ys.data.copy_(yb.data)
        g.replay()
        torch.cuda.synchronize()
        assert digest([s.reveal(p) for p in st.params]) == meta[f"digest_{it}"], f"replay {it}"


def test_alexnet_b128_eager_then_graph_matches_reference_digest():
    """bench.py's sequence: an eager step, then a CUDA graph captured after
    it and replayed on the next batch."""
    _, meta = need("alexnet_b128")
    s, st, batches = _alexnet_state()
    st.step(*batches[0])
    assert digest([s.reveal(p) for p in st.params]) == meta["digest_1"]
    xs = E.RssTensor(batches[1][0].data.clone())
    ys = E.RssTensor(batches[1][1].data.clone())
    g = st.capture(xs, ys)
    g.replay()
    torch.cuda.synchronize()
    assert digest([s.reveal(p) for p in st.params]) == meta["digest_2"]


def test_alexnet_b128_train_trio_matches_reference():
    _, meta = need("alexnet_b128")
    imgs, labels = alexnet_b128_data()
    res = nn.train_trio(TrioSession(0), M.alexnet_cifar(), M.TrainConfig(0.01, 128, 2, seed=0), imgs, labels)
    assert digest(res.weights) == meta["digest_2"]
    assert np.allclose(res.ce_history, meta["ce_2"], rtol=0, atol=1e-12)


# ---------------------------------------------------------------------------
# inference configs


def _deal_inference(model, batch, seed):
    s = TrioSession(seed)
    rin = np.random.default_rng(seed)
    params = [s.share(w, rin) for w in M.init_params(model, seed=seed)]
    x = s.share(M.fx_encode(rin.uniform(0, 1, (batch,) + model.input_shape)), rin)
    return s, params, x


@pytest.mark.parametrize("graph", [False, True])
@pytest.mark.parametrize("name,builder,batch,seed", [
    ("lenet_b64", M.lenet, 64, 3),
    ("vgg16ti_b32", M.vgg16, 32, 5),
    ("resnet50_b1", M.resnet50, 1, 11),
    ("resnet50_b64", M.resnet50, 64, 11),
])
def test_inference_configs_match_reference_shares(name, builder, batch, seed, graph):
    arrays, _ = need(name)
    model = builder()
    s, params, x = _deal_inference(model, batch, seed)
    if graph:
        out = nn.InferenceGraph(s, model, params, x).replay()
        torch.cuda.synchronize()
    else:
        out = nn.infer_trio(s, model, params, x)
    assert np.array_equal(host(out), arrays["logits"])


def test_lenet_b64_per_party_infer_private_matches_reference():
    arrays, _ = need("lenet_b64")
    model = M.lenet()
    w = M.init_params(model, seed=3)

    def job(ctx):
        rin = np.random.default_rng(3)
        priv = M.share_model(ctx, model.with_params(w), rin)
        xv = M.fx_encode(rin.uniform(0, 1, (64, 1, 28, 28))) if ctx.party == 0 else None
        xs = M.distribute_input(ctx, xv, rin, shape=(64, 1, 28, 28))
        return M.infer_private(ctx, priv, xs)

    res = M.run_in_process(job, seed=3)
    got = np.stack([np.asarray(r.lo) for r in res])
    assert np.array_equal(got, arrays["logits"])


@pytest.mark.parametrize("dgrad_rows", [None, 0, 1 << 62])
def test_vgg16ti_b32_training_step_matches_reference_digest(dgrad_rows, monkeypatch):
    """Eager train_trio at VGG-16-TI b32 = the reference's weights; with the
    engine's input-gradient choice per layer (None), and with every stride-1
    layer on the cropped correlation (0) or on the transposed convolution."""
    if dgrad_rows is not None:
        monkeypatch.setattr(E, "DGRAD_IM2COL_MIN_ROWS", dgrad_rows)
    _, meta = need("vgg16ti_train")
    imgs, labels = vgg16ti_train_data()
    res = nn.train_trio(TrioSession(5), M.vgg16(), M.TrainConfig(0.01, 32, 1, seed=5), imgs, labels)
    assert digest(res.weights) == meta["digest"]


def test_vgg16ti_b32_graph_step_matches_reference_digest():
    """The CUDA-graph training step bench.py times for VGG-16-TI, captured on
    fresh state and replayed once: the reference's weights."""
    _, meta = need("vgg16ti_train")
    imgs, labels = vgg16ti_train_data()
    s = TrioSession(5)
    st = nn.TrainState(s, M.vgg16(), M.TrainConfig(0.01, 32, 1, seed=5))
    xs, ys = st.deal_batch(M.fx_encode(imgs), M.fx_encode(nn.one_hot(labels, 200)))
    g = st.capture(E.RssTensor(xs.data.clone()), E.RssTensor(ys.data.clone()))
    g.xs.data.copy_(xs.data)
    g.ys.data.copy_(ys.data)
    g.replay()
    torch.cuda.synchronize()
    assert digest([s.reveal(p) for p in st.params]) == meta["digest"]


# ---------------------------------------------------------------------------
# max-pool (inference extension composed from the reference's max_tree)


@pytest.mark.parametrize("case", ["k3s2p1", "k2s2", "k3s1"])
def test_maxpool_matches_reference_composition(case):
    arrays, meta = need("maxpool")
    c = meta["cases"][case]
    s = TrioSession(meta["seed"])
    xs = s.share(arrays[f"{case}_in"], np.random.default_rng(meta["dealer"]))
    out = s.maxpool(xs, tuple(c["window"]), tuple(c["stride"]), tuple(c["padding"]))
    assert np.array_equal(host(out), arrays[f"{case}_out"])


def test_maxpool_per_party_api_matches_reference_composition():
    arrays, meta = need("maxpool")
    c = meta["cases"]["k3s2p1"]
    x = arrays["k3s2p1_in"]

    def job(ctx):
        rin = np.random.default_rng(meta["dealer"])
        xs = M.distribute_input(ctx, x if ctx.party == 0 else None, rin, shape=x.shape)
        return M.maxpool_shares(ctx, xs, tuple(c["window"]), tuple(c["stride"]), tuple(c["padding"]))

    res = M.run_in_process(job, seed=meta["seed"])
    assert np.array_equal(np.stack([np.asarray(r.lo) for r in res]), arrays["k3s2p1_out"])


def test_resnet50_maxpool_stem_matches_composed_oracle():
    """The torchvision-style max-pool stem (stem_pool_kind="max") of a small
    ResNet against the oracle's composition (forward_ext + maxpool_shares)."""
    from oracle import nnmirror as N

    model = M.models.tiny_resnet(stem_pool_kind="max")
    layers = tuple(N.from_spec(sp) for sp in model.layers)
    rin = np.random.default_rng(5)
    w = M.init_params(model, seed=4)
    P_o = [R.share(t, rin) for t in w]
    xs = R.share(R.fx_encode(rin.uniform(0, 1, (2, 3, 16, 16))), rin)
    ref = N.forward_ext(R.Session(8), layers, iter(P_o), xs)
    s = TrioSession(8)
    got = M.infer_trio(s, model, [s.from_components(t) for t in P_o], s.from_components(xs))
    assert np.array_equal(host(got), ref)


# ---------------------------------------------------------------------------
# the sign circuit at bench sizes, directly against the oracle


@pytest.mark.parametrize("n,shard", [(1_228_800, None), (3_000_001, None), (1_200_000, (1_000_000, 2_400_001))])
def test_relu_with_mask_large_vs_oracle(n, shard):
    """relu_with_mask at conv1's 1.2 M elements and at 3 M (each persistent
    thread runs many pairs), plus a batch shard of a larger odd tensor whose
    Kogge-Stone p-half straddles AES blocks, against oracle.rss."""
    from paper_2104_10949_b200 import _capi

    rng = np.random.default_rng(n)
    x = rng.integers(-(1 << 45), 1 << 45, n, dtype=np.int64).view(U64)
    x[:5] = [0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1]
    xs = R.share(x, rng)
    if shard is None:
        s = TrioSession(9)
        out, mask = s.relu_with_mask(s.from_components(xs))
        ro, rm = R.relu_with_mask(R.Session(9), xs)
        assert np.array_equal(host(out), ro)
        assert np.array_equal(host(mask), rm)
        return
    off, n_total = shard
    # the oracle over the full tensor (zeros outside the shard), the device on the shard only
    full = np.zeros((3, n_total), U64)
    full[:, off:off + n] = xs
    ro, rm = R.relu_with_mask(R.Session(9), full)
    s = TrioSession(9)
    d = s.from_components(xs)
    out, mask = E.empty((n,)), E.empty((n,))
    _capi.call("mpc3_rss_sign", s.rk, None, 3, 0, 0, 0, d.data.data_ptr(), out.data.data_ptr(),
               mask.data.data_ptr(), n, n_total, off, E._stream())
    assert np.array_equal(host(out), ro[:, off:off + n])
    assert np.array_equal(host(mask), rm[:, off:off + n])


@pytest.mark.parametrize("bias", [False, True])
def test_conv1_layer_sign_b128_vs_oracle(bias):
    """mpc3_rss_layer_sign at AlexNet conv1's shape (batch 128: 1.23 M
    outputs; the persistent fused reshare + truncate + ReLU kernel) against
    the oracle's conv2d_shares (+ shared bias) then relu_with_mask."""
    rng = np.random.default_rng(17 + bias)
    x = R.share(R.fx_encode(rng.uniform(0, 1, (128, 3, 32, 32))), rng)
    k = R.share(R.fx_encode(rng.uniform(-0.1, 0.1, (96, 3, 11, 11))), rng)
    b = R.share(R.fx_encode(rng.uniform(-0.1, 0.1, 96)), rng)
    o = R.Session(21)
    zr = R.conv2d_shares(o, x, k, (4, 4), (9, 9))
    if bias:
        zr = zr + b[:, None, :, None, None]
    ro, rm = R.relu_with_mask(o, zr)
    s = TrioSession(21)
    out, mask = s.conv2d(s.from_components(x), s.from_components(k), (4, 4), (9, 9),
                         bias=s.from_components(b) if bias else None, relu=True)
    assert out.numel == 1_228_800
    assert np.array_equal(host(out), ro)
    assert np.array_equal(host(mask), rm)


def test_maxpool_large_level_by_level_vs_oracle():
    """A ResNet-stem-sized max-pool (3x3 / s2 / p1 over 4 x 16 x 56 x 56: 50 K
    window rows, above the one-launch max_tree's row limit, so each level runs
    through the sign kernels) against the oracle's composition."""
    rng = np.random.default_rng(31)
    x = R.share(R.fx_encode(rng.uniform(-4, 4, (4, 16, 56, 56))), rng)
    ref = R.maxpool_shares(R.Session(13), x, (3, 3), (2, 2), (1, 1))
    s = TrioSession(13)
    out = s.maxpool(s.from_components(x), (3, 3), (2, 2), (1, 1))
    assert out.shape == (4, 16, 28, 28)
    assert np.array_equal(host(out), ref)
