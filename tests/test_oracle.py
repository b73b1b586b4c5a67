"""The CPU oracle against the reference-generated golden vectors (no GPU)."""

import hashlib

import numpy as np
import pytest

from golden_cases import CASE_NAMES, DEALER, G, META, SEED, case
from oracle import nnmirror as N
from oracle import rss as R

OPS = {
    "mul": R.mul, "mul_bcast": R.mul, "matmul": R.matmul_shares, "matmul_bits": R.matmul_shares,
    "conv": R.conv2d_shares, "conv11s4": R.conv2d_shares, "trunc20": R.truncate, "trunc1": R.truncate,
    "trunc61": R.truncate, "a2b": R.a2b, "msb": R.msb, "relu": R.relu, "relu_mask": R.relu_with_mask,
    "drelu": R.drelu, "max_tree": R.max_tree, "exp": R.exp_approx, "reciprocal": R.reciprocal,
    "softmax": R.softmax, "avgpool2": R.avgpool_shares, "avgpool3": R.avgpool_shares,
}


def test_prf_known_answer():
    key = G["prf_kat_key"].tobytes()
    assert np.array_equal(R.prf_words(key, 1, 0, 4), G["prf_kat_words"])
    # SURVEY.md 8(c) KAT
    assert [hex(int(v)) for v in G["prf_kat_words"]] == [
        "0xa0877cdd63d37ce3", "0x829ce0603e0eff9a", "0x19ff076bfae7e67f", "0x62f3c9d7c774a10d"]


def test_party_keys_and_streams():
    ks = R.party_keys(SEED)
    assert np.array_equal(np.stack([np.frombuffer(k, np.uint8) for k in ks]), G["party_keys_seed3"])
    assert np.array_equal(np.stack([np.frombuffer(k, np.uint8) for k in R.party_keys(0)]), G["party_keys_seed0"])
    for purpose, index, count in META["prf_rows"]:
        assert np.array_equal(R.prf_words(ks[1], purpose, index, count), G[f"prf_k1_{purpose}_{index}_{count}"])


def test_prf_prefix_and_range():
    k = R.party_keys(0)[0]
    assert np.array_equal(R.prf_words(k, 2, 7, 5), R.prf_words(k, 2, 7, 11)[:5])
    with pytest.raises(ValueError):
        R.prf_words(k, 1 << 16, 0, 1)
    with pytest.raises(ValueError):
        R.prf_words(k, 1, 1 << 48, 1)


def test_prf_words_at_offset():
    """prf_words_at (started mid-stream, for the far-offset GPU tests) equals
    the stream prefix it skips, for even and odd offsets."""
    k = R.party_keys(1)[2]
    full = R.prf_words(k, 3, 11, 600)
    for off, cnt in [(0, 5), (1, 9), (256, 300), (511, 89)]:
        assert np.array_equal(R.prf_words_at(k, 3, 11, off, cnt), full[off:off + cnt])


def test_bilinear_engine():
    assert np.array_equal(R.ring_matmul(G["mm_a"], G["mm_b"]), G["mm_out"])
    assert np.array_equal(R.wrap_matmul(G["mm_a"], G["mm_b"]), G["mm_out"])
    assert np.array_equal(R.ring_conv2d(G["cv_x"], G["cv_k"], (2, 2), (1, 1)), G["cv_out"])
    assert np.array_equal(R.wrap_conv2d(G["cv_x"], G["cv_k"], (2, 2), (1, 1)), G["cv_out"])
    assert np.array_equal(R.ring_sumpool(G["cv_x"], (3, 3), (2, 2)), G["sp_out"])


@pytest.mark.parametrize("name", CASE_NAMES)
def test_protocol_shares_bit_exact(name):
    ins, outs, kw, _ = case(name)
    s = R.Session(SEED)
    rin = np.random.default_rng(DEALER)
    sh = [R.share(x, rin) for x in ins]
    got = OPS[name](s, *sh, **kw)
    got = list(got) if isinstance(got, tuple) else [got]
    assert len(got) == len(outs)
    for a, b in zip(got, outs):
        assert np.array_equal(a, b)


def test_lenet_inference_shares():
    layers, ishape = N.lenet()
    w = N.init_params(layers, ishape, 20, 31)
    s = R.Session(SEED)
    rin = np.random.default_rng(DEALER)
    P = [R.share(x, rin) for x in w]
    xs = R.share(R.fx_encode(G["lenet_infer_x"]), rin)
    assert np.array_equal(N.infer_private(s, layers, P, xs), G["lenet_infer_logits"])


def test_lenet_train_step_weights():
    layers, ishape = N.lenet()
    s = R.Session(0)
    P, _ = N.train_private(s, layers, ishape, G["train_lenet_images"], G["train_lenet_labels"], 0.01, 3, 1, seed=5)
    for i, p in enumerate(P):
        assert np.array_equal(R.open_trio(p), G[f"train_lenet_w{i}"])
    fixed = N.train_plain_fixed(layers, ishape, G["train_lenet_images"], G["train_lenet_labels"], 0.01, 3, 1,
                                seed=5, offsets=R.TruncationRandomness(0))
    for i, p in enumerate(fixed):
        assert np.array_equal(p, G[f"train_lenet_w{i}"])


def test_composed_resnet_oracle_tracks_float():
    """The composed (bias / residual / padded-pool) oracle decodes to the float
    network it encodes, within fixed-point error (no GPU)."""
    torch = pytest.importorskip("torch")
    import torch.nn.functional as F

    from paper_2104_10949_b200.models import tiny_resnet
    from paper_2104_10949_b200.nn import init_params_float

    model = tiny_resnet()
    layers = tuple(N.from_spec(sp) for sp in model.layers)
    wf = init_params_float(model, seed=3)
    x = np.random.default_rng(0).uniform(0, 1, (2, 3, 16, 16))
    rin = np.random.default_rng(2)
    P = [R.share(R.fx_encode(t), rin) for t in wf]
    out = R.open_trio(N.forward_ext(R.Session(1), layers, iter(P), R.share(R.fx_encode(x), rin)))

    it = iter([torch.tensor(t) for t in wf])

    def run(ls, h):
        for L in ls:
            if L.kind == N.CONV:
                h = F.conv2d(h, next(it), stride=L.stride, padding=L.padding)
                if L.bias:
                    h = h + next(it)[None, :, None, None]
            elif L.kind == N.FC:
                h = h @ next(it).T
                if L.bias:
                    h = h + next(it)
            elif L.kind == N.POOL:
                h = F.avg_pool2d(h, L.window, L.stride, L.padding, count_include_pad=True)
            elif L.kind == N.RELU:
                h = torch.relu(h)
            elif L.kind == N.FLAT:
                h = h.reshape(h.shape[0], -1)
            elif L.kind == N.RES:
                hm = run(L.main, h) if L.main else h
                hs = run(L.shortcut, h) if L.shortcut else h
                h = hm + hs
        return h

    ref = run(layers, torch.tensor(x)).numpy()
    assert np.max(np.abs(R.fx_decode(out) - ref)) < 1e-3


@pytest.mark.slow
def test_alexnet_train_step_digest():
    layers, ishape = N.alexnet_cifar()
    fixed = N.train_plain_fixed(layers, ishape, G["train_alexnet_images"], G["train_alexnet_labels"], 0.01, 4, 1,
                                seed=5, offsets=R.TruncationRandomness(0))
    d = hashlib.sha256(b"".join(np.ascontiguousarray(x, "<u8").tobytes() for x in fixed)).hexdigest()
    assert d == META["train_alexnet_digest"]


# ---------------------------------------------------------------------------
# the oracle at the BASELINE configurations (tests/golden/make_golden_configs.py)


def test_maxpool_composition_matches_reference():
    from golden_configs import cfg

    arrays, meta = cfg("maxpool")
    for name, c in meta["cases"].items():
        xs = R.share(arrays[f"{name}_in"], np.random.default_rng(meta["dealer"]))
        out = R.maxpool_shares(R.Session(meta["seed"]), xs, tuple(c["window"]), tuple(c["stride"]),
                               tuple(c["padding"]))
        assert np.array_equal(out, arrays[f"{name}_out"]), name


def test_lenet_b64_inference_matches_reference():
    from golden_configs import cfg

    arrays, _ = cfg("lenet_b64")
    layers, ishape = N.lenet()
    rin = np.random.default_rng(3)
    P = [R.share(w, rin) for w in N.init_params(layers, ishape, 20, 3)]
    x = R.share(R.fx_encode(rin.uniform(0, 1, (64,) + ishape)), rin)
    assert np.array_equal(N.infer_private(R.Session(3), layers, P, x), arrays["logits"])


@pytest.mark.slow
def test_resnet50_b1_composed_oracle_matches_reference_composition():
    """forward_ext at ResNet-50 224x224 batch 1 = the reference's per-party
    protocols composed (cfg_resnet50_b1.npz); ~1 min of CPU."""
    from golden_configs import cfg

    from paper_2104_10949_b200 import models as BM
    from paper_2104_10949_b200 import nn as B

    arrays, _ = cfg("resnet50_b1")
    model = BM.resnet50()
    layers = tuple(N.from_spec(sp) for sp in model.layers)
    rin = np.random.default_rng(11)
    P = [R.share(t, rin) for t in B.init_params(model, seed=11)]
    x = R.share(R.fx_encode(rin.uniform(0, 1, (1, 3, 224, 224))), rin)
    assert np.array_equal(N.forward_ext(R.Session(11), layers, iter(P), x), arrays["logits"])
