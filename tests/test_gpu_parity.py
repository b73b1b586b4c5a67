"""Bit-exact parity of the B200 engine with the reference (needs a B200).

Golden fixtures come from the real reference (tests/golden/make_golden.py):
per-party replicated shares, opened outputs and communication accounting.
Both the per-party drop-in API (run_in_process + protocols) and the trio API
are checked against them.
"""

import hashlib

import numpy as np
import pytest

from golden_cases import CASE_NAMES, DEALER, G, META, SEED, case

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import nn, protocols as P  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402

U64 = np.uint64
OPS = {
    "mul": P.mul, "mul_bcast": P.mul, "matmul": P.matmul_shares, "matmul_bits": P.matmul_shares,
    "conv": P.conv2d_shares, "conv11s4": P.conv2d_shares, "trunc20": P.truncate, "trunc1": P.truncate,
    "trunc61": P.truncate, "a2b": P.a2b, "msb": P.msb, "relu": P.relu, "relu_mask": P.relu_with_mask,
    "drelu": P.drelu, "max_tree": P.max_tree, "exp": P.exp_approx, "reciprocal": P.reciprocal,
    "softmax": P.softmax, "avgpool2": P.avgpool_shares, "avgpool3": P.avgpool_shares,
}
TRIO = {
    "mul": "mul", "mul_bcast": "mul", "matmul": "matmul", "matmul_bits": "matmul", "conv": "conv2d",
    "conv11s4": "conv2d", "trunc20": "truncate", "trunc1": "truncate", "trunc61": "truncate", "a2b": "a2b",
    "msb": "msb", "relu": "relu", "relu_mask": "relu_with_mask", "drelu": "drelu", "max_tree": "max_tree",
    "exp": "exp_approx", "reciprocal": "reciprocal", "softmax": "softmax", "avgpool2": "avgpool",
    "avgpool3": "avgpool",
}


def comps(shares):
    out = np.stack([s.lo for s in shares])
    for p in range(3):
        assert isinstance(shares[p].lo, np.ndarray) and shares[p].lo.dtype == U64  # reference share type
        assert np.array_equal(shares[p].hi, out[(p + 1) % 3])
    return out


@pytest.mark.parametrize("name", CASE_NAMES)
def test_per_party_api_matches_reference_shares_and_accounting(name):
    ins, outs, kw, meta = case(name)
    op = OPS[name]

    def job(ctx):
        rin = np.random.default_rng(DEALER)
        sh = [M.distribute_input(ctx, x if ctx.party == 0 else None, rin, shape=x.shape) for x in ins]
        base = ctx.transport.stats.copy()
        out = op(ctx, *sh, **kw)
        d = ctx.transport.stats.since(base)
        return out, d.payload_bytes_sent(), d.round_labels

    res = M.run_in_process(job, seed=SEED)
    got = [r[0] for r in res]
    if isinstance(got[0], tuple):
        got = [comps([g[i] for g in got]) for i in range(len(got[0]))]
    else:
        got = [comps(got)]
    for a, b in zip(got, outs):
        assert np.array_equal(a, b)
    assert [r[1] for r in res] == meta["payload_bytes"]
    assert res[0][2] == meta["labels"]


@pytest.mark.parametrize("name", CASE_NAMES)
def test_trio_api_matches_reference_shares(name):
    ins, outs, kw, _ = case(name)
    s = TrioSession(SEED)
    rin = np.random.default_rng(DEALER)
    xs = [s.share(x, rin) for x in ins]
    fn = getattr(s, TRIO[name])
    if name.startswith("avgpool"):
        out = fn(*xs, kw["window"], kw.get("stride"))
    elif name.startswith("conv"):
        out = fn(*xs, kw["stride"], kw["padding"])
    else:
        out = fn(*xs, **kw)
    out = list(out) if isinstance(out, tuple) else [out]
    for a, b in zip(out, outs):
        assert np.array_equal(a.data.cpu().numpy().view(U64), b)


def test_lenet_private_inference_shares():
    m = M.lenet()
    w = nn.init_params(m, seed=31)
    xin = G["lenet_infer_x"]

    def job(ctx):
        rin = np.random.default_rng(DEALER)
        priv = M.share_model(ctx, m.with_params(w), rin)
        xs = M.distribute_input(ctx, M.fx_encode(xin) if ctx.party == 0 else None, rin, shape=xin.shape)
        return M.infer_private(ctx, priv, xs)

    assert np.array_equal(comps(M.run_in_process(job, seed=SEED)), G["lenet_infer_logits"])


def test_lenet_train_step_weights_bit_exact():
    cfg = M.TrainConfig(0.01, 3, 1, 5)
    imgs, labels = G["train_lenet_images"], G["train_lenet_labels"]
    res = M.run_in_process(lambda ctx: M.train_private(ctx, M.lenet(), cfg, (imgs, labels) if ctx.party == 0 else None))
    for i, w in enumerate(res[0].weights):
        assert np.array_equal(w, G[f"train_lenet_w{i}"])
    assert np.allclose(res[0].ce_history, META["train_lenet_ce"])


def test_alexnet_train_step_digest_bit_exact():
    s = TrioSession(0)
    cfg = M.TrainConfig(0.01, 4, 1, 5)
    res = nn.train_trio(s, M.alexnet_cifar(), cfg, G["train_alexnet_images"], G["train_alexnet_labels"])
    d = hashlib.sha256(b"".join(np.ascontiguousarray(x, "<u8").tobytes() for x in res.weights)).hexdigest()
    assert d == META["train_alexnet_digest"]
    assert np.allclose(res.ce_history, META["train_alexnet_ce"])


@pytest.mark.parametrize("flags", [{"REUSE_PACKS": False}, {"OVERLAP_PACK": False}, {"nn.OVERLAP": False},
                                   {"REUSE_PACKS": False, "nn.OVERLAP": False}, {"nn.FUSE_RELU": False},
                                   {"nn.FUSE_RELU_MIN": 0}, {"MAXTREE_FUSED": False}, {"CS_PACKS": False},
                                   {"T_PACKS": False}, {"WGRAD_SWAP_MIN_KC": 0}, {"DGRAD_IM2COL_MIN_ROWS": 0}])
def test_alexnet_train_step_digest_under_schedule_variants(flags, monkeypatch):
    """The engine's schedule choices (packs reused across the three GEMMs of a
    layer, weight packs one layer ahead, side-stream weight gradients, pack
    stream, transposed packs, every weight gradient as g^T x, every stride-1
    input gradient as the cropped padded-gradient correlation) change no
    share: the reference's digest under each variant."""
    from paper_2104_10949_b200 import engine as E

    for k, v in flags.items():
        mod, name = (nn, k[3:]) if k.startswith("nn.") else (E, k)
        monkeypatch.setattr(mod, name, v)
    s = TrioSession(0)
    cfg = M.TrainConfig(0.01, 4, 1, 5)
    res = nn.train_trio(s, M.alexnet_cifar(), cfg, G["train_alexnet_images"], G["train_alexnet_labels"])
    d = hashlib.sha256(b"".join(np.ascontiguousarray(x, "<u8").tobytes() for x in res.weights)).hexdigest()
    assert d == META["train_alexnet_digest"]


def test_bilinear_exact_device_matches_golden():
    assert np.array_equal(M.bilinear_exact(G["mm_a"], G["mm_b"], M.matmul_spec(9, 33, 7)), G["mm_out"])
    assert np.array_equal(M.bilinear_exact(G["cv_x"], G["cv_k"], M.conv2d_spec(3, (3, 3), (2, 2), (1, 1))),
                          G["cv_out"])
    assert np.array_equal(M.bilinear_exact(G["cv_x"], None, M.sumpool_spec((3, 3), (2, 2))), G["sp_out"])
    with pytest.raises(M.ExactnessError):
        M.bilinear_exact(np.zeros((1, 1), U64), np.zeros((1, 1), U64), M.matmul_spec(1, (1 << 20) + 1, 1))


def test_prf_words_known_answer():
    words = M.PrfKey(bytes(range(16))).words(1, 0, 4)
    assert np.array_equal(words, G["prf_kat_words"])
