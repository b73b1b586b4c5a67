"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) on the
B200 engine through the drop-in API (needs a B200).

Criterion 1 at the reference's sizes (100 random matmuls with k <= 4096 and
100 convs including the 11x11 / stride-4 / 64-channel microbenchmark
geometry), criterion 9 (100 private LeNet training iterations at batch 128
against the plaintext fixed-point trainer with the truncation offsets
replayed, within the reference's per-weight budget, and learning), and
criteria 7-8 (private inference of the trained model tracks the float model;
error shrinks monotonically with the fixed-point precision).  The digit data
set (data.py, out of scope) is replaced by a synthetic class-template set of
the same shape.
"""

import numpy as np
import pytest

from oracle import nnmirror as N
from oracle import rss as R

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import nn  # noqa: E402

U64 = np.uint64


def conv_oracle(x, w, stride, padding):
    """Wrapping integer conv2d: accumulate shifted products (test_acceptance.py:58-73)."""
    n, ci, h, wd = x.shape
    co, _, kh, kw = w.shape
    (sh, sw), (ph, pw) = stride, padding
    xp = np.zeros((n, ci, h + 2 * ph, wd + 2 * pw), U64)
    xp[:, :, ph:ph + h, pw:pw + wd] = x
    oh, ow = (h + 2 * ph - kh) // sh + 1, (wd + 2 * pw - kw) // sw + 1
    out = np.zeros((n, co, oh, ow), U64)
    for di in range(kh):
        for dj in range(kw):
            patch = xp[:, :, di:di + oh * sh:sh, dj:dj + ow * sw:sw]
            out += np.einsum("nchw,oc->nohw", patch, w[:, :, di, dj])
    return out


def test_criterion_01_exact_ring_bilinear_ops():
    rng = np.random.default_rng(101)
    for _ in range(100):
        m, n = (int(v) for v in rng.integers(1, 129, 2))
        k = int(rng.integers(1, 4097))
        a = rng.integers(0, 2**64, (m, k), dtype=U64)
        b = rng.integers(0, 2**64, (k, n), dtype=U64)
        assert np.array_equal(M.bilinear_exact(a, b, M.matmul_spec(m, k, n)), np.einsum("ik,kj->ij", a, b))
    for i in range(100):
        if i < 3:
            n = (16, 32, 64)[i]
            x = rng.integers(0, 2**64, (1, 3, n, n), dtype=U64)
            w = rng.integers(0, 2**64, (64, 3, 11, 11), dtype=U64)
            stride, padding = (4, 4), (0, 0)
        else:
            ci, co = (int(v) for v in rng.integers(1, 5, 2))
            kh, kw = (int(v) for v in rng.integers(1, 6, 2))
            ph, pw = (int(v) for v in rng.integers(0, 3, 2))
            sh, sw = (int(v) for v in rng.integers(1, 3, 2))
            h, wd = int(rng.integers(kh, kh + 16)), int(rng.integers(kw, kw + 16))
            batch = int(rng.integers(1, 4))
            x = rng.integers(0, 2**64, (batch, ci, h, wd), dtype=U64)
            w = rng.integers(0, 2**64, (co, ci, kh, kw), dtype=U64)
            stride, padding = (sh, sw), (ph, pw)
        got = M.bilinear_exact(x, w, M.conv2d_spec(x.shape[1], w.shape[2:], stride, padding))
        assert np.array_equal(got, conv_oracle(x, w, stride, padding)), i


def template_digits(n, seed):
    """A learnable stand-in for the synthetic digit set (data.py:92-145):
    one random 28x28 template per class plus noise, values in [0, 1]."""
    rng = np.random.default_rng(seed)
    templates = rng.uniform(0, 1, (10, 1, 28, 28)) > 0.6
    labels = rng.integers(0, 10, n)
    images = 0.75 * templates[labels] + 0.25 * rng.uniform(0, 1, (n, 1, 28, 28))
    return images.astype(np.float64), labels


@pytest.fixture(scope="module")
def trained():
    images, labels = template_digits(1280, 11)
    cfg = M.TrainConfig(learning_rate=0.3, batch_size=128, iterations=100, seed=11)
    outs = M.run_in_process(lambda ctx: M.train_private(ctx, M.lenet(), cfg, (images, labels) if ctx.party == 0 else None),
                            seed=cfg.seed, timeout=3500)
    return outs[0], (images, labels), cfg


def test_criterion_09_private_training_matches_fixed_trainer_and_learns(trained):
    priv, (images, labels), cfg = trained
    layers, ishape = N.lenet()
    ref = N.train_plain_fixed(layers, ishape, images, labels, cfg.learning_rate, cfg.batch_size, cfg.iterations,
                              seed=cfg.seed, t=20, offsets=R.TruncationRandomness(cfg.seed))
    bound = 100 * 2**-19 / 2.0**-20  # test_acceptance.py:239: per-weight budget in ring units
    for got, want in zip(priv.weights, ref):
        diff = np.abs(M.to_signed(got).astype(np.float64) - M.to_signed(want).astype(np.float64))
        assert diff.max() <= bound
    ma = nn.moving_average(priv.ce_history)
    assert 2.2 < ma[0] < 2.4
    assert ma[0] - ma.min() >= 0.05


def _private_logits(model_float, images, fp, seed=0):
    def job(ctx):
        rng = np.random.default_rng(4242) if ctx.party == 0 else None
        ring = [M.fx_encode(w, fp) for w in model_float.params]
        shared = M.share_model(ctx, model_float.with_params(ring if ctx.party == 0 else None), rng)
        xs = M.distribute_input(ctx, M.fx_encode(images, fp) if ctx.party == 0 else None, rng,
                                shape=(len(images),) + model_float.input_shape)
        return M.open_share(ctx, M.infer_private(ctx, shared, xs))

    outs = M.run_in_process(job, fp=fp, seed=seed)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    return M.fx_decode(outs[0], fp)


def test_criteria_07_08_private_inference_tracks_float_model(trained):
    priv, _, _ = trained
    model = M.lenet().with_params([M.fx_decode(w) for w in priv.weights])
    images, _ = template_digits(100, 12)
    got = _private_logits(model, images, M.DEFAULT_FP)
    ref = nn.infer_plain_float(model, images)
    assert int((got.argmax(axis=-1) == ref.argmax(axis=-1)).sum()) >= 99
    assert nn.mean_relative_error(got, ref) < 0.01
    errs = []
    for t in (10, 12, 14, 16, 18, 20):
        out = _private_logits(model, images[:32], M.FixedPointConfig(t))
        errs.append(nn.mean_relative_error(out, ref[:32]))
    assert all(b <= a for a, b in zip(errs, errs[1:])), errs
