"""CUDA-graph replay of the training step is bit-exact with eager steps (needs a B200)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.engine import RssTensor  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402


def _setup(batch):
    sess = M.TrioSession(5)
    st = TrainState(sess, M.lenet(), M.TrainConfig(0.05, batch, 4, seed=2))
    rng = np.random.default_rng(9)
    batches = []
    for _ in range(4):
        x = rng.uniform(0, 1, (batch, 1, 28, 28))
        y = one_hot(rng.integers(0, 10, batch), 10)
        batches.append(st.deal_batch(M.fx_encode(x), M.fx_encode(y)))
    return sess, st, batches


@pytest.mark.parametrize("batch", [8, 6])
def test_graph_replay_matches_eager_steps(batch):
    sess_a, st_a, batches_a = _setup(batch)
    eager_logits = [sess_a.reveal(st_a.step(*b)) for b in batches_a]
    eager_w = [sess_a.reveal(p) for p in st_a.params]

    sess_b, st_b, batches_b = _setup(batch)
    xs = RssTensor(batches_b[0][0].data.clone())
    ys = RssTensor(batches_b[0][1].data.clone())
    g = st_b.capture(xs, ys)
    for i, (xb, yb) in enumerate(batches_b):
        xs.data.copy_(xb.data)
        ys.data.copy_(yb.data)
        lg = g.replay()
        assert np.array_equal(sess_b.reveal(lg), eager_logits[i])
    for a, b in zip(eager_w, [sess_b.reveal(p) for p in st_b.params]):
        assert np.array_equal(a, b)
    assert sess_a.seq == sess_b.seq


def test_inference_graph_with_packed_weights_matches_eager():
    """InferenceGraph packs the weight operands once (frozen_weights) and
    every replay reproduces the eager forward's logits and consumes the same
    counters; a weight changed in place is repacked under frozen_weights."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.engine import TrioSession
    from paper_2104_10949_b200.nn import InferenceGraph, TrioNet

    model = M.models.tiny_resnet()
    rng = np.random.default_rng(4)
    w = M.init_params(model, seed=4)
    x_plain = M.fx_encode(rng.uniform(0, 1, (2,) + model.input_shape))

    def setup():
        s = TrioSession(6)
        r = np.random.default_rng(1)
        return s, [s.share(v, r) for v in w], s.share(x_plain, r)

    s0, p0, x0 = setup()
    net0 = TrioNet(s0)
    ref = [net0.forward(model, p0, x0, record=False)[0].data.cpu().numpy() for _ in range(3)]

    s1, p1, x1 = setup()
    g = InferenceGraph(s1, model, p1, x1)
    got = [g.replay().data.cpu().numpy() for _ in range(3)]
    # replay k equals eager call k (the warm-up ran on a scratch session: no counters consumed)
    assert all(np.array_equal(a, b) for a, b in zip(got, ref))
    assert s1.seq == s0.seq

    s2, p2, x2 = setup()
    net2 = TrioNet(s2)
    with s2.frozen_weights():
        a = net2.forward(model, p2, x2, record=False)[0].data.clone()
        p2[0].data.add_(1)  # in place: new tensor version -> repacked
        b = net2.forward(model, p2, x2, record=False)[0].data.clone()
    s3, p3, x3 = setup()
    net3 = TrioNet(s3)
    a3 = net3.forward(model, p3, x3, record=False)[0].data.clone()
    p3[0].data.add_(1)
    b3 = net3.forward(model, p3, x3, record=False)[0].data.clone()
    torch.cuda.synchronize()
    assert torch.equal(a, a3) and torch.equal(b, b3)


def test_train_trio_graph_replays_equal_eager_run(monkeypatch):
    """train_trio (the drop-in train_private's body) switching to CUDA-graph
    replays mid-run gives the eager run's weights, losses and CommStats."""
    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import nn
    from paper_2104_10949_b200.engine import TrioSession

    rng = np.random.default_rng(3)
    imgs, labels = rng.uniform(0, 1, (24, 1, 28, 28)), rng.integers(0, 10, 24)
    cfg = M.TrainConfig(0.05, 8, 5, seed=2)
    runs = []
    for min_steps in (2, 10 ** 9):
        monkeypatch.setattr(nn, "GRAPH_MIN_STEPS", min_steps)
        s = TrioSession(4)
        res = nn.train_trio(s, M.lenet(), cfg, imgs, labels)
        runs.append((res, [t.stats.as_dict() for t in s.ledger.parties], dict(s.seq)))
    (a, sa, qa), (b, sb, qb) = runs
    for wa, wb in zip(a.weights, b.weights):
        assert np.array_equal(wa, wb)
    assert a.ce_history == b.ce_history
    assert sa == sb and qa == qb
