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
