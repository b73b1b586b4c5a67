"""The data-parallel NCCL path inside a captured training step: a one-rank
NCCL process group on one B200 runs the same code as torchrun at N ranks
(all-reduce of the weight-gradient cross terms on the side stream, inside
CUDA-graph capture) and must reproduce the plain step bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import engine  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402
from paper_2104_10949_b200.nn import DataParallel, TrainState, one_hot  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_dp_step_captures_and_matches_plain():
    import torch.distributed as dist

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = M.TrainConfig(0.05, 8, 3, seed=3)
        rng = np.random.default_rng(2)
        x = M.fx_encode(rng.uniform(0, 1, (8, 3, 32, 32)))
        y = M.fx_encode(one_hot(rng.integers(0, 10, 8), 10))

        s0 = TrioSession(4)
        st0 = TrainState(s0, M.alexnet_cifar(), cfg)
        b0 = st0.deal_batch(x, y)
        ref = [s0.reveal(st0.step(*b0)) for _ in range(2)]

        s1 = TrioSession(4)
        s1.dp = DataParallel.from_process_group()
        st1 = TrainState(s1, M.alexnet_cifar(), cfg)
        b1 = st1.deal_batch(x, y)
        st1.step(*b1)  # eager step: NCCL communicator created outside capture
        xs = engine.RssTensor(b1[0].data.clone())
        ys = engine.RssTensor(b1[1].data.clone())
        g = st1.capture(xs, ys)
        got = s1.reveal(g.replay())
        torch.cuda.synchronize()
        assert np.array_equal(got, ref[1])
    finally:
        dist.destroy_process_group()
