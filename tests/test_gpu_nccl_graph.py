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


def test_nccl_tp_inference_graph_matches_eager():
    """Tensor-parallel batch-1 inference (TPNet) captured with its NCCL
    all-gathers as an InferenceGraph (bench.py's resnet50_b1_tp at N ranks):
    two replays equal the eager tensor-parallel passes and the one-GPU
    forward at the same counters."""
    import torch.distributed as dist

    from paper_2104_10949_b200.nn import InferenceGraph, TensorParallel, TPNet, TrioNet

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        model = M.models.tiny_resnet()
        rng = np.random.default_rng(3)
        w = M.init_params(model, seed=3)
        xin = M.fx_encode(rng.uniform(0, 1, (1,) + tuple(model.input_shape)))

        def fresh():
            s = TrioSession(6)
            r = np.random.default_rng(4)
            return s, [s.share(t, r) for t in w], s.share(xin, r)

        s0, p0, x0 = fresh()
        ref = [s0.reveal(TrioNet(s0).forward(model, p0, x0, record=False)[0]) for _ in range(2)]
        tp = TensorParallel.from_process_group()
        s1, p1, x1 = fresh()
        eager = [s1.reveal(TPNet(s1, tp).forward_tp(model, p1, x1)) for _ in range(2)]
        s2, p2, x2 = fresh()
        g = InferenceGraph(s2, model, p2, x2, forward=lambda s, m, p, xx: TPNet(s, tp).forward_tp(m, p, xx))
        got = [s2.reveal(g.replay()) for _ in range(2)]
        for a, b, c in zip(ref, eager, got):
            assert np.array_equal(a, b) and np.array_equal(a, c)
        assert s2.seq == s0.seq
    finally:
        dist.destroy_process_group()
