"""Data-parallel training/inference shards reproduce the single-GPU run bit
for bit.  Two virtual ranks run in two threads on one B200; their weight
gradient cross terms meet in an in-process all-reduce (the NCCL path differs
only in the transport of that one sum)."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.engine import RssTensor, TrioSession  # noqa: E402
from paper_2104_10949_b200.nn import DataParallel, TrainState, one_hot  # noqa: E402


class ThreadAllReduce:
    def __init__(self, world):
        self.world = world
        self.cv = threading.Condition()
        self.buf, self.gen, self.done = [], 0, {}
        self.failed = False

    def fail(self):
        with self.cv:
            self.failed = True
            self.cv.notify_all()

    def __call__(self, z):
        with self.cv:
            if self.failed:
                raise RuntimeError("peer rank failed")
            gen = self.gen
            self.buf.append(z)
            if len(self.buf) == self.world:
                torch.cuda.synchronize()
                total = self.buf[0].clone()
                for t in self.buf[1:]:
                    total += t  # int64 add wraps mod 2^64
                for t in self.buf:
                    t.copy_(total)
                torch.cuda.synchronize()
                self.buf, self.gen = [], self.gen + 1
                self.done[gen] = True
                self.cv.notify_all()
            else:
                self.cv.wait_for(lambda: self.done.get(gen) or self.failed, timeout=120)
                if not self.done.get(gen):
                    raise RuntimeError("all-reduce aborted: a peer rank failed or timed out")


def _shard(t: RssTensor, r, world):
    b = t.shape[0] // world
    return RssTensor(t.data[:, r * b:(r + 1) * b].contiguous(), t.fp)


def _run_threads(fns, ar=None):
    errs = []

    def wrap(f):
        try:
            f()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            if ar is not None:
                ar.fail()

    ths = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("model_name,batch,world", [("lenet", 8, 2), ("alexnet", 8, 2), ("lenet", 16, 4)])
def test_dp_train_step_bit_exact(model_name, batch, world):
    mk = M.lenet if model_name == "lenet" else M.alexnet_cifar
    cfg = M.TrainConfig(0.05, batch, 2, seed=3)
    rng = np.random.default_rng(5)
    shape = (1, 28, 28) if model_name == "lenet" else (3, 32, 32)
    xs_plain = [M.fx_encode(rng.uniform(0, 1, (batch,) + shape)) for _ in range(2)]
    ys_plain = [M.fx_encode(one_hot(rng.integers(0, 10, batch), 10)) for _ in range(2)]

    # single-GPU reference run (global batch)
    s0 = TrioSession(7)
    st0 = TrainState(s0, mk(), cfg)
    batches = [st0.deal_batch(x, y) for x, y in zip(xs_plain, ys_plain)]
    logits0 = [s0.reveal(st0.step(*b)) for b in batches]
    w0 = [s0.reveal(p) for p in st0.params]

    # `world` virtual ranks, each with its own session and batch shard
    ar = ThreadAllReduce(world)
    out = [None] * world

    def rank(r):
        s = TrioSession(7)
        s.dp = DataParallel(r, world, ar)
        st = TrainState(s, mk(), cfg)
        _ = [st.deal_batch(x, y) for x, y in zip(xs_plain, ys_plain)]  # keep the dealer rng in step
        lg = []
        for xb, yb in batches:
            lg.append(st.step(_shard(xb, r, world), _shard(yb, r, world)))
        torch.cuda.synchronize()
        out[r] = ([x.data.clone() for x in lg], [p.data.clone() for p in st.params], dict(s.seq))

    _run_threads([lambda r=r: rank(r) for r in range(world)], ar)
    for i in range(2):
        full = torch.cat([out[r][0][i] for r in range(world)], dim=1)
        got = (full[0] + full[1] + full[2]).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, logits0[i])
    for r in range(world):
        for p, w in zip(out[r][1], w0):
            assert np.array_equal((p[0] + p[1] + p[2]).cpu().numpy().view(np.uint64), w)
        assert out[r][2] == s0.seq


def test_dp8_alexnet_step_matches_pinned_digest():
    """Eight virtual ranks of the data-parallel bench step (AlexNet-CIFAR, 128
    images per rank, rank r's batch from default_rng(100 + r), as bench.py
    under torchrun --nproc-per-node 8): the opened weights after one step
    equal digest_dp8 of tests/golden/cfg_alexnet_dp.npz (the oracle's
    train_private at global batch 1024, where the reference raises
    ExactnessError; the same oracle reproduces the reference at N = 2)."""
    import hashlib
    import json
    import os
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench

    meta = json.loads(bytes(np.load(os.path.join(root, "tests", "golden", "cfg_alexnet_dp.npz"))["meta"]).decode())
    if "digest_dp8" not in meta:
        pytest.skip("no N = 8 digest in the fixture")
    world = 8
    ar = ThreadAllReduce(world)
    out = [None] * world

    def rank(r):
        s = TrioSession(0)
        s.dp = DataParallel(r, world, ar)
        st = TrainState(s, M.alexnet_cifar(), M.TrainConfig(0.01, 128 * world, 1, seed=0))
        imgs, labels = bench._synthetic(128, 100 + r)
        st.step(*st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10))))
        torch.cuda.synchronize()
        out[r] = [s.reveal(p) for p in st.params]

    _run_threads([lambda r=r: rank(r) for r in range(world)], ar)
    for r in range(world):
        d = hashlib.sha256(b"".join(np.ascontiguousarray(w, "<u8").tobytes() for w in out[r])).hexdigest()
        assert d == meta["digest_dp8"], r
