"""Output-channel sharding of batch-1 inference (TensorParallel, SURVEY.md
8(e) "ResNet-50 b=1"): the gathered logits and their per-party shares equal
the single-GPU run bit for bit.  Virtual ranks are threads on one B200 whose
slabs meet in an in-process all-gather (the NCCL path differs only in the
transport)."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402
from paper_2104_10949_b200.nn import TensorParallel, TPNet, TrioNet  # noqa: E402


class ThreadAllGather:
    def __init__(self, world):
        self.world = world
        self.cv = threading.Condition()
        self.buf, self.gen, self.out = {}, 0, {}
        self.failed = False

    def fail(self):
        with self.cv:
            self.failed = True
            self.cv.notify_all()

    def make(self, rank):
        def allgather(t):
            with self.cv:
                if self.failed:
                    raise RuntimeError("peer rank failed")
                gen = self.gen
                self.buf[rank] = t.contiguous()
                if len(self.buf) == self.world:
                    torch.cuda.synchronize()
                    self.out[gen] = torch.stack([self.buf[r] for r in range(self.world)])
                    self.buf, self.gen = {}, self.gen + 1
                    self.cv.notify_all()
                else:
                    self.cv.wait_for(lambda: gen in self.out or self.failed, timeout=120)
                    if gen not in self.out:
                        raise RuntimeError("all-gather aborted")
                return self.out[gen].clone()
        return allgather


@pytest.mark.parametrize("world,classes", [(2, 10), (4, 8)])
def test_tp_batch1_inference_bit_exact(world, classes):
    model = M.models.tiny_resnet(num_classes=classes)
    rng = np.random.default_rng(world)
    w_plain = M.init_params(model, seed=3)
    x_plain = M.fx_encode(rng.uniform(0, 1, (1,) + model.input_shape))

    def setup():
        s = TrioSession(5)
        r = np.random.default_rng(9)
        params = [s.share(w, r) for w in w_plain]
        x = s.share(x_plain, r)
        return s, params, x

    s0, p0, x0 = setup()
    ref = TrioNet(s0).forward(model, p0, x0, record=False)[0]
    ref_shares = ref.data.cpu().numpy().view(np.uint64)

    ag = ThreadAllGather(world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            s, p, x = setup()
            net = TPNet(s, TensorParallel(r, world, ag.make(r)))
            y = net.forward_tp(model, p, x)
            torch.cuda.synchronize()
            out[r] = (y.data.cpu().numpy().view(np.uint64), dict(s.seq))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ag.fail()

    ths = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if errs:
        raise errs[0]
    for r in range(world):
        assert np.array_equal(out[r][0], ref_shares)  # every party's share, every rank
        assert out[r][1] == s0.seq  # same counters consumed
