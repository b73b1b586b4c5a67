"""Per-call CUDA-event timeline of one eager AlexNet training step (streams as
in production, not serialised): every C-ABI call bracketed by events on its
launch stream; prints each call's start/end relative to the step start.

python tools/dbg/timeline.py [batch]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import _capi, engine  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402


def main(batch=128):
    sess = M.TrioSession(seed=0)
    st = TrainState(sess, M.alexnet_cifar(), M.TrainConfig(0.01, batch, 8, seed=0))
    rng = np.random.default_rng(100)
    imgs, labels = rng.uniform(0, 1, (batch, 3, 32, 32)), rng.integers(0, 10, batch)
    xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
    for _ in range(3):
        st.step(*xb)
    torch.cuda.synchronize()
    orig = _capi.call
    recs = []

    def traced(name, *a):
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the call's stream argument, when it is not the current stream (pack / side streams)
        sp = a[-1] if a and isinstance(a[-1], int) else None
        stream = s if sp in (None, s.cuda_stream) else torch.cuda.ExternalStream(sp)
        e0.record(stream)
        r = orig(name, *a)
        e1.record(stream)
        recs.append((name, stream.cuda_stream, e0, e1))
        return r

    _capi.call = traced
    engine.K.call = traced
    torch.cuda._sleep(int(2e8))
    base = torch.cuda.Event(enable_timing=True)
    base.record()
    st.step(*xb)
    end = torch.cuda.Event(enable_timing=True)
    end.record()
    torch.cuda.synchronize()
    _capi.call = orig
    engine.K.call = orig
    streams = {}
    print(f"step {base.elapsed_time(end) * 1e3:.0f} us (incl. the host-enqueue lead)")
    t0 = None
    for name, sid, e0, e1 in recs:
        a, b = base.elapsed_time(e0) * 1e3, base.elapsed_time(e1) * 1e3
        t0 = a if t0 is None else min(t0, a)
        streams.setdefault(sid, len(streams))
    for name, sid, e0, e1 in recs:
        a, b = base.elapsed_time(e0) * 1e3 - t0, base.elapsed_time(e1) * 1e3 - t0
        print(f"s{streams[sid]} {a:8.1f} {b:8.1f} {b - a:7.1f}  {name}")


if __name__ == "__main__":
    main(*map(int, sys.argv[1:]))
