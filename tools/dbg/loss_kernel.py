"""Drive mpc3_rss_softmax_loss at the AlexNet shape (128, 10) for ncu / timing."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import rss as R  # noqa: E402
from paper_2104_10949_b200.engine import TrioSession  # noqa: E402

rows, d = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (128, 10)
rng = np.random.default_rng(0)
z = R.share(R.fx_encode(rng.uniform(-6, 6, (rows, d))), rng)
y = R.share(R.fx_encode(np.eye(d)[rng.integers(0, d, rows)]), rng)
s = TrioSession(1)
zs, ys = s.from_components(z), s.from_components(y)
for _ in range(3):
    s.softmax_loss(zs, ys)
torch.cuda.synchronize()
for name, fn in (("fused", lambda: s.softmax_loss(zs, ys)), ("separate", lambda: s.sub(s.softmax(zs), ys))):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    e1.synchronize()
    print(name, e0.elapsed_time(e1) / 50 * 1e3, "us per loss gradient (graph)")
