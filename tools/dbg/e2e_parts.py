"""Where the e2e step's time over the graph replay goes (AlexNet b128, wall
clock over 30 pipelined steps, as bench.py's e2e): graph alone, + the input
D2D copies, + the copy-stream H2D / encode / deal, + the logits D2H."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import engine  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402

b, steps = 128, 30
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
sess = M.TrioSession(0)
st = TrainState(sess, M.alexnet_cifar(), M.TrainConfig(0.01, b, 10 ** 6, seed=0))
imgs, labels = bench._synthetic(b, 100)
xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
st.step(*xb)
xs, ys = engine.RssTensor(xb[0].data.clone()), engine.RssTensor(xb[1].data.clone())
graph = st.capture(xs, ys)
graph.replay()
torch.cuda.synchronize()

nbuf = 2
pin_img = [torch.empty(imgs.shape, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
pin_lab = [torch.empty((b, 10), dtype=torch.float64).pin_memory() for _ in range(nbuf)]
out_host = [torch.empty((b, 10), dtype=torch.int64).pin_memory() for _ in range(nbuf)]
dev_img = [torch.empty(imgs.shape, dtype=torch.float64, device=dev) for _ in range(nbuf)]
dev_lab = [torch.empty((b, 10), dtype=torch.float64, device=dev) for _ in range(nbuf)]
cs = torch.cuda.Stream(device=dev)
bad = torch.zeros(1, dtype=torch.int32, device=dev)
onehot = one_hot(labels, 10)
rng = np.random.default_rng(1)


def run(d2d, deal, h2d, d2h, fill):
    done, held = [None] * nbuf, [None] * nbuf

    def step(i):
        k = i % nbuf
        if done[k] is not None:
            done[k].synchronize()
        if fill:
            pin_img[k].numpy()[...] = imgs
            pin_lab[k].numpy()[...] = onehot
        main = torch.cuda.current_stream()
        if deal or h2d:
            with torch.cuda.stream(cs):
                if h2d:
                    dev_img[k].copy_(pin_img[k], non_blocking=True)
                    dev_lab[k].copy_(pin_lab[k], non_blocking=True)
                if deal:
                    xe = sess.fx_encode_device(dev_img[k], bad)
                    ye = sess.fx_encode_device(dev_lab[k], bad)
                    held[k] = (sess.share_device(xe, rng), sess.share_device(ye, rng))
                ev = torch.cuda.Event()
                ev.record(cs)
            main.wait_event(ev)
        if d2d:
            src = held[k] if deal else (xb[0], xb[1])
            xs.data.copy_(src[0].data)
            ys.data.copy_(src[1].data)
        logits = graph.replay()
        if d2h:
            out_host[k].copy_(engine.reconstruct_device(logits).view(b, 10), non_blocking=True)
        done[k] = torch.cuda.Event()
        done[k].record(main)

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / steps * 1e3


for name, kw in [("graph only", dict(d2d=False, deal=False, h2d=False, d2h=False, fill=False)),
                 ("+ D2D input copies", dict(d2d=True, deal=False, h2d=False, d2h=False, fill=False)),
                 ("+ D2H logits", dict(d2d=True, deal=False, h2d=False, d2h=True, fill=False)),
                 ("+ H2D (copy stream)", dict(d2d=True, deal=False, h2d=True, d2h=True, fill=False)),
                 ("+ encode + deal (copy stream)", dict(d2d=True, deal=True, h2d=True, d2h=True, fill=False)),
                 ("+ host fill of pinned inputs (= e2e)", dict(d2d=True, deal=True, h2d=True, d2h=True, fill=True)),
                 ("graph only", dict(d2d=False, deal=False, h2d=False, d2h=False, fill=False)),
                 ("= e2e", dict(d2d=True, deal=True, h2d=True, d2h=True, fill=True))]:
    print(f"{name:40s} {run(**kw):7.4f} ms/step", flush=True)
