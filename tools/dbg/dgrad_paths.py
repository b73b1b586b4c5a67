"""Input-gradient formulations per layer shape (CUDA-graph replays, warm):
the transposed convolution (GEMM + col2im) vs the cropped correlation of the
padded gradient (im2col + GEMM + reshare), and the engine's choice.
python tools/dbg/dgrad_paths.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2104_10949_b200 import engine as E  # noqa: E402
from paper_2104_10949_b200.engine import RssTensor, TrioSession  # noqa: E402

# (name, nb, o, oh, ow, c, k, p): g (nb, o, oh, ow), kernel (o, c, k, k), stride 1
SHAPES = [
    ("vgg conv1_2", 32, 64, 64, 64, 64, 3, 1), ("vgg conv2_1", 32, 128, 32, 32, 64, 3, 1),
    ("vgg conv2_2", 32, 128, 32, 32, 128, 3, 1), ("vgg conv3_1", 32, 256, 16, 16, 128, 3, 1),
    ("vgg conv3_2", 32, 256, 16, 16, 256, 3, 1), ("vgg conv4_1", 32, 512, 8, 8, 256, 3, 1),
    ("vgg conv4_2", 32, 512, 8, 8, 512, 3, 1), ("vgg conv5_2", 32, 512, 4, 4, 512, 3, 1),
    ("alex conv2", 128, 256, 2, 2, 96, 5, 1), ("alex conv3", 128, 384, 1, 1, 256, 3, 1),
    ("alex conv4", 128, 384, 1, 1, 384, 3, 1), ("alex conv5", 128, 256, 1, 1, 384, 3, 1),
]


def graph_us(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (3 * reps)


def main():
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    print(f"{'layer':14s} {'col2im us':>10s} {'im2col us':>10s}  engine picks   same")
    for name, nb, o, oh, ow, c, k, p in SHAPES:
        h, w = oh + k - 1 - 2 * p, ow + k - 1 - 2 * p
        g = RssTensor(torch.from_numpy(rng.integers(0, 1 << 64, (3, nb, o, oh, ow), dtype=np.uint64)
                                       .view(np.int64)).cuda())
        kk = RssTensor(torch.from_numpy(rng.integers(0, 1 << 64, (3, o, c, k, k), dtype=np.uint64)
                                        .view(np.int64)).cuda())
        res, outs = [], []
        for path in ("conv2d_dgrad_col2im", "conv2d_dgrad_im2col"):
            s = TrioSession(8)
            outs.append(getattr(s, path)(g, kk, (1, 1), (p, p), (nb, c, h, w), 20).data.clone())
            res.append(graph_us(lambda: getattr(s, path)(g, kk, (1, 1), (p, p), (nb, c, h, w), 20)))
        pick = "im2col" if E._dgrad_use_im2col(nb, oh, ow, k, k, (p, p)) else "col2im"
        print(f"{name:14s} {res[0]:10.1f} {res[1]:10.1f}  {pick:12s}  {bool(torch.equal(*outs))}", flush=True)


if __name__ == "__main__":
    main()
