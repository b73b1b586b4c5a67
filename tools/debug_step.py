"""Layer-by-layer comparison of one private training step: B200 engine vs oracle.

python tools/debug_step.py [--model alexnet|lenet] [--batch 4]
Prints the first op whose shares differ.
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10949_b200 as M  # noqa: E402
from oracle import nnmirror as N  # noqa: E402
from oracle import rss as R  # noqa: E402

U64 = np.uint64


def host(t):
    return t.data.cpu().numpy().view(U64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="alexnet")
    ap.add_argument("--batch", type=int, default=4)
    a = ap.parse_args()
    layers, ishape = N.alexnet_cifar() if a.model == "alexnet" else N.lenet()
    model = M.alexnet_cifar() if a.model == "alexnet" else M.lenet()
    rng = np.random.default_rng(1)
    b = a.batch
    imgs = rng.uniform(0, 1, (b,) + ishape)
    labels = rng.integers(0, 10, b)
    w = N.init_params(layers, ishape, 20, 5)
    rin = np.random.default_rng(5)
    P_o = [R.share(t, rin) for t in w]
    xs = R.share(R.fx_encode(imgs), rin)
    ys = R.share(R.fx_encode(N.one_hot(labels, 10)), rin)
    o = R.Session(0)
    s = M.TrioSession(0)
    eo = N.TrioEngine(o)
    net = M.TrioNet(s)
    Pd = [s.from_components(t) for t in P_o]
    h_o, h_d = xs, s.from_components(xs)
    pi = 0
    acts_o, acts_d = [], []
    for L, spec in zip(layers, model.layers):
        if L.kind == N.CONV:
            acts_o.append((h_o, P_o[pi]))
            acts_d.append((h_d, Pd[pi]))
            h_o = eo.conv2d(h_o, P_o[pi], L.stride, L.padding)
            h_d = s.conv2d(h_d, Pd[pi], spec.stride, spec.padding)
            pi += 1
        elif L.kind == N.FC:
            acts_o.append((h_o, P_o[pi]))
            acts_d.append((h_d, Pd[pi]))
            h_o = eo.matmul(h_o, eo.map_structural(P_o[pi], lambda q: q.T))
            h_d = s.matmul(h_d, Pd[pi].apply(lambda d: d.transpose(1, 2)))
            pi += 1
        elif L.kind == N.POOL:
            acts_o.append((eo.shape(h_o),))
            acts_d.append((h_d.shape,))
            h_o = eo.avgpool(h_o, L.window, L.stride)
            h_d = s.avgpool(h_d, spec.window, spec.stride)
        elif L.kind == N.RELU:
            h_o, m_o = eo.relu_mask(h_o)
            h_d, m_d = s.relu_with_mask(h_d)
            acts_o.append((m_o,))
            acts_d.append((m_d,))
        else:
            shp = eo.shape(h_o)
            acts_o.append((shp,))
            acts_d.append((h_d.shape,))
            h_o = eo.map_structural(h_o, lambda q: q.reshape(shp[0], -1))
            h_d = h_d.contiguous().reshape(shp[0], -1)
        ok = np.array_equal(host(h_d), h_o)
        print("fwd", L.kind, h_o.shape[1:], "OK" if ok else "MISMATCH", flush=True)
        if not ok:
            return
    g_o = R.softmax(o, h_o) - ys
    g_d = net.loss_grad(h_d, s.from_components(ys))
    print("loss_grad", "OK" if np.array_equal(host(g_d), g_o) else "MISMATCH")
    # backward, layer by layer
    bb = N.batch_bits(b)
    plist = [i for i, L in enumerate(layers) if L.kind in (N.CONV, N.FC)]
    pi = len(plist)
    for li in range(len(layers) - 1, -1, -1):
        L, spec = layers[li], model.layers[li]
        co, cd = acts_o[li], acts_d[li]
        if L.kind == N.FC:
            pi -= 1
            go = eo.matmul(eo.map_structural(g_o, lambda q: q.T), co[0], bits=20 + bb)
            gd = s.matmul(g_d.apply(lambda d: d.transpose(1, 2)), cd[0], bits=20 + bb)
            print("wgrad FC", pi, "OK" if np.array_equal(host(gd), go) else "MISMATCH")
            if li == plist[0]:
                break
            g_o = eo.matmul(g_o, co[1])
            g_d = s.matmul(g_d, cd[1])
        elif L.kind == N.CONV:
            pi -= 1
            go = N.conv_grad_kernel(eo, co[0], g_o, L, 20 + bb)
            gd = s.conv2d_wgrad(cd[0], g_d, spec.kernel, spec.stride, spec.padding, 20 + bb)
            print("wgrad conv", pi, "OK" if np.array_equal(host(gd), go) else "MISMATCH")
            if li == plist[0]:
                break
            g_o = N.conv_grad_input(eo, g_o, co[1], L, eo.shape(co[0]), 20)
            g_d = s.conv2d_dgrad(g_d, cd[1], spec.stride, spec.padding, cd[0].shape, 20)
        elif L.kind == N.POOL:
            g_o = N.avgpool_backward(eo, g_o, L.window, L.stride, co[0])
            g_d = s.avgpool_backward(g_d, spec.window, spec.stride, cd[0])
        elif L.kind == N.RELU:
            g_o = R.mul(o, g_o, co[0])
            g_d = s.mul(g_d, cd[0], "mul.mask")
        else:
            g_o = eo.map_structural(g_o, lambda q, sh=co[0]: q.reshape(sh))
            g_d = g_d.contiguous().reshape(cd[0])
        ok = np.array_equal(host(g_d), g_o)
        print("bwd", L.kind, g_o.shape[1:], "OK" if ok else "MISMATCH", flush=True)
        if not ok:
            diff = host(g_d) != g_o
            print("  mismatching elements:", int(diff.sum()), "of", diff.size, "first at", np.argwhere(diff)[:5])
            return


if __name__ == "__main__":
    main()
