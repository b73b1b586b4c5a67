"""Per-launch kernel times of one instrumented step (CUDA events, streams
serialised), grouped by C-ABI entry point: where a step's time goes.

python tools/step_breakdown.py alexnet [--out gpurun_out/breakdown_alexnet.json]
python tools/step_breakdown.py resnet50 64
python tools/step_breakdown.py vgg16 32
"""
import argparse
import json
import os
import sys
from collections import defaultdict

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import _capi, engine  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, TrioNet, one_hot  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", default="alexnet", nargs="?")
    ap.add_argument("batch", type=int, default=0, nargs="?")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rec = bench.Recorder(_capi, engine)
    if a.which == "alexnet":
        b = a.batch or 128
        sess = M.TrioSession(seed=0)
        st = TrainState(sess, M.alexnet_cifar(), M.TrainConfig(0.01, b, 8, seed=0))
        imgs, labels = bench._synthetic(b, 100)
        xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
        for _ in range(2):
            st.step(*xb)
        fn = lambda: st.step(*xb)  # noqa: E731
    elif a.which == "vgg16":  # VGG-16-TI training step (bench.vgg16_ti's)
        b = a.batch or 32
        sess = M.TrioSession(seed=5)
        trng = np.random.default_rng(5)
        imgs, labels = trng.uniform(0, 1, (b, 3, 64, 64)), trng.integers(0, 200, b)
        st = TrainState(sess, M.models.vgg16(), M.TrainConfig(0.01, b, 8, seed=5))
        xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 200)))
        for _ in range(2):
            st.step(*xb)
        fn = lambda: st.step(*xb)  # noqa: E731
    else:
        b = a.batch or 64
        sess = M.TrioSession(seed=11)
        model = M.models.resnet50()
        rng = np.random.default_rng(11)
        params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
        x = sess.share(M.fx_encode(rng.uniform(0, 1, (b, 3, 224, 224))), rng)
        net = TrioNet(sess)
        net.forward(model, params, x, record=False)
        fn = lambda: net.forward(model, params, x, record=False)  # noqa: E731
    torch.cuda.synchronize()
    bench._instrumented(fn, rec, torch)
    rows = []
    by = defaultdict(lambda: [0.0, 0])
    for i, (name, cat, e0, e1, work, shape) in enumerate(rec.events):
        us = (rec.ms[i] if rec.ms is not None else e0.elapsed_time(e1)) * 1e3  # shortest of the passes
        rows.append({"i": i, "call": name, "cat": cat, "us": round(us, 2), "shape": list(shape), "work": work})
        by[name][0] += us
        by[name][1] += 1
    total = sum(r["us"] for r in rows)
    summary = sorted(([k, round(v[0], 1), v[1], round(v[0] / total, 4)] for k, v in by.items()), key=lambda r: -r[1])
    print(f"{a.which} b{b}: {len(rows)} launches, {total:.1f} us kernel time (serialised)")
    for r in summary:
        print(f"  {r[0]:45s} {r[1]:9.1f} us  x{r[2]:3d}  {100 * r[3]:5.1f}%")
    for r in rows:
        print(f"  {r['i']:3d} {r['call']:42s} {r['us']:8.2f} us  {r['shape']}")
    if a.out:
        json.dump({"which": a.which, "batch": b, "total_us": total, "summary": summary, "launches": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
