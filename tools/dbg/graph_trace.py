"""Kernel timeline of CUDA-graph replays of the AlexNet training step
(torch.profiler / CUPTI activity records): per-kernel start/end on the device,
busy time vs idle gaps between consecutive kernels, overlap.

python tools/dbg/graph_trace.py [replays] [resnet50 batch: trace its inference graph instead]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import engine  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402


def main(reps=3, resnet_batch=0):
    torch.cuda.set_device(0)
    if resnet_batch:  # ResNet-50 inference graph at this batch instead
        from paper_2104_10949_b200.nn import InferenceGraph

        sess = M.TrioSession(seed=11)
        model = M.models.resnet50()
        rng = np.random.default_rng(11)
        params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
        x = sess.share(M.fx_encode(rng.uniform(0, 1, (resnet_batch, 3, 224, 224))), rng)
        g = InferenceGraph(sess, model, params, x)
    else:
        b = 128
        sess = M.TrioSession(seed=0)
        st = TrainState(sess, M.alexnet_cifar(), M.TrainConfig(0.01, b, 16, seed=0))
        imgs, labels = bench._synthetic(b, 100)
        xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
        for _ in range(2):
            st.step(*xb)
        xs = engine.RssTensor(xb[0].data.clone())
        ys = engine.RssTensor(xb[1].data.clone())
        g = st.capture(xs, ys)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            g.replay()
        torch.cuda.synchronize()
    path = "/tmp/graph_trace.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    ev.sort(key=lambda e: e["ts"])
    t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
    # union of busy intervals
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:
        s, d = e["ts"], e["ts"] + e["dur"]
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = s, d
        else:
            cur_e = max(cur_e, d)
    busy += cur_e - cur_s
    span = t1 - t0
    print(f"{len(ev)} kernels over {reps} replays: span {span:.0f} us, busy {busy:.0f} us, idle {span - busy:.0f} us "
          f"({100 * (span - busy) / span:.1f} %), per replay {span / reps:.0f} us")
    gaps = []
    for a, c in zip(ev, ev[1:]):
        gap = c["ts"] - (a["ts"] + a["dur"])
        if gap > 0:
            gaps.append((gap, a["name"][:50], c["name"][:50]))
    gaps.sort(reverse=True)
    print("largest gaps (us):")
    for gp in gaps[:15]:
        print(f"  {gp[0]:7.1f}  {gp[1]}  ->  {gp[2]}")
    # device time per kernel (durations overlap under PDL / side streams): by
    # name, total duration and the time it ran alone
    pts = sorted([(e["ts"], 1, i) for i, e in enumerate(ev)] + [(e["ts"] + e["dur"], -1, i) for i, e in enumerate(ev)])
    active, alone, last = set(), [0.0] * len(ev), None
    for t, kind, i in pts:
        if last is not None and len(active) == 1:
            alone[next(iter(active))] += t - last
        if kind == 1:
            active.add(i)
        else:
            active.discard(i)
        last = t
    by = {}
    for i, e in enumerate(ev):
        nm = e["name"].split("(")[0].replace("void ", "")[:48]
        d = by.setdefault(nm, [0, 0.0, 0.0])
        d[0] += 1
        d[1] += e["dur"]
        d[2] += alone[i]
    print(f"{'kernel':48s} {'n':>4s} {'dur us/replay':>14s} {'alone us/replay':>16s}")
    for nm, (n_, du, al) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"{nm:48s} {n_ // reps:4d} {du / reps:14.1f} {al / reps:16.1f}")
    tot = sum(x[0] for x in gaps)
    print(f"sum of positive gaps {tot:.0f} us ({len(gaps)} gaps), median {np.median([x[0] for x in gaps]):.1f} us")


if __name__ == "__main__":
    main(*map(int, sys.argv[1:]))
