"""Run warm-up steps, then ONE profiled step between cudaProfilerStart/Stop,
for launch lists of exactly one step:

ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/step.csv python tools/step_profile.py alexnet
python tools/step_profile.py resnet50 64     # one ResNet-50 inference pass at batch 64
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, TrioNet, one_hot  # noqa: E402


def main(which, batch):
    torch.cuda.set_device(0)
    cudart = torch.cuda.cudart()
    if which == "alexnet":
        sess = M.TrioSession(seed=0)
        st = TrainState(sess, M.alexnet_cifar(), M.TrainConfig(0.01, batch, 8, seed=0))
        rng = np.random.default_rng(100)
        imgs, labels = rng.uniform(0, 1, (batch, 3, 32, 32)), rng.integers(0, 10, batch)
        xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
        for _ in range(3):
            st.step(*xb)
        torch.cuda.synchronize()
        cudart.cudaProfilerStart()
        st.step(*xb)
        torch.cuda.synchronize()
        cudart.cudaProfilerStop()
    else:
        sess = M.TrioSession(seed=11)
        model = M.models.resnet50()
        rng = np.random.default_rng(11)
        params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
        x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 3, 224, 224))), rng)
        net = TrioNet(sess)
        net.forward(model, params, x, record=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStart()
        net.forward(model, params, x, record=False)
        torch.cuda.synchronize()
        cudart.cudaProfilerStop()
    print("ok", which, batch)


if __name__ == "__main__":
    w = sys.argv[1] if len(sys.argv) > 1 else "alexnet"
    main(w, int(sys.argv[2]) if len(sys.argv) > 2 else (128 if w == "alexnet" else 64))
