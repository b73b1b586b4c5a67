"""Host-side cost of an eager AlexNet b128 step (cProfile) and its wall time."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402

s = M.TrioSession(0)
st = TrainState(s, M.alexnet_cifar(), M.TrainConfig(0.01, 128, 30, seed=0))
imgs, labels = bench._synthetic(128, 100)
b = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10)))
for _ in range(3):
    st.step(*b)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    st.step(*b)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"eager: host enqueue {1e3 * (t1 - t0) / 10:.2f} ms/step, wall {1e3 * (t2 - t0) / 10:.2f} ms/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    st.step(*b)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats(os.environ.get("SORT", "tottime")).print_stats(int(os.environ.get("NSTAT", "25")))
