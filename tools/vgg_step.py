"""One VGG-16-TI private training step between cudaProfilerStart/Stop (ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200.nn import TrainState, one_hot  # noqa: E402

if __name__ == "__main__":
    b = 32
    sess = M.TrioSession(seed=5)
    st = TrainState(sess, M.models.vgg16(), M.TrainConfig(0.01, b, 4, seed=5))
    rng = np.random.default_rng(5)
    xb = st.deal_batch(M.fx_encode(rng.uniform(0, 1, (b, 3, 64, 64))), M.fx_encode(one_hot(rng.integers(0, 200, b), 200)))
    st.step(*xb)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    st.step(*xb)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok")
