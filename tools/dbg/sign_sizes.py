"""Device time of the sign circuit (ReLU mode) per size, CUDA-graph replays:
python tools/dbg/sign_sizes.py  (MPC3_SIGN2_PIPE=0 for the unpipelined two-phase kernel)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2104_10949_b200 import _capi  # noqa: E402

rk = np.zeros((3, 44), np.uint32)
for i in range(3):
    _capi.check(_capi.lib().mpc3_aes128_expand(C.c_char_p(bytes([i]) * 16), rk[i].ctypes.data_as(C.c_void_p)))
rkd = torch.from_numpy(rk.view(np.int32)).pin_memory()
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
res = {}
for n in (1024, 25088, 32768, 49152, 50176, 100352, 131072, 200704, 401408, 802816, 1228800):
    x = torch.randint(-(1 << 40), 1 << 40, (3 * n,), dtype=torch.int64, device="cuda")
    y, m = torch.empty_like(x), torch.empty_like(x)
    f = lambda: _capi.call("mpc3_rss_sign", rkd.data_ptr(), None, 3, 0, 0, 0, x.data_ptr(), y.data_ptr(),  # noqa: E731
                           m.data_ptr(), n, n, 0, st())
    f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            f()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 30 * 1e3
    res[n] = us
    print(f"n={n:8d} {us:8.1f} us  {23 * n / us / 1e3:6.1f} G blocks/s", flush=True)
