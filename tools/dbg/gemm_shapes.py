"""Device time of mpc3_ring_gemm_auto (3 groups, packed operands) on the
AlexNet / ResNet-50 forward shapes: compare MPC3_GEMM_NARROW=0 / 1 runs."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tools.microbench import graph_us, p, st  # noqa: E402
from paper_2104_10949_b200 import _capi  # noqa: E402

SHAPES = [(12800, 96, 736), (512, 256, 4800), (128, 384, 4608), (128, 256, 512), (3456, 256, 256),
          (200704, 64, 128), (200704, 256, 128), (50176, 128, 256), (802816, 64, 320), (12544, 512, 512),
          (3136, 512, 4608), (4096, 4096, 4096)]
for M, N, kp in SHAPES:
    A = torch.randint(0, 256, (3 * 8 * M * kp,), dtype=torch.uint8, device="cuda")
    B = torch.randint(0, 256, (3 * 8 * N * kp,), dtype=torch.uint8, device="cuda")
    C = torch.empty(3 * M * N, dtype=torch.int64, device="cuda")
    us = graph_us(lambda: _capi.call("mpc3_ring_gemm_auto", p(A), p(B), p(C), 3, M, N, kp, 1, st()), reps=5)
    print(f"M={M:7d} N={N:5d} K2={kp:5d} {us:9.1f} us {72 * 3 * M * N * kp / 2 / us / 1e6:7.0f} TOPS", flush=True)
    del A, B, C
