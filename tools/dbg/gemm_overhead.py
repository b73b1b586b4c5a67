import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st
M, N = 512, 2368
for R in (32, 64, 128, 256, 512, 1024, 2048):
    kc = (R + 31) // 32 * 32
    kpa, kpb = 2 * M, 2 * N
    A = torch.randint(0, 256, (8 * R * kpa,), dtype=torch.uint8, device="cuda")
    B = torch.randint(0, 256, (8 * R * kpb,), dtype=torch.uint8, device="cuda")
    Cm = torch.empty(M * N, dtype=torch.int64, device="cuda")
    t = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(A), 1, R, kpa, M, p(B), 1, R, kpb, N, p(Cm), 1, M, N, kc, 1, st()), reps=10)
    mma_us = (2 * kc // 32) * 1152 / 1.9e3
    print(f"R={R:5d} nkb={2*kc//32:4d} t={t:7.2f} us  ideal-mma={mma_us:6.2f} us  overhead={t-mma_us:6.2f}", flush=True)
