import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st
for (M, K, N) in [(128, 256, 256), (128, 256, 10), (256, 128, 256), (10, 128, 256), (128, 10, 256)]:
    x = torch.randint(-(1 << 62), 1 << 62, (3 * M * K,), dtype=torch.int64, device="cuda")
    y = torch.randint(-(1 << 62), 1 << 62, (3 * K * N,), dtype=torch.int64, device="cuda")
    z = torch.empty(3 * M * N, dtype=torch.int64, device="cuda")
    oa, ob = _capi.dense_operand(M, K, s_r=K, t2=1), _capi.dense_operand(N, K, s_r=1, t2=N)
    t = graph_us(lambda: _capi.call("mpc3_ring_gemm_cross_simt", p(x), M * K, C.byref(oa), p(y), K * N, C.byref(ob), p(z), 0, st()), reps=10)
    kp = (2 * K + 15) // 16 * 16
    A = torch.empty(3 * 8 * M * kp, dtype=torch.uint8, device="cuda")
    B = torch.empty(3 * 8 * N * kp, dtype=torch.uint8, device="cuda")
    def tc():
        _capi.call("mpc3_ring_pack", p(x), M * K, C.byref(oa), 0, p(A), kp, st())
        _capi.call("mpc3_ring_pack", p(y), K * N, C.byref(ob), 1, p(B), kp, st())
        _capi.call("mpc3_ring_gemm_auto", p(A), p(B), p(z), 3, M, N, kp, 0, st())
    t2 = graph_us(tc, reps=10)
    t3 = graph_us(lambda: _capi.call("mpc3_ring_gemm_cross", p(x), M * K, C.byref(oa), p(y), K * N, C.byref(ob), p(z), N, M * N, 1, st()), reps=10)
    print(f"M={M} K={K} N={N}: simt {t:6.1f} us   pack+pack+tcgen05 {t2:6.1f} us   implicit {t3:6.1f} us", flush=True)
