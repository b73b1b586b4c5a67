import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st
for (Mm, K, Nn) in [(12800, 363, 96), (512, 2400, 256), (128, 3456, 384)]:
    kc = (K + 31) // 32 * 32
    kpc = (K + 31) // 32 * 32 if len(sys.argv) > 1 else (K + 15) // 16 * 16
    Acs = torch.randint(0, 256, (3 * 8 * Mm * kpc,), dtype=torch.uint8, device="cuda")
    Akm = torch.randint(0, 256, (3 * 8 * Mm * 2 * kc,), dtype=torch.uint8, device="cuda")
    B = torch.randint(0, 256, (3 * 8 * Nn * 2 * kc,), dtype=torch.uint8, device="cuda")
    Cm = torch.empty(3 * Mm * Nn, dtype=torch.int64, device="cuda")
    t_cs = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(Acs), 2, Mm, kpc, 0, p(B), 0, Nn, 2 * kc, 0, p(Cm), 3, Mm, Nn, kc, 1, st()), reps=5)
    t_km = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(Akm), 0, Mm, 2 * kc, 0, p(B), 0, Nn, 2 * kc, 0, p(Cm), 3, Mm, Nn, kc, 1, st()), reps=5)
    t_au = graph_us(lambda: _capi.call("mpc3_ring_gemm_auto", p(Akm), p(B), p(Cm), 3, Mm, Nn, 2 * kc, 1, st()), reps=5)
    print(f"M={Mm} K={K} N={Nn}: cs {t_cs:.1f} us  kmajor(t) {t_km:.1f} us  auto {t_au:.1f} us", flush=True)
