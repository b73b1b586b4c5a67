import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st
nb = 128
x = torch.randint(-(1 << 62), 1 << 62, (3 * nb * 3 * 32 * 32,), dtype=torch.int64, device="cuda")
op = _capi.conv_operand(_capi.GATHER_IM2COL, nb * 100, 363, nb, 3, 32, 32, (3 * 1024, 1024, 32, 1), 11, 11, 4, 4, 9, 9, 10, 10)
kh, kp = 368, 736
out = torch.empty(3 * 8 * nb * 100 * kp, dtype=torch.uint8, device="cuda")
t = graph_us(lambda: _capi.call("mpc3_ring_pack_halves", p(x), nb * 3 * 1024, C.byref(op), 1, p(out), kp, kh, st()), reps=5)
print(f"conv1 pack {t:.1f} us  {out.numel() / t / 1e6:.2f} TB/s written")
