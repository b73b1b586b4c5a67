"""Time the operand packs of the AlexNet-CIFAR step (graph-replayed, warm)."""
import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import torch
from paper_2104_10949_b200 import _capi
from tools.microbench import graph_us, p, st


def run(name, src, plane, op, role, kp, kh):
    out = torch.empty(3 * 8 * op.rows * kp, dtype=torch.uint8, device="cuda")
    t = graph_us(lambda: _capi.call("mpc3_ring_pack_halves", p(src), plane, C.byref(op), role, p(out), kp, kh, st()),
                 reps=5)
    print(f"{name:28s} {t:7.1f} us  {out.numel() / t / 1e6:5.2f} TB/s written  ({out.numel() / 1e6:.0f} MB)", flush=True)


def r16(v):
    return (v + 15) // 16 * 16


nb = 128
x = torch.randint(-(1 << 62), 1 << 62, (3 * nb * 3 * 32 * 32,), dtype=torch.int64, device="cuda")
op = _capi.conv_operand(_capi.GATHER_IM2COL, nb * 100, 363, nb, 3, 32, 32, (3 * 1024, 1024, 32, 1), 11, 11, 4, 4, 9, 9, 10, 10)
run("conv1 x im2col s4 role1", x, nb * 3 * 1024, op, 1, 736, 368)
# conv2: input (128, 96, 4, 4), 5x5 pad 1 -> 2x2
x2 = torch.randint(-(1 << 62), 1 << 62, (3 * nb * 96 * 16,), dtype=torch.int64, device="cuda")
op = _capi.conv_operand(_capi.GATHER_IM2COL, nb * 4, 2400, nb, 96, 4, 4, (96 * 16, 16, 4, 1), 5, 5, 1, 1, 1, 1, 2, 2)
run("conv2 x im2col s1 role1", x2, nb * 96 * 16, op, 1, r16(r16(2400) + 2400), r16(2400))
# conv4 weights (384, 384, 3, 3) role 0
w = torch.randint(-(1 << 62), 1 << 62, (3 * 384 * 3456,), dtype=torch.int64, device="cuda")
op = _capi.dense_operand(384, 3456, s_r=3456, t0=9, t1=3, t2=1, K1=3, K2=3)
run("conv4 W dense role0", w, 384 * 3456, op, 0, r16(r16(3456) + 3456), r16(3456))
# conv1 g (128, 96, 10, 10) role 0 (im2col 1x1)
g = torch.randint(-(1 << 62), 1 << 62, (3 * nb * 96 * 100,), dtype=torch.int64, device="cuda")
op = _capi.conv_operand(_capi.GATHER_IM2COL, nb * 100, 96, nb, 96, 10, 10, (9600, 100, 10, 1), 1, 1, 1, 1, 0, 0, 10, 10)
run("conv1 g role0 (wgrad)", g, nb * 9600, op, 0, r16(r16(96) + 96), r16(96))
run("conv1 g role1 K-major halves", g, nb * 9600, op, 1, 2 * 128, 128)
