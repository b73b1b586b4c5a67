"""Raw cross-term products of the AlexNet conv1 weight gradient: split-K variants vs oracle."""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_10949_b200 import _capi as K  # noqa: E402
from paper_2104_10949_b200 import engine as E  # noqa: E402
from oracle import nnmirror as N  # noqa: E402
from oracle import rss as R  # noqa: E402

U64 = np.uint64
rng = np.random.default_rng(3)
nb, c, h, w, o, kh, kw, sh, ph = 4, 3, 32, 32, 96, 11, 11, 4, 9
oh = (h + 2 * ph - kh) // sh + 1
x = rng.integers(0, 1 << 64, (3, nb, c, h, w), dtype=U64)
g = rng.integers(0, 1 << 64, (3, nb, o, oh, oh), dtype=U64)


class Raw:
    t = 20

    def shape(self, v):
        return v.shape[1:]

    def map_structural(self, v, f):
        return np.stack([f(v[i]) for i in range(3)])

    def conv2d(self, a, b, stride, padding, bits=None):
        return R._bilinear3(lambda p, q: R.wrap_conv2d(p, q, stride, padding), a, b)


ref = N.conv_grad_kernel(Raw(), x, g, N.conv(o, kh, sh, ph), 20)  # (3, o, c, kh, kw)
xd, gd = E.to_device(x), E.to_device(g)
Kd = nb * oh * oh
a_op = K.conv_operand(K.GATHER_WGRAD, c * kh * kw, Kd, nb, c, h, w, xd.stride()[1:], kh, kw, sh, sh, ph, ph, oh, oh)
gs = gd.stride()
b_op = K.dense_operand(o, Kd, s_r=gs[2], t0=gs[1], t1=gs[3], t2=gs[4], K1=oh, K2=oh)
kp = E._round_up(2 * Kd, 16)
M, Nn = c * kh * kw, o
A = torch.empty(3 * 8 * M * kp, dtype=torch.uint8, device="cuda")
B = torch.empty(3 * 8 * Nn * kp, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
import ctypes as C  # noqa: E402

K.call("mpc3_ring_pack", xd.data_ptr(), xd.stride(0), C.byref(a_op), 0, A.data_ptr(), kp, st)
K.call("mpc3_ring_pack", gd.data_ptr(), gd.stride(0), C.byref(b_op), 1, B.data_ptr(), kp, st)
for splits in (1, 2, 3, 5):
    z = torch.zeros(3 * M * Nn, dtype=torch.int64, device="cuda")
    K.call("mpc3_ring_gemm_packed", A.data_ptr(), B.data_ptr(), z.data_ptr(), 3, M, Nn, kp, Nn, M * Nn, splits, st)
    zz = z.cpu().numpy().view(U64).reshape(3, c, kh, kw, o).transpose(0, 4, 1, 2, 3)
    bad = zz != ref
    print("splits", splits, "mismatch", int(bad.sum()), "of", bad.size,
          "parties", [int(bad[i].sum()) for i in range(3)], flush=True)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        print(" first", idx.tolist())
# groups=1 plain with splits
for splits in (1, 3):
    z = torch.zeros(M * Nn, dtype=torch.int64, device="cuda")
    K.call("mpc3_ring_gemm_packed", A.data_ptr(), B.data_ptr(), z.data_ptr(), 1, M, Nn, kp, Nn, M * Nn, splits, st)
    z1 = torch.zeros(M * Nn, dtype=torch.int64, device="cuda")
    K.call("mpc3_ring_gemm_packed", A.data_ptr(), B.data_ptr(), z1.data_ptr(), 1, M, Nn, kp, Nn, M * Nn, 1, st)
    print("group0 splits", splits, "equal to splits=1:", bool(torch.equal(z, z1)))
