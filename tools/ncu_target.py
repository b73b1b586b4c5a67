"""Launch one kernel a few times for an `ncu --set full` capture.

python tools/ncu_target.py gemm 4096      # mpc3_ring_gemm_packed, M=N=K=n (packed limb planes)
python tools/ncu_target.py gemm_mn 4096   # the same product with A read MN-major (the engine's forward layout)
python tools/ncu_target.py sign 16777216  # fused sign/ReLU circuit on n elements
python tools/ncu_target.py reshare 884736 # reshare + truncate of n cross terms (an AlexNet wgrad epilogue)
python tools/ncu_target.py sgd 0          # the AlexNet step's SGD over all parameters (one launch)
python tools/ncu_target.py poolbwd 128    # AlexNet conv1's avg-pool backward + ReLU mask at batch n
python tools/ncu_target.py layersign 128  # AlexNet conv1's fused reshare + truncate + ReLU at batch n
python tools/ncu_target.py pack 4096      # dense cross-term pack, 3 parties, M=K=n
python tools/ncu_target.py wgrad 128      # transposed-operand GEMM, AlexNet conv5 weight gradient (R=n)
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_10949_b200 import _capi  # noqa: E402
from tools.microbench import p, rk3, st  # noqa: E402


def main(kind, n, reps=3):
    if kind == "gemm":
        kp = (n + 15) // 16 * 16
        A = torch.randint(0, 256, (8 * n * kp,), dtype=torch.uint8, device="cuda")
        B = torch.randint(0, 256, (8 * n * kp,), dtype=torch.uint8, device="cuda")
        Cm = torch.empty(n * n, dtype=torch.int64, device="cuda")
        for _ in range(reps):
            _capi.call("mpc3_ring_gemm_packed", p(A), p(B), p(Cm), 1, n, n, kp, n, 0, 1, st())
    elif kind == "gemm_mn":  # the engine's forward layout: A read MN-major from a transposed pack
        kc = n // 2
        At = torch.randint(0, 256, (8 * kc * 2 * n,), dtype=torch.uint8, device="cuda")
        B = torch.randint(0, 256, (8 * n * n,), dtype=torch.uint8, device="cuda")
        Cm = torch.empty(n * n, dtype=torch.int64, device="cuda")
        for _ in range(reps):
            _capi.call("mpc3_ring_gemm_t", p(At), 1, kc, 2 * n, n, p(B), 0, n, n, 0, p(Cm), 1, n, n, kc, 0, st())
    elif kind == "reshare":  # reshare + truncate of n cross terms (a layer epilogue), row-major view
        rk = rk3()
        z = torch.randint(-(1 << 62), 1 << 62, (3 * n,), dtype=torch.int64, device="cuda")
        out = torch.empty_like(z)
        v = _capi.make_view((1, 1, n // 256, 256))
        for _ in range(reps):
            _capi.call("mpc3_rss_reshare_truncate", p(rk), None, 0, 0, 0, 20, p(z), C.byref(v), p(out), 0, st())
    elif kind == "sgd":  # the AlexNet-CIFAR step's one-launch SGD over every parameter (n unused)
        import paper_2104_10949_b200 as M
        sess = M.TrioSession(seed=0)
        params = [sess.share(w, __import__("numpy").random.default_rng(1)) for w in
                  M.init_params(M.alexnet_cifar(), seed=0)]
        grads = [M.engine.RssTensor(p.data.clone()) for p in params]
        for _ in range(reps):
            sess.sgd_inplace(params, grads, 3)
    elif kind == "poolbwd":  # AlexNet conv1's avg-pool backward + ReLU mask (batch n), one launch
        rk = rk3()
        N, Cc, H, W, OH, OW = n, 96, 10, 10, 4, 4
        g = torch.randint(-(1 << 40), 1 << 40, (3 * N * Cc * OH * OW,), dtype=torch.int64, device="cuda")
        m = torch.randint(0, 2, (3 * N * Cc * H * W,), dtype=torch.int64, device="cuda")
        out = torch.empty_like(m)
        for _ in range(reps):
            _capi.call("mpc3_rss_avgpool_backward_mask", p(rk), None, 0, 0, 20, 7282, p(g), p(m), 0, p(out), N, Cc, H, W,
                       OH, OW, 3, 3, 2, 2, 0, 0, 0, st())
    elif kind == "sign":
        rk = rk3()
        x = torch.randint(-(1 << 40), 1 << 40, (3 * n,), dtype=torch.int64, device="cuda")
        y, m = torch.empty_like(x), torch.empty_like(x)
        for _ in range(reps):
            _capi.call("mpc3_rss_sign", p(rk), None, 3, 0, 0, 0, p(x), p(y), p(m), n, n, 0, st())
    elif kind == "layersign":  # AlexNet conv1's fused reshare + truncate + ReLU (batch n): column-major z view
        rk = rk3()
        nb, o, oh, ow = n, 96, 10, 10
        m = nb * oh * ow
        z = torch.randint(-(1 << 62), 1 << 62, (3 * nb * o * oh * ow,), dtype=torch.int64, device="cuda")
        y, mk = torch.empty_like(z), torch.empty_like(z)
        v = _capi.make_view((nb, o, oh, ow), z_stride=(oh * ow, m, ow, 1))
        for _ in range(reps):
            _capi.call("mpc3_rss_layer_sign", p(rk), None, 1, 2, 3, 20, p(z), C.byref(v), None, 0, 1, 3, 4, 5, 6,
                       p(y), p(mk), 0, nb * o * oh * ow, st())
    elif kind == "pack":
        x = torch.randint(-(1 << 62), 1 << 62, (3 * n * n,), dtype=torch.int64, device="cuda")
        kp = 2 * n
        out = torch.empty(3 * 8 * n * kp, dtype=torch.uint8, device="cuda")
        op = _capi.Operand()
        op.mode, op.rows, op.k, op.s_r, op.t2 = 0, n, n, n, 1
        for _ in range(reps):
            _capi.call("mpc3_ring_pack", p(x), n * n, C.byref(op), 0, p(out), kp, st())
    elif kind == "pack_conv1":  # AlexNet conv1 im2col pack: x (n,3,32,32), 11x11 stride 4 pad 9, role 1
        nb = n
        x = torch.randint(-(1 << 62), 1 << 62, (3 * nb * 3 * 32 * 32,), dtype=torch.int64, device="cuda")
        op = _capi.conv_operand(_capi.GATHER_IM2COL, nb * 100, 363, nb, 3, 32, 32, (3 * 1024, 1024, 32, 1), 11, 11,
                                4, 4, 9, 9, 10, 10)
        kh, kp = 368, 736
        out = torch.empty(3 * 8 * nb * 100 * kp, dtype=torch.uint8, device="cuda")
        for _ in range(reps):
            _capi.call("mpc3_ring_pack_halves", p(x), nb * 3 * 1024, C.byref(op), 1, p(out), kp, kh, st())
    elif kind == "mul":  # RSS mul (reshare), n elements
        rk = rk3()
        x = torch.randint(-(1 << 62), 1 << 62, (3 * n,), dtype=torch.int64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(reps):
            _capi.call("mpc3_rss_mul", p(rk), None, 0, p(x), p(x), p(y), n, 0, st())
    elif kind == "wgrad":  # M = 256 (O), N = 2304 (C*3*3), contraction R = n rows, MN-read packs
        M, N, R = 256, 2304, n
        kc = (R + 31) // 32 * 32
        kha, khb = M, N
        kpa, kpb = 2 * M, 2 * N
        A = torch.randint(0, 256, (3 * 8 * R * kpa,), dtype=torch.uint8, device="cuda")
        B = torch.randint(0, 256, (3 * 8 * R * kpb,), dtype=torch.uint8, device="cuda")
        Cm = torch.empty(3 * M * N, dtype=torch.int64, device="cuda")
        for _ in range(reps):
            _capi.call("mpc3_ring_gemm_t", p(B), 1, R, kpb, khb, p(A), 1, R, kpa, kha, p(Cm), 3, N, M, kc, 1, st())
    else:
        raise SystemExit(f"unknown kernel {kind}")
    torch.cuda.synchronize()
    print("ok", kind, n)


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
