"""Per-CTA phase timeline of one gemm_tc_kernel launch (globaltimer, debug build).

python tools/dbg/gemm_trace.py build     # here: nvcc the traced library variant
python tools/dbg/gemm_trace.py M N R G   # on the GPU box
"""
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
LIB = os.path.join(ROOT, "tools", "dbg", "libmpc3trace.so")


def build():
    src = os.path.join(ROOT, "paper_2104_10949_b200", "csrc")
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-Xcompiler", "-fPIC"]
    obj = "/tmp/gemm_trace.o"
    subprocess.check_call(["nvcc", *flags, "-DMPC3_GEMM_TRACE", "-c", "-o", obj, os.path.join(src, "gemm.cu")])
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, obj,
                           os.path.join(ROOT, "build", "elementwise.o"), os.path.join(ROOT, "build", "deal.o")])


def run(M, N, R, G):
    import numpy as np
    import torch

    lib = C.CDLL(LIB)
    P, I64, INT = C.c_void_p, C.c_int64, C.c_int
    lib.mpc3_ring_gemm_t.argtypes = [P, INT, I64, I64, I64, P, INT, I64, I64, I64, P, INT, I64, I64, I64, INT, P]
    kc = (R + 31) // 32 * 32
    kpa, kpb = 2 * M, 2 * N
    A = torch.randint(0, 256, (G * 8 * R * kpa,), dtype=torch.uint8, device="cuda")
    B = torch.randint(0, 256, (G * 8 * R * kpb,), dtype=torch.uint8, device="cuda")
    Cm = torch.empty(G * M * N, dtype=torch.int64, device="cuda")
    for _ in range(5):
        assert lib.mpc3_ring_gemm_t(A.data_ptr(), 1, R, kpa, M, B.data_ptr(), 1, R, kpb, N, Cm.data_ptr(), G, M, N,
                                    kc, 1, None) == 0
    torch.cuda.synchronize()
    tr = np.zeros((8192, 8), np.uint64)
    lib.mpc3_debug_gemm_trace(tr.ctypes.data_as(C.c_void_p))
    ctas = ((M + 127) // 128) * ((N + 63) // 64) * G
    t = tr[:ctas, :6].astype(np.int64)
    t0 = t[:, 0].min()
    t = t - t0
    names = ["start", "after griddep_wait", "first stage full", "mma done", "epilogue done", "cta end"]
    print(f"M={M} N={N} R={R} G={G}: {ctas} CTAs, span {t[:, 5].max() / 1e3:.2f} us")
    for i, n in enumerate(names):
        print(f"  {n:20s} median {np.median(t[:, i]) / 1e3:7.2f} us  min {t[:, i].min() / 1e3:7.2f}  "
              f"max {t[:, i].max() / 1e3:7.2f}")
    d = np.diff(t, axis=1)
    for i in range(5):
        print(f"  phase {names[i]} -> {names[i + 1]}: median {np.median(d[:, i]) / 1e3:6.2f} us")


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build()
    else:
        run(*map(int, sys.argv[1:5]))
