"""ctypes access to the CPU self-check build of the device logic (tests only)."""

import ctypes as C
import os

import numpy as np

from paper_2104_10949_b200 import _capi

PATH = os.path.join(os.path.dirname(_capi.LIB_PATH), "libmpc3hostcheck.so")
_h = None


def lib():
    global _h
    if _h is None:
        _h = C.CDLL(PATH)
    return _h


def ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def keys48(keys):
    return C.c_char_p(b"".join(keys))


def prf_words(key, purpose, index, off, count):
    out = np.zeros(count, np.uint64)
    lib().hc_prf_words(C.c_char_p(key), C.c_uint32(purpose), C.c_uint64(index), C.c_uint64(off),
                       C.c_uint64(count), ptr(out))
    return out


def zero_share(keys, purpose, index, xor_mode, n):
    out = np.zeros((3, n), np.uint64)
    lib().hc_zero_share(keys48(keys), C.c_uint32(purpose), C.c_uint64(index), C.c_int(xor_mode),
                        C.c_uint64(n), ptr(out))
    return out


def arith(keys, kind, ja, jrho, jr, bits, x, y=None):
    x = np.ascontiguousarray(x, np.uint64)
    n = x.size // 3
    y = x if y is None else np.ascontiguousarray(y, np.uint64)
    out = np.zeros_like(x)
    lib().hc_arith(keys48(keys), C.c_int(kind), C.c_uint64(ja), C.c_uint64(jrho), C.c_uint64(jr),
                   C.c_int(bits), ptr(x), ptr(y), ptr(out), C.c_uint64(n))
    return out


def sign(keys, mode, jbin, jxor, ja, x, n_total=None, off=0):
    x = np.ascontiguousarray(x, np.uint64)
    n = x.size // 3
    out = np.zeros_like(x)
    mask = np.zeros_like(x)
    lib().hc_sign(keys48(keys), C.c_int(mode), C.c_uint64(jbin), C.c_uint64(jxor), C.c_uint64(ja),
                  ptr(x), ptr(out), ptr(mask), C.c_uint64(n), C.c_uint64(n if n_total is None else n_total),
                  C.c_uint64(off))
    return out, mask


def inject(keys, ja, bits):
    bits = np.ascontiguousarray(bits, np.uint64)
    out = np.zeros_like(bits)
    lib().hc_inject(keys48(keys), C.c_uint64(ja), ptr(bits), ptr(out), C.c_uint64(bits.size // 3))
    return out


def reshare_truncate(keys, ja, jrho, jr, bits, z, view, out_shape):
    z = np.ascontiguousarray(z, np.uint64)
    out = np.zeros(out_shape, np.uint64)
    lib().hc_reshare_truncate(keys48(keys), C.c_uint64(ja), C.c_uint64(jrho), C.c_uint64(jr), C.c_int(bits),
                              ptr(z), C.byref(view), ptr(out))
    return out


def pool(keys, backward, jrho, jr, bits, mulc, x, N, Cc, H, W, OH, OW, kh, kw, sh, sw, ph=0, pw=0):
    x = np.ascontiguousarray(x, np.uint64)
    n = N * Cc * (H * W if backward else OH * OW)
    out = np.zeros((3, n), np.uint64)
    lib().hc_pool(keys48(keys), C.c_int(backward), C.c_uint64(jrho), C.c_uint64(jr), C.c_int(bits),
                  C.c_uint64(mulc), ptr(x), ptr(out), C.c_int64(N), C.c_int64(Cc), C.c_int64(H), C.c_int64(W),
                  C.c_int64(OH), C.c_int64(OW), C.c_int(kh), C.c_int(kw), C.c_int(sh), C.c_int(sw),
                  C.c_int(ph), C.c_int(pw))
    return out


def pack(src, plane, op, role, kp, kh=-1):
    """kh: first packed column of the second half (-1: K, the adjacent layout)."""
    src = np.ascontiguousarray(src, np.uint64)
    groups = 1 if role == 2 else 3
    out = np.zeros((groups, 8, op.rows, kp), np.uint8)
    lib().hc_pack(ptr(src), C.c_int64(plane), C.byref(op), C.c_int(role), ptr(out), C.c_int64(kp), C.c_int64(kh))
    return out


def gemm_packed(A, B, split_k=16384):
    groups, _, M, kp = A.shape
    N = B.shape[2]
    Cm = np.zeros((groups, M, N), np.uint64)
    lib().hc_gemm_packed(ptr(A), ptr(B), ptr(Cm), C.c_int(groups), C.c_int64(M), C.c_int64(N), C.c_int64(kp),
                         C.c_int64(N), C.c_int64(M * N), C.c_int64(split_k))
    return Cm


def col2im(keys, ja, jrho, jr, bits, z, N, Cc, OH, OW, kh, kw, sh, sw, ph, pw, H, W):
    z = np.ascontiguousarray(z, np.uint64)
    out = np.zeros((3, N, Cc, H, W), np.uint64)
    lib().hc_col2im(keys48(keys), C.c_uint64(ja), C.c_uint64(jrho), C.c_uint64(jr), C.c_int(bits), ptr(z),
                    C.c_int64(N), C.c_int64(Cc), C.c_int64(OH), C.c_int64(OW), C.c_int(kh), C.c_int(kw), C.c_int(sh),
                    C.c_int(sw), C.c_int(ph), C.c_int(pw), C.c_int64(H), C.c_int64(W), ptr(out))
    return out
