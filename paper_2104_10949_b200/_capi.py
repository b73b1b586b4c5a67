"""ctypes binding of the C ABI declared in include/mpc3_b200.h.

The shared library `libmpc3b200.so` is built in-tree (`make`, or
`__graft_entry__.build()`); there is no fallback: every compute call goes
through it, and loading fails loudly if it is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import errors as E

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpc3b200.so")

OK = 0
_STATUS_EXC = {
    1: E.RangeError,
    2: E.ShapeError,
    3: E.ExactnessError,
    4: E.ConfigError,
    5: E.FreshnessError,
    6: E.TopologyError,
    7: E.IntegrityError,
}

EW_ADD, EW_SUB, EW_NEG, EW_MULC, EW_ADDC, EW_XOR, EW_SHL, EW_SHR, EW_SAR, EW_AXPY = range(10)
GATHER_DENSE, GATHER_IM2COL, GATHER_WGRAD = 0, 1, 2
MODE_A2B, MODE_MSB, MODE_DRELU, MODE_RELU = 0, 1, 2, 3


class View4(C.Structure):
    _fields_ = [
        ("full", C.c_int64 * 4),
        ("origin", C.c_int64 * 4),
        ("crop", C.c_int64 * 4),
        ("z_stride", C.c_int64 * 4),
        ("out_stride", C.c_int64 * 4),
        ("z_plane", C.c_int64),
        ("out_plane", C.c_int64),
    ]


class Operand(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "rows", "k", "off", "s_r", "t0", "t1", "t2", "K1", "K2",
        "n", "c", "h", "w", "sN", "sC", "sH", "sW",
        "kh", "kw", "sh", "sw", "ph", "pw", "dh", "dw", "oh", "ow")]
    _fields_ = [("mode", C.c_int)] + _fields_


class SgdTensor(C.Structure):
    """MPC3SgdTensor (include/mpc3_b200.h)."""
    _fields_ = [("param", C.c_void_p), ("grad", C.c_void_p), ("n", C.c_uint64), ("j_rho", C.c_uint64),
                ("j_r", C.c_uint64)]


SGD_MAX_TENSORS = 64


class ChainStep(C.Structure):
    """MPC3ChainStep (include/mpc3_b200.h): one step of a fused elementwise chain."""
    _fields_ = [("op", C.c_int), ("bits", C.c_int), ("c", C.c_uint64)]


class SoftmaxLossArgs(C.Structure):
    """mpc3_softmax_loss_args (include/mpc3_b200.h)."""
    _fields_ = [("levels", C.c_int), ("j_bin", C.c_uint64 * 16), ("j_xor", C.c_uint64 * 16),
                ("j_arith", C.c_uint64 * 16), ("exp_j", C.c_uint64 * 3), ("exp_steps", C.POINTER(ChainStep)),
                ("exp_count", C.c_int), ("rec_j", C.c_uint64 * 3), ("rec_steps", C.POINTER(ChainStep)),
                ("rec_count", C.c_int), ("fin_j", C.c_uint64 * 3), ("bits", C.c_int), ("row_off", C.c_uint64),
                ("rows_total", C.c_uint64)]


CHAIN_ADDC, CHAIN_SETC, CHAIN_SQ, CHAIN_MULX, CHAIN_NEWTON, CHAIN_SQT = range(6)
CHAIN_MAX_STEPS = 48


def chain_program(steps):
    """[(op, bits, c), ...] -> (ctypes array, count)."""
    arr = (ChainStep * max(1, len(steps)))()
    for i, (op, bits, c) in enumerate(steps):
        arr[i].op, arr[i].bits, arr[i].c = int(op), int(bits), int(c) % (1 << 64)
    return arr, len(steps)


def make_view(full, crop=None, z_stride=None, out_stride=None, z_plane=None, out_plane=None,
              origin=None) -> View4:
    full = [int(v) for v in full]
    while len(full) < 4:
        full.insert(0, 1)
    crop = full if crop is None else [int(v) for v in crop]
    while len(crop) < 4:
        crop.insert(0, 1)
    org = [0, 0, 0, 0] if origin is None else [int(v) for v in origin]
    while len(org) < 4:
        org.insert(0, 0)

    def cstrides(shape):
        s, acc = [0] * 4, 1
        for k in range(3, -1, -1):
            s[k] = acc
            acc *= shape[k]
        return s

    zs = cstrides(full) if z_stride is None else list(z_stride)
    os_ = cstrides(crop) if out_stride is None else list(out_stride)
    while len(zs) < 4:
        zs.insert(0, 0)
    while len(os_) < 4:
        os_.insert(0, 0)
    n_full = full[0] * full[1] * full[2] * full[3]
    n_crop = crop[0] * crop[1] * crop[2] * crop[3]
    v = View4()
    v.full[:] = full
    v.origin[:] = org
    v.crop[:] = crop
    v.z_stride[:] = zs
    v.out_stride[:] = os_
    v.z_plane = n_full if z_plane is None else int(z_plane)
    v.out_plane = n_crop if out_plane is None else int(out_plane)
    return v


def dense_operand(rows, k, s_r, t2, off=0, t0=0, t1=0, K1=1, K2=None) -> Operand:
    o = Operand()
    o.mode = GATHER_DENSE
    o.rows, o.k, o.off, o.s_r = int(rows), int(k), int(off), int(s_r)
    o.t0, o.t1, o.t2 = int(t0), int(t1), int(t2)
    o.K1 = int(K1)
    o.K2 = int(k) if K2 is None else int(K2)
    if K2 is None:  # plain 2-d view: k is a single digit of stride t2
        o.K1, o.K2, o.t0, o.t1 = 1, int(k), 0, 0
    return o


def conv_operand(mode, rows, k, n, c, h, w, strides, kh, kw, sh, sw, ph, pw, oh, ow, dh=1, dw=1) -> Operand:
    o = Operand()
    o.mode = mode
    o.rows, o.k = int(rows), int(k)
    o.n, o.c, o.h, o.w = int(n), int(c), int(h), int(w)
    o.sN, o.sC, o.sH, o.sW = (int(s) for s in strides)
    o.kh, o.kw, o.sh, o.sw = int(kh), int(kw), int(sh), int(sw)
    o.ph, o.pw, o.dh, o.dw, o.oh, o.ow = int(ph), int(pw), int(dh), int(dw), int(oh), int(ow)
    return o


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_U64 = C.c_uint64
_I64 = C.c_int64
_SIGS = {
    "mpc3_abi_version": (C.c_int, []),
    "mpc3_status_name": (C.c_char_p, [C.c_int]),
    "mpc3_last_error": (C.c_char_p, []),
    "mpc3_aes128_expand": (C.c_int, [C.c_char_p, _P]),
    "mpc3_prf_words": (C.c_int, [_P, C.c_uint32, _U64, _U64, _U64, _P, _P]),
    "mpc3_rss_zero_share": (C.c_int, [_P, _P, C.c_uint32, _U64, C.c_int, _U64, _P, _P]),
    "mpc3_fx_encode": (C.c_int, [_P, _P, _U64, C.c_int, _P, _P]),
    "mpc3_deal_pcg64": (C.c_int, [_U64, _U64, _U64, _U64, _P, _P, _U64, _P]),
    "mpc3_ring_ew": (C.c_int, [C.c_int, _P, _P, _U64, _P, _U64, _P]),
    "mpc3_ring_rowop": (C.c_int, [C.c_int, _P, _P, _P, _U64, _U64, _P]),
    "mpc3_ring_rowsum": (C.c_int, [_P, _P, _U64, _U64, _P]),
    "mpc3_rss_mul": (C.c_int, [_P, _P, _U64, _P, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_truncate": (C.c_int, [_P, _P, _U64, _U64, C.c_int, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_mul_truncate": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_sign": (C.c_int, [_P, _P, C.c_int, _U64, _U64, _U64, _P, _P, _P, _U64, _U64, _U64, _P]),
    "mpc3_rss_max_tree": (C.c_int, [_P, _P, C.c_int, _P, _P, _P, _P, _P, _P, _U64, _U64, _U64, _U64, _P]),
    "mpc3_rss_layer_sign": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, C.POINTER(View4), _P, _I64, C.c_int,
                                      C.c_int, _U64, _U64, _U64, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_layer_sign_residual": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, C.POINTER(View4), _P, _I64,
                                               C.c_int, _P, _I64, C.c_int, _U64, _U64, _U64, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_sgd_multi": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _U64, _P]),
    "mpc3_rss_softmax_loss_scratch": (C.c_size_t, [_U64, _U64]),
    "mpc3_rss_softmax_loss": (C.c_int, [_P, _P, _P, _P, _P, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_max_level": (C.c_int, [_P, _P, _U64, _U64, _U64, _P, _P, _U64, _U64, _U64, _U64, _P]),
    "mpc3_rss_chain": (C.c_int, [_P, _P, _P, C.c_int, _U64, _U64, _U64, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_bit_inject": (C.c_int, [_P, _P, _U64, _P, _P, _U64, _U64, _P]),
    "mpc3_rss_reshare_truncate": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, C.POINTER(View4), _P, _U64,
                                            _P]),
    "mpc3_rss_reshare_truncate_bias": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, C.POINTER(View4), _P, _I64,
                                                 C.c_int, _P, _U64, _P]),
    "mpc3_rss_avgpool": (C.c_int, [_P, _P, _U64, _U64, C.c_int, _U64, _P, _P, _I64, _I64, _I64, _I64,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _U64, _P]),
    "mpc3_rss_avgpool_backward": (C.c_int, [_P, _P, _U64, _U64, C.c_int, _U64, _P, _P, _I64, _I64, _I64, _I64,
                                            _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _U64,
                                            _P]),
    "mpc3_rss_avgpool_backward_mask": (C.c_int, [_P, _P, _U64, _U64, C.c_int, _U64, _P, _P, _U64, _P, _I64, _I64,
                                                 _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                 C.c_int, _U64, _P]),
    "mpc3_rss_col2im_reshare_truncate": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, _I64, _I64, _I64, _I64,
                                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _I64,
                                                   _I64, _P, _U64, _P]),
    "mpc3_rss_col2im_reshare_truncate_layout": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, C.c_int, _I64, _I64,
                                                          _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                                          C.c_int, _I64, _I64, _P, _U64, _P]),
    "mpc3_rss_window_gather": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_int, _U64, _P]),
    "mpc3_ring_sumpool": (C.c_int, [_P, _P, _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_int, _P]),
    "mpc3_ring_pack": (C.c_int, [_P, _I64, C.POINTER(Operand), C.c_int, _P, _I64, _P]),
    "mpc3_ring_pack_halves": (C.c_int, [_P, _I64, C.POINTER(Operand), C.c_int, _P, _I64, _I64, _P]),
    "mpc3_ring_pack_halves_z": (C.c_int, [_P, _I64, C.POINTER(Operand), C.c_int, _P, _I64, _I64, _P, _I64, _P]),
    "mpc3_ring_gemm_needs_zero": (C.c_int, [C.c_int, C.c_int, _I64, _I64, _I64]),
    "mpc3_ring_gemm_auto_z": (C.c_int, [_P, _P, _P, C.c_int, _I64, _I64, _I64, C.c_int, C.c_int, _P]),
    "mpc3_ring_gemm_t_z": (C.c_int, [_P, C.c_int, _I64, _I64, _I64, _P, C.c_int, _I64, _I64, _I64, _P, C.c_int, _I64,
                                     _I64, _I64, C.c_int, C.c_int, _P]),
    "mpc3_ring_gemm_packed": (C.c_int, [_P, _P, _P, C.c_int, _I64, _I64, _I64, _I64, _I64, C.c_int, _P]),
    "mpc3_ring_gemm_auto": (C.c_int, [_P, _P, _P, C.c_int, _I64, _I64, _I64, C.c_int, _P]),
    "mpc3_ring_gemm_t": (C.c_int, [_P, C.c_int, _I64, _I64, _I64, _P, C.c_int, _I64, _I64, _I64, _P, C.c_int, _I64,
                                   _I64, _I64, C.c_int, _P]),
    "mpc3_ring_gemm_packed_layout": (C.c_int, [_P, _P, _P, C.c_int, _I64, _I64, _I64, _I64, _I64, C.c_int, C.c_int,
                                               _P]),
    "mpc3_ring_gemm_simt": (C.c_int, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P]),
    "mpc3_ring_matmul_workspace": (C.c_size_t, [_I64, _I64, _I64]),
    "mpc3_ring_matmul_u64": (C.c_int, [_P, _P, _P, _I64, _I64, _I64, _P, _P]),
    "mpc3_ring_conv2d_workspace": (C.c_size_t, [_I64, _I64, _I64, _I64, _I64] + [C.c_int] * 6),
    "mpc3_ring_conv2d_u64": (C.c_int, [_P, _P, _P, _I64, _I64, _I64, _I64, _I64] + [C.c_int] * 6 + [_P, _P]),
    "mpc3_rss_matmul_workspace": (C.c_size_t, [_I64, _I64, _I64]),
    "mpc3_rss_matmul_reshare_trunc": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, _P, _P, _I64, _I64, _I64, _P,
                                                _P]),
    "mpc3_rss_conv2d_workspace": (C.c_size_t, [_I64, _I64, _I64, _I64, _I64] + [C.c_int] * 6),
    "mpc3_rss_conv2d_reshare_trunc": (C.c_int, [_P, _P, _U64, _U64, _U64, C.c_int, _P, _P, _P, _I64, _I64, _I64, _I64,
                                                _I64] + [C.c_int] * 6 + [_P, _P]),
}
EXPORTED = tuple(_SIGS)


def lib():
    """The loaded engine library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise E.ConfigError(
                        f"CUDA engine library missing: {LIB_PATH} (run `make` or __graft_entry__.build())")
                h = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    f = getattr(h, name)
                    f.restype = res
                    f.argtypes = args
                if h.mpc3_abi_version() != 1:
                    raise E.ConfigError("engine library ABI mismatch")
                _lib = h
    return _lib


class CudaError(E.Mpc3Error, RuntimeError):
    """A CUDA launch or runtime failure inside the engine library."""


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    exc = _STATUS_EXC.get(status)
    msg = f"{what}: {lib().mpc3_status_name(status).decode()}"
    if exc is None:
        raise CudaError(msg + f" ({lib().mpc3_last_error().decode()})")
    raise exc(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)
