"""Z_2^64 ring helpers and the exact bilinear entry point.

Host-side helpers keep the reference's semantics (ring.py:38-141): ring
tensors are numpy uint64 with wrapping arithmetic, reals are fixed point with
t fractional bits.  `bilinear_exact` (ring.py:183-200) keeps its contract —
same specs, same 2^20 accumulation refusal, same result bits — but runs on
the B200 ring GEMM (tcgen05 int8 limbs) instead of float64 limb dgemms.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

import numpy as np

from .errors import ExactnessError, RangeError, ShapeError

RING_BITS = 64
LIMB_BITS = 16
NUM_LIMBS = 4
MAX_ACCUMULATION = 1 << 20
U64 = np.uint64

# reference limb schedule, kept for API parity (ring.py:30-35); the device
# engine uses 8 byte limbs and 36 pairs instead (csrc/gemm.cu)
LIMB_PAIRS: tuple[tuple[int, int], ...] = tuple(
    (i, j) for i in range(NUM_LIMBS) for j in range(NUM_LIMBS - i)
)


def as_ring(x: Any) -> np.ndarray:
    """Any integer (array) as uint64 ring elements, python ints reduced mod 2^64."""
    if isinstance(x, np.ndarray) and x.dtype == U64:
        return x
    if isinstance(x, (int, np.integer)):
        return np.asarray(int(x) % (1 << 64), dtype=U64)
    arr = np.asarray(x)
    if arr.dtype == object or arr.dtype.kind not in "ui":
        raise ShapeError(f"dtype {arr.dtype} is not a ring tensor")
    return arr.astype(U64)


def to_signed(a) -> np.ndarray:
    return np.asarray(a, dtype=U64).view(np.int64)


def _bcast(a, b):
    try:
        np.broadcast_shapes(np.shape(a), np.shape(b))
    except ValueError as e:
        raise ShapeError(str(e)) from None


def ring_add(a, b):
    a, b = as_ring(a), as_ring(b)
    _bcast(a, b)
    return a + b


def ring_sub(a, b):
    a, b = as_ring(a), as_ring(b)
    _bcast(a, b)
    return a - b


def ring_neg(a):
    return U64(0) - as_ring(a)


def ring_scalar_mul(a, c: int):
    return as_ring(a) * U64(int(c) % (1 << 64))


def ring_shift_arith(a, bits: int):
    if not 0 <= bits < 64:
        raise RangeError(f"shift {bits} not in [0, 64)")
    return (to_signed(as_ring(a)) >> np.int64(bits)).view(U64)


@dataclass(frozen=True)
class FixedPointConfig:
    """t fractional bits (ring.py:89-101)."""

    t: int = 20

    def __post_init__(self):
        if not 0 < self.t < 32:
            raise RangeError(f"t={self.t} not in (0, 32)")

    @property
    def scale(self) -> int:
        return 1 << self.t


DEFAULT_FP = FixedPointConfig()


def fx_encode(x: Any, cfg: FixedPointConfig = DEFAULT_FP) -> np.ndarray:
    """Round-half-away-from-zero of x * 2^t, two's complement in Z_2^64."""
    v = np.asarray(x, dtype=np.float64)
    lim = float(1 << (63 - cfg.t))
    if not np.isfinite(v).all() or (np.abs(v) >= lim).any():
        raise RangeError(f"|x| must be < 2^{63 - cfg.t}")
    mag = np.floor(np.abs(v) * cfg.scale + 0.5).astype(U64)
    with np.errstate(over="ignore"):
        return np.where(v >= 0, mag, U64(0) - mag)


def fx_decode(v: Any, cfg: FixedPointConfig = DEFAULT_FP) -> np.ndarray:
    return to_signed(as_ring(v)).astype(np.float64) / cfg.scale


def limb_decompose(a) -> np.ndarray:
    """Reference-compatible 4 x 16-bit float limbs (ring.py:123-133)."""
    a = as_ring(a)
    return np.stack([((a >> U64(LIMB_BITS * i)) & U64(0xFFFF)).astype(np.float64) for i in range(NUM_LIMBS)])


def limb_recombine(limbs) -> np.ndarray:
    out = np.zeros(np.shape(limbs)[1:], dtype=U64)
    for i in range(NUM_LIMBS):
        out = out + (np.asarray(limbs[i]).astype(U64) << U64(LIMB_BITS * i))
    return out


@dataclass(frozen=True)
class BilinearOpSpec:
    kind: str
    geometry: dict = field(default_factory=dict)
    accumulation_count: int = 0

    def __post_init__(self):
        if self.kind not in ("matmul", "conv2d", "sum-pool"):
            raise ShapeError(f"unknown bilinear kind {self.kind!r}")


def matmul_spec(m: int, k: int, n: int) -> BilinearOpSpec:
    return BilinearOpSpec("matmul", {"m": m, "k": k, "n": n}, k)


def conv2d_spec(in_channels: int, kernel, stride=(1, 1), padding=(0, 0)) -> BilinearOpSpec:
    kh, kw = kernel
    geo = {"in_channels": in_channels, "kernel": (kh, kw), "stride": tuple(stride), "padding": tuple(padding)}
    return BilinearOpSpec("conv2d", geo, in_channels * kh * kw)


def sumpool_spec(window, stride=None) -> BilinearOpSpec:
    kh, kw = window
    return BilinearOpSpec("sum-pool", {"window": (kh, kw), "stride": tuple(stride or (kh, kw))}, kh * kw)


def check_accumulation(count: int) -> None:
    """The reference's float engine refuses accumulations beyond 2^20
    (ring.py:191-195); the device engine mirrors the contract."""
    if count > MAX_ACCUMULATION:
        raise ExactnessError(f"accumulation_count {count} exceeds 2^20")


def bilinear_exact(a, b, spec: BilinearOpSpec) -> np.ndarray:
    """Exact Z_2^64 matmul / conv2d / sum-pool of host tensors on the GPU."""
    from . import engine  # local import: needs torch + the CUDA library

    check_accumulation(spec.accumulation_count)
    a = as_ring(a)
    if spec.kind == "matmul":
        b = as_ring(b)
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
            raise ShapeError(f"matmul shapes {a.shape} x {b.shape}")
        if a.shape[1] != spec.accumulation_count:
            raise ShapeError("spec accumulation_count does not match inner dimension")
        return engine.plain_matmul(a, b)
    if spec.kind == "conv2d":
        b = as_ring(b)
        g = spec.geometry
        if a.ndim != 4 or b.ndim != 4:
            raise ShapeError("conv2d expects (N,C,H,W) and (O,C,kh,kw)")
        if tuple(b.shape[2:]) != tuple(g["kernel"]) or b.shape[1] != a.shape[1] or g["in_channels"] != a.shape[1]:
            raise ShapeError(f"kernel {b.shape} incompatible with input {a.shape}")
        return engine.plain_conv2d(a, b, g["stride"], g["padding"])
    g = spec.geometry
    if a.ndim != 4:
        raise ShapeError("sum-pool expects (N,C,H,W)")
    return engine.plain_sumpool(a, g["window"], g["stride"])
