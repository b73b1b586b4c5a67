"""Per-party protocol API (protocols.py:57-468 of the reference).

Same names, arguments, return types and exceptions as the reference; each
interactive call is a rendezvous of the three party threads that runs ONE
fused trio kernel on the GPU (engine.TrioSession).  Local operations
(add_const, mul_const, ...) stay per-party as in the reference.
"""

from __future__ import annotations

import numpy as np

from .engine import ExpConfig, ReciprocalConfig, RssTensor  # noqa: F401
from .errors import ConfigError, RangeError, ShapeError
from .ring import as_ring, fx_encode
from .sharing import ArithmeticShare, BinaryShare, PartyContext, assemble, split_trio

__all__ = [
    "ExpConfig", "ReciprocalConfig", "a2b", "add_const", "avgpool_shares", "bit_inject", "compare",
    "conv2d_shares", "division", "drelu", "exp_approx", "matmul_shares", "max_tree", "maxpool_shares", "msb", "mul", "mul_const",
    "reciprocal", "relu", "relu_with_mask", "softmax", "sub_from_const", "truncate", "truncation_offset",
]

U64 = np.uint64


def _dev_const(c, shape):
    import torch

    arr = np.ascontiguousarray(np.broadcast_to(as_ring(c), shape)).view(np.int64)
    return torch.from_numpy(arr.copy()).cuda()


# ---------------------------------------------------------------------------
# local ops (protocols.py:57-72)


def add_const(x: ArithmeticShare, c) -> ArithmeticShare:
    """x + public c, the constant in component 0 (held by party 0 as lo and party 2 as hi)."""
    cd = _dev_const(c, x.shape)
    lo = x.dlo + cd if x.owner == 0 else x.dlo
    hi = x.dhi + cd if x.owner == 2 else x.dhi
    return ArithmeticShare(x.owner, lo, hi, x.fp)


def sub_from_const(c, x: ArithmeticShare) -> ArithmeticShare:
    return add_const(-x, c)


def mul_const(x: ArithmeticShare, c: int) -> ArithmeticShare:
    c = int(c) % (1 << 64)
    cs = c - (1 << 64) if c >= 1 << 63 else c
    return x.map(lambda v: v * cs)


def truncation_offset(raw):
    return (np.asarray(raw, U64) >> U64(2)) - U64(1 << 61)


# ---------------------------------------------------------------------------
# interactive protocols


def _arith(ps, i=0, fp=None):
    return assemble({p: ps[p][i] for p in range(3)}, fp)


def _run(ctx: PartyContext, name: str, args: tuple, fn, binary=False):
    """Rendezvous on `name`; fn(session, trio_args) -> RssTensor | tuple."""

    def body(sess, ps):
        trios = [assemble({p: ps[p][i] for p in range(3)}, getattr(args[i], "fp", None))
                 for i in range(len(args))]
        out = fn(sess, *trios)
        if isinstance(out, tuple):
            return tuple(split_trio(o, binary) if isinstance(o, RssTensor) else o for o in out)
        return split_trio(out, binary)

    res = ctx.collective(name, args, body)
    if isinstance(res, tuple):
        return tuple(r[ctx.party] if isinstance(r, list) else r for r in res)
    return res[ctx.party]


def mul(ctx: PartyContext, x: ArithmeticShare, y: ArithmeticShare, label: str = "mul.reshare") -> ArithmeticShare:
    try:
        np.broadcast_shapes(x.shape, y.shape)
    except ValueError as e:
        raise ShapeError(str(e)) from None
    return _run(ctx, "mul", (x, y), lambda s, a, b: s.mul(a, b, label))


def matmul_shares(ctx: PartyContext, x: ArithmeticShare, y: ArithmeticShare, bits: int | None = None):
    if len(x.shape) != 2 or len(y.shape) != 2 or x.shape[1] != y.shape[0]:
        raise ShapeError(f"matmul shapes {x.shape} x {y.shape}")
    return _run(ctx, "matmul", (x, y), lambda s, a, b: s.matmul(a, b, bits))


def conv2d_shares(ctx: PartyContext, x: ArithmeticShare, k: ArithmeticShare, stride=(1, 1), padding=(0, 0),
                  bits: int | None = None):
    return _run(ctx, "conv2d", (x, k), lambda s, a, b: s.conv2d(a, b, tuple(stride), tuple(padding), bits))


def avgpool_shares(ctx: PartyContext, x: ArithmeticShare, window, stride=None):
    return _run(ctx, "avgpool", (x,), lambda s, a: s.avgpool(a, tuple(window), tuple(stride or window)))


def maxpool_shares(ctx: PartyContext, x: ArithmeticShare, window, stride=None, padding=(0, 0)):
    """Max-pooling extension (the reference has none): windows flattened
    row-major into max_tree (protocols.py:356-380); padded positions hold the
    public constant -2^60 in component 0."""
    return _run(ctx, "maxpool", (x,), lambda s, a: s.maxpool(a, tuple(window), tuple(stride or window),
                                                             tuple(padding)))


def truncate(ctx: PartyContext, x: ArithmeticShare, bits: int | None = None) -> ArithmeticShare:
    b = ctx.fp.t if bits is None else bits
    if not 1 <= b <= 61:
        raise RangeError(f"truncation by {b} bits outside [1, 61]")
    return _run(ctx, "truncate", (x,), lambda s, a: s.truncate(a, b))


def a2b(ctx: PartyContext, x: ArithmeticShare) -> BinaryShare:
    return _run(ctx, "a2b", (x,), lambda s, a: s.a2b(a), binary=True)


def msb(ctx: PartyContext, x: ArithmeticShare) -> BinaryShare:
    return _run(ctx, "msb", (x,), lambda s, a: s.msb(a), binary=True)


def bit_inject(ctx: PartyContext, b: BinaryShare) -> ArithmeticShare:
    return _run(ctx, "bit_inject", (b,), lambda s, a: s.bit_inject(a))


def drelu(ctx: PartyContext, x: ArithmeticShare) -> ArithmeticShare:
    return _run(ctx, "drelu", (x,), lambda s, a: s.drelu(a))


def relu(ctx: PartyContext, x: ArithmeticShare) -> ArithmeticShare:
    return _run(ctx, "relu", (x,), lambda s, a: s.relu(a))


def relu_with_mask(ctx: PartyContext, x: ArithmeticShare):
    return _run(ctx, "relu_with_mask", (x,), lambda s, a: s.relu_with_mask(a))


def compare(ctx: PartyContext, x: ArithmeticShare, y: ArithmeticShare) -> ArithmeticShare:
    return _run(ctx, "compare", (x, y), lambda s, a, b: s.compare(a, b))


def max_tree(ctx: PartyContext, v: ArithmeticShare) -> ArithmeticShare:
    if not v.shape or v.shape[-1] < 1:
        raise ShapeError("max_tree needs at least one element")
    return _run(ctx, "max_tree", (v,), lambda s, a: s.max_tree(a))


def exp_approx(ctx: PartyContext, x: ArithmeticShare, cfg: ExpConfig = ExpConfig()) -> ArithmeticShare:
    if ctx.fp.t + 2 * cfg.squarings > 61:
        raise ConfigError(f"m={cfg.m} too large for t={ctx.fp.t}")
    return _run(ctx, "exp_approx", (x,), lambda s, a: s.exp_approx(a, cfg))


def reciprocal(ctx: PartyContext, y: ArithmeticShare, cfg: ReciprocalConfig = ReciprocalConfig()):
    return _run(ctx, "reciprocal", (y,), lambda s, a: s.reciprocal(a, cfg))


def division(ctx: PartyContext, x: ArithmeticShare, y: ArithmeticShare, cfg: ReciprocalConfig = ReciprocalConfig()):
    return _run(ctx, "division", (x, y), lambda s, a, b: s.division(a, b, cfg))


def softmax(ctx: PartyContext, z: ArithmeticShare, cfg: ReciprocalConfig = ReciprocalConfig()):
    if z.shape[-1] > cfg.Y:
        raise ConfigError(f"class count {z.shape[-1]} exceeds reciprocal domain Y={cfg.Y}")
    return _run(ctx, "softmax", (z,), lambda s, a: s.softmax(a, cfg))


_ = fx_encode
