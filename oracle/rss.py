"""Trio-form CPU restatement of the reference RSS protocols (TEST ORACLE ONLY).

A shared tensor is held as its three additive components, an array of shape
(3,) + shape of uint64; party i's replicated share (lo, hi) is
(C[i], C[(i+1) % 3]) (sharing.py:1-12, 37-49).  All three parties run in
lockstep in one thread, so each per-purpose stream counter is one integer
(sharing.py:225-230: parties that take a purpose take it in lockstep).

References are to /root/reference/pkg/src/mpc3/<file>:<line>.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
from cryptography.hazmat.primitives.ciphers import Cipher, algorithms, modes

U64 = np.uint64
F64 = np.float64

# purpose tags (prf.py:24-28)
ARITH_ZERO, XOR_ZERO, TRUNC_RHO, TRUNC_R, BIN_INPUT = 1, 2, 3, 4, 5

MAX_ACCUM = 1 << 20  # ring.py:22 exactness budget of the float-limb engine


class OracleError(ValueError):
    """Raised where the reference raises one of its Mpc3Error subclasses."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---------------------------------------------------------------------------
# PRF (prf.py:31-61, session.py:29-32, 55)


def prf_words(key: bytes, purpose: int, index: int, count: int) -> np.ndarray:
    """AES-128-CTR word stream; initial counter block is
    purpose_LE16 || index_LE48 || 0^64 (prf.py:40-49)."""
    if not 0 <= purpose < 1 << 16:
        raise OracleError("RangeError", "purpose outside 16 bits")
    if not 0 <= index < 1 << 48:
        raise OracleError("RangeError", "index outside 48 bits")
    block0 = purpose.to_bytes(2, "little") + index.to_bytes(6, "little") + bytes(8)
    enc = Cipher(algorithms.AES(key), modes.CTR(block0)).encryptor()
    raw = enc.update(bytes(8 * int(count)))
    return np.frombuffer(raw, dtype="<u8").astype(U64)


def prf_words_at(key: bytes, purpose: int, index: int, word_off: int, count: int) -> np.ndarray:
    """Words [word_off, word_off + count) of the prf_words stream without
    generating the prefix: CTR mode started at block word_off // 2 (the
    counter runs over the big-endian low 64 bits of the block, prf.py:40-49)."""
    b0 = word_off // 2
    block0 = purpose.to_bytes(2, "little") + index.to_bytes(6, "little") + b0.to_bytes(8, "big")
    enc = Cipher(algorithms.AES(key), modes.CTR(block0)).encryptor()
    skip = word_off - 2 * b0
    raw = enc.update(bytes(8 * (int(count) + skip)))
    return np.frombuffer(raw, dtype="<u8").astype(U64)[skip:]


def session_id(seed: int) -> bytes:
    """session.py:29-32."""
    return hashlib.sha256(f"mpc3-session|{seed}".encode()).digest()[:16]


def derive_key(seed: bytes, session: bytes, label: str) -> bytes:
    """prf.py:58-61."""
    return hashlib.sha256(b"mpc3-key|" + seed + b"|" + session + b"|" + label.encode()).digest()[:16]


def party_keys(seed: int) -> list[bytes]:
    """k_0, k_1, k_2 of a seeded session (session.py:43-59)."""
    sid = session_id(seed)
    return [derive_key(f"seed{seed}".encode(), sid, f"party{i}") for i in range(3)]


class Session:
    """Three co-resident parties: keys, lockstep counters, fixed point t."""

    def __init__(self, seed: int = 0, t: int = 20):
        self.keys = party_keys(seed)
        self.t = t
        self.seq: dict[int, int] = {}

    def take(self, purpose: int) -> int:  # sharing.py:225-230
        j = self.seq.get(purpose, 0)
        self.seq[purpose] = j + 1
        return j

    def words(self, key_idx: int, purpose: int, j: int, n: int) -> np.ndarray:
        return prf_words(self.keys[key_idx], purpose, j, n)


# ---------------------------------------------------------------------------
# ring helpers (ring.py:50-120)


def sar(a: np.ndarray, bits: int) -> np.ndarray:
    """Arithmetic right shift of the two's-complement view (ring.py:75-79)."""
    if not 0 <= bits < 64:
        raise OracleError("RangeError", "shift outside [0, 64)")
    return (np.asarray(a, U64).view(np.int64) >> np.int64(bits)).view(U64)


def fx_encode(x, t: int = 20) -> np.ndarray:
    """Round-half-away-from-zero of x*2^t (ring.py:104-115)."""
    arr = np.asarray(x, dtype=F64)
    if not np.all(np.isfinite(arr)) or np.any(np.abs(arr) >= float(1 << (63 - t))):
        raise OracleError("RangeError", "value outside encodable range")
    mag = np.floor(np.abs(arr) * (1 << t) + 0.5).astype(U64)
    with np.errstate(over="ignore"):
        return np.where(arr >= 0, mag, U64(0) - mag)


def fx_decode(v, t: int = 20) -> np.ndarray:
    return np.asarray(v, U64).view(np.int64).astype(F64) / (1 << t)


# ---------------------------------------------------------------------------
# float-limb bilinear engine (ring.py:123-268): 4 x 16-bit limbs as float64,
# the 10 limb pairs with shift < 64, recombined mod 2^64.

_PAIRS = [(i, j) for i in range(4) for j in range(4) if i + j < 4]


def _limbs(a: np.ndarray) -> np.ndarray:
    a = np.asarray(a, U64)
    return np.stack([((a >> U64(16 * i)) & U64(0xFFFF)).astype(F64) for i in range(4)])


def _pair_sum(fa, fb, kern) -> np.ndarray:
    acc = None
    for i, j in _PAIRS:
        prod = kern(fa[i], fb[j])
        if prod.size and float(prod.max(initial=0.0)) >= 2.0**53:
            raise OracleError("ExactnessError", "float intermediate exceeded 2^53")
        term = prod.astype(U64) << U64(16 * (i + j))
        acc = term if acc is None else acc + term
    return acc


def ring_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """(m,k) @ (k,n) mod 2^64 via limb dgemms (ring.py:183-222)."""
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise OracleError("ShapeError", f"matmul shapes {a.shape} x {b.shape}")
    if a.shape[1] > MAX_ACCUM:
        raise OracleError("ExactnessError", "accumulation exceeds 2^20")
    return _pair_sum(_limbs(a), _limbs(b), lambda x, y: x @ y)


def conv_out_hw(h, w, kh, kw, stride, padding):
    sh, sw = stride
    ph, pw = padding
    return (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1


def ring_conv2d(x: np.ndarray, k: np.ndarray, stride=(1, 1), padding=(0, 0)) -> np.ndarray:
    """NCHW cross-correlation mod 2^64 via im2col + limb dgemms (ring.py:225-256)."""
    if x.ndim != 4 or k.ndim != 4 or x.shape[1] != k.shape[1]:
        raise OracleError("ShapeError", f"conv shapes {x.shape} x {k.shape}")
    n, c, h, w = x.shape
    o, _, kh, kw = k.shape
    sh, sw = stride
    ph, pw = padding
    if c * kh * kw > MAX_ACCUM:
        raise OracleError("ExactnessError", "accumulation exceeds 2^20")
    if h + 2 * ph < kh or w + 2 * pw < kw:
        raise OracleError("ShapeError", "kernel larger than padded input")
    oh, ow = conv_out_hw(h, w, kh, kw, stride, padding)
    fx = _limbs(x)
    if ph or pw:
        fx = np.pad(fx, ((0, 0), (0, 0), (0, 0), (ph, ph), (pw, pw)))
    fk = _limbs(k).reshape(4, o, c * kh * kw)
    cols = np.empty((4, n * oh * ow, c * kh * kw), dtype=F64)
    for i in range(4):
        win = np.lib.stride_tricks.sliding_window_view(fx[i], (kh, kw), axis=(2, 3))
        win = win[:, :, ::sh, ::sw].transpose(0, 2, 3, 1, 4, 5)
        cols[i] = win.reshape(n * oh * ow, c * kh * kw)
    flat = _pair_sum(cols, fk, lambda p, q: p @ q.T)
    return flat.reshape(n, oh, ow, o).transpose(0, 3, 1, 2)


def ring_sumpool(x: np.ndarray, window, stride=None) -> np.ndarray:
    """Window sums mod 2^64 (ring.py:259-268)."""
    kh, kw = window
    sh, sw = stride or window
    if x.ndim != 4 or x.shape[2] < kh or x.shape[3] < kw:
        raise OracleError("ShapeError", "window larger than input")
    win = np.lib.stride_tricks.sliding_window_view(x, (kh, kw), axis=(2, 3))[:, :, ::sh, ::sw]
    return win.sum(axis=(-1, -2), dtype=U64)


def wrap_matmul(a, b):
    """Independent einsum oracle (tests/oracles.py:15-17)."""
    return np.einsum("ik,kj->ij", np.asarray(a, U64), np.asarray(b, U64))


def wrap_conv2d(x, k, stride=(1, 1), padding=(0, 0)):
    """Independent einsum conv oracle (tests/oracles.py:34-45)."""
    ph, pw = padding
    xp = np.pad(np.asarray(x, U64), ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    kh, kw = k.shape[2:]
    win = np.lib.stride_tricks.sliding_window_view(xp, (kh, kw), axis=(2, 3))
    win = win[:, :, :: stride[0], :: stride[1]]
    return np.einsum("ncxyuv,ocuv->noxy", win, np.asarray(k, U64))


# ---------------------------------------------------------------------------
# sharing (sharing.py:113-187)


def share(x, rng: np.random.Generator) -> np.ndarray:
    """Dealer draws c0, c1 then sets c2 = x - c0 - c1 (sharing.py:113-118)."""
    x = np.asarray(x, U64)
    c0 = rng.integers(0, 1 << 64, size=x.shape, dtype=U64)
    c1 = rng.integers(0, 1 << 64, size=x.shape, dtype=U64)
    return np.stack([c0, c1, x - c0 - c1])


def reconstruct(c: np.ndarray) -> np.ndarray:
    return c[0] + c[1] + c[2]


def xor_reconstruct(c: np.ndarray) -> np.ndarray:
    return c[0] ^ c[1] ^ c[2]


def party_view(c: np.ndarray, p: int) -> tuple[np.ndarray, np.ndarray]:
    """Party p's (lo, hi) (sharing.py:37-43)."""
    return c[p], c[(p + 1) % 3]


def _nxt(c):
    return c[[1, 2, 0]]


def _relabel(z):
    """Party i keeps (z_{i-1}, z_i): new component i+1 is z_i (protocols.py:88-94)."""
    return z[[2, 0, 1]]


def _numel(shape) -> int:
    return int(np.prod(shape, dtype=np.int64)) if shape else 1


def zero_share(s: Session, purpose: int, shape, xor: bool = False) -> np.ndarray:
    """z_i = F(k_i) -/^ F(k_{i-1}) (sharing.py:233-250)."""
    j = s.take(purpose)
    n = _numel(shape)
    f = [s.words(i, purpose, j, n).reshape(shape) for i in range(3)]
    if xor:
        return np.stack([f[i] ^ f[(i - 1) % 3] for i in range(3)])
    return np.stack([f[i] - f[(i - 1) % 3] for i in range(3)])


# ---------------------------------------------------------------------------
# local ops (protocols.py:57-72)


def add_const(x: np.ndarray, c) -> np.ndarray:
    out = x.copy()
    out[0] = x[0] + np.broadcast_to(np.asarray(c, U64), x.shape[1:])
    return out


def sub_from_const(c, x):
    return add_const(U64(0) - x, c)


def mul_const(x, c: int):
    return x * U64(int(c) & ((1 << 64) - 1))


def const_share(value, shape) -> np.ndarray:
    """Components (c, 0, 0) (sharing.py:184-187)."""
    out = np.zeros((3,) + tuple(shape), U64)
    out[0] = np.broadcast_to(np.asarray(value, U64), shape)
    return out


# ---------------------------------------------------------------------------
# multiplication / bilinear (protocols.py:79-159)


def reshare(s: Session, z: np.ndarray) -> np.ndarray:
    return _relabel(z + zero_share(s, ARITH_ZERO, z.shape[1:]))


def mul(s: Session, x, y):
    shape = np.broadcast_shapes(x.shape[1:], y.shape[1:])
    xb = np.broadcast_to(x.reshape((3,) + (1,) * (len(shape) + 1 - x.ndim) + x.shape[1:]), (3,) + shape)
    yb = np.broadcast_to(y.reshape((3,) + (1,) * (len(shape) + 1 - y.ndim) + y.shape[1:]), (3,) + shape)
    z = xb * yb + _nxt(xb) * yb + xb * _nxt(yb)
    return reshare(s, z)


_POOL = None


def _bilinear3(fn, x, y):
    """z_i = f(x_i, y_i) + f(x_{i+1}, y_i) + f(x_i, y_{i+1}) per party
    (protocols.py:110-115).  The three parties run concurrently, as the
    reference's three party threads do (session.py:141-152)."""
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(3)

    def party(i):
        return fn(x[i], y[i]) + fn(x[(i + 1) % 3], y[i]) + fn(x[i], y[(i + 1) % 3])

    return np.stack(list(_POOL.map(party, range(3))))


def matmul_shares(s: Session, x, y, bits=None):
    if x.ndim != 3 or y.ndim != 3 or x.shape[2] != y.shape[1]:
        raise OracleError("ShapeError", f"matmul shapes {x.shape[1:]} x {y.shape[1:]}")
    return truncate(s, reshare(s, _bilinear3(ring_matmul, x, y)), bits)


def conv2d_shares(s: Session, x, k, stride=(1, 1), padding=(0, 0), bits=None):
    z = _bilinear3(lambda a, b: ring_conv2d(a, b, stride, padding), x, k)
    return truncate(s, reshare(s, z), bits)


def avgpool_shares(s: Session, x, window, stride=None):
    summed = np.stack([ring_sumpool(x[i], window, stride) for i in range(3)])
    return div_area(s, summed, window[0] * window[1])


def div_area(s: Session, x, area: int):
    """protocols.py:154-159 / nn.py:239-243."""
    if area & (area - 1) == 0:
        return truncate(s, x, area.bit_length() - 1)
    return truncate(s, mul_const(x, int(fx_encode(1.0 / area, s.t))))


# ---------------------------------------------------------------------------
# truncation (protocols.py:166-216)


def truncation_offset(raw):
    return (raw >> U64(2)) - U64(1 << 61)


def truncate(s: Session, x, bits=None):
    bits = s.t if bits is None else bits
    if not 1 <= bits <= 61:
        raise OracleError("RangeError", f"truncation by {bits} bits outside [1, 61]")
    shape = x.shape[1:]
    n = _numel(shape)
    half = U64(1 << (bits - 1))
    rho = truncation_offset(s.words(2, TRUNC_RHO, s.take(TRUNC_RHO), n).reshape(shape))
    r = s.words(1, TRUNC_R, s.take(TRUNC_R), n).reshape(shape)
    z0 = sar(rho + half, bits)
    b = (x[0] - rho) + x[1] + x[2]
    z1 = sar(b + half, bits) - r
    return np.stack([z0, z1, r])


class TruncationRandomness:
    """rho replay from k_2's TRUNC_RHO stream (session.py:94-113)."""

    def __init__(self, seed: int):
        self._key = party_keys(seed)[2]
        self._index = 0

    def draw(self, shape):
        raw = prf_words(self._key, TRUNC_RHO, self._index, _numel(shape)).reshape(shape)
        self._index += 1
        return truncation_offset(raw)


# ---------------------------------------------------------------------------
# binary world (protocols.py:223-353)


def and_gate(s: Session, a, b):
    z = (a & b) ^ (_nxt(a) & b) ^ (a & _nxt(b))
    return _relabel(z ^ zero_share(s, XOR_ZERO, z.shape[1:], xor=True))


def ks_add(s: Session, a, b):
    """64-bit Kogge-Stone on XOR shares: leaf AND + 6 fused levels whose AND
    runs over 2n words [g-part | p-part] (protocols.py:233-263)."""
    shape = a.shape[1:]
    n = _numel(shape)
    p = (a ^ b).reshape(3, n)
    g = and_gate(s, a, b).reshape(3, n)
    p_leaf = p
    for d in (1, 2, 4, 8, 16, 32):
        dd = U64(d)
        lhs = np.concatenate([p, p], axis=1)
        rhs = np.concatenate([g << dd, p << dd], axis=1)
        prod = and_gate(s, lhs, rhs)
        g = g ^ prod[:, :n]
        p = prod[:, n:]
    return (p_leaf ^ (g << U64(1))).reshape((3,) + shape)


def a2b(s: Session, x):
    shape = x.shape[1:]
    r = s.words(0, BIN_INPUT, s.take(BIN_INPUT), _numel(shape)).reshape(shape)
    zero = np.zeros(shape, U64)
    w = np.stack([(x[0] + x[1]) ^ r, r, zero])
    x2 = np.stack([zero, zero, x[2]])
    return ks_add(s, w, x2)


def msb(s: Session, x):
    return a2b(s, x) >> U64(63)


def bit_inject(s: Session, b):
    shape = b.shape[1:]
    slots = []
    for j in range(3):
        t = np.zeros((3,) + shape, U64)
        t[j] = b[j]
        slots.append(t)

    def xor_arith(u, v):
        return u + v - mul_const(mul(s, u, v), 2)

    return xor_arith(xor_arith(slots[0], slots[1]), slots[2])


def drelu(s: Session, x):
    return sub_from_const(U64(1), bit_inject(s, msb(s, x)))


def relu_with_mask(s: Session, x):
    mask = drelu(s, x)
    return mul(s, x, mask), mask


def relu(s: Session, x):
    return relu_with_mask(s, x)[0]


def compare(s: Session, x, y):
    return drelu(s, x - y)


def max_tree(s: Session, v):
    """Last-axis tournament max(a,b) = b + relu(a-b) (protocols.py:356-380)."""
    m = v.shape[-1] if v.ndim > 1 else 0
    if m < 1:
        raise OracleError("ShapeError", "max_tree needs at least one element")
    while m > 1:
        k = m // 2
        a = v[..., 0 : 2 * k : 2]
        b = v[..., 1 : 2 * k : 2]
        mx = b + relu(s, a - b)
        if m % 2:
            mx = np.concatenate([mx, v[..., -1:]], axis=-1)
        v = mx
        m = v.shape[-1]
    return v[..., 0]


MAXPOOL_PAD = (1 << 64) - (1 << 60)  # public padding constant (ring encoding of -2^60)


def maxpool_shares(s: Session, x, window, stride=None, padding=(0, 0)):
    """Max-pool composed from reference primitives (the reference has no
    max-pool layer): each component's (kh, kw) windows gathered
    row-major (a local structural op; padded positions hold the public
    constant in component 0, sharing.py:184-187), then max_tree
    (protocols.py:356-380) over the window axis."""
    (kh, kw), (ph, pw) = window, padding
    sh, sw = stride or window
    outs = []
    for i in range(3):
        v = x[i]
        if ph or pw:
            v = np.pad(v, ((0, 0), (0, 0), (ph, ph), (pw, pw)), constant_values=MAXPOOL_PAD if i == 0 else 0)
        win = np.lib.stride_tricks.sliding_window_view(v, (kh, kw), axis=(2, 3))[:, :, ::sh, ::sw]
        outs.append(win.reshape(win.shape[:4] + (kh * kw,)))
    return max_tree(s, np.ascontiguousarray(np.stack(outs)))


# ---------------------------------------------------------------------------
# function approximations (protocols.py:387-468)


def exp_approx(s: Session, x, m: int = 512):
    sq = m.bit_length() - 1
    if s.t + 2 * sq > 61:
        raise OracleError("ConfigError", "m too large for t")
    y = add_const(x, fx_encode(float(m), s.t))
    y = truncate(s, mul(s, y, y), s.t + 2 * sq)
    for _ in range(sq - 1):
        y = truncate(s, mul(s, y, y))
    return y


def reciprocal(s: Session, y, Y: float = 200.0, iterations: int = 13):
    z = const_share(fx_encode(1.0 / Y, s.t), y.shape[1:])
    for _ in range(iterations):
        z2 = truncate(s, mul(s, z, z))
        yz2 = truncate(s, mul(s, y, z2))
        z = mul_const(z, 2) - yz2
    return z


def division(s: Session, x, y, Y: float = 200.0, iterations: int = 13):
    return truncate(s, mul(s, x, reciprocal(s, y, Y, iterations)))


def softmax(s: Session, z, Y: float = 200.0, iterations: int = 13):
    d = z.shape[-1]
    if d > Y:
        raise OracleError("ConfigError", "class count exceeds reciprocal domain")
    mx = max_tree(s, z)
    x = z - mx[..., None]
    e = exp_approx(s, x)
    tot = e.sum(axis=-1, keepdims=True, dtype=U64)
    r = reciprocal(s, tot, Y, iterations)
    return truncate(s, mul(s, e, r))


def open_trio(c: np.ndarray) -> np.ndarray:
    """session.py:116-121: every party ends with c0 + c1 + c2."""
    return reconstruct(c)
