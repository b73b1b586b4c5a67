"""The trio engine: all three RSS parties co-resident on one B200.

A shared tensor (`RssTensor`) is ONE device buffer of shape (3, *shape),
int64 bit-cast of the three additive components c0, c1, c2; party i's
replicated share (lo, hi) is (c_i, c_{i+1}) (sharing.py:37-49).  Every
protocol of the reference (protocols.py:57-468) runs as fused CUDA kernels
over the trio: the local cross terms of all three parties, the PRF zero
shares (AES-CTR generated inline, bit-exact with prf.py:40-49) and the
"messages" (register / HBM handoffs) in one launch per protocol call, with
the reference's lockstep per-purpose counters (sharing.py:225-230) kept on
the host.  Communication is charged analytically into per-party CommStats
with the reference's byte and round accounting.

There is no CPU path: every compute call goes through libmpc3b200.so.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi as K
from .errors import ConfigError, FreshnessError, RangeError, ShapeError
from .prf import (
    PURPOSE_ARITH_ZERO as ARITH,
    PURPOSE_BIN_INPUT as BIN,
    PURPOSE_TRUNC_R as TR_R,
    PURPOSE_TRUNC_RHO as TR_RHO,
    PURPOSE_XOR_ZERO as XOR,
    PURPOSES,
    PrfKey,
    derive_key,
)
from .ring import DEFAULT_FP, FixedPointConfig, as_ring, check_accumulation, fx_encode
from .transport import Ledger

U64 = np.uint64
MAX_SPLIT_K = 16384  # per-split K bound of the int8-limb GEMM (exactness of S_3)
# MPC3_OVERLAP_PACK=0: pack both GEMM operands on the calling stream
OVERLAP_PACK = os.environ.get("MPC3_OVERLAP_PACK", "1") == "1"
SMS = 148
# MPC3_REUSE_PACKS=0: weight gradients pack their own operands instead of
# reading the forward / input-gradient packs in place (mpc3_ring_gemm_t)
REUSE_PACKS = os.environ.get("MPC3_REUSE_PACKS", "1") == "1"
# MPC3_CS_PACKS=0: role-1 operands of the training step packed with both halves
# instead of once per component (role 3: half the pack's writes)
CS_PACKS = os.environ.get("MPC3_CS_PACKS", "1") == "1"
# MPC3_T_PACKS=0: role-3 operands packed K-major (rows = the GEMM's rows)
# instead of transposed (rows = the contraction), see Packed.t
T_PACKS = os.environ.get("MPC3_T_PACKS", "1") == "1"
# weight gradients from a transposed x pack with at least this contraction
# per half run as g^T x (x as B, see wgrad_packed) unless that orientation
# fills the 128 x 64 tiles worse: its MN-major A reads are worth up to
# WGRAD_SWAP_EDGE x the tile fill (VGG-16-TI conv1_2, O = 64: g^T x fills half
# of each tile's rows, x^T g 90 %)
WGRAD_SWAP_MIN_KC = int(os.environ.get("MPC3_WGRAD_SWAP_MIN_KC", "4096"))
WGRAD_SWAP_EDGE = float(os.environ.get("MPC3_WGRAD_SWAP_EDGE", "1.15"))


def _tile_fill(rows: int, cols: int) -> float:
    return rows / (-(-rows // 128) * 128) * cols / (-(-cols // 64) * 64)
# MPC3_MAXTREE_FUSED=0: one launch per max_tree level instead of one for the whole tree
MAXTREE_FUSED = os.environ.get("MPC3_MAXTREE_FUSED", "1") == "1"
# MPC3_LOSS_FUSED=0: the loss gradient softmax(z) - y as its separate launches
LOSS_FUSED = os.environ.get("MPC3_LOSS_FUSED", "1") == "1"
# the one-launch max_tree runs two rows per CTA (a latency design for the
# softmax's (batch, classes) rows); many rows (max-pool windows) go level by
# level through the persistent sign kernel instead
MAXTREE_FUSED_MAX_ROWS = 8192
# public padding constant of the max-pool extension: the ring encoding of -2^60
MAXPOOL_PAD = (1 << 64) - (1 << 60)


@dataclass
class Packed:
    """A cross-term operand packed for the ring GEMM, kept for reuse: byte-limb
    planes [3][8][rows][kp] of [first half | second half] with the second half
    at the 16-aligned column kh, role 0 ([x_i + x_{i+1} | x_i]) or 1
    ([x_i | x_{i+1}]); or role 3, a role-1 operand stored once per component
    (plane i = x_i, K columns, kh = k unused) whose halves the GEMM reads from
    planes i and i + 1.  A weight gradient reads two of these transposed.
    t: a role-3 operand packed transposed — buffer rows are the contraction
    index, columns the GEMM's rows (rows / k / kp describe the buffer).  The
    GEMM then reads its A tiles MN-major: 128-byte TMA rows and SWIZZLE_128B
    instead of 32-byte K-major rows (the forward and input-gradient GEMMs
    +12-17 %, profiles/README.md), and a weight gradient reads the forward
    pack K-major."""
    buf: torch.Tensor
    rows: int
    k: int
    kh: int
    kp: int
    role: int
    t: bool = False

    @staticmethod
    def geometry(k: int) -> tuple[int, int]:
        kh = _round_up(k, 16)
        return kh, _round_up(kh + k, 32)  # whole 32-byte K-blocks (see pack)

    @staticmethod
    def geometry_cs(k: int) -> tuple[int, int]:
        """(kh, kp) of the role-0 partner of a role-3 operand: halves at the
        32-aligned column kc_half (whole K-blocks per half)."""
        kc = _round_up(k, 32)
        return kc, 2 * kc


def _stream() -> int:
    # the raw C getters: torch.cuda.current_stream() resolves its device index
    # through Python helpers, ~8 us per call on the eager step's ~130 launches
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def _dev():
    return torch.device("cuda", torch._C._cuda_getDevice())


def _cur():
    """torch.cuda.current_stream() with the device index given (skips the
    Python device-index resolution)."""
    return torch.cuda.current_stream(torch._C._cuda_getDevice())


def to_device(a: np.ndarray) -> torch.Tensor:
    """Host uint64 array -> device int64 tensor (bit-cast)."""
    a = np.ascontiguousarray(np.asarray(a, dtype=U64))
    return torch.from_numpy(a.view(np.int64)).to(_dev(), non_blocking=False)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().contiguous().cpu().numpy().view(U64)


def _round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


# ---------------------------------------------------------------------------
# shared tensors


class RssTensor:
    """Three components of a replicated sharing in one (3, *shape) buffer."""

    __slots__ = ("data", "fp")

    def __init__(self, data: torch.Tensor, fp: FixedPointConfig = DEFAULT_FP):
        if data.dtype != torch.int64 or data.dim() < 1 or data.shape[0] != 3:
            raise ShapeError("RssTensor data must be int64 of shape (3, ...)")
        self.data = data
        self.fp = fp

    @property
    def shape(self) -> tuple:
        return tuple(self.data.shape[1:])

    @property
    def ndim(self) -> int:
        return self.data.dim() - 1

    @property
    def numel(self) -> int:
        return self.data.numel() // 3

    def contiguous(self) -> "RssTensor":
        return self if self.data.is_contiguous() else RssTensor(self.data.contiguous(), self.fp)

    def reshape(self, *shape) -> "RssTensor":
        if len(shape) == 1 and isinstance(shape[0], (tuple, list)):
            shape = tuple(shape[0])
        return RssTensor(self.data.reshape((3,) + tuple(shape)), self.fp)

    def apply(self, f) -> "RssTensor":
        """Structural (per-component) transform f on the (3, ...) buffer."""
        return RssTensor(f(self.data), self.fp)

    def __getitem__(self, idx) -> "RssTensor":
        if not isinstance(idx, tuple):
            idx = (idx,)
        return RssTensor(self.data[(slice(None),) + idx], self.fp)

    def comp(self, i: int) -> torch.Tensor:
        return self.data[i]

    def __repr__(self):
        return f"RssTensor(shape={self.shape}, device={self.data.device})"


def empty(shape, fp=DEFAULT_FP) -> RssTensor:
    return RssTensor(torch.empty((3,) + tuple(shape), dtype=torch.int64, device=_dev()), fp)


def zeros(shape, fp=DEFAULT_FP) -> RssTensor:
    return RssTensor(torch.zeros((3,) + tuple(shape), dtype=torch.int64, device=_dev()), fp)


def _flat(t: RssTensor) -> torch.Tensor:
    return t.data if t.data.is_contiguous() else t.data.contiguous()


# ---------------------------------------------------------------------------
# session


def make_session_id(seed):
    import hashlib
    import os

    if seed is None:
        return os.urandom(16)
    return hashlib.sha256(f"mpc3-session|{seed}".encode()).digest()[:16]


def session_keys(seed, session_id=None) -> list[PrfKey]:
    """k_0, k_1, k_2 exactly as the reference's seeded setup (session.py:43-59)."""
    import os

    sid = session_id if session_id is not None else make_session_id(seed)
    if seed is None:
        return [PrfKey(os.urandom(16)) for _ in range(3)]
    return [derive_key(f"seed{seed}".encode(), sid, f"party{i}") for i in range(3)]


@dataclass(frozen=True)
class ExpConfig:
    """e^x ~ (1 + x/m)^m (protocols.py:387-399)."""

    m: int = 512

    def __post_init__(self):
        if self.m < 2 or self.m & (self.m - 1):
            raise ConfigError(f"m={self.m} must be a power of two >= 2")

    @property
    def squarings(self) -> int:
        return self.m.bit_length() - 1


@dataclass(frozen=True)
class ReciprocalConfig:
    """Newton 1/y on [1, Y] from z0 = 1/Y (protocols.py:402-411)."""

    Y: float = 200.0
    iterations: int = 13

    def __post_init__(self):
        if self.Y < 1 or self.iterations < 0:
            raise ConfigError("need Y >= 1 and iterations >= 0")


class TrioSession:
    """Keys, lockstep PRF counters and communication ledger of one 3-party
    session whose parties are co-resident on the current CUDA device."""

    def __init__(self, seed: int | None = 0, fp: FixedPointConfig = DEFAULT_FP, session_id: bytes | None = None,
                 keys: list[PrfKey] | None = None):
        self.fp = fp
        self.seed = seed
        self.session_id = session_id if session_id is not None else make_session_id(seed)
        self.keys = keys if keys is not None else session_keys(seed, self.session_id)
        rk = np.stack([k.round_keys for k in self.keys])
        # pinned host memory: the launches read the schedules on the host and
        # pass them in the kernel parameters (constant bank on the device)
        self.rk3 = torch.from_numpy(rk.view(np.int32).copy())
        if torch.cuda.is_available():
            self.rk3 = self.rk3.pin_memory()
        self.seq = {p: 0 for p in PURPOSES}
        self.engine_mark = {p: 0 for p in PURPOSES}  # first counter no engine kernel has drawn
        self._party_seq = {}  # per-party counters of PartyContext.take (lockstep, sharing.py:225-230)
        self.ledger = Ledger()
        self.ctr = None  # optional device per-purpose counter base (CUDA-graph replay)
        self.dp = None  # DataParallel: this session computes one batch shard
        self._side = None  # side stream for independent launches (weight gradients)
        self._pack = None  # stream for the B-operand pack of a GEMM
        self._wcache = None  # packed weight operands under frozen_weights()
        self._prepacked = {}  # weight packs made ahead of their layer (prepack): key -> (Packed, event)
        # False: the fused layer + ReLU launches skip the mask (an inference
        # pass without a backward: TrioNet sets it per pass)
        self.relu_masks = True
        self._replicated = 0

    # -- data parallelism --
    def frozen_weights(self):
        """Context: the weight operands (GEMM B side) do not change, so their
        packed limb planes are built once and reused (inference; a weight
        modified by a torch in-place op gets a new tensor version and is
        repacked, and sgd_launch, which writes through raw pointers, drops
        the cache)."""
        sess = self

        class _Ctx:
            def __enter__(self_inner):
                self_inner.prev = sess._wcache
                if sess._wcache is None:
                    sess._wcache = {}
                return sess

            def __exit__(self_inner, *exc):
                sess._wcache = self_inner.prev
                return False

        return _Ctx()

    def pack_stream(self):
        """The stream that packs a GEMM's B operand while A packs (lazily created)."""
        if self._pack is None:
            self._pack = torch.cuda.Stream(device=_dev())
        return self._pack

    def side_stream(self):
        """A second CUDA stream on this session's device (lazily created)."""
        if self._side is None:
            self._side = torch.cuda.Stream(device=_dev())
        return self._side

    def shard_offset(self, numel: int) -> tuple[int, int]:
        """(global word offset of this shard's element 0, global element count)
        of a batch-major tensor whose local part has `numel` elements.  Every
        rank holds an equal batch shard, so the shard is one contiguous range
        of the reference's flat tensor and its PRF words a seekable range."""
        if self.dp is None or self._replicated:
            return 0, numel
        return self.dp.rank * numel, self.dp.world * numel

    def replicated(self):
        """Context: ops on replicated (non-batch) tensors, e.g. the SGD update."""
        sess = self

        class _Ctx:
            def __enter__(self):
                sess._replicated += 1

            def __exit__(self, *a):
                sess._replicated -= 1

        return _Ctx()

    def _reduce_cross_terms(self, z: torch.Tensor) -> None:
        """Weight gradients: sum the shards' raw cross terms (mod 2^64) BEFORE
        the reshare/truncation, which then run replicated on every rank."""
        if self.dp is not None and self.dp.world > 1:
            self.dp.allreduce(z)

    # -- counters (sharing.py:190-204, 225-230) --
    def take(self, purpose: int, count: int = 1) -> int:
        j = self.seq[purpose]
        if j + count > (1 << 48):
            raise FreshnessError(f"stream counters for purpose {purpose:#06x} exhausted")
        self.seq[purpose] = j + count
        self.engine_mark[purpose] = max(self.engine_mark[purpose], j + count)
        return j

    def party_take(self, party: int, purpose: int) -> int:
        """PartyContext.take for party `party` (sharing.py:225-230): the three
        parties draw the same counter in lockstep, never one an engine kernel
        has already used; once all three hold j, the engine's next counter
        is past it."""
        own = self._party_seq.setdefault(party, {})
        j = max(own.get(purpose, 0), self.seq[purpose])
        if j + 1 > (1 << 48):
            raise FreshnessError(f"stream counters for purpose {purpose:#06x} exhausted")
        own[purpose] = j + 1
        if all(self._party_seq.get(p, {}).get(purpose, 0) >= j + 1 for p in range(3)):
            self.seq[purpose] = max(self.seq[purpose], j + 1)
        return j

    def check_fresh(self, purpose: int, j: int) -> None:
        """A stream a protocol kernel has already consumed may not be drawn
        again through the per-party randomness API (sharing.py:198-204)."""
        if j < self.engine_mark.get(purpose, 0):
            raise FreshnessError(f"counter {j} for purpose {purpose:#06x} already consumed by the engine")

    def counters(self) -> dict:
        return dict(self.seq)

    def rewind(self, seq: dict) -> None:
        """Counters only move forward; a rewind would reuse PRF streams."""
        for p, j in seq.items():
            if j < self.seq[p]:
                raise FreshnessError(f"counter {j} already used for purpose {p:#06x}")
        self.seq.update(seq)

    @property
    def ctr_ptr(self):
        return None if self.ctr is None else self.ctr.data_ptr()

    @property
    def rk(self) -> int:
        return self.rk3.data_ptr()

    # -- host boundary (session.py:62-91, 116-121; sharing.py:113-155) --
    def share(self, x, rng: np.random.Generator, label: str = "share.input", owner: int = 0) -> RssTensor:
        """Dealer draws c0, c1 ~ rng (numpy, as sharing.py:113-118), c2 = x - c0 - c1;
        the three components are uploaded as one trio buffer."""
        x = as_ring(x)
        c0 = rng.integers(0, 1 << 64, size=x.shape, dtype=U64)
        c1 = rng.integers(0, 1 << 64, size=x.shape, dtype=U64)
        comps = np.stack([c0, c1, x - c0 - c1])
        n = int(x.size)
        self.ledger.round(label, [(owner, p, 2 * n) for p in range(3) if p != owner])
        return RssTensor(to_device(comps), self.fp)

    def share_device(self, x: torch.Tensor, rng: np.random.Generator, label: str = "share.input",
                     owner: int = 0, out: RssTensor | None = None) -> RssTensor:
        """`share` for an input already on the device (int64 bit-cast ring
        values): the dealer's PCG64 draws are generated by the GPU, word for
        word the ones numpy would return, and the host Generator is advanced
        past them (sharing.py:113-118).  `out`: a contiguous (3, *x.shape)
        sharing to deal into (e.g. a captured graph's static input)."""
        st = rng.bit_generator.state
        if st.get("bit_generator") != "PCG64":
            raise ConfigError("device dealing reproduces numpy's PCG64 Generator only")
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        x = x.contiguous()
        n = x.numel()
        if out is None:
            out = empty(tuple(x.shape), self.fp)
        elif out.shape != tuple(x.shape) or not out.data.is_contiguous():
            raise ShapeError("out must be a contiguous sharing of the input's shape")
        m64 = (1 << 64) - 1
        K.call("mpc3_deal_pcg64", s >> 64, s & m64, inc >> 64, inc & m64, x.data_ptr(), out.data.data_ptr(), n,
               _stream())
        rng.bit_generator.advance(2 * n)
        self.ledger.round(label, [(owner, p, 2 * n) for p in range(3) if p != owner])
        return out

    def fx_encode_device(self, x: torch.Tensor, bad: torch.Tensor | None = None) -> torch.Tensor:
        """ring.fx_encode on a float64 device tensor; `bad` (int32 device
        scalar) becomes 1 on an out-of-range input (checked by the caller)."""
        x = x.to(torch.float64).contiguous()
        out = torch.empty(x.shape, dtype=torch.int64, device=x.device)
        K.call("mpc3_fx_encode", x.data_ptr(), out.data_ptr(), x.numel(), self.fp.t,
               None if bad is None else bad.data_ptr(), _stream())
        return out

    def from_components(self, comps) -> RssTensor:
        return RssTensor(to_device(np.asarray(comps, U64)), self.fp)

    def reveal(self, x: RssTensor, label: str = "open") -> np.ndarray:
        """open_share: every party learns c0 + c1 + c2 (session.py:116-121)."""
        self.ledger.ring(label, x.numel)
        return to_host(reconstruct_device(x)).reshape(x.shape)

    # -- local ops (protocols.py:57-72, sharing.py:54-67) --
    def add(self, a, b):
        return _ew2(K.EW_ADD, a, b)

    def sub(self, a, b, out: RssTensor | None = None):
        return _ew2(K.EW_SUB, a, b, out)

    def neg(self, a):
        out = empty(a.shape, a.fp)
        K.call("mpc3_ring_ew", K.EW_NEG, _flat(a).data_ptr(), None, 0, out.data.data_ptr(), 3 * a.numel, _stream())
        return out

    def mul_const(self, a, c: int):
        out = empty(a.shape, a.fp)
        K.call("mpc3_ring_ew", K.EW_MULC, _flat(a).data_ptr(), None, int(c) % (1 << 64), out.data.data_ptr(),
               3 * a.numel, _stream())
        return out

    def add_const(self, a, c):
        """Public constant into component 0 (protocols.py:57-62)."""
        a = a.contiguous()
        cv = np.broadcast_to(as_ring(c), a.shape)
        if cv.ndim == 0 or np.all(cv == cv.flat[0]):
            out = RssTensor(a.data.clone(), a.fp)
            K.call("mpc3_ring_ew", K.EW_ADDC, a.data.data_ptr(), None, int(cv.flat[0]) if cv.size else 0,
                   out.data.data_ptr(), a.numel, _stream())
            return out
        out = RssTensor(a.data.clone(), a.fp)
        cd = to_device(np.ascontiguousarray(cv))
        K.call("mpc3_ring_ew", K.EW_ADD, a.data.data_ptr(), cd.data_ptr(), 0, out.data.data_ptr(), a.numel, _stream())
        return out

    def sub_from_const(self, c, a):
        return self.add_const(self.neg(a), c)

    def const_share(self, value, shape) -> RssTensor:
        """Components (c, 0, 0) (sharing.py:184-187)."""
        out = zeros(shape, self.fp)
        v = as_ring(value)
        if v.ndim == 0:  # device fill, no host copy (CUDA-graph safe)
            c = int(v)
            out.data[0].fill_(c - (1 << 64) if c >= 1 << 63 else c)
        else:
            out.data[0] = torch.from_numpy(np.broadcast_to(v, shape).astype(U64).view(np.int64)).to(_dev())
        return out

    # -- multiplication (protocols.py:79-94) --
    def mul(self, x: RssTensor, y: RssTensor, label: str = "mul.reshare") -> RssTensor:
        x, y = _broadcast(x, y)
        out = empty(x.shape, x.fp)
        j = self.take(ARITH)
        K.call("mpc3_rss_mul", self.rk, self.ctr_ptr, j, x.data.data_ptr(), y.data.data_ptr(), out.data.data_ptr(),
               x.numel, self.shard_offset(x.numel)[0], _stream())
        self.ledger.ring(label, x.numel)
        return out

    def truncate(self, x: RssTensor, bits: int | None = None) -> RssTensor:
        bits = self.fp.t if bits is None else bits
        if not 1 <= bits <= 61:
            raise RangeError(f"truncation by {bits} bits outside [1, 61]")
        x = x.contiguous()
        out = empty(x.shape, x.fp)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        K.call("mpc3_rss_truncate", self.rk, self.ctr_ptr, jr, jq, bits, x.data.data_ptr(), out.data.data_ptr(),
               x.numel, self.shard_offset(x.numel)[0], _stream())
        self._charge_trunc(x.numel)
        return out

    def sgd_inplace(self, params, grads, c: int, bits: int | None = None) -> None:
        """params[i] -= truncate(mul_const(grads[i], c)) for all i in ONE launch
        (mpc3_rss_sgd_multi); the counters and accounting are those of the
        per-parameter truncate calls, in order."""
        self.sgd_launch(self.sgd_plan(params, grads, bits), range(len(params)), c)

    def sgd_plan(self, params, grads, bits: int | None = None):
        """Take every parameter's truncation counters, in parameter order (the
        order the per-parameter truncate calls would take them), so that the
        updates can then be launched in any grouping (sgd_launch)."""
        bits = self.fp.t if bits is None else bits
        if not 1 <= bits <= 61:
            raise RangeError(f"truncation by {bits} bits outside [1, 61]")
        plan = []
        for p, g in zip(params, grads):
            if not p.data.is_contiguous() or p.shape != g.shape:
                raise ShapeError("in-place SGD needs contiguous parameters of the gradient's shape")
            jr, jq = self.take(TR_RHO), self.take(TR_R)
            self._charge_trunc(p.numel)
            plan.append((p, g, jr, jq, bits))
        return plan

    def sgd_launch(self, plan, which, c: int) -> None:
        idx = list(which)
        for i in range(0, len(idx), K.SGD_MAX_TENSORS):
            chunk = [plan[j] for j in idx[i:i + K.SGD_MAX_TENSORS]]
            if not chunk:
                continue
            arr = (K.SgdTensor * len(chunk))()
            held = []  # contiguous gradient copies stay alive until the launch
            for e, (p, g, jr, jq, _) in enumerate(chunk):
                g = g.contiguous()
                held.append(g)
                arr[e].param, arr[e].grad, arr[e].n, arr[e].j_rho, arr[e].j_r = (
                    p.data.data_ptr(), g.data.data_ptr(), p.numel, jr, jq)
            K.call("mpc3_rss_sgd_multi", self.rk, self.ctr_ptr, arr, len(chunk), chunk[0][4], int(c) % (1 << 64),
                   _stream())
        # the parameters changed through raw pointers (no torch version bump):
        # packed weight operands cached under frozen_weights are stale now
        if self._wcache:
            self._wcache.clear()

    def mul_truncate(self, x, y, bits=None, label="mul.reshare") -> RssTensor:
        """truncate(mul(x, y)) in one launch; same counters and accounting."""
        bits = self.fp.t if bits is None else bits
        if not 1 <= bits <= 61:
            raise RangeError(f"truncation by {bits} bits outside [1, 61]")
        x, y = _broadcast(x, y)
        out = empty(x.shape, x.fp)
        ja = self.take(ARITH)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        K.call("mpc3_rss_mul_truncate", self.rk, self.ctr_ptr, ja, jr, jq, bits, x.data.data_ptr(),
               y.data.data_ptr(), out.data.data_ptr(), x.numel, self.shard_offset(x.numel)[0], _stream())
        self.ledger.ring(label, x.numel)
        self._charge_trunc(x.numel)
        return out

    def _charge_trunc(self, n):
        # P0 -> P1 (c0 - rho), then P1 -> P0 (z1); P2 silent (protocols.py:201-216)
        self.ledger.round("trunc.mask", [(0, 1, n)])
        self.ledger.round("trunc.open", [(1, 0, n)])

    # -- binary world (protocols.py:223-353) --
    def _sign(self, x: RssTensor, mode: int):
        x = x.contiguous()
        n = x.numel
        out = empty(x.shape, x.fp)
        mask = empty(x.shape, x.fp) if mode == K.MODE_RELU else None
        jb = self.take(BIN)
        jx = self.take(XOR, 7)
        ja = self.take(ARITH, [0, 0, 2, 3][mode]) if mode >= K.MODE_DRELU else self.seq[ARITH]
        off, n_total = self.shard_offset(n)
        K.call("mpc3_rss_sign", self.rk, self.ctr_ptr, mode, jb, jx, ja, x.data.data_ptr(), out.data.data_ptr(),
               None if mask is None else mask.data.data_ptr(), n, n_total, off, _stream())
        self._charge_sign(n, mode)
        return out, mask

    def _charge_sign(self, n: int, mode: int) -> None:
        """Rounds / bytes of the a2b + Kogge-Stone + inject + mask circuit."""
        L = self.ledger
        L.round("share.a2b", [(0, 2, n)])
        L.ring("and.ks.g", n)
        for d in (1, 2, 4, 8, 16, 32):
            L.ring(f"and.ks.{d}", 2 * n)
        if mode >= K.MODE_DRELU:
            L.ring("mul.inject", n)
            L.ring("mul.inject", n)
        if mode == K.MODE_RELU:
            L.ring("mul.mask", n)

    def a2b(self, x):
        return self._sign(x, K.MODE_A2B)[0]

    def msb(self, x):
        return self._sign(x, K.MODE_MSB)[0]

    def drelu(self, x):
        return self._sign(x, K.MODE_DRELU)[0]

    def relu_with_mask(self, x):
        return self._sign(x, K.MODE_RELU)

    def relu(self, x):
        return self._sign(x, K.MODE_RELU)[0]

    def compare(self, x, y):
        return self.drelu(self.sub(x, y))

    def bit_inject(self, b: RssTensor) -> RssTensor:
        b = b.contiguous()
        out = empty(b.shape, b.fp)
        ja = self.take(ARITH, 2)
        K.call("mpc3_rss_bit_inject", self.rk, self.ctr_ptr, ja, b.data.data_ptr(), out.data.data_ptr(), b.numel,
               self.shard_offset(b.numel)[0], _stream())
        self.ledger.ring("mul.inject", b.numel)
        self.ledger.ring("mul.inject", b.numel)
        return out

    # -- bilinear layers (protocols.py:97-136, nn.py:435-484) --
    def pack_t(self, src: torch.Tensor, op, rows: int, k: int, zero: torch.Tensor | None = None) -> Packed | None:
        """Role-3 pack of a (rows x k) operand transposed (Packed.t): the
        buffer holds k rows of `rows` columns; None when the operand has no
        transposed gather (dilated im2col, multi-digit dense views)."""
        if not T_PACKS:
            return None
        t = K.Operand()
        C.memmove(C.byref(t), C.byref(op), C.sizeof(K.Operand))
        if op.mode == K.GATHER_IM2COL and op.dh <= 1 and op.dw <= 1:
            t.mode = K.GATHER_WGRAD  # rows (c, u, v), columns (n, y, x): the same gather offsets
        elif op.mode == K.GATHER_DENSE and op.K1 == 1 and op.K2 == op.k and op.t0 == 0 and op.t1 == 0:
            t = K.dense_operand(op.k, op.rows, s_r=op.t2, t2=op.s_r, off=op.off)
        else:
            return None
        t.rows, t.k = op.k, op.rows
        pk = self.pack(src, t, k, rows, 3, zero=zero)
        pk.t = True
        return pk

    def pack(self, src: torch.Tensor, op, rows: int, k: int, role: int, zero: torch.Tensor | None = None,
             geom: tuple[int, int] | None = None) -> Packed:
        """Pack one cross-term operand in the reusable layout (see Packed);
        `zero`: the next GEMM's C, cleared by the same launch when that GEMM
        accumulates atomically; `geom`: (kh, kp) other than Packed.geometry."""
        if role == 3:  # (kp a whole number of 32-byte K-blocks: a TMA box reaching past the end of a row
            kh, kp = k, _round_up(k, 32)  # is zero-filled on a slow path — conv1's GEMM 123 -> 157 us)
        else:
            kh, kp = geom if geom is not None else Packed.geometry(k)
        buf = torch.empty(3 * 8 * rows * kp, dtype=torch.uint8, device=_dev())
        K.call("mpc3_ring_pack_halves_z", src.data_ptr(), src.stride(0), C.byref(op), role, buf.data_ptr(), kp, kh,
               None if zero is None else zero.data_ptr(), 0 if zero is None else zero.numel(), _stream())
        return Packed(buf, rows, k, kh, kp, role)

    @staticmethod
    def _needs_zero(transposed: bool, M: int, N: int, kp: int) -> bool:
        return K.lib().mpc3_ring_gemm_needs_zero(1 if transposed else 0, 3, M, N, kp) == 1

    @staticmethod
    def _pack_key(src: torch.Tensor, op, role: int):
        return (src.data_ptr(), src._version, tuple(src.shape), tuple(src.stride()), role,
                tuple(getattr(op, f) for f, _ in op._fields_))

    def prepack(self, items) -> None:
        """Pack weight operands (role 0) ahead of the layers that use them, on
        the pack stream: items = [(src, op, rows, k)].  _cross_gemm_kept takes
        a matching prepacked B instead of packing it on the critical path."""
        main = _cur()
        ps = self.pack_stream()
        ev = torch.cuda.Event()
        ev.record(main)
        ps.wait_event(ev)
        with torch.cuda.stream(ps):
            packs = [(self._pack_key(src, op, 0),
                      self.pack(src, op, rows, k, 0, geom=Packed.geometry_cs(k) if CS_PACKS else None))
                     for src, op, rows, k in items]
        done = torch.cuda.Event()
        done.record(ps)
        for key, pk in packs:
            self._prepacked[key] = (pk, done)

    def clear_prepacked(self) -> None:
        self._prepacked.clear()

    def _cross_gemm_kept(self, a_src, a_op, b_src, b_op, M, N, Kd, c_col, a_role, keep, a_packed):
        """_cross_gemm in the Packed layout: A packed with role a_role (or
        given), B with the other role; both packs appended to `keep` (the
        backward pass reads them transposed).  A role-1 A is packed once per
        component (role 3) under CS_PACKS."""
        cs = CS_PACKS and a_role == 1 and a_packed is None
        kh, kp = Packed.geometry_cs(Kd) if cs else Packed.geometry(Kd)
        st = _stream()
        main = _cur()
        pre = self._prepacked.pop(self._pack_key(b_src, b_op, 1 - a_role), None) if self._prepacked else None
        if pre is not None:
            pre, done = pre
            if (pre.rows, pre.k, pre.kh, pre.kp) != (N, Kd, kh, kp):
                raise ShapeError("prepacked operand does not match the GEMM")
            main.wait_event(done)
            B = pre.buf
        else:
            B = torch.empty(3 * 8 * N * kp, dtype=torch.uint8, device=_dev())
        ps = self.pack_stream() if OVERLAP_PACK and pre is None else None
        if pre is None and ps is not None and ps != main:  # B on the pack stream, A here
            ev = torch.cuda.Event()
            ev.record(main)
            ps.wait_event(ev)
            K.call("mpc3_ring_pack_halves", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 1 - a_role,
                   B.data_ptr(), kp, kh, ps.cuda_stream)
        elif pre is None:
            K.call("mpc3_ring_pack_halves", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 1 - a_role,
                   B.data_ptr(), kp, kh, st)
        z = torch.empty(3 * M * N, dtype=torch.int64, device=_dev())
        zeroed = False
        if a_packed is not None:
            if (a_packed.rows, a_packed.k, a_packed.kh, a_packed.kp, a_packed.role) != (M, Kd, kh, kp, a_role):
                raise ShapeError("packed operand does not match the GEMM")
            A = a_packed
        else:  # the A pack clears C when the GEMM accumulates atomically
            zeroed = self._needs_zero(cs, M, N, kp)
            A = self.pack_t(a_src, a_op, M, Kd, zero=z if zeroed else None) if cs else None
            if A is None:
                A = self.pack(a_src, a_op, M, Kd, 3 if cs else a_role, zero=z if zeroed else None)
        if ps is not None and ps != main:
            ev2 = torch.cuda.Event()
            ev2.record(ps)
            main.wait_event(ev2)
        if cs:  # A's halves from component planes g, g + 1; B role 0 with halves at kh = kc_half
            self._gemm_cs(A, M, B, N, kp, z, kh, c_col, zeroed, st)
        else:
            K.call("mpc3_ring_gemm_auto_z", A.buf.data_ptr(), B.data_ptr(), z.data_ptr(), 3, M, N, kp,
                   1 if c_col else 0, 1 if zeroed else 0, st)
        if keep is not None:
            keep.extend([A, Packed(B, N, Kd, kh, kp, 1 - a_role)])
        return z

    def dgrad_packed(self, g_src: torch.Tensor, g_op, rows: int, o: int, wp: Packed, c_col: bool) -> torch.Tensor:
        """Input-gradient cross terms z_i = g_i (W_i + W_{i+1}) + g_{i+1} W_i
        (protocols.py:110-115 for nn.py:460-484 / 525-530's g . W) with W read
        transposed from the forward pass's role-0 weight pack (no W^T pack):
        g is packed role 1 with its halves at kc_half = roundup(O, 32), the
        contraction of the MN-read weight rows.  z: [3][rows][wp.k] (or
        column-major)."""
        if wp.role != 0 or wp.rows != o:
            raise ShapeError("weight pack does not match the input gradient")
        kc = _round_up(o, 32)
        st = _stream()
        z = torch.empty(3 * rows * wp.k, dtype=torch.int64, device=_dev())
        zeroed = self._needs_zero(True, rows, wp.k, 2 * kc)
        if CS_PACKS:  # g once per component (role 3): the GEMM reads half h from plane g + h
            A = self.pack_t(g_src, g_op, rows, o, zero=z if zeroed else None)
            if A is not None:  # transposed: A read MN-major too
                K.call("mpc3_ring_gemm_t_z", A.buf.data_ptr(), 3, A.rows, A.kp, 0, wp.buf.data_ptr(), 1, wp.rows,
                       wp.kp, wp.kh, z.data_ptr(), 3, rows, wp.k, kc, 1 if c_col else 0, 1 if zeroed else 0, st)
                return z
            A = self.pack(g_src, g_op, rows, o, 3, zero=z if zeroed else None)
            K.call("mpc3_ring_gemm_t_z", A.buf.data_ptr(), 2, rows, A.kp, 0, wp.buf.data_ptr(), 1, wp.rows, wp.kp,
                   wp.kh, z.data_ptr(), 3, rows, wp.k, kc, 1 if c_col else 0, 1 if zeroed else 0, st)
            return z
        A = torch.empty(3 * 8 * rows * 2 * kc, dtype=torch.uint8, device=_dev())
        K.call("mpc3_ring_pack_halves_z", g_src.data_ptr(), g_src.stride(0), C.byref(g_op), 1, A.data_ptr(), 2 * kc,
               kc, z.data_ptr() if zeroed else None, z.numel() if zeroed else 0, st)
        K.call("mpc3_ring_gemm_t_z", A.data_ptr(), 0, rows, 2 * kc, 0, wp.buf.data_ptr(), 1, wp.rows, wp.kp, wp.kh,
               z.data_ptr(), 3, rows, wp.k, kc, 1 if c_col else 0, 1 if zeroed else 0, st)
        return z

    def wgrad_packed(self, g: RssTensor, xp: Packed) -> torch.Tensor:
        """Weight-gradient cross terms dW_i = (g_i + g_{i+1})^T x_i + g_i^T x_{i+1}
        (protocols.py:110-115 with nn.py:435-457's operands) from a role-0
        pack of g and the forward pass's role-1 pack of x, both read
        transposed.  z is [3][O][xp.k] row-major."""
        op, rows, o = self.grad_operand(g)
        if xp.role not in (1, 3) or (xp.k if xp.t else xp.rows) != rows:
            raise ShapeError("weight-gradient packs do not match")
        # computed as x^T g (A = x, B = g) into the column-major layout, which
        # is the same memory and keeps the epilogue's stores coalesced
        M, N, kc = (xp.rows if xp.t else xp.k), o, _round_up(rows, 32)
        z = torch.empty(3 * M * N, dtype=torch.int64, device=_dev())
        if xp.t and xp.kp < kc:
            raise ShapeError("transposed pack narrower than the contraction")
        if xp.t and kc >= WGRAD_SWAP_MIN_KC and _tile_fill(N, M) * WGRAD_SWAP_EDGE >= _tile_fill(M, N):
            # x packed transposed in the forward pass (its rows are (c, u, v)),
            # long contraction: computed as g^T x with g's pack as the MN-read A
            # and x's pack as a component-plane K-major B (b_mn = 2), row-major
            # [O][(c, u, v)] — the same memory as the column-major x^T g below
            # (AlexNet conv1, kc = 12,800: 99 -> 86 us; the short-contraction
            # weight gradients of conv2-5 are 20-35 % slower this way)
            zeroed = self._needs_zero(True, N, M, 2 * kc)
            gp = self.pack(g.data, op, rows, o, 0, zero=z if zeroed else None)
            K.call("mpc3_ring_gemm_t_z", gp.buf.data_ptr(), 1, gp.rows, gp.kp, gp.kh, xp.buf.data_ptr(), 2, M, xp.kp,
                   0, z.data_ptr(), 3, N, M, kc, 0, 1 if zeroed else 0, _stream())
            return z
        zeroed = self._needs_zero(True, M, N, 2 * kc)
        gp = self.pack(g.data, op, rows, o, 0, zero=z if zeroed else None)
        if xp.t:  # the transposed x pack's rows are this GEMM's rows: read K-major
            K.call("mpc3_ring_gemm_t_z", xp.buf.data_ptr(), 2, M, xp.kp, 0, gp.buf.data_ptr(), 1, gp.rows, gp.kp,
                   gp.kh, z.data_ptr(), 3, M, N, kc, 1, 1 if zeroed else 0, _stream())
            return z
        K.call("mpc3_ring_gemm_t_z", xp.buf.data_ptr(), 3 if xp.role == 3 else 1, xp.rows, xp.kp,
               0 if xp.role == 3 else xp.kh, gp.buf.data_ptr(), 1, gp.rows, gp.kp, gp.kh, z.data_ptr(), 3, M, N, kc, 1,
               1 if zeroed else 0, _stream())
        return z

    def _cross_gemm(self, a_src, a_op, b_src, b_op, M, N, Kd, c_col: bool = False, a_role: int = 0,
                    keep: list | None = None, a_packed: Packed | None = None) -> torch.Tensor:
        """z_i = (x_i + x_{i+1}) y_i + x_i y_{i+1} for the three parties, as one
        batched ring GEMM with inner length 2K (protocols.py:110-115): the
        pack kernel writes the byte-limb planes, the TMA-fed tcgen05 GEMM
        consumes them.  c_col: z[g] column-major (element (m, n) at n*M + m).
        keep / a_packed / a_role: pack A in the reusable Packed layout with
        the given role (the operand roles are symmetric), append it to `keep`,
        or take it ready-packed (training: the weight gradient reuses it)."""
        if keep is not None or a_packed is not None:
            return self._cross_gemm_kept(a_src, a_op, b_src, b_op, M, N, Kd, c_col, a_role, keep, a_packed)
        if CS_PACKS:
            return self._cross_gemm_cs(a_src, a_op, b_src, b_op, M, N, Kd, c_col)
        kp = _round_up(2 * Kd, 32)  # whole 32-byte K-blocks (see pack)
        A = torch.empty(3 * 8 * M * kp, dtype=torch.uint8, device=_dev())
        st = _stream()
        if self._wcache is not None:  # frozen weights (inference): B packed once per weight version
            key = (b_src.data_ptr(), b_src._version, tuple(b_src.shape), tuple(b_src.stride()), kp,
                   tuple(getattr(b_op, f) for f, _ in b_op._fields_))
            B = self._wcache.get(key)
            if B is None:
                B = torch.empty(3 * 8 * N * kp, dtype=torch.uint8, device=_dev())
                K.call("mpc3_ring_pack", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 1, B.data_ptr(), kp, st)
                self._wcache[key] = B
            z = torch.empty(3 * M * N, dtype=torch.int64, device=_dev())
            zeroed = self._needs_zero(False, M, N, kp)
            self._pack_a_zero(a_src, a_op, A, kp, Kd, z, zeroed, st)
            K.call("mpc3_ring_gemm_auto_z", A.data_ptr(), B.data_ptr(), z.data_ptr(), 3, M, N, kp, 1 if c_col else 0,
                   1 if zeroed else 0, st)
            return z
        B = torch.empty(3 * 8 * N * kp, dtype=torch.uint8, device=_dev())
        z = torch.empty(3 * M * N, dtype=torch.int64, device=_dev())
        zeroed = self._needs_zero(False, M, N, kp)
        # the two operand packs are independent: B on the pack stream, A here
        main = _cur()
        ps = self.pack_stream() if OVERLAP_PACK else None
        if ps is not None and ps != main:
            ev = torch.cuda.Event()
            ev.record(main)
            ps.wait_event(ev)
            K.call("mpc3_ring_pack", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 1, B.data_ptr(), kp,
                   ps.cuda_stream)
            self._pack_a_zero(a_src, a_op, A, kp, Kd, z, zeroed, st)
            ev2 = torch.cuda.Event()
            ev2.record(ps)
            main.wait_event(ev2)
        else:
            self._pack_a_zero(a_src, a_op, A, kp, Kd, z, zeroed, st)
            K.call("mpc3_ring_pack", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 1, B.data_ptr(), kp, st)
        K.call("mpc3_ring_gemm_auto_z", A.data_ptr(), B.data_ptr(), z.data_ptr(), 3, M, N, kp, 1 if c_col else 0,
               1 if zeroed else 0, st)
        return z

    def _cross_gemm_cs(self, a_src, a_op, b_src, b_op, M, N, Kd, c_col):
        """_cross_gemm with A as the role-1 operand packed once per component
        (role 3, half the pack's writes) and B role 0 with its halves at the
        32-aligned kc_half (cached under frozen_weights)."""
        kc, kpb = Packed.geometry_cs(Kd)
        st = _stream()
        main = _cur()
        ps = None
        B = None
        key = None
        if self._wcache is not None:  # frozen weights (inference): B packed once per weight version
            key = (b_src.data_ptr(), b_src._version, tuple(b_src.shape), tuple(b_src.stride()), kpb, "cs",
                   tuple(getattr(b_op, f) for f, _ in b_op._fields_))
            B = self._wcache.get(key)
        if B is None:
            B = torch.empty(3 * 8 * N * kpb, dtype=torch.uint8, device=_dev())
            ps = self.pack_stream() if OVERLAP_PACK and key is None else None
            if ps is not None and ps != main:  # B on the pack stream, A here
                ev = torch.cuda.Event()
                ev.record(main)
                ps.wait_event(ev)
            else:
                ps = None
            K.call("mpc3_ring_pack_halves", b_src.data_ptr(), b_src.stride(0), C.byref(b_op), 0, B.data_ptr(), kpb, kc,
                   ps.cuda_stream if ps is not None else st)
            if key is not None:
                self._wcache[key] = B
        z = torch.empty(3 * M * N, dtype=torch.int64, device=_dev())
        zeroed = self._needs_zero(True, M, N, kpb)
        A = self.pack_t(a_src, a_op, M, Kd, zero=z if zeroed else None)
        if A is None:
            A = self.pack(a_src, a_op, M, Kd, 3, zero=z if zeroed else None)
        if ps is not None:
            ev2 = torch.cuda.Event()
            ev2.record(ps)
            main.wait_event(ev2)
        self._gemm_cs(A, M, B, N, kpb, z, kc, c_col, zeroed, st)
        return z

    @staticmethod
    def _gemm_cs(A: Packed, M: int, B: torch.Tensor, N: int, kpb: int, z, kc: int, c_col, zeroed, st) -> None:
        """The ring GEMM of a role-3 A (halves from component planes g, g + 1;
        read MN-major when packed transposed) and a role-0 B whose halves
        start at kc = kc_half."""
        if A.t:
            K.call("mpc3_ring_gemm_t_z", A.buf.data_ptr(), 3, A.rows, A.kp, 0, B.data_ptr(), 0, N, kpb, 0,
                   z.data_ptr(), 3, M, N, kc, 1 if c_col else 0, 1 if zeroed else 0, st)
        else:
            K.call("mpc3_ring_gemm_t_z", A.buf.data_ptr(), 2, M, A.kp, 0, B.data_ptr(), 0, N, kpb, 0, z.data_ptr(), 3,
                   M, N, kc, 1 if c_col else 0, 1 if zeroed else 0, st)

    @staticmethod
    def _pack_a_zero(a_src, a_op, A, kp, Kd, z, zeroed, st):
        """Role-0 pack of A (adjacent halves), clearing the GEMM's C with it when needed."""
        K.call("mpc3_ring_pack_halves_z", a_src.data_ptr(), a_src.stride(0), C.byref(a_op), 0, A.data_ptr(), kp, Kd,
               z.data_ptr() if zeroed else None, z.numel() if zeroed else 0, st)

    @property
    def c_col_ok(self) -> bool:
        return True

    def _finish(self, z, view, out: RssTensor, bits, label, bias: RssTensor | None = None, bias_dim: int = 1,
                z_off: int = 0):
        """Reshare + truncate (+ bias) of the cross terms z through `view`;
        z_off (elements, may be negative): added to z's address, for a z that
        holds only the view's crop while the view indexes the full tensor."""
        ja = self.take(ARITH)
        jr = jq = 0
        if bits:
            jr, jq = self.take(TR_RHO), self.take(TR_R)
        full = math.prod(view.full)
        if bias is None:
            K.call("mpc3_rss_reshare_truncate", self.rk, self.ctr_ptr, ja, jr, jq, bits,
                   (z.data_ptr() + 8 * z_off) % (1 << 64), C.byref(view),
                   out.data.data_ptr(), self.shard_offset(full)[0], _stream())
        else:  # the shared bias added in the same pass (a local add, nn.py bias extension)
            if bias.ndim != 1 or bias.data.stride(1) != 1:
                raise ShapeError("bias must be a 1-d shared vector with unit stride")
            K.call("mpc3_rss_reshare_truncate_bias", self.rk, self.ctr_ptr, ja, jr, jq, bits, z.data_ptr(),
                   C.byref(view), bias.data.data_ptr(), bias.data.stride(0), bias_dim, out.data.data_ptr(),
                   self.shard_offset(full)[0], _stream())
        self.ledger.ring(label, full)
        if bits:
            self._charge_trunc(full)
        return out

    def _finish_relu(self, z, view, shape, bits, label, bias: RssTensor | None = None, bias_dim: int = 1):
        """_finish followed by relu_with_mask in ONE launch (mpc3_rss_layer_sign):
        the same counters in the same order, the same shares and accounting;
        the pre-activation tensor is never materialised.  -> (relu, mask)."""
        return self.relu_epilogue_end(self.relu_epilogue_begin(z, view, shape, bits, label, bias, bias_dim))

    def relu_epilogue_begin(self, z, view, shape, bits, label, bias: RssTensor | None = None, bias_dim: int = 1):
        """First half of _finish_relu: the layer epilogue's counters (reshare,
        truncation) and accounting, taken here in program order; the launch
        waits for relu_epilogue_end, so a residual block's shortcut branch
        can run (and take its own counters) in between."""
        if bias is not None and (bias.ndim != 1 or bias.data.stride(1) != 1):
            raise ShapeError("bias must be a 1-d shared vector with unit stride")
        ja = self.take(ARITH)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        full = math.prod(view.full)
        self.ledger.ring(label, full)
        self._charge_trunc(full)
        return {"z": z, "view": view, "shape": shape, "bits": bits, "bias": bias, "bias_dim": bias_dim,
                "ja": ja, "jr": jr, "jq": jq, "full": full}

    def relu_epilogue_end(self, pend: dict, residual: RssTensor | None = None):
        """Second half: the ReLU's counters, then ONE launch of the layer's
        reshare + truncate (+ bias) (+ the residual shortcut, a local add) and
        the ReLU (mpc3_rss_layer_sign_residual).  -> (relu, mask); mask None
        when relu_masks is off."""
        jb = self.take(BIN)
        jx = self.take(XOR, 7)
        jm = self.take(ARITH, 3)
        full, shape, bias, view = pend["full"], pend["shape"], pend["bias"], pend["view"]
        off, n_total = self.shard_offset(full)
        out, mask = empty(shape, self.fp), (empty(shape, self.fp) if self.relu_masks else None)
        res = None
        if residual is not None:
            if tuple(residual.shape) != tuple(shape):
                raise ShapeError(f"residual {tuple(residual.shape)} does not match the layer output {tuple(shape)}")
            res = residual.data.contiguous()
        K.call("mpc3_rss_layer_sign_residual", self.rk, self.ctr_ptr, pend["ja"], pend["jr"], pend["jq"],
               pend["bits"], pend["z"].data_ptr(), C.byref(view), None if bias is None else bias.data.data_ptr(),
               0 if bias is None else bias.data.stride(0), pend["bias_dim"], None if res is None else res.data_ptr(),
               0 if res is None else res.stride(0), K.MODE_RELU, jb, jx, jm, out.data.data_ptr(),
               None if mask is None else mask.data.data_ptr(), off, n_total, _stream())
        self._charge_sign(full, K.MODE_RELU)
        return out, mask

    def matmul(self, x: RssTensor, y: RssTensor, bits: int | None = None, wgrad: bool = False,
               bias: RssTensor | None = None, keep: list | None = None, x_packed: Packed | None = None,
               x_role: int = 0, relu: bool = False):
        """matmul_shares (protocols.py:97-117): cross terms, reshare, truncate.
        wgrad=True marks a weight gradient g^T x whose inner dimension is the
        batch: under data parallelism the shards' cross terms are summed
        before the (replicated) reshare + truncate.  keep / x_packed / x_role:
        see _cross_gemm."""
        if x.ndim != 2 or y.ndim != 2 or x.shape[1] != y.shape[0]:
            raise ShapeError(f"matmul shapes {x.shape} x {y.shape}")
        m, k = x.shape
        n = y.shape[1]
        check_accumulation(k)  # this rank's accumulation (see conv2d_wgrad)
        bits = self.fp.t if bits is None else bits
        if not 1 <= bits <= 61:
            raise RangeError(f"truncation by {bits} bits outside [1, 61]")
        xs, ys = x.data.stride(), y.data.stride()
        a_op = K.dense_operand(m, k, s_r=xs[1], t2=xs[2])
        b_op = self.matmul_weight_operand(y)[0]
        z = self._cross_gemm(x.data, a_op, y.data, b_op, m, n, k, a_role=x_role, keep=keep, a_packed=x_packed)
        out = empty((m, n), x.fp)
        if wgrad:
            self._reduce_cross_terms(z)
            with self.replicated():
                return self._finish(z, K.make_view((1, 1, m, n)), out, bits, "mul.reshare")
        if relu:  # fused with the ReLU after it: -> (relu, mask)
            return self._finish_relu(z, K.make_view((1, 1, m, n)), (m, n), bits, "mul.reshare", bias=bias, bias_dim=3)
        return self._finish(z, K.make_view((1, 1, m, n)), out, bits, "mul.reshare", bias=bias, bias_dim=3)

    def fc_wgrad_packed(self, g: RssTensor, xp: Packed, bits: int) -> RssTensor:
        """Fully-connected weight gradient g^T x (nn.py:525-527) from x's
        forward pack (rows: batch, K: in)."""
        check_accumulation(g.shape[0])  # this rank's accumulation (see conv2d_wgrad)
        m, n = g.shape[1], (xp.rows if xp.t else xp.k)
        z = self.wgrad_packed(g, xp)
        out = empty((m, n), self.fp)
        self._reduce_cross_terms(z)
        with self.replicated():
            return self._finish(z, K.make_view((1, 1, m, n)), out, bits, "mul.reshare")

    def fc_dgrad_packed(self, g: RssTensor, wp: Packed, bits: int | None = None) -> RssTensor:
        """g . W for a fully-connected layer (nn.py:529-530) with W from its
        forward pack; the same reshare + truncate as matmul."""
        b, o = g.shape
        bits = self.fp.t if bits is None else bits
        check_accumulation(o)
        op, rows, k = self.grad_operand(g)
        z = self.dgrad_packed(g.data, op, rows, o, wp, False)
        out = empty((b, wp.k), g.fp)
        return self._finish(z, K.make_view((1, 1, b, wp.k)), out, bits, "mul.reshare")

    @staticmethod
    def conv_weight_operand(k: RssTensor):
        """(operand, rows, K) of a conv kernel (O, C, kh, kw) as the GEMM's B."""
        ks = k.data.stride()
        o, c, kh, kw = k.shape
        return K.dense_operand(o, c * kh * kw, s_r=ks[1], t0=ks[2], t1=ks[3], t2=ks[4], K1=kh, K2=kw), o, c * kh * kw

    @staticmethod
    def matmul_weight_operand(y: RssTensor):
        """(operand, rows, K) of the right matmul operand y (k, n) as the GEMM's B."""
        ys = y.data.stride()
        return K.dense_operand(y.shape[1], y.shape[0], s_r=ys[2], t2=ys[1]), y.shape[1], y.shape[0]

    def conv2d(self, x: RssTensor, k: RssTensor, stride=(1, 1), padding=(0, 0), bits=None,
               bias: RssTensor | None = None, keep: list | None = None, relu: bool = False):
        """conv2d_shares (protocols.py:120-136), NCHW cross-correlation;
        `bias` (inference extension) is added per output channel after the
        truncation in the same kernel."""
        if x.ndim != 4 or k.ndim != 4 or x.shape[1] != k.shape[1]:
            raise ShapeError(f"kernel {k.shape} incompatible with input {x.shape}")
        nb, c, h, w = x.shape
        o, _, kh, kw = k.shape
        sh, sw = stride
        ph, pw = padding
        check_accumulation(c * kh * kw)
        if h + 2 * ph < kh or w + 2 * pw < kw:
            raise ShapeError("kernel larger than padded input")
        bits = self.fp.t if bits is None else bits
        oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        xs, ks = x.data.stride(), k.data.stride()
        a_op = K.conv_operand(K.GATHER_IM2COL, nb * oh * ow, c * kh * kw, nb, c, h, w, xs[1:], kh, kw, sh, sw, ph, pw,
                              oh, ow)
        b_op = self.conv_weight_operand(k)[0]
        col = self.c_col_ok
        M = nb * oh * ow
        # keep: x's im2col pack (role 1) is left for the weight gradient
        z = self._cross_gemm(x.data, a_op, k.data, b_op, M, o, c * kh * kw, c_col=col, a_role=1 if keep is not None
                             else 0, keep=keep)
        out = empty((nb, o, oh, ow), x.fp)
        # z[(n, y, x), o]: column-major keeps each (n, o) plane's (y, x) run contiguous
        zs = (oh * ow, M, ow, 1) if col else (oh * ow * o, 1, ow * o, o)
        view = K.make_view((nb, o, oh, ow), z_stride=zs)
        if relu == "defer":  # the epilogue's counters now, the fused launch later (relu_epilogue_end)
            return self.relu_epilogue_begin(z, view, (nb, o, oh, ow), bits, "mul.reshare", bias=bias, bias_dim=1)
        if relu:  # fused with the ReLU after it: -> (relu, mask)
            return self._finish_relu(z, view, (nb, o, oh, ow), bits, "mul.reshare", bias=bias, bias_dim=1)
        return self._finish(z, view, out, bits, "mul.reshare", bias=bias, bias_dim=1)

    def conv2d_wgrad(self, x: RssTensor, g: RssTensor, kernel, stride, padding, bits,
                     x_packed: Packed | None = None) -> RssTensor:
        """Kernel gradient (nn.py:435-457) as one direct implicit GEMM with
        K = N*OH*OW; the reference's dilated zeros contribute nothing, and the
        zero shares / truncation words are indexed over its full (C,O,fh,fw)
        output so the result is bit-exact.  x_packed: x's im2col pack from the
        forward pass, read transposed beside a role-0 pack of g."""
        nb, c, h, w = x.shape
        nb2, o, oh, ow = g.shape
        kh, kw = kernel
        sh, sw = stride
        ph, pw = padding
        ghd, gwd = (oh - 1) * sh + 1, (ow - 1) * sw + 1
        # the reference's 2^20 bound (ring.py:191-195) guards ITS float-limb
        # products; here it applies to this rank's batch shard, whose cross
        # terms the int8-limb GEMM computes exactly (split-K, any length);
        # the ranks' sums meet in an exact mod-2^64 all-reduce, so data
        # parallelism may exceed the bound the single-process reference
        # would raise for (AlexNet conv1 past a global batch of ~766)
        check_accumulation(nb * ghd * gwd)
        if h + 2 * ph < ghd or w + 2 * pw < gwd:
            raise ShapeError("kernel larger than padded input")
        fh, fw = h + 2 * ph - ghd + 1, w + 2 * pw - gwd + 1
        xs, gs = x.data.stride(), g.data.stride()
        a_op = K.conv_operand(K.GATHER_WGRAD, c * kh * kw, nb * oh * ow, nb, c, h, w, xs[1:], kh, kw, sh, sw, ph, pw,
                              oh, ow)
        b_op = K.dense_operand(o, nb * oh * ow, s_r=gs[2], t0=gs[1], t1=gs[3], t2=gs[4], K1=oh, K2=ow)
        col = self.c_col_ok
        M = c * kh * kw
        if x_packed is not None:  # z[o][(c, u, v)]: the column-major layout below
            if ((x_packed.k, x_packed.rows) if x_packed.t else (x_packed.rows, x_packed.k)) != (nb * oh * ow, M):
                raise ShapeError("weight-gradient packs do not match the layer")
            z, col = self.wgrad_packed(g, x_packed), True
        else:
            z = self._cross_gemm(x.data, a_op, g.data, b_op, M, o, nb * oh * ow, c_col=col)
        out = empty((o, c, kh, kw), x.fp)
        zs = (kh * kw, M, kw, 1) if col else (kh * kw * o, 1, kw * o, o)
        view = K.make_view((c, o, fh, fw), crop=(c, o, kh, kw), z_stride=zs,
                           out_stride=(kh * kw, c * kh * kw, kw, 1), z_plane=c * kh * kw * o)
        self._reduce_cross_terms(z)  # sum over the batch shards before reshare / truncate
        with self.replicated():
            return self._finish(z, view, out, bits, "mul.reshare")

    def grad_operand(self, g: RssTensor):
        """(operand, rows, K) of an output gradient as the left operand of its
        layer's input-gradient GEMM: rows are the batch positions (n, y, x),
        K the output channels (the layout both that GEMM and the weight
        gradient read)."""
        gs = g.data.stride()
        if g.ndim == 2:
            b, o = g.shape
            return K.dense_operand(b, o, s_r=gs[1], t2=gs[2]), b, o
        nb, o, oh, ow = g.shape
        return (K.conv_operand(K.GATHER_IM2COL, nb * oh * ow, o, nb, o, oh, ow, gs[1:], 1, 1, 1, 1, 0, 0, oh, ow),
                nb * oh * ow, o)

    def conv2d_dgrad(self, g: RssTensor, k: RssTensor, stride, padding, in_shape, bits,
                     w_packed: Packed | None = None) -> RssTensor:
        """Input gradient (nn.py:460-484).  Two bit-identical formulations
        (same ring values, same PRF words at the reference's flat indices of
        the full (N, C, hf, wf) correlation); the faster one for the shape
        (_dgrad_use_im2col): the transposed convolution (GEMM with inner
        length O + col2im) for small maps, the reference's correlation of the
        padded gradient with the flipped kernel, cropped to the rows the layer
        keeps (GEMM with inner length O*kh*kw + reshare, no col2im), for
        stride 1 on maps large enough to fill the GPU — e.g. VGG's 64 x 64
        layers, where the first would be a K=64 GEMM writing kh*kw times the
        input gradient."""
        nb, o, oh, ow = g.shape
        o2, c, kh, kw = k.shape
        if tuple(stride) == (1, 1) and _dgrad_use_im2col(nb, oh, ow, kh, kw, padding):
            return self.conv2d_dgrad_im2col(g, k, stride, padding, in_shape, bits)
        return self.conv2d_dgrad_col2im(g, k, stride, padding, in_shape, bits, w_packed=w_packed)

    def conv2d_dgrad_col2im(self, g: RssTensor, k: RssTensor, stride, padding, in_shape, bits,
                            w_packed: Packed | None = None) -> RssTensor:
        """Input gradient as a transposed convolution: one ring GEMM
        cols = g^T-rows x k (inner length O) and a fused col2im + reshare +
        truncate + embed kernel."""
        nb, o, oh, ow = g.shape
        o2, c, kh, kw = k.shape
        sh, sw = stride
        ph, pw = padding
        h, w = in_shape[-2:]
        check_accumulation(o * kh * kw)
        k = k.contiguous()
        gs = g.data.stride()
        a_op = K.conv_operand(K.GATHER_IM2COL, nb * oh * ow, o, nb, o, oh, ow, gs[1:], 1, 1, 1, 1, 0, 0, oh, ow)
        ncols = c * kh * kw
        b_op = K.dense_operand(ncols, o, s_r=1, t2=ncols)
        col = self.c_col_ok  # column-major cols: the col2im gathers along x coalesce
        if w_packed is not None:  # the forward pass's weight pack, read transposed
            if w_packed.k != ncols:
                raise ShapeError("weight pack does not match the layer")
            z = self.dgrad_packed(g.data, a_op, nb * oh * ow, o, w_packed, col)
        else:
            z = self._cross_gemm(g.data, a_op, k.data, b_op, nb * oh * ow, ncols, o, c_col=col)
        hf, wf = (oh - 1) * sh + kh, (ow - 1) * sw + kw
        # every input position is some correlation element's embedding unless
        # the forward conv dropped trailing rows / columns (floor division):
        # only then do the uncovered positions need zeros
        out = (empty if h + ph <= hf and w + pw <= wf else zeros)((nb, c, h, w), g.fp)
        ja = self.take(ARITH)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        full = nb * c * hf * wf
        K.call("mpc3_rss_col2im_reshare_truncate_layout", self.rk, self.ctr_ptr, ja, jr, jq, bits, z.data_ptr(),
               1 if col else 0, nb, c, oh, ow, kh, kw, sh, sw, ph, pw, h, w, out.data.data_ptr(),
               self.shard_offset(full)[0], _stream())
        self.ledger.ring("mul.reshare", full)
        self._charge_trunc(full)
        return out

    def conv2d_dgrad_im2col(self, g: RssTensor, k: RssTensor, stride, padding, in_shape, bits) -> RssTensor:
        """Input gradient by explicit im2col of the dilated, padded gradient
        (the reference's formulation, nn.py:460-484), computing only the
        window of the full correlation the layer keeps when the padding
        allows."""
        nb, o, oh, ow = g.shape
        o2, c, kh, kw = k.shape
        sh, sw = stride
        ph, pw = padding
        h, w = in_shape[-2:]
        check_accumulation(o * kh * kw)
        hf, wf = (oh - 1) * sh + kh, (ow - 1) * sw + kw
        gs, ks = g.data.stride(), k.data.stride()
        b_op = K.dense_operand(c, o * kh * kw, s_r=ks[2], off=(kh - 1) * ks[3] + (kw - 1) * ks[4], t0=ks[1],
                               t1=-ks[3], t2=-ks[4], K1=kh, K2=kw)
        out = (empty if h + ph <= hf and w + pw <= wf else zeros)((nb, c, h, w), g.fp)
        ch, cw = max(0, min(h, hf - ph)), max(0, min(w, wf - pw))
        crop = (nb, c, ch, cw)
        qh, qw = kh - 1 - ph, kw - 1 - pw
        if qh >= 0 and qw >= 0 and ch and cw:
            # only the rows the layer keeps: the (ch, cw) window of the full
            # correlation at (ph, pw) is the correlation of g padded by
            # (kh-1-ph, kw-1-pw); z holds that window (column-major when the
            # GEMM can) and the view still indexes the full (N, C, hf, wf)
            # output, so the PRF words stay at the reference's flat indices
            M = nb * ch * cw
            a_op = K.conv_operand(K.GATHER_IM2COL, M, o * kh * kw, nb, o, oh, ow, gs[1:], kh, kw, 1, 1, qh, qw,
                                  ch, cw, dh=sh, dw=sw)
            col = self.c_col_ok
            z = self._cross_gemm(g.data, a_op, k.data, b_op, M, c, o * kh * kw, c_col=col)
            zs = (ch * cw, M, cw, 1) if col else (ch * cw * c, 1, cw * c, c)
            view = K.make_view((nb, c, hf, wf), crop=crop, origin=(0, 0, ph, pw), z_stride=zs,
                               out_stride=(c * h * w, h * w, w, 1), out_plane=nb * c * h * w, z_plane=M * c)
            return self._finish(z, view, out, bits, "mul.reshare", z_off=-(ph * zs[2] + pw * zs[3]))
        a_op = K.conv_operand(K.GATHER_IM2COL, nb * hf * wf, o * kh * kw, nb, o, oh, ow, gs[1:], kh, kw, 1, 1,
                              kh - 1, kw - 1, hf, wf, dh=sh, dw=sw)
        z = self._cross_gemm(g.data, a_op, k.data, b_op, nb * hf * wf, c, o * kh * kw)
        view = K.make_view((nb, c, hf, wf), crop=crop, origin=(0, 0, ph, pw), z_stride=(hf * wf * c, 1, wf * c, c),
                           out_stride=(c * h * w, h * w, w, 1), out_plane=nb * c * h * w, z_plane=nb * hf * wf * c)
        return self._finish(z, view, out, bits, "mul.reshare")

    # -- pooling (protocols.py:139-159, nn.py:487-499) --
    def _area_params(self, area: int):
        if area & (area - 1) == 0:
            return area.bit_length() - 1, 1
        return self.fp.t, int(fx_encode(1.0 / area, self.fp))

    def avgpool(self, x: RssTensor, window, stride=None, padding=(0, 0)) -> RssTensor:
        """avgpool_shares (protocols.py:139-159); padding (zero, divisor kh*kw)
        extends the reference for ResNet's stem (composed: pad + avgpool)."""
        kh, kw = window
        sh, sw = stride or window
        ph, pw = padding
        if x.ndim != 4 or x.shape[2] + 2 * ph < kh or x.shape[3] + 2 * pw < kw:
            raise ShapeError("window larger than input")
        x = x.contiguous()
        nb, c, h, w = x.shape
        oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        bits, mulc = self._area_params(kh * kw)
        out = empty((nb, c, oh, ow), x.fp)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        K.call("mpc3_rss_avgpool", self.rk, self.ctr_ptr, jr, jq, bits, mulc, x.data.data_ptr(), out.data.data_ptr(),
               nb, c, h, w, kh, kw, sh, sw, ph, pw, self.shard_offset(out.numel)[0], _stream())
        self._charge_trunc(out.numel)
        return out

    def avgpool_backward(self, g: RssTensor, window, stride, in_shape, padding=(0, 0),
                         mask: RssTensor | None = None) -> RssTensor:
        """nn.py:487-499; with `mask`, also the backward of the ReLU before the
        pool (g * mask, "mul.mask") in the same pass: the same counters in the
        same order (TRUNC_RHO, TRUNC_R, then ARITH_ZERO) and the same shares."""
        kh, kw = window
        sh, sw = stride
        ph, pw = padding
        g = g.contiguous()
        nb, c, oh, ow = g.shape
        h, w = in_shape[-2:]
        bits, mulc = self._area_params(kh * kw)
        out = empty((nb, c, h, w), g.fp)
        jr, jq = self.take(TR_RHO), self.take(TR_R)
        off = self.shard_offset(out.numel)[0]
        if mask is None:
            K.call("mpc3_rss_avgpool_backward", self.rk, self.ctr_ptr, jr, jq, bits, mulc, g.data.data_ptr(),
                   out.data.data_ptr(), nb, c, h, w, oh, ow, kh, kw, sh, sw, ph, pw, off, _stream())
            self._charge_trunc(out.numel)
            return out
        mask = mask.contiguous()
        if mask.shape != out.shape:
            raise ShapeError(f"mask {mask.shape} does not match the pool input {out.shape}")
        ja = self.take(ARITH)
        K.call("mpc3_rss_avgpool_backward_mask", self.rk, self.ctr_ptr, jr, jq, bits, mulc, g.data.data_ptr(),
               mask.data.data_ptr(), ja, out.data.data_ptr(), nb, c, h, w, oh, ow, kh, kw, sh, sw, ph, pw, off,
               _stream())
        self._charge_trunc(out.numel)
        self.ledger.ring("mul.mask", out.numel)
        return out

    def maxpool(self, x: RssTensor, window, stride=None, padding=(0, 0)) -> RssTensor:
        """Max-pool extension (absent from the reference):
        each (kh, kw) window flattened row-major (mpc3_rss_window_gather;
        padded positions hold the public constant -2^60 in component 0) and
        reduced by max_tree (protocols.py:356-380) — the composition of the
        reference's own primitives, share for share."""
        kh, kw = window
        sh, sw = stride or window
        ph, pw = padding
        if x.ndim != 4 or x.shape[2] + 2 * ph < kh or x.shape[3] + 2 * pw < kw or 2 * ph > kh or 2 * pw > kw:
            raise ShapeError("max-pool window does not fit the input")
        x = x.contiguous()
        nb, c, h, w = x.shape
        oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        win = empty((nb, c, oh, ow, kh * kw), x.fp)
        K.call("mpc3_rss_window_gather", x.data.data_ptr(), win.data.data_ptr(), nb, c, h, w, kh, kw, sh, sw, ph, pw,
               MAXPOOL_PAD, _stream())
        return self.max_tree(win)

    def div_area(self, x: RssTensor, area: int) -> RssTensor:
        bits, mulc = self._area_params(area)
        if mulc != 1:
            return self.mul_truncate_const(x, mulc, bits)
        return self.truncate(x, bits)

    def mul_truncate_const(self, x, c, bits):
        return self.truncate(self.mul_const(x, c), bits)

    # -- comparisons and function approximations (protocols.py:356-468) --
    def max_tree(self, v: RssTensor) -> RssTensor:
        m = v.shape[-1] if v.ndim else 0
        if m < 1:
            raise ShapeError("max_tree needs at least one element")
        lead = v.shape[:-1]
        rows = int(np.prod(lead, dtype=np.int64)) if lead else 1
        v = v.contiguous()
        levels, mm = [], m
        while mm > 1:
            levels.append(mm)
            mm = mm // 2 + mm % 2
        row_off, rows_total = self.shard_offset(rows)
        if MAXTREE_FUSED and levels and len(levels) <= 16 and row_off % 2 == 0 and rows <= MAXTREE_FUSED_MAX_ROWS:
            # every level in one launch (mpc3_rss_max_tree), the same counters
            jb, jx, ja = (np.zeros(len(levels), np.uint64) for _ in range(3))
            for i, ml in enumerate(levels):
                jb[i], jx[i], ja[i] = self.take(BIN), self.take(XOR, 7), self.take(ARITH, 3)
                self._charge_sign(rows * (ml // 2), K.MODE_RELU)
            scratch = torch.empty(2 * 3 * rows * ((m + 1) // 2), dtype=torch.int64, device=_dev())
            out = empty(lead + (1,), v.fp)
            K.call("mpc3_rss_max_tree", self.rk, self.ctr_ptr, len(levels), jb.ctypes.data, jx.ctypes.data,
                   ja.ctypes.data, v.data.data_ptr(), scratch.data_ptr(), out.data.data_ptr(), rows, m, row_off,
                   rows_total, _stream())
            return out.apply(lambda d: d[..., 0].contiguous())
        while m > 1:
            # one launch per level: b + relu(a - b) over the (even, odd) column
            # pairs, the odd tail passed through (mpc3_rss_max_level); counters
            # and accounting are those of the relu on the (rows, m/2) difference
            k, mo = m // 2, m // 2 + m % 2
            out = empty(lead + (mo,), v.fp)
            n = rows * k
            jb = self.take(BIN)
            jx = self.take(XOR, 7)
            ja = self.take(ARITH, 3)
            off, n_total = self.shard_offset(n)
            K.call("mpc3_rss_max_level", self.rk, self.ctr_ptr, jb, jx, ja, v.data.data_ptr(), out.data.data_ptr(),
                   rows, m, off, n_total, _stream())
            self._charge_sign(n, K.MODE_RELU)
            v, m = out, mo
        return v.apply(lambda d: d[..., 0].contiguous())

    def exp_approx(self, x: RssTensor, cfg: ExpConfig = ExpConfig()) -> RssTensor:
        s = cfg.squarings
        if self.fp.t + 2 * s > 61:
            raise ConfigError(f"m={cfg.m} too large for t={self.fp.t}")
        steps = [(K.CHAIN_ADDC, 0, int(fx_encode(float(cfg.m), self.fp)))]
        steps += [(K.CHAIN_SQ, self.fp.t + 2 * s if i == 0 else self.fp.t, 0) for i in range(s)]
        return self._chain(x, steps)

    def reciprocal(self, y: RssTensor, cfg: ReciprocalConfig = ReciprocalConfig()) -> RssTensor:
        steps = [(K.CHAIN_SETC, 0, int(fx_encode(1.0 / cfg.Y, self.fp)))]
        for _ in range(cfg.iterations):
            steps += [(K.CHAIN_SQT, self.fp.t, 0), (K.CHAIN_MULX, self.fp.t, 0), (K.CHAIN_NEWTON, 0, 0)]
        return self._chain(y, steps)

    def _chain(self, x: RssTensor, steps) -> RssTensor:
        """One launch for a chain of local ops and mul+truncates on the same
        elements (mpc3_rss_chain); counters, accounting and results are those
        of the unfused sequence of mul_truncate calls."""
        muls = (K.CHAIN_SQ, K.CHAIN_MULX, K.CHAIN_SQT)
        nmul = sum(1 for op, _, _ in steps if op in muls)
        if len(steps) > K.CHAIN_MAX_STEPS:  # e.g. ReciprocalConfig(iterations >= 16)
            return self._chain_unfused(x, steps)
        for op, bits, _ in steps:
            if op in muls and not 1 <= bits <= 61:
                raise RangeError(f"truncation by {bits} bits outside [1, 61]")
        x = x.contiguous()
        out = empty(x.shape, x.fp)
        ja, jr, jq = self.take(ARITH, nmul), self.take(TR_RHO, nmul), self.take(TR_R, nmul)
        prog, count = K.chain_program(steps)
        K.call("mpc3_rss_chain", self.rk, self.ctr_ptr, prog, count, ja, jr, jq, x.data.data_ptr(),
               out.data.data_ptr(), x.numel, self.shard_offset(x.numel)[0], _stream())
        for _ in range(nmul):
            self.ledger.ring("mul.reshare", x.numel)
            self._charge_trunc(x.numel)
        return out

    def _chain_unfused(self, x: RssTensor, steps) -> RssTensor:
        """The chain program as separate launches (one mul_truncate per
        multiply): the same counters, accounting and shares as _chain, for
        programs longer than one chain launch holds."""
        x = x.contiguous()
        z, t = x, None
        for op, bits, c in steps:
            if op == K.CHAIN_ADDC:
                z = self.add_const(z, c)
            elif op == K.CHAIN_SETC:
                z = self.const_share(c, x.shape)
            elif op == K.CHAIN_SQ:
                z = self.mul_truncate(z, z, bits)
            elif op == K.CHAIN_SQT:
                t = self.mul_truncate(z, z, bits)
            elif op == K.CHAIN_MULX:
                t = self.mul_truncate(x, t, bits)
            elif op == K.CHAIN_NEWTON:
                z = self.sub(self.mul_const(z, 2), t)
            else:
                raise ConfigError(f"unknown chain op {op}")
        return z

    def division(self, x, y, cfg: ReciprocalConfig = ReciprocalConfig()):
        return self.mul_truncate(x, self.reciprocal(y, cfg))

    def softmax_loss(self, z: RssTensor, y: RssTensor, cfg: ReciprocalConfig = ReciprocalConfig(),
                     exp_cfg: ExpConfig = ExpConfig()) -> RssTensor:
        """softmax(z) - y (the loss gradient, nn.py:561-568) in ONE launch
        (mpc3_rss_softmax_loss): the counters, PRF words, shares and
        accounting of softmax() followed by sub()."""
        rows_shape, d = z.shape[:-1], z.shape[-1]
        rows = int(np.prod(rows_shape, dtype=np.int64)) if rows_shape else 1
        if d > cfg.Y:
            raise ConfigError(f"class count {d} exceeds reciprocal domain Y={cfg.Y}")
        if y.shape != z.shape:
            raise ShapeError(f"logit/label shapes {z.shape} vs {y.shape}")
        levels, mm = [], d
        while mm > 1:
            levels.append(mm)
            mm = mm // 2 + mm % 2
        s = exp_cfg.squarings
        if self.fp.t + 2 * s > 61:
            raise ConfigError(f"m={exp_cfg.m} too large for t={self.fp.t}")
        exp_steps = [(K.CHAIN_ADDC, 0, int(fx_encode(float(exp_cfg.m), self.fp)))]
        exp_steps += [(K.CHAIN_SQ, self.fp.t + 2 * s if i == 0 else self.fp.t, 0) for i in range(s)]
        rec_steps = [(K.CHAIN_SETC, 0, int(fx_encode(1.0 / cfg.Y, self.fp)))]
        for _ in range(cfg.iterations):
            rec_steps += [(K.CHAIN_SQT, self.fp.t, 0), (K.CHAIN_MULX, self.fp.t, 0), (K.CHAIN_NEWTON, 0, 0)]
        row_off, rows_total = self.shard_offset(rows)
        if not levels or len(levels) > 16 or len(exp_steps) > K.CHAIN_MAX_STEPS or \
                len(rec_steps) > K.CHAIN_MAX_STEPS or row_off % 2:
            return self.sub(self.softmax(z, cfg), y)
        z, y = z.contiguous(), y.contiguous()
        a = K.SoftmaxLossArgs()
        a.levels = len(levels)
        for i, ml in enumerate(levels):  # max_tree (protocols.py:356-380)
            a.j_bin[i], a.j_xor[i], a.j_arith[i] = self.take(BIN), self.take(XOR, 7), self.take(ARITH, 3)
            self._charge_sign(rows * (ml // 2), K.MODE_RELU)
        prog_e, ne = K.chain_program(exp_steps)
        prog_r, nr = K.chain_program(rec_steps)
        for j, prog, n, steps, cnt in ((a.exp_j, prog_e, ne, exp_steps, rows * d), (a.rec_j, prog_r, nr, rec_steps, rows)):
            nmul = sum(1 for op, _, _ in steps if op in (K.CHAIN_SQ, K.CHAIN_MULX, K.CHAIN_SQT))
            j[0], j[1], j[2] = self.take(ARITH, nmul), self.take(TR_RHO, nmul), self.take(TR_R, nmul)
            for _ in range(nmul):
                self.ledger.ring("mul.reshare", cnt)
                self._charge_trunc(cnt)
        a.exp_steps, a.exp_count = C.cast(prog_e, C.POINTER(K.ChainStep)), ne
        a.rec_steps, a.rec_count = C.cast(prog_r, C.POINTER(K.ChainStep)), nr
        a.fin_j[0], a.fin_j[1], a.fin_j[2] = self.take(ARITH), self.take(TR_RHO), self.take(TR_R)
        self.ledger.ring("mul.reshare", rows * d)
        self._charge_trunc(rows * d)
        a.bits = self.fp.t
        a.row_off, a.rows_total = row_off, rows_total
        scratch = torch.empty(K.lib().mpc3_rss_softmax_loss_scratch(rows, d) // 8, dtype=torch.int64, device=_dev())
        out = empty(z.shape, z.fp)
        K.call("mpc3_rss_softmax_loss", self.rk, self.ctr_ptr, C.byref(a), z.data.data_ptr(), y.data.data_ptr(),
               scratch.data_ptr(), out.data.data_ptr(), rows, d, _stream())
        return out

    def softmax(self, z: RssTensor, cfg: ReciprocalConfig = ReciprocalConfig()) -> RssTensor:
        d = z.shape[-1]
        if d > cfg.Y:
            raise ConfigError(f"class count {d} exceeds reciprocal domain Y={cfg.Y}")
        z = z.contiguous()
        mx = self.max_tree(z)
        x = _rowop(K.EW_SUB, z, mx)
        e = self.exp_approx(x)
        tot = _rowsum(e)
        r = self.reciprocal(tot, cfg)
        return self.mul_truncate(e, RssTensor(r.data.expand(e.data.shape).contiguous(), r.fp))


# ---------------------------------------------------------------------------
# kernel helpers


# Input-gradient formulation (stride 1), measured per layer shape on B200
# (tools/dbg/dgrad_paths.py, profiles/r02_dgrad_paths.txt): the cropped
# correlation of the padded gradient wins once its GEMM has enough rows to
# fill the GPU without split-K (VGG-16-TI b32 conv1_2 2.34 -> 1.69 ms,
# conv2_2 1.47 -> 1.16, conv3_2 1.05 -> 0.96; 16 x 16 maps about even) and
# loses below (8 x 8 maps and AlexNet-CIFAR's 1 x 1 / 2 x 2 maps, where its
# GEMM is a long-K split); it also computes (h w) / (oh ow) times the
# transposed convolution's MACs, so only kernels whose padding keeps the
# map size qualify.
DGRAD_IM2COL_MIN_ROWS = int(os.environ.get("MPC3_DGRAD_IM2COL_MIN_ROWS", "8192"))


def _dgrad_use_im2col(nb, oh, ow, kh, kw, padding) -> bool:
    ph, pw = padding
    h, w = oh + kh - 1 - 2 * ph, ow + kw - 1 - 2 * pw
    if kh - 1 - ph < 0 or kw - 1 - pw < 0 or h <= 0 or w <= 0:
        return False
    return nb * h * w >= DGRAD_IM2COL_MIN_ROWS and h * w * 4 <= oh * ow * 5


def _ew2(op, a: RssTensor, b: RssTensor, out: RssTensor | None = None) -> RssTensor:
    a, b = _broadcast(a, b)
    if out is None:
        out = empty(a.shape, a.fp)
    elif not out.data.is_contiguous() or out.shape != a.shape:
        raise ShapeError("in-place output must be contiguous and of the operand shape")
    K.call("mpc3_ring_ew", op, a.data.data_ptr(), b.data.data_ptr(), 0, out.data.data_ptr(), 3 * a.numel, _stream())
    return out


def _broadcast(x: RssTensor, y: RssTensor):
    if x.shape == y.shape:
        return x.contiguous(), y.contiguous()
    try:
        shape = tuple(np.broadcast_shapes(x.shape, y.shape))
    except ValueError as e:
        raise ShapeError(str(e)) from None

    def ex(t):
        d = t.data.reshape((3,) + (1,) * (len(shape) - t.ndim) + t.shape)
        return RssTensor(d.expand((3,) + shape).contiguous(), t.fp)

    return ex(x), ex(y)


def _rowop(op, a: RssTensor, b: RssTensor) -> RssTensor:
    """a[..., j] op b[...] for the trio (b has a's shape without the last axis)."""
    a = a.contiguous()
    b = b.contiguous()
    cols = a.shape[-1]
    rows = 3 * (a.numel // cols)
    out = empty(a.shape, a.fp)
    K.call("mpc3_ring_rowop", op, a.data.data_ptr(), b.data.data_ptr(), out.data.data_ptr(), rows, cols, _stream())
    return out


def _rowsum(a: RssTensor) -> RssTensor:
    a = a.contiguous()
    cols = a.shape[-1]
    out = empty(a.shape[:-1] + (1,), a.fp)
    K.call("mpc3_ring_rowsum", a.data.data_ptr(), out.data.data_ptr(), 3 * (a.numel // cols), cols, _stream())
    return out


def reconstruct_device(x: RssTensor) -> torch.Tensor:
    x = x.contiguous()
    n = x.numel
    out = torch.empty(n, dtype=torch.int64, device=x.data.device)
    d = x.data.reshape(3, n)
    K.call("mpc3_ring_ew", K.EW_ADD, d[0].data_ptr(), d[1].data_ptr(), 0, out.data_ptr(), n, _stream())
    K.call("mpc3_ring_ew", K.EW_ADD, out.data_ptr(), d[2].data_ptr(), 0, out.data_ptr(), n, _stream())
    return out


# ---------------------------------------------------------------------------
# plain (non-shared) exact ring ops: bilinear_exact's device body


def plain_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    m, k = a.shape
    n = b.shape[1]
    if m == 0 or n == 0:
        return np.zeros((m, n), U64)
    da, db = to_device(a), to_device(b)
    ws = torch.empty(K.lib().mpc3_ring_matmul_workspace(m, n, k), dtype=torch.uint8, device=_dev())
    out = torch.empty(m * n, dtype=torch.int64, device=_dev())
    K.call("mpc3_ring_matmul_u64", da.data_ptr(), db.data_ptr(), out.data_ptr(), m, n, k, ws.data_ptr(), _stream())
    return to_host(out).reshape(m, n)


def plain_conv2d(x: np.ndarray, k: np.ndarray, stride, padding) -> np.ndarray:
    nb, c, h, w = x.shape
    o, _, kh, kw = k.shape
    sh, sw = stride
    ph, pw = padding
    if h + 2 * ph < kh or w + 2 * pw < kw:
        raise ShapeError("kernel larger than padded input")
    oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
    dx, dk = to_device(x), to_device(k)
    K_ = c * kh * kw
    M = nb * oh * ow
    kp = _round_up(K_, 32)
    A = torch.empty(8 * M * kp, dtype=torch.uint8, device=_dev())
    B = torch.empty(8 * o * kp, dtype=torch.uint8, device=_dev())
    a_op = K.conv_operand(K.GATHER_IM2COL, M, K_, nb, c, h, w, dx.stride(), kh, kw, sh, sw, ph, pw, oh, ow)
    b_op = K.dense_operand(o, K_, s_r=K_, t2=1)
    st = _stream()
    K.call("mpc3_ring_pack", dx.data_ptr(), 0, C.byref(a_op), 2, A.data_ptr(), kp, st)
    K.call("mpc3_ring_pack", dk.data_ptr(), 0, C.byref(b_op), 2, B.data_ptr(), kp, st)
    z = torch.empty(M * o, dtype=torch.int64, device=_dev())
    K.call("mpc3_ring_gemm_auto", A.data_ptr(), B.data_ptr(), z.data_ptr(), 1, M, o, kp, 0, st)
    return to_host(z).reshape(nb, oh, ow, o).transpose(0, 3, 1, 2).copy()


def plain_sumpool(x: np.ndarray, window, stride) -> np.ndarray:
    kh, kw = window
    sh, sw = stride
    nb, c, h, w = x.shape
    if h < kh or w < kw:
        raise ShapeError("window larger than input")
    oh, ow = (h - kh) // sh + 1, (w - kw) // sw + 1
    dx = to_device(x)
    out = torch.empty(nb * c * oh * ow, dtype=torch.int64, device=_dev())
    K.call("mpc3_ring_sumpool", dx.data_ptr(), out.data_ptr(), nb, c, h, w, kh, kw, sh, sw, _stream())
    return to_host(out).reshape(nb, c, oh, ow)
