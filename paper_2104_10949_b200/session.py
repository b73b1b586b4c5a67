"""Session setup, dealing, opening and the three-party runner (session.py API).

`run_in_process` keeps the reference's model — three party threads, each
running `party_fn(ctx)` — but the parties share ONE trio session on the GPU:
every protocol call is a rendezvous of the three threads, and the last to
arrive launches the fused trio kernel (the "messages" are device handoffs).
"""

from __future__ import annotations

import threading
from typing import Callable

import numpy as np

from .engine import TrioSession, make_session_id, session_keys
from .errors import ProtocolError, TopologyError
from .prf import PURPOSE_TRUNC_RHO, derive_key
from .ring import DEFAULT_FP, FixedPointConfig, as_ring
from .sharing import NUM_PARTIES, ArithmeticShare, PartyContext, PrfKeySet, assemble, split_trio

__all__ = ["make_session_id", "setup_context", "distribute_input", "open_share", "run_in_process",
           "TruncationRandomness", "InProcessNetwork", "Rendezvous"]


class Rendezvous:
    """Barrier-with-payload for the three party threads of one session."""

    def __init__(self, timeout: float = 600.0):
        self.cv = threading.Condition()
        self.timeout = timeout
        self.gen = 0
        self.payloads: dict = {}
        self.names: dict = {}
        self.results: dict = {}
        self.reads: dict = {}

    def run(self, party: int, name: str, payload, fn):
        with self.cv:
            gen = self.gen
            if party in self.payloads:
                raise ProtocolError(f"party {party} entered {name!r} twice")
            self.payloads[party] = payload
            self.names[party] = name
            if len(self.payloads) == NUM_PARTIES:
                if len(set(self.names.values())) != 1:
                    res = (False, ProtocolError(f"parties out of lockstep: {sorted(set(self.names.values()))}"))
                else:
                    try:
                        res = (True, fn(dict(self.payloads)))
                    except BaseException as e:  # noqa: BLE001 - re-raised in every party
                        res = (False, e)
                self.results[gen] = res
                self.reads[gen] = 0
                self.payloads, self.names = {}, {}
                self.gen += 1
                self.cv.notify_all()
            else:
                if not self.cv.wait_for(lambda: gen in self.results, timeout=self.timeout):
                    raise ProtocolError(f"party {party} timed out waiting in {name!r}")
            ok, val = self.results[gen]
            self.reads[gen] += 1
            if self.reads[gen] == NUM_PARTIES:
                del self.results[gen], self.reads[gen]
        if not ok:
            raise val
        return val


class InProcessNetwork:
    """The three co-resident parties of one session (transport.py:151-175 API)."""

    def __init__(self, timeout: float = 600.0):
        self.rendezvous = Rendezvous(timeout)
        self._session = None
        self._lock = threading.Lock()

    def session(self, fp, seed, session_id) -> TrioSession:
        with self._lock:
            if self._session is None:
                self._session = TrioSession(seed, fp, session_id)
            return self._session

    def transport(self, party: int) -> "Endpoint":
        if party not in range(NUM_PARTIES):
            raise TopologyError(f"party id {party} outside 0..2")
        return Endpoint(party, self)


class Endpoint:
    def __init__(self, party, net):
        self.party = party
        self.net = net


def setup_context(transport: Endpoint, fp: FixedPointConfig = DEFAULT_FP, seed: int | None = None,
                  session_id: bytes | None = None) -> PartyContext:
    """Keys k_i derived as the reference does (session.py:43-59); the k_i ->
    successor exchange is charged as its 2-word setup round."""
    sess = transport.net.session(fp, seed, session_id)
    p = transport.party
    t = sess.ledger.parties[p]
    # setup.keys: each party sends its 16-byte key to its successor
    t.round_mark("setup.keys")
    t.charge_send((p + 1) % 3, 2)
    t.charge_recv((p + 2) % 3, 2)
    keys = PrfKeySet(sess.keys[p], sess.keys[(p + 2) % 3])
    return PartyContext(p, t, keys, fp, session=sess, rendezvous=transport.net.rendezvous)


def distribute_input(ctx: PartyContext, x, rng: np.random.Generator | None = None, owner: int = 0,
                     shape: tuple | None = None) -> ArithmeticShare:
    """Owner deals (numpy draws, as the reference) and every party gets its pair."""
    if ctx.party == owner and (x is None or rng is None):
        raise ProtocolError("input owner must supply data and randomness")

    def fn(sess, ps):
        data, r = ps[owner]
        return split_trio(sess.share(as_ring(data), r, owner=owner))

    res = ctx.collective("share.input", (x, rng) if ctx.party == owner else None, fn)
    return res[ctx.party]


def open_share(ctx: PartyContext, x: ArithmeticShare) -> np.ndarray:
    """Every party learns the secret (session.py:116-121)."""
    return ctx.collective("open", x, lambda sess, ps: sess.reveal(assemble(ps, x.fp)))


class TruncationRandomness:
    """Replay of the truncation offsets of a seeded session (session.py:94-113)."""

    def __init__(self, seed: int, session_id: bytes | None = None):
        sid = session_id if session_id is not None else make_session_id(seed)
        self._key = derive_key(f"seed{seed}".encode(), sid, "party2")
        self._index = 0

    def draw(self, shape: tuple) -> np.ndarray:
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        raw = self._key.words(PURPOSE_TRUNC_RHO, self._index, n).reshape(shape)
        self._index += 1
        return (raw >> np.uint64(2)) - np.uint64(1 << 61)


def run_in_process(party_fn: Callable[[PartyContext], object], fp: FixedPointConfig = DEFAULT_FP,
                   seed: int | None = 0, timeout: float = 600.0) -> list:
    """Run the three parties as threads sharing one co-resident trio session."""
    import torch

    net = InProcessNetwork(timeout)
    session = make_session_id(seed)
    results: list = [None] * NUM_PARTIES
    errors: list = [None] * NUM_PARTIES
    dev = torch.cuda.current_device()

    def runner(p: int) -> None:
        try:
            torch.cuda.set_device(dev)
            ctx = setup_context(net.transport(p), fp, seed, session)
            results[p] = party_fn(ctx)
        except BaseException as e:  # noqa: BLE001
            errors[p] = e

    threads = [threading.Thread(target=runner, args=(p,), daemon=True) for p in range(NUM_PARTIES)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=timeout)
    for p, e in enumerate(errors):
        if e is not None:
            raise ProtocolError(f"party {p} failed: {e!r}") from e
    if any(th.is_alive() for th in threads):
        raise ProtocolError("party thread hung")
    return results


_ = session_keys  # re-exported helper
