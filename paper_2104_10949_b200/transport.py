"""Communication accounting for co-resident parties (transport.py:26-175).

On the B200 engine the three parties share one GPU, so a protocol "send" is a
register/HBM handoff inside a fused kernel.  What the reference measures on
its wire — bytes per ordered pair, messages, rounds and the ordered round
labels — is charged analytically here with the reference's exact frame
format (8-byte LE length header + LE u64 words), so `CommStats` numbers are
identical to an in-process or TCP run of the reference.  The TCP backend
(transport.py:178-319) is out of scope: multi-host LAN parties are not a B200
path.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import FrameError, TopologyError

NUM_PARTIES = 3
FRAME_HEADER_BYTES = 8
MAX_FRAME_BYTES = 1 << 32


def encode_frame(words: np.ndarray) -> bytes:
    payload = np.ascontiguousarray(words, dtype="<u8").tobytes()
    if len(payload) > MAX_FRAME_BYTES:
        raise FrameError(f"frame of {len(payload)} bytes exceeds 2^32")
    return struct.pack("<Q", len(payload)) + payload


def decode_frame(frame: bytes) -> np.ndarray:
    if len(frame) < FRAME_HEADER_BYTES:
        raise FrameError("truncated frame header")
    (n,) = struct.unpack_from("<Q", frame)
    if n % 8 or len(frame) != FRAME_HEADER_BYTES + n:
        raise FrameError("frame length mismatch")
    return np.frombuffer(frame, dtype="<u8", offset=FRAME_HEADER_BYTES).astype(np.uint64)


@dataclass
class CommStats:
    """Per-party traffic and round counters (transport.py:52-105)."""

    bytes_sent: dict = field(default_factory=dict)
    bytes_received: dict = field(default_factory=dict)
    messages: int = 0
    messages_received: int = 0
    rounds: int = 0
    round_labels: list = field(default_factory=list)

    def total_bytes_sent(self) -> int:
        return sum(self.bytes_sent.values())

    def total_bytes_received(self) -> int:
        return sum(self.bytes_received.values())

    def payload_bytes_sent(self) -> int:
        return self.total_bytes_sent() - FRAME_HEADER_BYTES * self.messages

    def and_rounds(self) -> int:
        return sum(lab.startswith("and.") for lab in self.round_labels)

    def copy(self) -> "CommStats":
        return CommStats(dict(self.bytes_sent), dict(self.bytes_received), self.messages,
                         self.messages_received, self.rounds, list(self.round_labels))

    def since(self, base: "CommStats") -> "CommStats":
        return CommStats(
            {p: v - base.bytes_sent.get(p, 0) for p, v in self.bytes_sent.items()},
            {p: v - base.bytes_received.get(p, 0) for p, v in self.bytes_received.items()},
            self.messages - base.messages,
            self.messages_received - base.messages_received,
            self.rounds - base.rounds,
            self.round_labels[len(base.round_labels):],
        )

    def as_dict(self) -> dict:
        return {
            "bytes_sent": {str(k): v for k, v in sorted(self.bytes_sent.items())},
            "bytes_received": {str(k): v for k, v in sorted(self.bytes_received.items())},
            "messages": self.messages,
            "messages_received": self.messages_received,
            "rounds": self.rounds,
            "round_labels": list(self.round_labels),
        }


class Transport:
    """A party's endpoint: identity plus the CommStats the engine charges."""

    def __init__(self, party: int):
        if party not in range(NUM_PARTIES):
            raise TopologyError(f"party id {party} outside 0..2")
        self.party = party
        self.stats = CommStats()

    @property
    def peers(self) -> tuple:
        return tuple(p for p in range(NUM_PARTIES) if p != self.party)

    def round_mark(self, label: str) -> None:
        self.stats.rounds += 1
        self.stats.round_labels.append(label)

    def charge_send(self, to: int, words: int) -> None:
        if to == self.party or to not in range(NUM_PARTIES):
            raise TopologyError(f"cannot send to party {to}")
        nbytes = FRAME_HEADER_BYTES + 8 * int(words)
        self.stats.bytes_sent[to] = self.stats.bytes_sent.get(to, 0) + nbytes
        self.stats.messages += 1

    def charge_recv(self, frm: int, words: int) -> None:
        nbytes = FRAME_HEADER_BYTES + 8 * int(words)
        self.stats.bytes_received[frm] = self.stats.bytes_received.get(frm, 0) + nbytes
        self.stats.messages_received += 1

    def close(self) -> None:
        pass


class Ledger:
    """The three parties' transports; protocols charge rounds through it."""

    def __init__(self):
        self.parties = [Transport(i) for i in range(NUM_PARTIES)]
        self.enabled = True
        self._rec = None

    def round(self, label: str, sends=()) -> None:
        """One round: every party marks `label`; sends = [(src, dst, words)]."""
        if self._rec is not None:
            self._rec.append((label, tuple(sends)))
            return
        if not self.enabled:
            return
        for t in self.parties:
            t.round_mark(label)
        for src, dst, words in sends:
            self.parties[src].charge_send(dst, words)
            self.parties[dst].charge_recv(src, words)

    def capture(self):
        """Context for a CUDA-graph capture: the rounds the captured calls
        charge are recorded instead of applied; `.charge` (per-party CommStats
        of one replay) is then applied by `apply` on every replay."""
        led = self

        class _Cap:
            charge = None

            def __enter__(self_inner):
                led._rec = []
                return self_inner

            def __exit__(self_inner, *exc):
                rec, led._rec = led._rec, None
                tmp = [Transport(i) for i in range(NUM_PARTIES)]
                for label, sends in rec:
                    for t in tmp:
                        t.round_mark(label)
                    for src, dst, words in sends:
                        tmp[src].charge_send(dst, words)
                        tmp[dst].charge_recv(src, words)
                self_inner.charge = [t.stats for t in tmp]
                return False

        return _Cap()

    def apply(self, charge) -> None:
        """Add one replay's per-party CommStats (from capture) to the parties."""
        if not self.enabled or charge is None:
            return
        for t, d in zip(self.parties, charge):
            st = t.stats
            for k, v in d.bytes_sent.items():
                st.bytes_sent[k] = st.bytes_sent.get(k, 0) + v
            for k, v in d.bytes_received.items():
                st.bytes_received[k] = st.bytes_received.get(k, 0) + v
            st.messages += d.messages
            st.messages_received += d.messages_received
            st.rounds += d.rounds
            st.round_labels.extend(d.round_labels)

    def ring(self, label: str, words: int) -> None:
        """Every party i sends `words` to i+1 (reshare / AND / open).  The same
        charges as round(label, [(i, i+1, words)]) without the per-send
        topology checks (a ring's sends are valid by construction): this runs
        once per protocol call on the eager path."""
        if self._rec is not None or not self.enabled:
            self.round(label, [(i, (i + 1) % 3, words) for i in range(3)])
            return
        nbytes = FRAME_HEADER_BYTES + 8 * int(words)
        for i, t in enumerate(self.parties):
            st = t.stats
            st.rounds += 1
            st.round_labels.append(label)
            j, k = (i + 1) % 3, (i + 2) % 3
            st.bytes_sent[j] = st.bytes_sent.get(j, 0) + nbytes
            st.messages += 1
            st.bytes_received[k] = st.bytes_received.get(k, 0) + nbytes
            st.messages_received += 1
