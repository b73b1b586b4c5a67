"""Generate golden fixtures by running the REAL reference (`mpc3`).

Run in the build container, where /root/reference is readable:

    python tests/golden/make_golden.py

It writes tests/golden/golden.npz (+ golden_meta.json).  The fixtures hold
per-party replicated shares, opened outputs, PRF words and communication
accounting produced by the reference's own code path
(run_in_process + distribute_input + the protocol), so that the CPU oracle
(`oracle/`) and the CUDA engine are both pinned to the reference, and the
fixtures travel to the GPU box where /root/reference does not exist.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import mpc3.protocols as P  # noqa: E402
from mpc3 import models, nn  # noqa: E402
from mpc3.prf import PrfKey  # noqa: E402
from mpc3.ring import bilinear_exact, conv2d_spec, fx_encode, matmul_spec, sumpool_spec  # noqa: E402
from mpc3.session import distribute_input, make_session_id, open_share, run_in_process  # noqa: E402
from mpc3.prf import derive_key  # noqa: E402

U64 = np.uint64
OUT = Path(__file__).resolve().parent
SEED, DEALER = 3, 7


def comps(shares):
    """Per-party shares -> (3, ...) components, checking replication."""
    c = np.stack([s.lo for s in shares])
    for p in range(3):
        assert np.array_equal(shares[p].hi, c[(p + 1) % 3])
    return c


def run_case(op, xs, seed=SEED, **kw):
    def job(ctx):
        rin = np.random.default_rng(DEALER)
        sh = [distribute_input(ctx, x if ctx.party == 0 else None, rin, shape=x.shape) for x in xs]
        base = ctx.transport.stats.copy()
        out = op(ctx, *sh, **kw)
        d = ctx.transport.stats.since(base)
        return out, d.payload_bytes_sent(), d.round_labels

    res = run_in_process(job, seed=seed)
    outs = [r[0] for r in res]
    if isinstance(outs[0], tuple):
        c = [comps([o[i] for o in outs]) for i in range(len(outs[0]))]
    else:
        c = [comps(outs)]
    acct = {"payload_bytes": [r[1] for r in res], "labels": res[0][2]}
    return c, acct


def main():
    g: dict[str, np.ndarray] = {}
    meta: dict = {"seed": SEED, "dealer": DEALER, "cases": {}}
    rng = np.random.default_rng(2026)

    # PRF known-answer vectors (prf.py:40-49)
    kat_key = bytes(range(16))
    g["prf_kat_key"] = np.frombuffer(kat_key, np.uint8).copy()
    g["prf_kat_words"] = PrfKey(kat_key).words(1, 0, 4)
    sid = make_session_id(SEED)
    keys = [derive_key(f"seed{SEED}".encode(), sid, f"party{i}").key for i in range(3)]
    g["party_keys_seed3"] = np.stack([np.frombuffer(k, np.uint8) for k in keys])
    sid0 = make_session_id(0)
    g["party_keys_seed0"] = np.stack(
        [np.frombuffer(derive_key(b"seed0", sid0, f"party{i}").key, np.uint8) for i in range(3)]
    )
    prf_rows = []
    for purpose, index, count in [(1, 0, 9), (2, 5, 16), (3, 1, 7), (4, 123456, 33), (5, (1 << 48) - 1, 5)]:
        w = PrfKey(keys[1]).words(purpose, index, count)
        prf_rows.append((purpose, index, count))
        g[f"prf_k1_{purpose}_{index}_{count}"] = w
    meta["prf_rows"] = prf_rows

    # ring bilinear engine (ring.py:183-268)
    a = rng.integers(0, 1 << 64, (9, 33), dtype=U64)
    b = rng.integers(0, 1 << 64, (33, 7), dtype=U64)
    g["mm_a"], g["mm_b"] = a, b
    g["mm_out"] = bilinear_exact(a, b, matmul_spec(9, 33, 7))
    x = rng.integers(0, 1 << 64, (2, 3, 10, 10), dtype=U64)
    k = rng.integers(0, 1 << 64, (4, 3, 3, 3), dtype=U64)
    g["cv_x"], g["cv_k"] = x, k
    g["cv_out"] = bilinear_exact(x, k, conv2d_spec(3, (3, 3), (2, 2), (1, 1)))
    g["sp_out"] = bilinear_exact(x, None, sumpool_spec((3, 3), (2, 2)))

    # protocols: per-party components of the outputs
    edges = np.array([0, 1, (1 << 63) - 1, 1 << 63, (1 << 64) - 1, 123456789], dtype=U64)
    cases = {
        "mul": (P.mul, [rng.integers(0, 1 << 64, (5, 7), dtype=U64), rng.integers(0, 1 << 64, (5, 7), dtype=U64)], {}),
        "mul_bcast": (P.mul, [rng.integers(0, 1 << 64, (3, 1), dtype=U64), rng.integers(0, 1 << 64, (4,), dtype=U64)], {}),
        "matmul": (P.matmul_shares, [fx_encode(rng.uniform(-4, 4, (12, 32))), fx_encode(rng.uniform(-4, 4, (32, 9)))], {}),
        "matmul_bits": (P.matmul_shares, [fx_encode(rng.uniform(-2, 2, (6, 8))), fx_encode(rng.uniform(-2, 2, (8, 5)))], {"bits": 23}),
        "conv": (P.conv2d_shares, [fx_encode(rng.uniform(-2, 2, (2, 3, 10, 10))), fx_encode(rng.uniform(-1, 1, (4, 3, 3, 3)))], {"stride": (2, 2), "padding": (1, 1)}),
        "conv11s4": (P.conv2d_shares, [fx_encode(rng.uniform(-1, 1, (1, 3, 16, 16))), fx_encode(rng.uniform(-1, 1, (8, 3, 11, 11)) / 19)], {"stride": (4, 4), "padding": (0, 0)}),
        "trunc20": (P.truncate, [rng.integers(-(1 << 61), 1 << 61, 257, dtype=np.int64).view(U64)], {}),
        "trunc1": (P.truncate, [rng.integers(-(1 << 61), 1 << 61, 64, dtype=np.int64).view(U64)], {"bits": 1}),
        "trunc61": (P.truncate, [rng.integers(-(1 << 61), 1 << 61, 64, dtype=np.int64).view(U64)], {"bits": 61}),
        "a2b": (P.a2b, [np.concatenate([edges, rng.integers(0, 1 << 64, 121, dtype=U64)])], {}),
        "msb": (P.msb, [np.concatenate([edges, rng.integers(0, 1 << 64, 57, dtype=U64)])], {}),
        "relu": (P.relu, [np.concatenate([edges, rng.integers(0, 1 << 64, 301, dtype=U64)])], {}),
        "relu_mask": (P.relu_with_mask, [fx_encode(rng.uniform(-8, 8, (3, 17)))], {}),
        "drelu": (P.drelu, [fx_encode(np.array([-1.0, 1.0, 0.0, -0.5, 2.0]))], {}),
        "max_tree": (P.max_tree, [fx_encode(rng.uniform(-30, 30, (6, 7)))], {}),
        "exp": (P.exp_approx, [fx_encode(np.linspace(-8, 0, 33))], {}),
        "reciprocal": (P.reciprocal, [fx_encode(np.linspace(1, 200, 17))], {}),
        "softmax": (P.softmax, [fx_encode(rng.uniform(-5, 5, (4, 10)))], {}),
        "avgpool2": (P.avgpool_shares, [fx_encode(rng.uniform(-4, 4, (1, 2, 6, 6)))], {"window": (2, 2)}),
        "avgpool3": (P.avgpool_shares, [fx_encode(rng.uniform(-4, 4, (1, 2, 9, 9)))], {"window": (3, 3)}),
    }
    for name, (op, xs, kw) in cases.items():
        outs, acct = run_case(op, xs, **kw)
        for i, x in enumerate(xs):
            g[f"{name}_in{i}"] = x
        for i, c in enumerate(outs):
            g[f"{name}_out{i}"] = c
        meta["cases"][name] = {"kw": {k: list(v) if isinstance(v, tuple) else v for k, v in kw.items()},
                               "n_in": len(xs), "n_out": len(outs), **acct}

    # nn: LeNet private inference (b=2) per-party logits, and one training
    # step of LeNet (b=3, non-power-of-two) and AlexNet-CIFAR (b=4): opened
    # weights (LeNet raw, AlexNet as a SHA-256 digest to keep the file small).
    lenet = models.lenet()
    w = nn.init_params(lenet, seed=31)
    xin = rng.uniform(0, 1, (2, 1, 28, 28))
    g["lenet_infer_x"] = xin

    def infer_job(ctx):
        rin = np.random.default_rng(DEALER)
        priv = nn.share_model(ctx, lenet.with_params(w), rin)
        xs = distribute_input(ctx, fx_encode(xin) if ctx.party == 0 else None, rin, shape=xin.shape)
        return nn.infer_private(ctx, priv, xs)

    g["lenet_infer_logits"] = comps(run_in_process(infer_job, seed=SEED))

    for name, mk, bsz in [("lenet", models.lenet, 3), ("alexnet", models.alexnet_cifar, 4)]:
        m = mk()
        imgs = rng.uniform(0, 1, (bsz,) + m.input_shape)
        labels = rng.integers(0, 10, bsz)
        cfg = nn.TrainConfig(0.01, bsz, 1, 5)
        res = run_in_process(
            lambda ctx: nn.train_private(ctx, mk(), cfg, (imgs, labels) if ctx.party == 0 else None),
            seed=0, timeout=6000,
        )
        weights = res[0].weights
        g[f"train_{name}_images"] = imgs
        g[f"train_{name}_labels"] = labels
        digest = hashlib.sha256(b"".join(np.ascontiguousarray(x, "<u8").tobytes() for x in weights)).hexdigest()
        meta[f"train_{name}_digest"] = digest
        meta[f"train_{name}_ce"] = res[0].ce_history
        if name == "lenet":
            for i, x in enumerate(weights):
                g[f"train_lenet_w{i}"] = x

    np.savez_compressed(OUT / "golden.npz", **g)
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=1))
    print("wrote", OUT / "golden.npz", sum(v.nbytes for v in g.values()), "bytes raw")


if __name__ == "__main__":
    main()
