"""Reference-generated fixtures at the BASELINE.json configurations
(tests/golden/make_golden_configs.py): cfg(name) -> (arrays, meta)."""

import hashlib
import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "golden"


def cfg(name):
    z = np.load(HERE / f"cfg_{name}.npz")
    meta = json.loads(bytes(z["meta"]).decode())
    return {k: z[k] for k in z.files if k != "meta"}, meta


def available(name) -> bool:
    return (HERE / f"cfg_{name}.npz").exists()


def digest(ws) -> str:
    """SHA-256 over the little-endian u64 words of each array, in order
    (the digest make_golden_configs.py records)."""
    return hashlib.sha256(b"".join(np.ascontiguousarray(np.asarray(x, np.uint64), "<u8").tobytes()
                                   for x in ws)).hexdigest()


def alexnet_b128_data():
    """bench.py's synthetic AlexNet-CIFAR batch (_synthetic(128, 100))."""
    rng = np.random.default_rng(100)
    return rng.uniform(0, 1, (128, 3, 32, 32)), rng.integers(0, 10, 128)


def vgg16ti_train_data():
    rng = np.random.default_rng(5)
    return rng.uniform(0, 1, (32, 3, 64, 64)), rng.integers(0, 200, 32)
