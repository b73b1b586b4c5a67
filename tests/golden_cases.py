"""Shared access to the reference-generated golden fixtures (tests/golden)."""

import json
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "golden"
G = np.load(HERE / "golden.npz")
META = json.loads((HERE / "golden_meta.json").read_text())
SEED = META["seed"]
DEALER = META["dealer"]


def case(name):
    m = META["cases"][name]
    ins = [G[f"{name}_in{i}"] for i in range(m["n_in"])]
    outs = [G[f"{name}_out{i}"] for i in range(m["n_out"])]
    kw = {k: tuple(v) if isinstance(v, list) else v for k, v in m["kw"].items()}
    return ins, outs, kw, m


CASE_NAMES = list(META["cases"].keys())
