"""The reference's own CPU path, driven through its public API for bench.py.

The reference (`mpc3`, pure Python: numpy/OpenBLAS float64 limb GEMMs and
OpenSSL AES-CTR, three party threads) is installed unmodified into
`baseline/_ref`; `/root/reference/pkg/src` is the fallback in
the build container.  Nothing here touches the B200 engine: the reference
arm (`bench.py --impl reference`) and the `cpu_baseline` legs call these.

* `alexnet_train`  — `mpc3.nn.train_private` (nn.py:679-751), AlexNet-CIFAR,
  batch 128, through `run_in_process` (session.py:124-158);
* `lenet_infer`    — `share_model` + `distribute_input` + `infer_private`
  (nn.py:550) at batch 64;
* `resnet50_composed` — ResNet-50 v1.5 224x224 inference COMPOSED from the
  reference's per-party protocols (`conv2d_shares` protocols.py:120 + a local
  bias add, `relu` :340, zero-padded `avgpool_shares` :139, `matmul_shares`
  :97, residual = local add): the reference graph has no residual / bias /
  padded-pool layers, so this is the "composed" baseline
  BASELINE.md §2 prescribes.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
_CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def load():
    """Import the unmodified reference package; returns (module, source path) or (None, reason)."""
    for path in _CANDIDATES:
        if os.path.isdir(os.path.join(path, "mpc3")):
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import mpc3  # noqa: F401
                import mpc3.nn  # noqa: F401
                import mpc3.protocols  # noqa: F401
                import mpc3.session  # noqa: F401
            except ImportError as e:  # e.g. `cryptography` missing
                return None, f"mpc3 at {path} does not import: {e!r}"
            return sys.modules["mpc3"], path
    return None, "reference package not installed (baseline/_ref) and /root/reference absent"


def threads() -> dict:
    return {"cores": os.cpu_count(), "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset (all)"),
            "party_threads": 3}


def alexnet_train(batch: int, iterations: int, images, labels) -> float:
    """Seconds for one `train_private` call of `iterations` iterations at
    `batch` (session seed 0, TrainConfig(0.01, batch, iterations, 0)); the
    call also deals the weights and opens them at the end (<1 % here)."""
    from mpc3 import models, nn
    from mpc3.session import run_in_process

    cfg = nn.TrainConfig(0.01, batch, iterations, 0)
    t0 = time.perf_counter()
    run_in_process(lambda ctx: nn.train_private(ctx, models.alexnet_cifar(), cfg,
                                                (images, labels) if ctx.party == 0 else None),
                   seed=0, timeout=1e5)
    return time.perf_counter() - t0


def lenet_infer(batch: int = 64, seed: int = 3) -> float:
    from mpc3 import models, nn
    from mpc3.ring import fx_encode
    from mpc3.session import distribute_input, run_in_process

    model = models.lenet()
    w = nn.init_params(model, seed=seed)
    shape = (batch,) + model.input_shape

    def job(ctx):
        rin = np.random.default_rng(seed)
        priv = nn.share_model(ctx, model.with_params(w), rin)
        x = fx_encode(rin.uniform(0, 1, shape)) if ctx.party == 0 else None
        t0 = time.perf_counter()
        nn.infer_private(ctx, priv, distribute_input(ctx, x, rin, shape=shape))
        return time.perf_counter() - t0

    return max(run_in_process(job, seed=seed, timeout=1e5))


def _composed_forward(ctx, layers, it, h):
    import mpc3.protocols as P
    from mpc3.sharing import ArithmeticShare

    from paper_2104_10949_b200 import nn as B  # layer specs only (host data, no engine call)

    for L in layers:
        if L.kind == B.CONV2D:
            h = P.conv2d_shares(ctx, h, next(it), L.stride, L.padding)
            if L.bias:
                b = next(it)
                h = ArithmeticShare(h.owner, h.lo + b.lo[None, :, None, None], h.hi + b.hi[None, :, None, None], h.fp)
        elif L.kind == B.FULLY_CONNECTED:
            w = next(it)
            h = P.matmul_shares(ctx, h, w.map(lambda v: np.ascontiguousarray(v.T)))
            if L.bias:
                b = next(it)
                h = ArithmeticShare(h.owner, h.lo + b.lo[None, :], h.hi + b.hi[None, :], h.fp)
        elif L.kind == B.AVGPOOL:
            ph, pw = L.padding
            if ph or pw:
                h = h.map(lambda v: np.pad(v, ((0, 0), (0, 0), (ph, ph), (pw, pw))))
            h = P.avgpool_shares(ctx, h, L.window, L.stride)
        elif L.kind == B.RELU:
            h = P.relu(ctx, h)
        elif L.kind == B.FLATTEN:
            h = h.map(lambda v: v.reshape(v.shape[0], -1))
        elif L.kind == B.RESIDUAL:
            hm = _composed_forward(ctx, L.main, it, h) if L.main else h
            hs = _composed_forward(ctx, L.shortcut, it, h) if L.shortcut else h
            h = hm + hs
        else:
            raise ValueError(f"no reference composition for {L.kind}")
    return h


def resnet50_composed(batch: int = 1, seed: int = 11) -> float:
    """Seconds of the composed reference ResNet-50 forward (dealing excluded)."""
    from mpc3.ring import fx_encode
    from mpc3.session import distribute_input, run_in_process

    from paper_2104_10949_b200 import models as BM
    from paper_2104_10949_b200 import nn as B

    model = BM.resnet50()
    w = B.init_params(model, seed=seed)
    shape = (batch, 3, 224, 224)

    def job(ctx):
        rin = np.random.default_rng(seed)
        params = [distribute_input(ctx, w[i] if ctx.party == 0 else None, rin, shape=w[i].shape)
                  for i in range(len(w))]
        x = fx_encode(rin.uniform(0, 1, shape)) if ctx.party == 0 else None
        xs = distribute_input(ctx, x, rin, shape=shape)
        t0 = time.perf_counter()
        _composed_forward(ctx, model.layers, iter(params), xs)
        return time.perf_counter() - t0

    return max(run_in_process(job, seed=seed, timeout=1e5))
