"""Layer graphs and the private forward / backward / SGD schedule on the GPU.

API of the reference's nn.py (nn.py:43-793): LayerSpec builders, ModelGraph
shape inference, parameter init, the per-party entry points
(infer_private, forward_private, loss_grad_output, backward, sgd_step,
share_model, train_private) and TrainConfig / TrainResult.

The schedule runs on `TrioNet`, the B200 engine behind the reference's
duck-typed engine seam (nn.py:209-253): conv/FC layers are one batched
tcgen05 ring GEMM over the three parties' cross terms plus one fused
reshare+truncate kernel; conv gradients are direct implicit GEMMs (no
materialised dilation / padding / flips, nn.py:435-484); ReLU is one fused
sign-circuit kernel; pooling forward/backward are one fused kernel each.
PRF counters are consumed in exactly the reference's order, so opened
results — and per-party shares — are bit-identical to the reference.
"""

from __future__ import annotations

import contextlib
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine as E
from .engine import ReciprocalConfig, RssTensor, TrioSession
from .errors import ConfigError, ProtocolError, RangeError, ShapeError
from .ring import DEFAULT_FP, FixedPointConfig, fx_decode, fx_encode
from .sharing import ArithmeticShare, PartyContext, assemble, split_trio

CONV2D = "Conv2d"
FULLY_CONNECTED = "FullyConnected"
AVGPOOL = "AvgPool"
RELU = "ReLU"
FLATTEN = "Flatten"
# inference-only extensions for ResNet (absent from the reference, nn.py:43-47;
# composed from its primitives: bias = local add after the truncation,
# residual = local add of two branches, padded avg-pool = zero pad + avg-pool)
RESIDUAL = "Residual"
# max-pooling (absent from the reference; the paper swaps it for avg-pooling,
# PAPER.md:1405-1420): each window flattened row-major into max_tree
# (protocols.py:356-380), padded positions holding a public -2^60
MAXPOOL = "MaxPool"
# MPC3_OVERLAP=0: weight gradients on the main stream (no side-stream overlap)
OVERLAP = os.environ.get("MPC3_OVERLAP", "1") == "1"
# MPC3_FUSE_RELU=0: a conv / linear layer's epilogue and the ReLU after it as two launches
FUSE_RELU = os.environ.get("MPC3_FUSE_RELU", "1") == "1"
# only for outputs of at least this many elements: the persistent sign kernel
# absorbs the 5 extra AES blocks per pair; the small tensors' two-phase kernel
# (two more keystream slots, smaller chunks) does not (AlexNet step: fused
# everywhere 2.559 ms, from 100 K elements 2.530 ms, never 2.541 ms)
FUSE_RELU_MIN = int(os.environ.get("MPC3_FUSE_RELU_MIN", "100000"))  # output elements
# inference (no backward pass recorded) fuses at every size: ResNet-50 b1's
# 25-50 K-element ReLUs 140.1 -> 141.4 img/s (profiles/README.md)
FUSE_RELU_MIN_INFER = int(os.environ.get("MPC3_FUSE_RELU_MIN_INFER", "0"))
# MPC3_FUSE_RESIDUAL=0: a residual block's last conv, shortcut add and ReLU as three launches
FUSE_RESIDUAL = os.environ.get("MPC3_FUSE_RESIDUAL", "1") == "1"
FUSE_RESIDUAL_MAX = 4 << 20  # block input elements
# train_trio replays a CUDA graph once this many iterations remain (the
# capture's host cost pays off after ~110 AlexNet steps: eager 3.9 ms
# (host-bound) vs replay 2.36 ms per step, capture ~170 ms)
GRAPH_MIN_STEPS = 112


def _pair(v) -> tuple:
    if isinstance(v, (tuple, list)):
        a, b = v
        return (int(a), int(b))
    return (int(v), int(v))


@dataclass(frozen=True)
class LayerSpec:
    kind: str
    out_channels: int = 0
    out_features: int = 0
    kernel: tuple = ()
    stride: tuple = (1, 1)
    padding: tuple = (0, 0)
    window: tuple = ()
    bias: bool = False
    main: tuple = ()
    shortcut: tuple = ()


def conv2d(out_channels: int, kernel, stride=1, padding=0, bias: bool = False) -> LayerSpec:
    return LayerSpec(CONV2D, out_channels=int(out_channels), kernel=_pair(kernel), stride=_pair(stride),
                     padding=_pair(padding), bias=bool(bias))


def fully_connected(out_features: int, bias: bool = False) -> LayerSpec:
    return LayerSpec(FULLY_CONNECTED, out_features=int(out_features), bias=bool(bias))


def avgpool(window, stride=None, padding=0) -> LayerSpec:
    w = _pair(window)
    return LayerSpec(AVGPOOL, window=w, stride=_pair(stride) if stride is not None else w, padding=_pair(padding))


def maxpool(window, stride=None, padding=0) -> LayerSpec:
    """Max-pool (inference extension): max_tree over each flattened window."""
    w = _pair(window)
    return LayerSpec(MAXPOOL, window=w, stride=_pair(stride) if stride is not None else w, padding=_pair(padding))


def residual(main, shortcut=()) -> LayerSpec:
    """out = main(x) + shortcut(x) (identity when shortcut is empty)."""
    return LayerSpec(RESIDUAL, main=tuple(main), shortcut=tuple(shortcut))


def relu() -> LayerSpec:
    return LayerSpec(RELU)


def flatten() -> LayerSpec:
    return LayerSpec(FLATTEN)


@dataclass
class ModelGraph:
    """Ordered layers, input shape (C,H,W) and per-layer parameters."""

    layers: tuple
    input_shape: tuple
    params: list | None = None

    def __post_init__(self):
        self.layers = tuple(self.layers)
        self.input_shape = tuple(int(d) for d in self.input_shape)
        self._shapes = self._infer_shapes()

    def _infer_shapes(self) -> list:
        return _infer(self.layers, self.input_shape)

    @property
    def output_shapes(self) -> list:
        return list(self._shapes)

    @property
    def num_classes(self) -> int:
        last = self._shapes[-1]
        if len(last) != 1:
            raise ShapeError(f"model output {last} is not a logit vector")
        return last[0]

    def param_shapes(self) -> list:
        return _param_shapes(self.layers, self.input_shape)

    def validate(self, recip: ReciprocalConfig | None = ReciprocalConfig()) -> None:
        """Shapes of the parameters; with `recip`, also the softmax domain
        (training, nn.py:167-172).  Inference-only graphs (ResNet-50's 1000
        classes) pass recip=None."""
        if recip is not None and self.num_classes > recip.Y:
            raise ConfigError(f"{self.num_classes} classes exceed the reciprocal domain")
        if self.params is not None:
            want = self.param_shapes()
            if len(self.params) != len(want):
                raise ShapeError(f"expected {len(want)} parameter tensors, got {len(self.params)}")
            for p, w in zip(self.params, want):
                if tuple(p.shape) != w:
                    raise ShapeError(f"parameter shape {tuple(p.shape)} != {w}")

    def with_params(self, params) -> "ModelGraph":
        return ModelGraph(self.layers, self.input_shape, params)

    @property
    def trainable(self) -> bool:
        """The reference's layer kinds only (backward is defined for them)."""
        return all(s.kind not in (RESIDUAL, MAXPOOL) and not s.bias for s in self.layers)


def _infer(layers, shape) -> list:
    """Per-layer output shapes (nn.py:99-143, extended with Residual / padding)."""
    shape = tuple(shape)
    out = []
    if True:
        for s in layers:
            if s.kind == RESIDUAL:
                m = _infer(s.main, shape)[-1] if s.main else shape
                sc = _infer(s.shortcut, shape)[-1] if s.shortcut else shape
                if m != sc:
                    raise ShapeError(f"residual branches disagree: {m} vs {sc}")
                shape = m
            elif s.kind == CONV2D:
                if len(shape) != 3:
                    raise ShapeError(f"Conv2d needs (C,H,W), got {shape}")
                c, h, w = shape
                (kh, kw), (sh, sw), (ph, pw) = s.kernel, s.stride, s.padding
                ho, wo = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
                if h + 2 * ph < kh or w + 2 * pw < kw or ho < 1 or wo < 1:
                    raise ShapeError(f"Conv2d kernel {s.kernel} does not fit {shape}")
                shape = (s.out_channels, ho, wo)
            elif s.kind in (AVGPOOL, MAXPOOL):
                if len(shape) != 3:
                    raise ShapeError(f"{s.kind} needs (C,H,W), got {shape}")
                c, h, w = shape
                ph, pw = s.padding
                ho = (h + 2 * ph - s.window[0]) // s.stride[0] + 1
                wo = (w + 2 * pw - s.window[1]) // s.stride[1] + 1
                if ho < 1 or wo < 1:
                    raise ShapeError(f"{s.kind} window {s.window} does not fit {shape}")
                shape = (c, ho, wo)
            elif s.kind == FULLY_CONNECTED:
                if len(shape) != 1:
                    raise ShapeError(f"FullyConnected needs a flat input, got {shape}")
                shape = (s.out_features,)
            elif s.kind == FLATTEN:
                shape = (int(np.prod(shape)),)
            elif s.kind != RELU:
                raise ConfigError(f"unknown layer kind {s.kind!r}")
            out.append(shape)
        return out


def _param_shapes(layers, shape) -> list:
    """Parameter shapes in schedule order (nn.py:145-153): conv weight
    (O,C,kh,kw) / FC weight (out,in), each followed by its (O,) bias when
    present; residual blocks list main then shortcut parameters."""
    out = []
    for s, nxt in zip(layers, _infer(layers, shape)):
        if s.kind == CONV2D:
            out.append((s.out_channels, shape[0]) + s.kernel)
            if s.bias:
                out.append((s.out_channels,))
        elif s.kind == FULLY_CONNECTED:
            out.append((s.out_features, shape[0]))
            if s.bias:
                out.append((s.out_features,))
        elif s.kind == RESIDUAL:
            out += _param_shapes(s.main, shape) + _param_shapes(s.shortcut, shape)
        shape = nxt
    return out


def init_params_float(model: ModelGraph, seed: int = 0) -> list:
    """U(-1/sqrt(fan_in), 1/sqrt(fan_in)) per parameter, in order (nn.py:190-198)."""
    rng = np.random.default_rng(seed)
    out = []
    for shp in model.param_shapes():
        # 1-d parameters are the (folded-BN) biases of the ResNet extension
        bound = 1.0 / np.sqrt(int(np.prod(shp[1:]))) if len(shp) > 1 else 0.05
        out.append(rng.uniform(-bound, bound, shp))
    return out


def init_params(model: ModelGraph, fp: FixedPointConfig = DEFAULT_FP, seed: int = 0) -> list:
    return [fx_encode(w, fp) for w in init_params_float(model, seed)]


# ---------------------------------------------------------------------------
# the B200 engine behind the seam


class TrioNet:
    """Forward / backward / SGD of a ModelGraph on trio tensors."""

    def __init__(self, sess: TrioSession):
        self.s = sess
        self.t = sess.fp.t
        self._ahead = []  # weight operands still to be prepacked (training forward)

    def forward(self, model: ModelGraph, params: list, x: RssTensor, record: bool):
        """nn.py:405-432 (plus the inference-only bias / residual / padded pool).
        Recording (training): each layer's weight is packed on the pack
        stream while the layer before it runs, off the critical path."""
        S = self.s
        if record and E.REUSE_PACKS and E.OVERLAP_PACK and all(sp.kind != RESIDUAL for sp in model.layers):
            items, it = [], iter(params)
            for spec in model.layers:
                if spec.kind == CONV2D:
                    k = next(it)
                    items.append((k.data,) + S.conv_weight_operand(k))
                elif spec.kind == FULLY_CONNECTED:
                    y = next(it).apply(lambda d: d.transpose(1, 2))  # the view _run hands to matmul
                    items.append((y.data,) + S.matmul_weight_operand(y))
                else:
                    continue
                if spec.bias:
                    next(it)
            S.prepack(items[:1])
            self._ahead = items[1:]  # packed one layer ahead (_run), beside the layer before
        try:
            return self._run(model.layers, iter(params), x, record)
        finally:
            S.clear_prepacked()
            self._ahead = []

    def _bias(self, h: RssTensor, b: RssTensor) -> RssTensor:
        """Shared bias, local add after the truncation (scale t)."""
        shape = (3, 1, b.shape[0]) + (1,) * (h.ndim - 2)
        return self.s.add(h, RssTensor(b.data.reshape(shape).expand(h.data.shape), h.fp))

    @staticmethod
    def _out_numel(spec, h: RssTensor) -> int:
        if spec.kind == CONV2D:
            (kh, kw), (sh, sw), (ph, pw) = spec.kernel, spec.stride, spec.padding
            return h.shape[0] * spec.out_channels * ((h.shape[2] + 2 * ph - kh) // sh + 1) * \
                ((h.shape[3] + 2 * pw - kw) // sw + 1)
        if spec.kind == FULLY_CONNECTED:
            return h.shape[0] * spec.out_features
        return 0

    def _run(self, layers, it, h: RssTensor, record: bool):
        saved = self.s.relu_masks
        self.s.relu_masks = record  # an inference pass keeps no ReLU masks
        try:
            return self._run_layers(layers, it, h, record)
        finally:
            self.s.relu_masks = saved

    def _run_layers(self, layers, it, h: RssTensor, record: bool):
        S, acts = self.s, []
        fused = None  # mask of a ReLU already computed with the layer before it
        for li, spec in enumerate(layers):
            # recording keeps each layer input's packed GEMM operand (role 1)
            # for the weight gradient, which reads it in place
            keep = [] if record and E.REUSE_PACKS else None
            # a conv / linear layer followed by a ReLU runs as one launch for
            # the layer's reshare + truncate and the ReLU (mpc3_rss_layer_sign)
            relu_next = FUSE_RELU and li + 1 < len(layers) and layers[li + 1].kind == RELU \
                and self._out_numel(spec, h) >= (FUSE_RELU_MIN if record else FUSE_RELU_MIN_INFER)
            if spec.kind == RELU and fused is not None:
                acts.append((fused,) if record else None)
                fused = None
                continue
            if spec.kind == CONV2D:
                k = next(it)
                x = h
                h = S.conv2d(h, k, spec.stride, spec.padding, bias=next(it) if spec.bias else None, keep=keep,
                             relu=relu_next)
                if relu_next:
                    h, fused = h
                    fused = True if fused is None else fused  # no mask kept (inference)
                acts.append(((x, k) + tuple(keep or ())) if record else None)
                if self._ahead:
                    S.prepack([self._ahead.pop(0)])
            elif spec.kind == FULLY_CONNECTED:
                w = next(it)
                x = h
                h = S.matmul(h, w.apply(lambda d: d.transpose(1, 2)), bias=next(it) if spec.bias else None,
                             keep=keep, x_role=1 if keep is not None else 0, relu=relu_next)
                if relu_next:
                    h, fused = h
                    fused = True if fused is None else fused  # no mask kept (inference)
                acts.append(((x, w) + tuple(keep or ())) if record else None)
                if self._ahead:
                    S.prepack([self._ahead.pop(0)])
            elif spec.kind == AVGPOOL:
                acts.append((h.shape,) if record else None)
                h = S.avgpool(h, spec.window, spec.stride, spec.padding)
            elif spec.kind == MAXPOOL:
                acts.append((h.shape,) if record else None)
                h = S.maxpool(h, spec.window, spec.stride, spec.padding)
            elif spec.kind == RELU:
                h, mask = S.relu_with_mask(h)
                acts.append((mask,) if record else None)
            elif spec.kind == FLATTEN:
                shp = h.shape
                acts.append((shp,) if record else None)
                h = h.contiguous().reshape(shp[0], -1)
            elif spec.kind == RESIDUAL:
                last = spec.main[-1] if spec.main else None
                if FUSE_RESIDUAL and li + 1 < len(layers) and layers[li + 1].kind == RELU and last is not None \
                        and last.kind == CONV2D and h.numel <= FUSE_RESIDUAL_MAX:
                    # the main branch's last conv, the shortcut add and the ReLU
                    # after the block in one launch (mpc3_rss_layer_sign_residual);
                    # counters in the unfused order: the conv's epilogue, then
                    # the shortcut branch, then the ReLU.  (ResNet-50 b1 138.4 ->
                    # 139.4 img/s; at b64 the fused epilogue in the persistent
                    # sign kernel is slower than the separate reshare: 186.9 ->
                    # 186.4, so large blocks stay unfused.)
                    hm = self._run(spec.main[:-1], it, h, False)[0] if len(spec.main) > 1 else h
                    k = next(it)
                    pend = S.conv2d(hm, k, last.stride, last.padding, bias=next(it) if last.bias else None,
                                    relu="defer")
                    hs = self._run(spec.shortcut, it, h, False)[0] if spec.shortcut else h
                    h, fused = S.relu_epilogue_end(pend, residual=hs)
                    fused = True if fused is None else fused
                else:
                    hm = self._run(spec.main, it, h, False)[0] if spec.main else h
                    hs = self._run(spec.shortcut, it, h, False)[0] if spec.shortcut else h
                    h = S.add(hm, hs)
                acts.append(("residual",) if record else None)
        return h, acts

    def backward(self, model: ModelGraph, acts, grad_out: RssTensor, batch_bits: int = 0, sgd=None) -> list:
        """nn.py:502-536.  sgd = (params, lr): also apply the in-place SGD
        update (nn.py:539-543) — every parameter but the first layer's is
        updated on the main stream while the first layer's weight gradient
        (the last one, on the side stream) is still running."""
        if acts is None or len(acts) != len(model.layers) or any(a is None for a in acts):
            raise ProtocolError("missing activation cache; run the forward pass with recording")
        if not model.trainable:
            raise ConfigError("backward is defined for the reference's layer kinds only "
                              "(bias / residual layers are an inference extension)")
        S, t = self.s, self.t
        plist = [i for i, s in enumerate(model.layers) if s.kind in (CONV2D, FULLY_CONNECTED)]
        grads = [None] * len(plist)
        pi, g = len(plist), grad_out
        # The weight gradient of a layer and the input-gradient chain below it
        # are independent: wgrads run on a side stream (forked from the main
        # stream once g is ready) while the chain continues on the main stream.
        # Counters are taken on the host in program order, so results, shares
        # and accounting are unchanged; the inputs of each side-stream launch
        # stay referenced until the join (no allocator reuse under it).
        main = torch.cuda.current_stream()
        side = S.side_stream() if OVERLAP else None
        keep = []

        def wgrad(fn, *args):
            if side is None:
                return fn(*args)
            ev = torch.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            keep.append(args)
            with torch.cuda.stream(side):
                return fn(*args)

        rest_done = None  # side-stream event: every weight gradient but the first layer's

        def mark_rest():
            nonlocal rest_done
            if side is not None:
                rest_done = torch.cuda.Event()
                rest_done.record(side)

        skip = False  # a ReLU whose backward already ran with the pool after it
        for li in range(len(model.layers) - 1, -1, -1):
            spec, cached = model.layers[li], acts[li]
            if skip:
                skip = False
                continue
            if li == plist[0]:
                mark_rest()
            if spec.kind == FULLY_CONNECTED:
                x, w = cached[:2]
                xp, wp = cached[2:4] if len(cached) > 3 else (None, None)
                pi -= 1
                if xp is not None:  # g's role-0 pack is made on the side stream, beside the input gradient
                    grads[pi] = wgrad(lambda gg, b: S.fc_wgrad_packed(gg, b, t + batch_bits), g, xp)
                else:
                    grads[pi] = wgrad(lambda gg, xx: S.matmul(gg.apply(lambda d: d.transpose(1, 2)), xx,
                                                              bits=t + batch_bits, wgrad=True), g, x)
                if li == plist[0]:
                    break
                g = S.fc_dgrad_packed(g, wp) if wp is not None else S.matmul(g, w)
            elif spec.kind == CONV2D:
                x, k = cached[:2]
                xp, wp = cached[2:4] if len(cached) > 3 else (None, None)
                pi -= 1
                grads[pi] = wgrad(lambda xx, gg, b: S.conv2d_wgrad(
                    xx, gg, spec.kernel, spec.stride, spec.padding, bits=t + batch_bits,
                    x_packed=b), x, g, xp)
                if li == plist[0]:
                    break
                g = S.conv2d_dgrad(g, k, spec.stride, spec.padding, x.shape, bits=t, w_packed=wp)
            elif spec.kind == AVGPOOL:
                # a ReLU right before the pool: its mask multiply runs in the pool's pass
                skip = FUSE_RELU and li > 0 and model.layers[li - 1].kind == RELU
                g = S.avgpool_backward(g, spec.window, spec.stride, cached[0],
                                       mask=acts[li - 1][0] if skip else None)
            elif spec.kind == RELU:
                g = S.mul(g, cached[0], "mul.mask")
            elif spec.kind == FLATTEN:
                g = g.contiguous().reshape(cached[0])
        plan = None
        if sgd is not None:
            params, lr = sgd
            c = int(fx_encode(lr, S.fp))
            if c != 0:
                with S.replicated():  # parameters are replicated, not batch-sharded
                    plan = S.sgd_plan(params, grads)
                    if rest_done is not None and len(params) > 1:
                        main.wait_event(rest_done)
                        S.sgd_launch(plan, range(1, len(params)), c)  # overlaps the first layer's wgrad
                        rest = [0]
                    else:
                        rest = range(len(params))
        if side is not None:
            main.wait_stream(side)
        if plan is not None:
            with S.replicated():
                S.sgd_launch(plan, rest, c)
        del keep
        return grads

    def sgd(self, params: list, grads: list, lr: float, inplace: bool = False) -> list:
        """W <- W - truncate(c * grad), c = enc(lr) (nn.py:539-543).  inplace
        writes the new shares into the parameter buffers (static addresses
        for CUDA-graph replay)."""
        c = int(fx_encode(lr, self.s.fp))
        if c == 0:
            return list(params)
        S = self.s
        with S.replicated():  # parameters are replicated, not batch-sharded
            if inplace:  # every parameter in one launch, in place
                S.sgd_inplace(params, grads, c)
                return list(params)
            return [S.sub(p, S.truncate(S.mul_const(g, c)), out=p if inplace else None)
                    for p, g in zip(params, grads)]

    def loss_grad(self, logits: RssTensor, y: RssTensor) -> RssTensor:
        """softmax(logits) - y (nn.py:561-568)."""
        if logits.shape[-1] != y.shape[-1]:
            raise ShapeError(f"logit/label length mismatch {logits.shape} vs {y.shape}")
        if E.LOSS_FUSED and logits.shape == y.shape:  # one launch (mpc3_rss_softmax_loss), same shares
            return self.s.softmax_loss(logits, y)
        return self.s.sub(self.s.softmax(logits), y)


# ---------------------------------------------------------------------------
# training configuration and helpers (nn.py:625-676)


@dataclass(frozen=True)
class TrainConfig:
    learning_rate: float
    batch_size: int
    iterations: int
    seed: int = 0

    def __post_init__(self):
        if not self.learning_rate > 0:
            raise ConfigError("learning_rate must be positive")
        if self.batch_size < 1 or self.iterations < 0:
            raise ConfigError("batch_size must be >= 1 and iterations >= 0")


@dataclass
class TrainResult:
    weights: list
    ce_history: list = field(default_factory=list)


def batch_indices(iteration: int, batch_size: int, n: int) -> np.ndarray:
    return (np.arange(batch_size) + iteration * batch_size) % n


def cross_entropy(logits: np.ndarray, labels: np.ndarray) -> float:
    z = logits - logits.max(axis=-1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=-1, keepdims=True))
    return float(-logp[np.arange(len(labels)), labels].mean())


def moving_average(values, window: int = 20) -> np.ndarray:
    v = np.asarray(values, dtype=np.float64)
    half = window // 2
    return np.array([v[max(0, i - half): i + window - half].mean() for i in range(len(v))])


def one_hot(labels: np.ndarray, num_classes: int) -> np.ndarray:
    labels = np.asarray(labels)
    out = np.zeros((len(labels), num_classes))
    out[np.arange(len(labels)), labels] = 1.0
    return out


def mean_relative_error(test, ref) -> float:
    test, ref = np.asarray(test, np.float64), np.asarray(ref, np.float64)
    return float((np.abs(test - ref).max(axis=-1) / np.abs(ref).max(axis=-1)).mean())


def batch_bits(batch_size: int) -> int:
    return batch_size.bit_length() - 1 if batch_size & (batch_size - 1) == 0 else 0


# ---------------------------------------------------------------------------
# trio drivers (single thread; what bench.py and the facade call)


class TrainState:
    """Shared weights + the dealer of one private training run (nn.py:679-751)."""

    def __init__(self, sess: TrioSession, model: ModelGraph, cfg: TrainConfig, owner: int = 0, params=None):
        model.validate()
        self.sess, self.model, self.cfg, self.owner = sess, model, cfg, owner
        self.net = TrioNet(sess)
        self.rng = np.random.default_rng(cfg.seed)
        # encoded (ring.py:104-115) and dealt on the device: the PCG64 draws
        # numpy's Generator would make (sharing.py:113-118), the host
        # Generator advanced past them; init_params = fx_encode of these
        # floats (nn.py:190-202), |w| <= 1 so always in range
        if params is None:
            dev = torch.device("cuda", torch.cuda.current_device())
            plain = [sess.fx_encode_device(torch.from_numpy(w).to(dev)) for w in init_params_float(model, cfg.seed)]
        else:
            plain = [E.to_device(w) for w in params]
        self.params = [sess.share_device(w, self.rng, owner=owner) for w in plain]
        self.bbits = batch_bits(cfg.batch_size)
        self.inv_b = int(fx_encode(1.0 / cfg.batch_size, sess.fp)) if self.bbits == 0 else 0

    def deal_batch(self, xb_enc: np.ndarray, yb_enc: np.ndarray):
        S = self.sess
        return S.share(xb_enc, self.rng, owner=self.owner), S.share(yb_enc, self.rng, owner=self.owner)

    def step(self, xs: RssTensor, ys: RssTensor) -> RssTensor:
        """One private SGD iteration on dealt shares; returns the shared logits."""
        S, net = self.sess, self.net
        logits, acts = net.forward(self.model, self.params, xs, record=True)
        g = net.loss_grad(logits, ys)
        if self.bbits == 0:
            g = S.truncate(S.mul_const(g, self.inv_b))
        net.backward(self.model, acts, g, self.bbits, sgd=(self.params, self.cfg.learning_rate))
        return logits

    def capture(self, xs: RssTensor, ys: RssTensor) -> "GraphStep":
        """Record one step as a CUDA graph (see GraphStep)."""
        return GraphStep(self, xs, ys)


class GraphStep:
    """One training iteration captured as a CUDA graph.

    The ~200 launches of a step replay with one cudaGraphLaunch.  PRF stream
    counters advance exactly as in the sequential schedule: kernels read
    j = j_capture + ctr[purpose] where `ctr` is a device buffer set to
    k * (per-step consumption) before replay k, so replay k draws the same
    words the k-th eager step would (sharing.py:225-230).  Parameters are
    updated in place; inputs are read from the static buffers xs / ys.
    """

    def __init__(self, st: TrainState, xs: RssTensor, ys: RssTensor):
        import torch

        S = st.sess
        self.st, self.xs, self.ys = st, xs, ys
        self.seq0 = dict(S.seq)
        S.ctr = torch.zeros(8, dtype=torch.int64, device=xs.data.device)
        self.ctr = S.ctr
        self.graph = torch.cuda.CUDAGraph()
        try:
            # the step's rounds are recorded, not charged, at capture and
            # charged on every replay (CommStats as the eager steps')
            with S.ledger.capture() as cap, torch.cuda.graph(self.graph):
                self.logits = st.step(xs, ys)
        except BaseException:
            S.seq = dict(self.seq0)  # a refused capture consumes nothing (the caller may step eagerly)
            raise
        finally:
            S.ctr = None  # the graph keeps the buffer's address; eager calls stay absolute
        self.charge = cap.charge
        self.delta = {p: S.seq[p] - self.seq0[p] for p in S.seq}
        S.seq = dict(self.seq0)  # nothing consumed until a replay
        self.replays = 0
        # ring of pinned counter buffers; an event guards each against reuse
        self._host = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(4)]
        self._done = [None] * 4

    def replay(self):
        """Run one iteration at the session's current counters, then advance
        them by one step's consumption (eager calls may interleave)."""
        import torch

        S = self.st.sess
        slot = self.replays % 4
        if self._done[slot] is not None:
            self._done[slot].synchronize()
        hv = self._host[slot].numpy()
        for p in self.delta:
            hv[p] = S.seq[p] - self.seq0[p]
        self.ctr.copy_(self._host[slot], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._done[slot] = ev
        self.graph.replay()
        self.replays += 1
        for p, d in self.delta.items():
            S.seq[p] += d
        S.ledger.apply(self.charge)
        return self.logits


class DataParallel:
    """Batch-sharded private training/inference across GPUs.

    Every rank hosts all three parties for an equal contiguous batch shard.
    Batch-major tensors are contiguous ranges of the reference's flat tensors,
    so each kernel draws its PRF words at the shard's global offset
    (TrioSession.shard_offset) and the shards together reproduce the
    single-GPU run bit for bit.  The only exchange is the weight gradient:
    the raw per-party cross terms are summed mod 2^64 across ranks before the
    (replicated) reshare + truncation.  `allreduce(z)` sums an int64 CUDA
    tensor in place (NCCL sum wraps like the ring)."""

    def __init__(self, rank: int, world: int, allreduce):
        self.rank, self.world, self.allreduce = rank, world, allreduce

    @classmethod
    def from_process_group(cls, group=None):
        """Ranks of an initialised torch.distributed group (NCCL on the GPUs;
        gloo in the CPU tests of the host-side logic)."""
        import torch.distributed as dist

        def allreduce(z):
            dist.all_reduce(z, op=dist.ReduceOp.SUM, group=group)

        return cls(dist.get_rank(group), dist.get_world_size(group), allreduce)

    nccl = from_process_group

    def shard_rows(self, global_batch: int) -> slice:
        """This rank's contiguous batch rows."""
        if global_batch % self.world:
            raise ConfigError(f"global batch {global_batch} not divisible by {self.world} ranks")
        b = global_batch // self.world
        return slice(self.rank * b, (self.rank + 1) * b)


class TensorParallel:
    """Output-channel sharding of batch-1 private inference (SURVEY.md 8(e),
    ResNet-50 b=1): every rank computes an equal slab of each conv / FC
    layer's output channels from the full (replicated) input.  With batch 1
    a channel slab is one contiguous range of the reference's flat output,
    so the reshare / truncation / ReLU / pooling PRF words are drawn at the
    slab's global offset exactly like a batch shard (TrioSession.shard_offset)
    and the gathered activations are bit-identical to the single-GPU run.
    The one exchange per layer is an all-gather of the slabs before the next
    layer that needs every input channel.  `allgather(t)` takes an int64
    (3, S) CUDA tensor and returns (world, 3, S) in rank order."""

    def __init__(self, rank: int, world: int, allgather):
        self.rank, self.world, self.allgather = rank, world, allgather

    @classmethod
    def from_process_group(cls, group=None):
        import torch.distributed as dist

        world = dist.get_world_size(group)

        def allgather(t):
            out = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(out, t.contiguous(), group=group)
            return out.view((world,) + tuple(t.shape))

        return cls(dist.get_rank(group), world, allgather)

    def slab(self, n: int) -> slice:
        if n % self.world:
            raise ConfigError(f"{n} channels not divisible by {self.world} ranks")
        b = n // self.world
        return slice(self.rank * b, (self.rank + 1) * b)

    def gather(self, h: RssTensor) -> RssTensor:
        """Slab (3, 1, c, ...) -> full (3, 1, world*c, ...) in channel order."""
        shp = h.shape
        g = self.allgather(h.data.reshape(3, -1))  # (world, 3, S)
        full = g.permute(1, 0, 2).contiguous()
        return RssTensor(full.reshape((3, shp[0], shp[1] * self.world) + tuple(shp[2:])), h.fp)


class TPNet(TrioNet):
    """Batch-1 private inference with output-channel slabs (TensorParallel)."""

    def __init__(self, sess: TrioSession, tp: TensorParallel):
        super().__init__(sess)
        self.tp = tp

    def forward_tp(self, model: ModelGraph, params: list, x: RssTensor) -> RssTensor:
        if x.shape[0] != 1:
            raise ConfigError("output-channel sharding is defined for batch 1")
        S = self.s
        saved = S.dp
        S.dp = DataParallel(self.tp.rank, self.tp.world, None)  # slab offsets = batch-shard offsets
        try:
            h, slab = self._run_tp(model.layers, iter(params), x, False)
            return self.tp.gather(h) if slab else h
        finally:
            S.dp = saved

    def _full(self, h, slab):
        return self.tp.gather(h) if slab else h

    def _run_tp(self, layers, it, h: RssTensor, slab: bool):
        """Returns (h, is_slab)."""
        S, tp = self.s, self.tp
        for spec in layers:
            if spec.kind in (CONV2D, FULLY_CONNECTED):
                k = next(it)
                b = next(it) if spec.bias else None
                h = self._full(h, slab)
                if spec.kind == CONV2D:
                    (kh, kw), (sh, sw), (ph, pw) = k.shape[2:], spec.stride, spec.padding
                    spatial = ((h.shape[2] + 2 * ph - kh) // sh + 1) * ((h.shape[3] + 2 * pw - kw) // sw + 1)
                else:
                    spatial = 1
                # shard only into slabs whose PRF words start at an even word (one
                # AES block = two adjacent elements); otherwise compute replicated
                split = k.shape[0] % tp.world == 0 and (k.shape[0] // tp.world * spatial) % 2 == 0
                cs = tp.slab(k.shape[0]) if split else slice(None)
                kk = RssTensor(k.data[:, cs], k.fp)
                ctx = contextlib.nullcontext() if split else S.replicated()
                bb = RssTensor(b.data[:, cs], b.fp) if b is not None else None
                with ctx:
                    if spec.kind == CONV2D:
                        h = S.conv2d(h, kk, spec.stride, spec.padding, bias=bb)
                    else:
                        h = S.matmul(h, kk.apply(lambda d: d.transpose(1, 2)), bias=bb)
                if not split:  # replicated output: this rank's slab for the slab-local layers after it
                    if h.shape[1] % tp.world == 0 and (h.numel // tp.world) % 2 == 0:
                        h = RssTensor(h.data[:, :, tp.slab(h.shape[1])].contiguous(), h.fp)
                        split = True
                slab = split
            elif spec.kind in (AVGPOOL, MAXPOOL):
                pool = S.avgpool if spec.kind == AVGPOOL else S.maxpool
                if slab:
                    h = pool(h, spec.window, spec.stride, spec.padding)
                else:
                    with S.replicated():
                        h = pool(h, spec.window, spec.stride, spec.padding)
            elif spec.kind == RELU:
                if slab:
                    h = S.relu(h)
                else:
                    with S.replicated():
                        h = S.relu(h)
            elif spec.kind == FLATTEN:
                h = h.contiguous().reshape(h.shape[0], -1)
            elif spec.kind == RESIDUAL:
                full = self._full(h, slab)
                hm, ms = self._run_tp(spec.main, it, full, False) if spec.main else (full, False)
                hs, ss = self._run_tp(spec.shortcut, it, full, False) if spec.shortcut else (full, False)
                if not ms:
                    hm = RssTensor(hm.data[:, :, tp.slab(hm.shape[1])].contiguous(), hm.fp)
                if not ss:
                    hs = RssTensor(hs.data[:, :, tp.slab(hs.shape[1])].contiguous(), hs.fp)
                h, slab = S.add(hm, hs), True
        return h, slab


class InferenceGraph:
    """Private inference of a fixed-shape batch captured as a CUDA graph.

    Same counter mechanism as GraphStep: each replay draws the PRF words the
    next eager inference would.  `x` is the static input buffer.  `forward`
    (sess, model, params, x) -> logits replaces TrioNet.forward, e.g. a
    TPNet's tensor-parallel pass whose NCCL all-gathers are captured too."""

    def __init__(self, sess: TrioSession, model: ModelGraph, params: list, x: RssTensor, forward=None):
        import torch

        if forward is None:
            def forward(s, m, p, xx):
                return TrioNet(s).forward(m, p, xx, record=False)[0]
        self.sess, self.x = sess, x
        self.seq0 = dict(sess.seq)
        self.ctr = sess.ctr = torch.zeros(8, dtype=torch.int64, device=x.data.device)
        self._frozen = sess.frozen_weights()
        self._frozen.__enter__()  # weights packed once (here, outside the graph) and reused by every replay
        try:
            # warm-up outside the capture (allocations, kernel attributes, the
            # frozen weight packs) on a scratch session with throwaway keys
            # that shares this session's weight-pack cache: this session's
            # counters stay untouched, so the first replay is its next
            # inference exactly (tests/test_gpu_configs.py)
            scratch = TrioSession(None, sess.fp)
            scratch.dp, scratch._wcache = sess.dp, sess._wcache
            forward(scratch, model, params, x)
            torch.cuda.synchronize()
            self.seq0 = dict(sess.seq)
            self.graph = torch.cuda.CUDAGraph()
            try:
                with sess.ledger.capture() as cap, torch.cuda.graph(self.graph):
                    self.logits = forward(sess, model, params, x)
            except BaseException:
                sess.seq = dict(self.seq0)  # a refused capture consumes nothing (the caller may run eagerly)
                raise
            finally:
                sess.ctr = None
            self.charge = cap.charge
        finally:
            self._wpacks = sess._wcache  # the graph reads these buffers: keep them alive
            self._frozen.__exit__(None, None, None)
        self.delta = {p: sess.seq[p] - self.seq0[p] for p in sess.seq}
        sess.seq = dict(self.seq0)
        # ring of pinned counter buffers, an event guarding each against reuse
        # (as GraphStep): replays queue back to back, no host-device sync
        self._host = [torch.zeros(8, dtype=torch.int64).pin_memory() for _ in range(4)]
        self._done = [None] * 4
        self.replays = 0

    def replay(self) -> RssTensor:
        import torch

        S = self.sess
        slot = self.replays % 4
        if self._done[slot] is not None:
            self._done[slot].synchronize()
        hv = self._host[slot].numpy()
        for p in self.delta:
            hv[p] = S.seq[p] - self.seq0[p]
        self.ctr.copy_(self._host[slot], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._done[slot] = ev
        self.graph.replay()
        self.replays += 1
        for p, d in self.delta.items():
            S.seq[p] += d
        S.ledger.apply(self.charge)
        return self.logits


def train_trio(sess: TrioSession, model: ModelGraph, cfg: TrainConfig, images: np.ndarray, labels: np.ndarray,
               owner: int = 0, graph: bool = True) -> TrainResult:
    """train_private with all three parties in one thread (nn.py:679-751).

    The owner's batches go to the device as float64 and are fx-encoded and
    dealt there (mpc3_fx_encode; the PCG64 dealer reproduces numpy's draws,
    sharing.py:113-118), and from the second iteration on the step replays a
    CUDA graph when at least GRAPH_MIN_STEPS iterations remain (GraphStep:
    the same counters, shares and CommStats as the eager step; a capture
    costs ~170 ms of host time against ~2 ms saved per replayed step)."""
    st = TrainState(sess, model, cfg, owner)
    n = len(images)
    if n < 1:
        raise ConfigError("empty training set")
    d = model.num_classes
    ce = []
    dev = torch.device("cuda", torch.cuda.current_device())
    bad = torch.zeros(1, dtype=torch.int32, device=dev)  # (range checked on the host per batch)
    images = np.asarray(images, dtype=np.float64)
    lim = float(1 << (63 - sess.fp.t))
    step_graph, xs_static, ys_static = None, None, None
    for it in range(cfg.iterations):
        idx = batch_indices(it, cfg.batch_size, n)
        batch = np.ascontiguousarray(images[idx])
        if not np.isfinite(batch).all() or np.abs(batch).max(initial=0.0) >= lim:  # fx_encode's check, ring.py:107-115
            raise RangeError(f"|x| must be < 2^{63 - sess.fp.t}")
        xb = torch.from_numpy(batch).to(dev, non_blocking=True)
        yb = torch.from_numpy(one_hot(labels[idx], d)).to(dev, non_blocking=True)
        xs = sess.share_device(sess.fx_encode_device(xb, bad), st.rng, owner=owner)
        ys = sess.share_device(sess.fx_encode_device(yb, bad), st.rng, owner=owner)
        if graph and step_graph is None and it >= 1 and cfg.iterations - it >= GRAPH_MIN_STEPS:
            xs_static, ys_static = RssTensor(xs.data.clone()), RssTensor(ys.data.clone())
            step_graph = st.capture(xs_static, ys_static)
        if step_graph is not None:
            xs_static.data.copy_(xs.data)
            ys_static.data.copy_(ys.data)
            logits = step_graph.replay()
        else:
            logits = st.step(xs, ys)
        ce.append(cross_entropy(fx_decode(sess.reveal(logits), sess.fp), labels[idx]))
    weights = [sess.reveal(p) for p in st.params]
    return TrainResult(weights=weights, ce_history=ce)


def infer_trio(sess: TrioSession, model: ModelGraph, params: list, x: RssTensor) -> RssTensor:
    return TrioNet(sess).forward(model, params, x, record=False)[0]


# ---------------------------------------------------------------------------
# per-party entry points (nn.py:550-609, 679-751)


def _params_payload(model):
    if model.params is None:
        raise ProtocolError("model has no parameters")
    return list(model.params)


def _assemble_list(ps, key, fp):
    n = len(ps[0][key])
    return [assemble({p: ps[p][key][i] for p in range(3)}, fp) for i in range(n)]


def infer_private(ctx: PartyContext, model: ModelGraph, x: ArithmeticShare) -> ArithmeticShare:
    def fn(sess, ps):
        params = _assemble_list(ps, 0, ctx.fp)
        return split_trio(infer_trio(sess, model, params, assemble({p: ps[p][1] for p in range(3)}, ctx.fp)))

    return ctx.collective("infer_private", (_params_payload(model), x), fn)[ctx.party]


class _Acts:
    """Per-party activation cache: per-party views of the trio cache."""

    def __init__(self, items):
        self.items = items

    def __len__(self):
        return len(self.items)

    def __iter__(self):
        return iter(self.items)

    def __getitem__(self, i):
        return self.items[i]


def _split_acts(acts):
    per = [[], [], []]
    for a in acts:
        for p in range(3):
            if a is None:
                per[p].append(None)
            else:
                # packed trio operands (E.Packed) hold every party's share: not split out
                per[p].append(tuple(split_trio(v)[p] if isinstance(v, RssTensor) else v for v in a
                                    if not isinstance(v, E.Packed)))
    return [_Acts(v) for v in per]


def _join_acts(ps, key, fp):
    n = len(ps[0][key])
    out = []
    for i in range(n):
        a0 = ps[0][key][i]
        if a0 is None:
            out.append(None)
            continue
        out.append(tuple(assemble({p: ps[p][key][i][j] for p in range(3)}, fp)
                         if isinstance(a0[j], ArithmeticShare) else a0[j] for j in range(len(a0))))
    return out


def forward_private(ctx: PartyContext, model: ModelGraph, x: ArithmeticShare):
    def fn(sess, ps):
        params = _assemble_list(ps, 0, ctx.fp)
        logits, acts = TrioNet(sess).forward(model, params, assemble({p: ps[p][1] for p in range(3)}, ctx.fp), True)
        return split_trio(logits), _split_acts(acts)

    logits, acts = ctx.collective("forward_private", (_params_payload(model), x), fn)
    return logits[ctx.party], acts[ctx.party]


def loss_grad_output(ctx: PartyContext, logits: ArithmeticShare, y: ArithmeticShare) -> ArithmeticShare:
    if logits.shape[-1] != y.shape[-1]:
        raise ShapeError(f"logit/label length mismatch {logits.shape} vs {y.shape}")

    def fn(sess, ps):
        lg = assemble({p: ps[p][0] for p in range(3)}, ctx.fp)
        yy = assemble({p: ps[p][1] for p in range(3)}, ctx.fp)
        return split_trio(TrioNet(sess).loss_grad(lg, yy))

    return ctx.collective("loss_grad_output", (logits, y), fn)[ctx.party]


def backward(ctx: PartyContext, model: ModelGraph, acts, grad_out: ArithmeticShare, batch_bits: int = 0) -> list:
    if acts is None or len(acts) != len(model.layers) or any(a is None for a in acts):
        raise ProtocolError("missing activation cache; run the forward pass with recording")

    def fn(sess, ps):
        cache = _join_acts(ps, 0, ctx.fp)
        g = assemble({p: ps[p][1] for p in range(3)}, ctx.fp)
        grads = TrioNet(sess).backward(model, cache, g, batch_bits)
        return [split_trio(t) for t in grads]

    res = ctx.collective("backward", (list(acts), grad_out), fn)
    return [r[ctx.party] for r in res]


def sgd_step(ctx: PartyContext, params: list, grads: list, lr: float) -> list:
    def fn(sess, ps):
        P = _assemble_list(ps, 0, ctx.fp)
        G = _assemble_list(ps, 1, ctx.fp)
        return [split_trio(t) for t in TrioNet(sess).sgd(P, G, lr)]

    res = ctx.collective("sgd_step", (list(params), list(grads)), fn)
    return [r[ctx.party] for r in res]


def share_model(ctx: PartyContext, model: ModelGraph, rng=None, owner: int = 0) -> ModelGraph:
    from .session import distribute_input

    shapes = model.param_shapes()
    params = [distribute_input(ctx, model.params[i] if ctx.party == owner else None, rng, owner, shape=shapes[i])
              for i in range(len(shapes))]
    return model.with_params(params)


def train_private(ctx: PartyContext, model: ModelGraph, cfg: TrainConfig, data=None, owner: int = 0) -> TrainResult:
    """Minibatch SGD on shares; weights opened at the end (nn.py:679-751)."""
    model.validate()
    if ctx.party == owner and data is None:
        raise ProtocolError("owner must supply the training data")

    def fn(sess, ps):
        images, labels = ps[owner]
        res = train_trio(sess, model.with_params(None), cfg, np.asarray(images), np.asarray(labels), owner)
        return res

    res = ctx.collective("train_private", data if ctx.party == owner else None, fn)
    return TrainResult(weights=res.weights, ce_history=res.ce_history if ctx.party == owner else [])


def infer_plain_float(model: ModelGraph, x: np.ndarray) -> np.ndarray:
    """float64 reference forward pass (nn.py:360-398), evaluated on the GPU."""
    import torch
    import torch.nn.functional as F

    h = torch.as_tensor(np.asarray(x, np.float64), device="cuda")
    pi = 0
    for s in model.layers:
        if s.kind == CONV2D:
            h = F.conv2d(h, torch.as_tensor(np.asarray(model.params[pi], np.float64), device="cuda"),
                         stride=s.stride, padding=s.padding)
            pi += 1
        elif s.kind == FULLY_CONNECTED:
            h = h @ torch.as_tensor(np.asarray(model.params[pi], np.float64), device="cuda").T
            pi += 1
        elif s.kind == AVGPOOL:
            h = F.avg_pool2d(h, s.window, s.stride)
        elif s.kind == MAXPOOL:
            h = F.max_pool2d(h, s.window, s.stride, s.padding)
        elif s.kind == RELU:
            h = h * (h >= 0)
        elif s.kind == FLATTEN:
            h = h.reshape(h.shape[0], -1)
    return h.cpu().numpy()


__all__ = [
    "LayerSpec", "ModelGraph", "TrainConfig", "TrainResult", "TrioNet", "TrainState", "avgpool", "backward",
    "maxpool", "residual",
    "conv2d", "flatten", "forward_private", "fully_connected", "infer_plain_float", "infer_private", "infer_trio",
    "init_params", "init_params_float", "loss_grad_output", "mean_relative_error", "relu", "sgd_step",
    "share_model", "train_private", "train_trio", "one_hot", "cross_entropy", "batch_indices", "moving_average",
]
_ = E
