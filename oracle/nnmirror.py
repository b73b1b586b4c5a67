"""Layer schedule of private inference/training, restated (TEST ORACLE ONLY).

Restates nn.py: model graphs (nn.py:43-187, models.py:39-84), the
engine-generic forward/backward schedule (nn.py:405-543) and the drivers
infer_private / train_private / train_plain_fixed (nn.py:550-793).  Two
engines: `TrioEngine` runs the trio-form protocols of `oracle.rss` (the CPU
reference arm of bench.py); `FixedEngine` is the plaintext ring mirror with
optional rho replay (nn.py:256-357).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.lib.stride_tricks import sliding_window_view

from . import rss as R

U64 = R.U64

CONV, FC, POOL, RELU, FLAT = "Conv2d", "FullyConnected", "AvgPool", "ReLU", "Flatten"


RES = "Residual"
MAXP = "MaxPool"


@dataclass(frozen=True)
class Layer:
    kind: str
    out: int = 0
    kernel: tuple = ()
    stride: tuple = (1, 1)
    padding: tuple = (0, 0)
    window: tuple = ()
    bias: bool = False
    main: tuple = ()
    shortcut: tuple = ()


def from_spec(spec):
    """Oracle layer from a product LayerSpec (so composed models are built once)."""
    kind = spec.kind
    return Layer(kind, out=spec.out_channels or spec.out_features, kernel=tuple(spec.kernel),
                 stride=tuple(spec.stride), padding=tuple(spec.padding), window=tuple(spec.window),
                 bias=bool(getattr(spec, "bias", False)),
                 main=tuple(from_spec(s) for s in getattr(spec, "main", ())),
                 shortcut=tuple(from_spec(s) for s in getattr(spec, "shortcut", ())))


def _p(v):
    return tuple(int(a) for a in v) if isinstance(v, (tuple, list)) else (int(v), int(v))


def conv(o, k, stride=1, padding=0):
    return Layer(CONV, out=o, kernel=_p(k), stride=_p(stride), padding=_p(padding))


def fc(o):
    return Layer(FC, out=o)


def pool(w, stride=None):
    return Layer(POOL, window=_p(w), stride=_p(stride) if stride is not None else _p(w))


def relu():
    return Layer(RELU)


def flat():
    return Layer(FLAT)


def lenet():
    """models.py:39-56."""
    return (conv(6, 5), relu(), pool(2), conv(16, 5), relu(), pool(2), flat(), fc(100), relu(), fc(10)), (1, 28, 28)


def alexnet_cifar():
    """models.py:59-84."""
    return (
        conv(96, 11, 4, 9), relu(), pool(3, 2),
        conv(256, 5, 1, 1), relu(), pool(2, 1),
        conv(384, 3, 1, 1), relu(), conv(384, 3, 1, 1), relu(), conv(256, 3, 1, 1), relu(),
        flat(), fc(256), relu(), fc(256), relu(), fc(10),
    ), (3, 32, 32)


def shapes(layers, input_shape):
    """Per-layer output shapes and parameter shapes (nn.py:99-164)."""
    shape = tuple(input_shape)
    outs, params = [], []
    for L in layers:
        if L.kind == CONV:
            c, h, w = shape
            oh, ow = R.conv_out_hw(h, w, *L.kernel, L.stride, L.padding)
            params.append((L.out, c) + L.kernel)
            shape = (L.out, oh, ow)
        elif L.kind == POOL:
            c, h, w = shape
            shape = (c, (h - L.window[0]) // L.stride[0] + 1, (w - L.window[1]) // L.stride[1] + 1)
        elif L.kind == FC:
            params.append((L.out, shape[0]))
            shape = (L.out,)
        elif L.kind == FLAT:
            shape = (int(np.prod(shape)),)
        outs.append(shape)
    return outs, params


def init_params_float(layers, input_shape, seed=0):
    """nn.py:190-198."""
    rng = np.random.default_rng(seed)
    out = []
    for shp in shapes(layers, input_shape)[1]:
        b = 1.0 / np.sqrt(int(np.prod(shp[1:])))
        out.append(rng.uniform(-b, b, shp))
    return out


def init_params(layers, input_shape, t=20, seed=0):
    return [R.fx_encode(w, t) for w in init_params_float(layers, input_shape, seed)]


# ---------------------------------------------------------------------------
# engines


class TrioEngine:
    """Private engine on trio arrays (nn.py:209-253)."""

    def __init__(self, s: R.Session):
        self.s = s
        self.t = s.t

    def shape(self, x):
        return x.shape[1:]

    def map_structural(self, x, f):
        return np.stack([f(x[i]) for i in range(3)])

    def conv2d(self, x, k, stride, padding, bits=None):
        return R.conv2d_shares(self.s, x, k, stride, padding, bits)

    def matmul(self, a, b, bits=None):
        return R.matmul_shares(self.s, a, b, bits)

    def avgpool(self, x, window, stride):
        return R.avgpool_shares(self.s, x, window, stride)

    def relu_mask(self, x):
        return R.relu_with_mask(self.s, x)

    def apply_mask(self, g, mask):
        return R.mul(self.s, g, mask)

    def sub(self, a, b):
        return a - b

    def truncate(self, x, bits=None):
        return R.truncate(self.s, x, bits)

    def mul_ring_const(self, x, c):
        return R.mul_const(x, c)

    def div_area(self, x, area):
        return R.div_area(self.s, x, area)

    def softmax(self, z):
        return R.softmax(self.s, z)


def _wrap_sumpool(x, window, stride):
    win = sliding_window_view(x, window, axis=(2, 3))[:, :, :: stride[0], :: stride[1]]
    return np.einsum("ncxyuv->ncxy", win, dtype=U64, casting="unsafe")


class FixedEngine:
    """Plaintext ring mirror (nn.py:274-357)."""

    def __init__(self, t=20, offsets=None):
        self.t = t
        self.offsets = offsets

    def shape(self, x):
        return x.shape

    def map_structural(self, x, f):
        return f(x)

    def truncate(self, x, bits=None):
        bits = self.t if bits is None else bits
        half = U64(1 << (bits - 1))
        if self.offsets is None:
            return R.sar(x + half, bits)
        rho = self.offsets.draw(np.shape(x))
        return R.sar(rho + half, bits) + R.sar(x - rho + half, bits)

    def conv2d(self, x, k, stride, padding, bits=None):
        return self.truncate(R.wrap_conv2d(x, k, stride, padding), bits)

    def matmul(self, a, b, bits=None):
        return self.truncate(R.wrap_matmul(a, b), bits)

    def div_area(self, x, area):
        if area & (area - 1) == 0:
            return self.truncate(x, area.bit_length() - 1)
        return self.truncate(x * U64(int(R.fx_encode(1.0 / area, self.t))))

    def avgpool(self, x, window, stride):
        return self.div_area(_wrap_sumpool(x, window, stride), window[0] * window[1])

    def relu_mask(self, x):
        mask = U64(1) - (x >> U64(63))
        return x * mask, mask

    def apply_mask(self, g, mask):
        return g * mask

    def sub(self, a, b):
        return a - b

    def mul_ring_const(self, x, c):
        return x * U64(c & ((1 << 64) - 1))

    def exp_approx(self, x, m=512):
        sq = m.bit_length() - 1
        y = x + R.fx_encode(float(m), self.t)
        y = self.truncate(y * y, self.t + 2 * sq)
        for _ in range(sq - 1):
            y = self.truncate(y * y)
        return y

    def reciprocal(self, y, Y=200.0, iterations=13):
        z = np.broadcast_to(R.fx_encode(1.0 / Y, self.t), y.shape).copy()
        for _ in range(iterations):
            z2 = self.truncate(z * z)
            yz2 = self.truncate(y * z2)
            z = z * U64(2) - yz2
        return z

    def softmax(self, z):
        mx = np.max(z.view(np.int64), axis=-1, keepdims=True).view(U64)
        e = self.exp_approx(z - mx)
        r = self.reciprocal(e.sum(axis=-1, keepdims=True, dtype=U64))
        return self.truncate(e * r)


# ---------------------------------------------------------------------------
# schedule (nn.py:405-543)


def forward(eng, layers, params, x, record):
    acts, h, pi = [], x, 0
    for L in layers:
        if L.kind == CONV:
            k = params[pi]
            pi += 1
            acts.append((h, k) if record else None)
            h = eng.conv2d(h, k, L.stride, L.padding)
        elif L.kind == FC:
            w = params[pi]
            pi += 1
            acts.append((h, w) if record else None)
            h = eng.matmul(h, eng.map_structural(w, lambda a: a.T))
        elif L.kind == POOL:
            acts.append((eng.shape(h),) if record else None)
            h = eng.avgpool(h, L.window, L.stride)
        elif L.kind == RELU:
            h, mask = eng.relu_mask(h)
            acts.append((mask,) if record else None)
        elif L.kind == FLAT:
            shp = eng.shape(h)
            acts.append((shp,) if record else None)
            h = eng.map_structural(h, lambda a: a.reshape(shp[0], -1))
    return h, acts


def dilate(a, stride):
    sh, sw = stride
    if sh == 1 and sw == 1:
        return a
    n, c, h, w = a.shape
    out = np.zeros((n, c, (h - 1) * sh + 1, (w - 1) * sw + 1), a.dtype)
    out[:, :, ::sh, ::sw] = a
    return out


def conv_grad_kernel(eng, x, g, L, bits):
    """nn.py:435-457."""
    kh, kw = L.kernel
    a = eng.map_structural(x, lambda v: v.transpose(1, 0, 2, 3))
    b = eng.map_structural(g, lambda v: dilate(v, L.stride).transpose(1, 0, 2, 3))
    full = eng.conv2d(a, b, (1, 1), L.padding, bits=bits)
    return eng.map_structural(full, lambda v: v[:, :, :kh, :kw].transpose(1, 0, 2, 3))


def conv_grad_input(eng, g, k, L, in_shape, bits):
    """nn.py:460-484."""
    kh, kw = L.kernel
    ph, pw = L.padding
    h, w = in_shape[-2:]
    gp = eng.map_structural(
        g, lambda v: np.pad(dilate(v, L.stride), ((0, 0), (0, 0), (kh - 1, kh - 1), (kw - 1, kw - 1)))
    )
    kf = eng.map_structural(k, lambda v: v.transpose(1, 0, 2, 3)[:, :, ::-1, ::-1])
    full = eng.conv2d(gp, kf, (1, 1), (0, 0), bits=bits)

    def embed(v):
        canvas = np.zeros(v.shape[:2] + (h + 2 * ph, w + 2 * pw), v.dtype)
        canvas[:, :, : v.shape[2], : v.shape[3]] = v
        return canvas[:, :, ph : ph + h, pw : pw + w]

    return eng.map_structural(full, embed)


def avgpool_backward(eng, g, window, stride, in_shape):
    """nn.py:487-499."""
    wh, ww = window
    sh, sw = stride
    ho, wo = eng.shape(g)[-2:]

    def up(a):
        out = np.zeros(in_shape, a.dtype)
        for u in range(wh):
            for v in range(ww):
                out[:, :, u : u + sh * (ho - 1) + 1 : sh, v : v + sw * (wo - 1) + 1 : sw] += a
        return out

    return eng.div_area(eng.map_structural(g, up), wh * ww)


def backward(eng, layers, acts, grad_out, batch_bits=0):
    """nn.py:502-536."""
    t = eng.t
    plist = [i for i, L in enumerate(layers) if L.kind in (CONV, FC)]
    grads = [None] * len(plist)
    pi = len(plist)
    g = grad_out
    for li in range(len(layers) - 1, -1, -1):
        L, cached = layers[li], acts[li]
        if L.kind == FC:
            x, w = cached
            pi -= 1
            grads[pi] = eng.matmul(eng.map_structural(g, lambda a: a.T), x, bits=t + batch_bits)
            if li == plist[0]:
                break
            g = eng.matmul(g, w)
        elif L.kind == CONV:
            x, k = cached
            pi -= 1
            grads[pi] = conv_grad_kernel(eng, x, g, L, bits=t + batch_bits)
            if li == plist[0]:
                break
            g = conv_grad_input(eng, g, k, L, eng.shape(x), bits=t)
        elif L.kind == POOL:
            g = avgpool_backward(eng, g, L.window, L.stride, cached[0])
        elif L.kind == RELU:
            g = eng.apply_mask(g, cached[0])
        elif L.kind == FLAT:
            g = eng.map_structural(g, lambda a, s=cached[0]: a.reshape(s))
    return grads


def sgd(eng, params, grads, lr):
    """nn.py:539-543."""
    c = int(R.fx_encode(lr, eng.t))
    if c == 0:
        return list(params)
    return [eng.sub(p, eng.truncate(eng.mul_ring_const(g, c))) for p, g in zip(params, grads)]


def one_hot(labels, d):
    out = np.zeros((len(labels), d))
    out[np.arange(len(labels)), labels] = 1.0
    return out


def batch_bits(b):
    return b.bit_length() - 1 if b & (b - 1) == 0 else 0


def train_private(s: R.Session, layers, input_shape, images, labels, lr, batch, iterations, seed=0, params=None):
    """Trio restatement of nn.py:679-751: owner deals params then each batch
    (x then y) from default_rng(seed); returns the trio weights and opened logits."""
    outs, pshapes = shapes(layers, input_shape)
    d = outs[-1][0]
    rng = np.random.default_rng(seed)
    plain = init_params(layers, input_shape, s.t, seed) if params is None else params
    P = [R.share(w, rng) for w in plain]
    bb = batch_bits(batch)
    inv_b = int(R.fx_encode(1.0 / batch, s.t)) if bb == 0 else 0
    eng = TrioEngine(s)
    n = len(images)
    logits_hist = []
    for it in range(iterations):
        idx = (np.arange(batch) + it * batch) % n
        xs = R.share(R.fx_encode(images[idx], s.t), rng)
        ys = R.share(R.fx_encode(one_hot(labels[idx], d), s.t), rng)
        logits, acts = forward(eng, layers, P, xs, True)
        g = R.softmax(s, logits) - ys
        if bb == 0:
            g = R.truncate(s, R.mul_const(g, inv_b))
        grads = backward(eng, layers, acts, g, bb)
        P = sgd(eng, P, grads, lr)
        logits_hist.append(R.open_trio(logits))
    return P, logits_hist


class TrainLoop:
    """train_private split into setup (param dealing) and per-iteration steps,
    so the CPU baseline times iterations the way bench.py times the GPU."""

    def __init__(self, s: R.Session, layers, input_shape, lr, batch, seed=0):
        self.s, self.layers, self.lr, self.batch = s, layers, lr, batch
        outs, _ = shapes(layers, input_shape)
        self.d = outs[-1][0]
        self.rng = np.random.default_rng(seed)
        self.P = [R.share(w, self.rng) for w in init_params(layers, input_shape, s.t, seed)]
        self.bb = batch_bits(batch)
        self.inv_b = int(R.fx_encode(1.0 / batch, s.t)) if self.bb == 0 else 0
        self.eng = TrioEngine(s)

    def step(self, images, labels):
        s, eng = self.s, self.eng
        xs = R.share(R.fx_encode(images, s.t), self.rng)
        ys = R.share(R.fx_encode(one_hot(labels, self.d), s.t), self.rng)
        logits, acts = forward(eng, self.layers, self.P, xs, True)
        g = R.softmax(s, logits) - ys
        if self.bb == 0:
            g = R.truncate(s, R.mul_const(g, self.inv_b))
        grads = backward(eng, self.layers, acts, g, self.bb)
        self.P = sgd(eng, self.P, grads, self.lr)
        return R.open_trio(logits)


def train_plain_fixed(layers, input_shape, images, labels, lr, batch, iterations, seed=0, t=20, offsets=None):
    """nn.py:754-793."""
    outs, _ = shapes(layers, input_shape)
    d = outs[-1][0]
    eng = FixedEngine(t, offsets)
    params = init_params(layers, input_shape, t, seed)
    bb = batch_bits(batch)
    inv_b = int(R.fx_encode(1.0 / batch, t)) if bb == 0 else 0
    n = len(images)
    for it in range(iterations):
        idx = (np.arange(batch) + it * batch) % n
        xs = R.fx_encode(images[idx], t)
        ys = R.fx_encode(one_hot(labels[idx], d), t)
        logits, acts = forward(eng, layers, params, xs, True)
        g = eng.softmax(logits) - ys
        if bb == 0:
            g = eng.truncate(eng.mul_ring_const(g, inv_b))
        grads = backward(eng, layers, acts, g, bb)
        params = sgd(eng, params, grads, lr)
    return params


def infer_private(s: R.Session, layers, params_trio, x_trio):
    return forward(TrioEngine(s), layers, params_trio, x_trio, False)[0]


def forward_ext(s: R.Session, layers, it, h):
    """Inference with the ResNet extensions, COMPOSED from reference
    primitives (no reference model has them): conv2d_shares /
    matmul_shares then a local add of the shared bias; residual = local add of
    the two branches; padded average pool = zero-pad each component, then
    avgpool_shares (protocols.py:139-159)."""
    for L in layers:
        if L.kind == CONV:
            h = R.conv2d_shares(s, h, next(it), L.stride, L.padding)
            if L.bias:
                b = next(it)
                h = h + b[:, None, :, None, None]
        elif L.kind == FC:
            w = next(it)
            h = R.matmul_shares(s, h, np.stack([w[i].T for i in range(3)]))
            if L.bias:
                b = next(it)
                h = h + b[:, None, :]
        elif L.kind == POOL:
            ph, pw = L.padding
            if ph or pw:
                h = np.pad(h, ((0, 0), (0, 0), (0, 0), (ph, ph), (pw, pw)))
            h = R.avgpool_shares(s, h, L.window, L.stride)
        elif L.kind == MAXP:
            h = R.maxpool_shares(s, h, L.window, L.stride, L.padding)
        elif L.kind == RELU:
            h = R.relu(s, h)
        elif L.kind == FLAT:
            h = h.reshape(3, h.shape[1], -1)
        elif L.kind == RES:
            hm = forward_ext(s, L.main, it, h) if L.main else h
            hs = forward_ext(s, L.shortcut, it, h) if L.shortcut else h
            h = hm + hs
    return h
