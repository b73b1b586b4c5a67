"""Ring conv2d microbench over the distinct ResNet-50 convolution shapes
(BASELINE configs[4]): for each shape at batch 1 and 64,
the secure conv2d_shares of the engine (operand packs + tcgen05 ring GEMM of
the three parties' cross terms + reshare / truncate / bias) timed with CUDA
events, warm, L2 flushed between repetitions.

python tools/resnet_convs.py [--out gpurun_out/resnet_convs.json] [--batches 1 64]

Reported per shape: multiplicity in the network, GEMM dims (M = N*OH*OW,
N = O, K = C*kh*kw), secure-conv time, ring-TOPS (2*M*N*K per party-product,
3 parties x 2 cross-term products) and int8-TOPS (72 int8 ops per ring MAC,
3 parties x M x N x 2K), against the measured int8 roofline; and the same
for the packs + ring GEMM alone (the rest is the AES-bound reshare /
truncate over the M x N outputs, which dominates the small-K layers).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import engine as E  # noqa: E402
from paper_2104_10949_b200.nn import CONV2D, RESIDUAL, AVGPOOL  # noqa: E402


def conv_shapes(layers, c, h, w, out):
    """Walk the graph: (C, H, W, O, k, stride, pad) of every conv, in order."""
    for s in layers:
        if s.kind == CONV2D:
            (kh, kw), (sh, sw), (ph, pw) = s.kernel, s.stride, s.padding
            out.append((c, h, w, s.out_channels, kh, sh, ph))
            h, w, c = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1, s.out_channels
        elif s.kind == AVGPOOL:
            (kh, kw), (sh, sw), (ph, pw) = s.window, s.stride, s.padding
            h, w = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
        elif s.kind == RESIDUAL:
            c0, h0, w0 = c, h, w
            c, h, w = conv_shapes(s.main, c0, h0, w0, out)
            if s.shortcut:
                conv_shapes(s.shortcut, c0, h0, w0, out)
    return c, h, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/resnet_convs.json")
    ap.add_argument("--batches", type=int, nargs="*", default=[1, 64])
    args = ap.parse_args()
    model = M.models.resnet50()
    shapes = []
    conv_shapes(model.layers, *model.input_shape, shapes)
    distinct = {}
    for sh in shapes:
        distinct[sh] = distinct.get(sh, 0) + 1
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                            "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        peaks = {"bf16_tflops": 1590.0}  # B200_PROFILING.md fallback
    int8_peak = 2 * peaks["bf16_tflops"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    S = M.TrioSession(seed=0)
    rng = np.random.default_rng(0)
    res = {"device": torch.cuda.get_device_name(), "when": time.time(), "int8_peak_tops": int8_peak,
           "distinct_shapes": len(distinct), "convs": len(shapes), "rows": []}
    for b in args.batches:
        for (c, h, w, o, k, st, pd), mult in distinct.items():
            x = E.RssTensor(torch.from_numpy(rng.integers(-(1 << 40), 1 << 40, (3, b, c, h, w))).cuda())
            kk = E.RssTensor(torch.from_numpy(rng.integers(-(1 << 30), 1 << 30, (3, o, c, k, k))).cuda())
            bias = E.RssTensor(torch.from_numpy(rng.integers(-(1 << 30), 1 << 30, (3, o))).cuda())
            oh, ow = (h + 2 * pd - k) // st + 1, (w + 2 * pd - k) // st + 1
            Mm, Nn, Kk = b * oh * ow, o, c * k * k

            def run():
                S.conv2d(x, kk, (st, st), (pd, pd), bias=bias)

            xs, ks = x.data.stride(), kk.data.stride()
            a_op = E.K.conv_operand(E.K.GATHER_IM2COL, Mm, Kk, b, c, h, w, xs[1:], k, k, st, st, pd, pd, oh, ow)
            b_op = S.conv_weight_operand(kk)[0]

            def gemm():  # the operand packs + the ring GEMM of the three parties' cross terms only
                S._cross_gemm(x.data, a_op, kk.data, b_op, Mm, Nn, Kk, c_col=True)

            def timed(fn):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                ts = []
                for _ in range(5 if b > 1 else 10):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 1e3)
                return float(np.median(ts))

            t, tg = timed(run), timed(gemm)
            ops = 72 * 3 * Mm * Nn * 2 * Kk
            row = {"batch": b, "C": c, "H": h, "W": w, "O": o, "k": k, "stride": st, "pad": pd, "count": mult,
                   "M": Mm, "N": Nn, "K": Kk, "secure_conv_us": round(t * 1e6, 1),
                   "ring_tops": round(2 * 3 * 2 * Mm * Nn * Kk / t / 1e12, 2), "int8_tops": round(ops / t / 1e12, 1),
                   "frac_of_int8_peak": round(ops / t / 1e12 / int8_peak, 3),
                   "packs_plus_gemm_us": round(tg * 1e6, 1), "gemm_path_int8_tops": round(ops / tg / 1e12, 1),
                   "epilogue_share": round(1 - tg / t, 3)}
            res["rows"].append(row)
            print(row, flush=True)
            del x, kk, bias
    for b in args.batches:
        rows = [r for r in res["rows"] if r["batch"] == b]
        tot_us = sum(r["secure_conv_us"] * r["count"] for r in rows)
        tot_ops = sum(72 * 3 * r["M"] * r["N"] * 2 * r["K"] * r["count"] for r in rows)
        res[f"b{b}_all_53_convs_us"] = round(tot_us, 1)
        res[f"b{b}_weighted_int8_tops"] = round(tot_ops / (tot_us / 1e6) / 1e12, 1)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)
    print({k: v for k, v in res.items() if k.startswith("b")})


if __name__ == "__main__":
    main()
