"""Kernel microbenchmarks on one B200 (CUDA-event timed, warm, L2-flushed).

python tools/microbench.py [--out gpurun_out/microbench.json] [--quick]

Reports: ring GEMM (tcgen05 kind::i8) ring-TOPS and int8-op rate for the
M=N=K sweep, cuBLASLt int8 (torch._int_mm) as the measured int8 roofline,
AES-CTR PRF blocks/s, and the fused sign (ReLU) / truncate kernels.
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_10949_b200 import _capi  # noqa: E402

L2_FLUSH = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def p(t):
    return C.c_void_p(t.data_ptr())


def st():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def timeit(fn, iters=10, warmup=3, flush=True):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush:
            L2_FLUSH.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b) / 1e3)
    return float(np.median(times)), float(np.min(times))


def rk3():
    rk = np.zeros((3, 44), np.uint32)
    for i in range(3):
        _capi.check(_capi.lib().mpc3_aes128_expand(C.c_char_p(bytes([i]) * 16), rk[i].ctypes.data_as(C.c_void_p)))
    return torch.from_numpy(rk.view(np.int32)).pin_memory()  # keys are read on the host at launch


def gemm_sweep(sizes):
    """M = N = K = n ring GEMMs (72 int8 ops per ring MAC) on random packed
    operands in the layout the engine's forward GEMMs use (A read MN-major
    from a transposed pack, B K-major: mpc3_ring_gemm_t with a_mn = 1, the
    contraction as two halves of n/2 source rows each), and for reference
    the all-K-major form (mpc3_ring_gemm_auto)."""
    out = []
    for n in sizes:
        kc = n // 2
        At = torch.randint(0, 256, (8 * kc * 2 * n,), dtype=torch.uint8, device="cuda")  # [8][n/2][2n]
        B = torch.randint(0, 256, (8 * n * n,), dtype=torch.uint8, device="cuda")         # [8][n][n]
        Cm = torch.empty(n * n, dtype=torch.int64, device="cuda")

        def run():
            _capi.call("mpc3_ring_gemm_t", p(At), 1, kc, 2 * n, n, p(B), 0, n, n, 0, p(Cm), 1, n, n, kc, 0, st())

        def run_k():
            _capi.call("mpc3_ring_gemm_auto", p(At), p(B), p(Cm), 1, n, n, n, 0, st())

        med, best = timeit(run, iters=5 if n >= 4096 else 10)
        med_k, _ = timeit(run_k, iters=5 if n >= 4096 else 10)
        ring_macs = n ** 3
        out.append({"n": n, "ms": med * 1e3, "ring_tops": 2 * ring_macs / med / 1e12,
                    "int8_tops": 72 * ring_macs / med / 1e12, "best_ms": best * 1e3,
                    "kmajor_ms": med_k * 1e3, "kmajor_int8_tops": 72 * ring_macs / med_k / 1e12})
        print("gemm", out[-1], flush=True)
        del At, B, Cm
    return out


def gemm_t_compare(shapes):
    """Weight-gradient GEMM read transposed from packed buffers (mpc3_ring_gemm_t,
    MN-major tiles) vs the same product from K-major packs (gemm_auto)."""
    out = []
    for (M, N, R) in shapes:
        kc = (R + 31) // 32 * 32
        kha, khb = (M + 15) // 16 * 16, (N + 15) // 16 * 16
        kpa, kpb = (kha + M + 15) // 16 * 16, (khb + N + 15) // 16 * 16
        A = torch.randint(0, 256, (3 * 8 * R * kpa,), dtype=torch.uint8, device="cuda")
        B = torch.randint(0, 256, (3 * 8 * R * kpb,), dtype=torch.uint8, device="cuda")
        Ak = torch.randint(0, 256, (3 * 8 * M * 2 * kc,), dtype=torch.uint8, device="cuda")
        Bk = torch.randint(0, 256, (3 * 8 * N * 2 * kc,), dtype=torch.uint8, device="cuda")
        Cm = torch.empty(3 * M * N, dtype=torch.int64, device="cuda")
        t_mn = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(A), 1, R, kpa, kha, p(B), 1, R, kpb, khb, p(Cm), 3,
                                           M, N, kc, 0, st()), reps=5)
        t_k = graph_us(lambda: _capi.call("mpc3_ring_gemm_auto", p(Ak), p(Bk), p(Cm), 3, M, N, 2 * kc, 0, st()), reps=5)
        t_amn = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(A), 1, R, kpa, kha, p(Bk), 0, N, 2 * kc, 0, p(Cm),
                                            3, M, N, kc, 0, st()), reps=5)
        t_bmn = graph_us(lambda: _capi.call("mpc3_ring_gemm_t", p(Ak), 0, M, 2 * kc, 0, p(B), 1, R, kpb, khb, p(Cm),
                                            3, M, N, kc, 0, st()), reps=5)
        ops = 72 * 3 * M * N * 2 * R
        out.append({"M": M, "N": N, "R": R, "mn_us": t_mn, "kmajor_us": t_k, "mn_tops": ops / t_mn / 1e6,
                    "kmajor_tops": ops / t_k / 1e6, "a_mn_tops": ops / t_amn / 1e6, "b_mn_tops": ops / t_bmn / 1e6})
        print("gemm_t", out[-1], flush=True)
    return out


def int8_peak():
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    try:
        med, best = timeit(lambda: torch._int_mm(a, b), iters=10, flush=False)
    except Exception as e:  # noqa: BLE001
        return {"error": repr(e)}
    return {"n": n, "ms": med * 1e3, "tops": 2 * n ** 3 / med / 1e12, "best_tops": 2 * n ** 3 / best / 1e12}


def aes_rate():
    rk = rk3()
    count = 1 << 28  # words -> 2^27 blocks
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    med, _ = timeit(lambda: _capi.call("mpc3_prf_words", p(rk), 1, 0, 0, count, p(out), st()), iters=5)
    return {"blocks": count // 2, "ms": med * 1e3, "gblocks_s": count / 2 / med / 1e9,
            "gbytes_s": count * 8 / med / 1e9}


def protocol_rates():
    rk = rk3()
    res = {}
    n = 1 << 24
    x = torch.randint(-(1 << 40), 1 << 40, (3 * n,), dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    m = torch.empty_like(x)
    med, _ = timeit(lambda: _capi.call("mpc3_rss_sign", p(rk), None, 3, 0, 0, 0, p(x), p(y), p(m), n, n, 0, st()), iters=5)
    # 23 AES-128 blocks per element (46 PRF words: BIN 1, XOR 36, ARITH 9)
    res["relu"] = {"n": n, "ms": med * 1e3, "gelem_s": n / med / 1e9, "aes_gblocks_s": 23 * n / med / 1e9,
                   "hbm_gbs": 72 * n / med / 1e9}
    med, _ = timeit(lambda: _capi.call("mpc3_rss_truncate", p(rk), None, 0, 0, 20, p(x), p(y), n, 0, st()), iters=5)
    res["truncate"] = {"n": n, "ms": med * 1e3, "gelem_s": n / med / 1e9, "hbm_gbs": 48 * n / med / 1e9}
    med, _ = timeit(lambda: _capi.call("mpc3_rss_mul", p(rk), None, 0, p(x), p(x), p(y), n, 0, st()), iters=5)
    res["mul"] = {"n": n, "ms": med * 1e3, "gelem_s": n / med / 1e9, "hbm_gbs": 72 * n / med / 1e9}
    # device time of the small launches of a training step: 20 launches captured
    # in a CUDA graph, replayed back to back (no host launch gaps, no L2 flush)
    for small in (64, 1024, 16384, 262144):
        xs, ys, ms = x[:3 * small], y[:3 * small], m[:3 * small]
        res[f"relu_n{small}_us"] = graph_us(lambda: _capi.call(
            "mpc3_rss_sign", p(rk), None, 3, 0, 0, 0, p(xs), p(ys), p(ms), small, small, 0, st()))
        res[f"mul_n{small}_us"] = graph_us(lambda: _capi.call(
            "mpc3_rss_mul", p(rk), None, 0, p(xs), p(xs), p(ys), small, 0, st()))
    return res


def cpu_reference(sizes, relu_n=1 << 20):
    """The reference's CPU path beside the GPU sweep: the
    unmodified mpc3 (baseline/_ref, refarm.py) `bilinear_exact(a, b,
    matmul_spec(n, n, n))` on rand_u64 inputs (tests/test_ring.py:15-16), one
    warm-up call, and its 3-party `relu` / `truncate` on fx_encode(U(-8, 8))
    (cli.py:250-251) through run_in_process."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import refarm

    mod, src = refarm.load()
    if mod is None:
        return {"unavailable": src}
    from mpc3 import protocols as P
    from mpc3.ring import bilinear_exact, fx_encode, matmul_spec
    from mpc3.session import distribute_input, run_in_process

    res = {"source": src, "threads": refarm.threads(), "gemm": []}
    for n in sizes:
        rng = np.random.default_rng(n)
        a = rng.integers(0, 1 << 64, (n, n), dtype=np.uint64)
        b = rng.integers(0, 1 << 64, (n, n), dtype=np.uint64)
        bilinear_exact(a[:64, :64], b[:64, :64], matmul_spec(64, 64, 64))
        t0 = time.perf_counter()
        bilinear_exact(a, b, matmul_spec(n, n, n))
        dt = time.perf_counter() - t0
        res["gemm"].append({"n": n, "s": dt, "ring_gops": 2 * n ** 3 / dt / 1e9})
        print("cpu gemm", res["gemm"][-1], flush=True)
    x = fx_encode(np.random.default_rng(1).uniform(-8, 8, relu_n))
    for name, op in (("relu", P.relu), ("truncate", P.truncate)):
        def job(ctx, op=op):
            xs = distribute_input(ctx, x if ctx.party == 0 else None, np.random.default_rng(2), shape=x.shape)
            t0 = time.perf_counter()
            op(ctx, xs)
            return time.perf_counter() - t0
        dt = max(run_in_process(job, seed=0, timeout=1e5))
        res[name] = {"n": relu_n, "s": dt, "melem_s": relu_n / dt / 1e6}
        print("cpu", name, res[name], flush=True)
    return res


def graph_us(launch, reps=20):
    launch()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            launch()
    med, _ = timeit(g.replay, iters=10, flush=False)
    return med * 1e6 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/microbench.json")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--gemm-t", action="store_true", help="only the transposed-operand GEMM comparison")
    ap.add_argument("--aes", action="store_true", help="only the AES keystream and protocol-kernel rates")
    ap.add_argument("--cpu", action="store_true", help="also time the reference's CPU bilinear_exact / relu / truncate")
    args = ap.parse_args()
    if args.gemm_t:
        shapes = [(256, 3456, 128), (384, 3456, 128), (96, 363, 12800), (256, 2400, 512),
                  (256, 256, 128), (1024, 1024, 4096), (4096, 4096, 4096)]
        if os.environ.get("GEMM_T_FWD"):  # the AlexNet forward / input-gradient shapes (M, N, contraction)
            shapes = [(12800, 96, 384), (512, 256, 2400), (128, 384, 2304), (128, 384, 3456), (128, 3456, 256),
                      (512, 2400, 256)]
        res = gemm_t_compare(shapes)
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
        return
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    res = {"device": torch.cuda.get_device_name(), "when": time.time()}
    res["aes"] = aes_rate()
    print("aes", res["aes"], flush=True)
    res["protocols"] = protocol_rates()
    print("protocols", res["protocols"], flush=True)
    if args.aes:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
        return
    res["int8_cublaslt"] = int8_peak()
    print("int8", res["int8_cublaslt"], flush=True)
    res["gemm"] = gemm_sweep([1024, 2048, 4096] if args.quick else [256, 512, 1024, 2048, 4096, 8192])
    if args.cpu:  # bounded: n <= 4096 (8192 is ~1 min of dgemm on 16 cores)
        res["cpu_reference"] = cpu_reference([256, 512, 1024, 2048] if args.quick else [256, 512, 1024, 2048, 4096])
        for g in res["gemm"]:
            c = next((c for c in res["cpu_reference"].get("gemm", []) if c["n"] == g["n"]), None)
            if c:
                g["speedup_vs_cpu_reference"] = c["s"] / (g["ms"] / 1e3)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
