"""Headline benchmark: AlexNet-CIFAR private training step (3-party RSS over
Z_2^64, batch 128 per GPU), images/s — BASELINE.json configs[1].

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

One "step" = one private SGD iteration (forward, softmax loss gradient,
backward, SGD update, all on shares) over one synthetic CIFAR-shaped batch.
`value`: device-resident dealt batches, CUDA-event timed per step with an L2
flush (256 MiB write) before each timed step, outside its events; max over
ranks.  `e2e`: the same step through the public API with host inputs: the
owner's fx-encoding + dealing on the host, pinned H2D of the shares, the
step, and the D2H of the opened logits (nn.py:746) inside the timed region.
Multi-GPU (N>1): each rank trains an independent replica on its own batch
(replicas; no data-path collective yet — see DESIGN.md), "scaling": "weak".

`--impl reference` times the reference algorithm's CPU implementation (the
oracle port, oracle/nnmirror.py) on the host cores on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "private images/sec (ResNet-50 inf, AlexNet train) at 1/2/4/8 B200; ring-GEMM TOPS"
UNIT = "images/s"
BATCH = 128
CPU_SAMPLE_BATCH = 32


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-resnet", action="store_true", help="skip the ResNet-50 inference side measurement")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _config(args, ws):
    return {"workload": "AlexNet-CIFAR private training step (3-party RSS, Z_2^64, t=20)",
            "model": "alexnet_cifar", "global_batch": args.batch * ws, "per_gpu_batch": args.batch,
            "input": "3x32x32", "classes": 10, "parallelism": f"dp{ws} (batch shards, NCCL all-reduce of weight-"
                                                             f"gradient cross terms)" if ws > 1 else "single",
            "l2": "flushed (256 MiB write) before every timed step, outside its events"}


def _synthetic(batch, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, (batch, 3, 32, 32)), rng.integers(0, 10, batch)


# ---------------------------------------------------------------------------
# CPU: the reference algorithm (oracle port)


def cpu_steps(batch, steps, warmup):
    from oracle import nnmirror as N
    from oracle import rss as R

    layers, ish = N.alexnet_cifar()
    imgs, labels = _synthetic(batch, 0)
    loop = N.TrainLoop(R.Session(0), layers, ish, 0.01, batch)
    if warmup:
        wi, wl = _synthetic(4, 1)
        wloop = N.TrainLoop(R.Session(1), layers, ish, 0.01, 4)
        for _ in range(warmup):
            wloop.step(wi, wl)
    t0 = time.perf_counter()
    for _ in range(steps):
        loop.step(imgs, labels)
    dt = time.perf_counter() - t0
    return batch * steps / dt, dt / steps


def run_reference(args, ws, rank):
    if rank != 0:
        return
    steps = max(1, args.steps)
    value, per_step = cpu_steps(CPU_SAMPLE_BATCH, steps, min(args.warmup, 1))
    cores = os.cpu_count()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 ring (int)", "data": "synthetic", "config": _config(args, ws), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"AlexNet-CIFAR private train step at batch {CPU_SAMPLE_BATCH} per step "
                                   f"(numpy/OpenBLAS float-limb restatement of the reference, 3 party threads "
                                   f"for bilinear ops; warm-up at batch 4)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU


class Clocks:
    """SM clock + throttle-reason sampling DURING the timed region: an NVML
    polling thread (2 ms period) so even a sub-second region is sampled; falls
    back to an nvidia-smi subprocess when NVML is unavailable."""

    def __new__(cls, index):
        try:
            import pynvml

            pynvml.nvmlInit()
            return super().__new__(NvmlClocks)
        except Exception:  # noqa: BLE001
            return super().__new__(cls)

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 8 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) > 8:
                for i, nm in enumerate(names):
                    if r[5 + i].strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


class NvmlClocks(Clocks):
    def __init__(self, index):
        import threading

        import pynvml

        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
        self.samples, self.reasons = [], set()
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.stop_ev = threading.Event()
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:  # noqa: BLE001
                pass
            self.stop_ev.wait(0.002)

    def stop(self):
        self.stop_ev.set()
        self.t.join()
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "NVML"}


def run_b200(args, ws, rank, local):
    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import _capi, engine
    from paper_2104_10949_b200.nn import TrainState, one_hot

    b = args.batch
    dev = torch.device("cuda", local)
    # one 3-party session across all ranks (same keys); each rank computes an
    # equal contiguous batch shard; weight-gradient cross terms are summed with
    # NCCL before the replicated reshare/truncation (nn.DataParallel)
    sess = M.TrioSession(seed=0)
    if ws > 1:
        from paper_2104_10949_b200.nn import DataParallel

        sess.dp = DataParallel.nccl()
    model = M.alexnet_cifar()
    cfg = M.TrainConfig(0.01, b * ws, args.warmup + args.steps, seed=0)  # global batch b * ws
    st = TrainState(sess, model, cfg)
    imgs, labels = _synthetic(b, 100 + rank)
    xe, ye = M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10))

    # device-resident dealt batches (dealing outside the timed region)
    batches = [st.deal_batch(xe, ye) for _ in range(args.warmup + args.steps)]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    counter = {"n": 0}
    orig_call = _capi.call

    def counting_call(name, *a):
        if name not in ("mpc3_aes128_expand",):
            counter["n"] += 1
        return orig_call(name, *a)

    # roofline instrumentation: CUDA events around every launch of the
    # dominant kernel (the tcgen05 ring GEMM) and of the fused sign circuit,
    # on their launch stream (torch's current stream)
    gemm_events, sign_events, gemm_bytes, gemm_shapes = [], [], [], []
    instrument = {"on": False, "k": 0}

    def traced_call(name, *a):
        if instrument["on"] and name in ("mpc3_ring_pack", "mpc3_ring_pack_halves", "mpc3_ring_pack_halves_z") \
                and a[3] in (0, 1, 3):
            instrument["k"] = int(a[2]._obj.k)  # logical K of the cross-term operand (inner length 2K)
        if instrument["on"] and name in ("mpc3_rss_sign", "mpc3_rss_layer_sign", "mpc3_ring_gemm_auto",
                                         "mpc3_ring_gemm_auto_z", "mpc3_ring_gemm_t", "mpc3_ring_gemm_t_z"):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            counting_call(name, *a)
            e1.record()
            if name == "mpc3_rss_sign":  # 23 AES blocks per element
                sign_events.append((e0, e1, int(a[9]), 23.0 * int(a[9])))
            elif name == "mpc3_rss_layer_sign":  # + the fused layer epilogue's 2.5 blocks per element
                n_el = 1
                for d in a[7]._obj.full:
                    n_el *= int(d)
                sign_events.append((e0, e1, n_el, 25.5 * n_el))
            elif name.startswith("mpc3_ring_gemm_t"):  # transposed operands: the contraction is an MN operand's rows
                groups, M, N, kc_half = int(a[11]), int(a[12]), int(a[13]), int(a[14])
                # contraction per half: an MN operand's source rows, else the logical K of the
                # operand packed just before (a_mn bit 1 = component-plane A, K-major when bit 0 is 0)
                rows = int(a[2]) if int(a[1]) & 1 else (int(a[7]) if a[6] else (instrument["k"] or kc_half))
                gemm_events.append((e0, e1, 72 * groups * M * N * 2 * rows))
                gemm_bytes.append(groups * ((M + N) * 8 * 2 * kc_half + M * N * 8))
                gemm_shapes.append((name, groups, M, N, 2 * rows))
            else:  # groups x M x N x 2K ring MACs, 72 int8 ops each (36 limb-pair MACs)
                groups, M, N = int(a[3]), int(a[4]), int(a[5])
                sign_k = instrument["k"] if instrument["k"] else int(a[6]) // 2
                kp = int(a[6])
                gemm_events.append((e0, e1, 72 * groups * M * N * 2 * sign_k))
                gemm_bytes.append(groups * ((M + N) * 8 * kp + M * N * 8))  # packed A, B (8 limb planes) + C
                gemm_shapes.append((name, groups, M, N, 2 * sign_k))
            return
        return counting_call(name, *a)

    _capi.call = traced_call
    engine.K.call = traced_call

    for i in range(max(0, args.warmup - 1)):
        st.step(*batches[i])
    # capture one iteration as a CUDA graph (static input buffers)
    xs_static = engine.RssTensor(batches[0][0].data.clone())
    ys_static = engine.RssTensor(batches[0][1].data.clone())
    counter["n"] = 0
    try:
        graph = st.capture(xs_static, ys_static)
    except Exception as e:  # noqa: BLE001 - e.g. a collective that refuses capture: time eagerly
        print(f"[bench] CUDA-graph capture failed ({e!r}); timing eager steps", file=sys.stderr)
        torch.cuda.synchronize()

        class _Eager:
            def replay(self_inner):
                return st.step(xs_static, ys_static)

        graph = _Eager()
    launches_per_step = counter["n"]
    graph.replay()  # last warm-up step, through the graph
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = Clocks(local)
    step_ms = []
    for i in range(args.steps):
        flush.zero_()
        xb, yb = batches[args.warmup + i]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        xs_static.data.copy_(xb.data)
        ys_static.data.copy_(yb.data)
        graph.replay()
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = launches_per_step * args.steps
    # eager instrumented pass (outside the timed region): per-launch CUDA
    # events around the dominant kernel on its launch stream
    # The GPU is first held by a spin kernel long enough for the host to
    # enqueue the whole step, so each launch's events bracket device time
    # only (no host enqueue gaps inside them).
    # Streams are serialised for this pass (no side-stream overlap), so each
    # kernel's events measure it alone.
    from paper_2104_10949_b200 import nn as nn_mod

    saved = (nn_mod.OVERLAP, engine.OVERLAP_PACK)
    nn_mod.OVERLAP, engine.OVERLAP_PACK = False, False
    instrument["on"] = True
    torch.cuda._sleep(int(2e8))  # ~0.1 s of GPU spin
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.step(*batches[-1])
    e1.record()
    torch.cuda.synchronize()
    instrument["on"] = False
    nn_mod.OVERLAP, engine.OVERLAP_PACK = saved
    eager_ms = e0.elapsed_time(e1)
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    value = b * args.steps * ws / (total_ms / 1e3)

    # roofline of the dominant kernel (largest share of the step): the
    # tcgen05 ring GEMM, tensor-bound.  Algorithmic work per launch =
    # 72 int8 ops (36 u8 x u8 limb-pair MACs) per ring MAC x groups * M * N * 2K.
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    traffic = {}
    try:  # one ncu capture of the same step's GEMM launches (tools/traffic.py)
        tj = json.load(open(os.path.join(ROOT, "profiles", "r01_gemm_traffic.json")))
        traffic = {"traffic_bytes_per_launch": tj["traffic_bytes_per_launch"],
                   "source_note": "profiles/r01_gemm_traffic.json: ncu dram__bytes_read.sum + dram__bytes_write.sum, "
                                  f"mean over the {tj['launches']} GEMM launches of one AlexNet step"}
    except (OSError, KeyError, ValueError):
        pass
    gemm_ms = sum(a.elapsed_time(c) for a, c, _ in gemm_events)
    gemm_ops = sum(w for _, _, w in gemm_events)
    nl = max(1, len(gemm_events))
    int8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0 * 0.7225)  # dense int8 = 2x dense bf16 on B200
    achieved = (gemm_ops / nl) / (gemm_ms / nl / 1e3) / 1e12 if gemm_ms else None
    roofline = {"kernel": "gemm_tc_kernel (tcgen05.mma kind::i8, 8 TMEM diagonal accumulators, TMA SWIZZLE_32B)",
                "bound": "tensor", "achieved": achieved, "peak": int8_peak, "unit": "TFLOP/s",
                "frac": (achieved / int8_peak) if achieved else None,
                "traffic": traffic.get("traffic_bytes_per_launch"),
                "traffic_source": traffic.get("source_note"),
                "operand_bytes_per_launch": sum(gemm_bytes) / nl if gemm_bytes else None,
                "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops (dense int8 = 2x dense bf16 on B200; "
                                "cuBLASLt int8 measured 2,924-3,063 TOPS, profiles/r01_microbench_quick.json)"),
                "launches": len(gemm_events), "kernel_ms_per_step": gemm_ms,
                "per_launch": [{"call": nm[len("mpc3_ring_"):], "groups": g_, "M": m_, "N": n_, "K2": k_,
                                "us": round(a.elapsed_time(c) * 1e3, 2),
                                "tops": round(w / (a.elapsed_time(c) / 1e3) / 1e12, 1)}
                               for (a, c, w), (nm, g_, m_, n_, k_) in zip(gemm_events, gemm_shapes)],
                "share_of_step": gemm_ms / max(total_ms / args.steps, 1e-9),
                "algorithmic": "72 int8 ops per ring MAC x groups*M*N*2K per launch (TOPS; TFLOP/s column = int8 TOPS)",
                "measured": "per-launch CUDA events on the launch stream in one eager step after the graph-timed region "
                            "(streams serialised, enqueued behind a GPU spin: the events bracket each kernel alone)"}
    # secondary bound: the nonlinear layers are AES-bound (23 AES-128 blocks
    # per ReLU element); peak = the standalone AES-CTR keystream kernel's rate
    sign_ms = sum(a.elapsed_time(c) for a, c, _, _ in sign_events)
    sign_elems = sum(n for _, _, n, _ in sign_events)
    sign_blocks = sum(bl for _, _, _, bl in sign_events)
    aes_peak = _aes_peak_gblocks()
    aes_rate = sign_blocks / (sign_ms / 1e3) / 1e9 if sign_ms else None
    roofline["secondary"] = {"kernel": "sign circuit (a2b + Kogge-Stone + bit_inject + ReLU, AES-CTR inline; "
                                       "with the layer epilogue fused for large outputs: mpc3_rss_layer_sign)",
                             "bound": "aes", "achieved": aes_rate, "peak": aes_peak, "unit": "G AES blocks/s",
                             "frac": aes_rate / aes_peak if aes_rate and aes_peak else None,
                             "share_of_step": sign_ms / max(total_ms / args.steps, 1e-9),
                             "hbm_gbs": 72.0 * sign_elems / (sign_ms / 1e3) / 1e9 if sign_ms else None,
                             "peak_source": "mpc3_prf_words AES-128-CTR keystream kernel, 2^27 blocks, this run"}

    # end-to-end through the public API with host inputs
    e2e = None
    if not args.no_e2e:
        _capi.call = orig_call
        engine.K.call = orig_call
        # the owner's raw inputs arrive from pinned host memory every step: the
        # float64 images (encoded on the device, ring.py:104-115) and the
        # one-hot labels; the dealer (PCG64, bit-exact with numpy) runs on the
        # device; the step's opened logits (nn.py:746) come back to the host.
        # Double-buffered: step i's host->device copy (own stream) overlaps
        # step i-1's graph; step i's opened logits are read back once its D2H
        # event completes (two steps later at the latest).  Every step copies
        # its own inputs in and its own result out.
        nbuf = 2
        pin_img = [torch.empty(imgs.shape, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
        pin_lab = [torch.empty((b, 10), dtype=torch.float64).pin_memory() for _ in range(nbuf)]
        out_host = [torch.empty((b, 10), dtype=torch.int64).pin_memory() for _ in range(nbuf)]
        dev_img = [torch.empty(imgs.shape, dtype=torch.float64, device=dev) for _ in range(nbuf)]
        dev_lab = [torch.empty((b, 10), dtype=torch.float64, device=dev) for _ in range(nbuf)]
        copy_stream = torch.cuda.Stream(device=dev)
        done = [None] * nbuf
        results = []
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        rng = st.rng
        onehot = one_hot(labels, 10)

        def e2e_step(i):
            k = i % nbuf
            if done[k] is not None:  # slot free: step i-2's logits are on the host
                done[k].synchronize()
                results.append(out_host[k].numpy().view(np.uint64).copy())
            pin_img[k].numpy()[...] = imgs
            pin_lab[k].numpy()[...] = onehot
            with torch.cuda.stream(copy_stream):
                dev_img[k].copy_(pin_img[k], non_blocking=True)
                dev_lab[k].copy_(pin_lab[k], non_blocking=True)
                h2d = torch.cuda.Event()
                h2d.record(copy_stream)
            main = torch.cuda.current_stream()
            main.wait_event(h2d)
            x_enc = sess.fx_encode_device(dev_img[k], bad)
            y_enc = sess.fx_encode_device(dev_lab[k], bad)
            xs_static.data.copy_(sess.share_device(x_enc, rng).data)
            ys_static.data.copy_(sess.share_device(y_enc, rng).data)
            logits = graph.replay()
            out_host[k].copy_(engine.reconstruct_device(logits).view(b, 10), non_blocking=True)
            done[k] = torch.cuda.Event()
            done[k].record(main)

        def drain():
            for k in range(nbuf):
                if done[k] is not None:
                    done[k].synchronize()
                    done[k] = None

        for i in range(2):
            e2e_step(i)
        drain()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        results.clear()
        t0 = time.perf_counter()
        for i in range(args.steps):
            e2e_step(i)
        for k in range(nbuf):  # the last steps' logits
            if done[k] is not None:
                done[k].synchronize()
                results.append(out_host[k].numpy().view(np.uint64).copy())
        dt = time.perf_counter() - t0
        assert len(results) == args.steps
        if ws > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": b * args.steps * ws / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(pin_img[0].numel() * 8 + pin_lab[0].numel() * 8),
               "d2h_bytes_per_step": int(out_host[0].numel() * 8),
               "note": "per step: host images+labels into pinned memory, H2D on a copy stream (double-buffered, "
                       "overlapping the previous step), device fx-encode, device PCG64 dealer (bit-exact with "
                       "sharing.py:113-118), graph step, opened logits D2H read on the host; wall clock"}
        if int(bad.item()):
            raise RuntimeError("input outside the encodable range")

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, _ = cpu_steps(CPU_SAMPLE_BATCH, 1, 0)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
               "sample": f"one AlexNet-CIFAR private train step at batch {CPU_SAMPLE_BATCH} "
                         f"(oracle port of the reference, numpy/OpenBLAS, 3 party threads)"}

    also = {}
    if not args.no_resnet:
        try:
            also["lenet_b64"] = lenet_inference(dev)
            also["vgg16_ti_b32"] = vgg16_ti(dev)
        except Exception as e:  # noqa: BLE001 - reported, not fatal to the headline
            also["side_error"] = repr(e)[:300]
        try:
            also["resnet50_b64"] = resnet50_inference(dev, 64, 2, use_graph=True)
            also["resnet50_b1"] = resnet50_inference(dev, 1, 5, use_graph=True)
        except Exception as e:  # noqa: BLE001 - reported, not fatal to the headline
            also["resnet50_error"] = repr(e)[:300]

    if ws > 1 and not args.no_resnet:
        try:
            tp = resnet50_b1_tp(dev)
        except Exception as e:  # noqa: BLE001
            tp = {"error": repr(e)[:300]}
    if ws > 1 and also:
        # every rank ran the same side workloads as an independent replica:
        # report the aggregate (sum of batches / slowest rank), weak scaling
        for key, rec in also.items():
            for sub in ([rec] + [v for v in rec.values() if isinstance(v, dict)] if isinstance(rec, dict) else []):
                if "ms_per_batch" in sub and "value" in sub:
                    t = torch.tensor([sub["ms_per_batch"]], device=dev, dtype=torch.float64)
                    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                    sub["value"] = sub["value"] * sub["ms_per_batch"] / float(t.item()) * ws
                    sub["ms_per_batch"] = float(t.item())
                    sub["scaling"] = f"weak: {ws} independent replicas, slowest rank"
    if ws > 1 and not args.no_resnet:
        also["resnet50_b1_tensor_parallel"] = tp
    if rank == 0:
        line = {
            "also": also,
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 ring (int)", "data": "synthetic",
            "config": _config(args, ws), "clocks": clk, "gpu_launches": launches, "roofline": roofline,
            "e2e": e2e, "cpu_baseline": cpu,
            "step_ms": [round(v, 3) for v in step_ms],
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _aes_peak_gblocks():
    """Measured rate of the standalone AES-128-CTR keystream kernel (the
    nonlinear protocols' roofline): 2^27 blocks, CUDA events, best of 3."""
    import ctypes as C

    import torch

    from paper_2104_10949_b200 import _capi

    rk = np.zeros((3, 44), np.uint32)
    for i in range(3):
        _capi.check(_capi.lib().mpc3_aes128_expand(C.c_char_p(bytes([i]) * 16), rk[i].ctypes.data_as(C.c_void_p)))
    rkd = torch.from_numpy(rk.view(np.int32)).pin_memory()  # read on the host at launch
    count = 1 << 28
    out = torch.empty(count, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    best = None
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _capi.call("mpc3_prf_words", rkd.data_ptr(), 1, 0, 0, count, out.data_ptr(), st)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return count / 2 / (best / 1e3) / 1e9


def lenet_inference(dev, batch: int = 64, steps: int = 5):
    """LeNet private inference (configs[0]), MNIST shape, device-resident input."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import InferenceGraph

    sess = M.TrioSession(seed=3)
    model = M.lenet()
    rng = np.random.default_rng(3)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=3)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 1, 28, 28))), rng)
    g = InferenceGraph(sess, model, params, x)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / steps
    return {"workload": f"LeNet private inference, MNIST 1x28x28, batch {batch}", "value": batch / (t / 1e3),
            "unit": "images/s", "ms_per_batch": t, "steps": steps, "cuda_graph": True}


def vgg16_ti(dev, batch: int = 32, steps: int = 3):
    """VGG-16 (avg-pool variant) on Tiny-ImageNet shape (configs[2]): private
    inference and one private training step (SGD), batch 32, images/s; both
    captured as CUDA graphs like the headline step."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import engine
    from paper_2104_10949_b200.nn import InferenceGraph, TrainState, one_hot

    sess = M.TrioSession(seed=5)
    model = M.models.vgg16()
    rng = np.random.default_rng(5)
    imgs, labels = rng.uniform(0, 1, (batch, 3, 64, 64)), rng.integers(0, 200, batch)
    st = TrainState(sess, model, M.TrainConfig(0.01, batch, steps + 4, seed=5))
    xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 200)))
    xs = engine.RssTensor(xb[0].data.clone())
    ys = engine.RssTensor(xb[1].data.clone())
    # inference first: its graph packs the weights once (frozen at capture)
    infer_graph = InferenceGraph(sess, model, st.params, xs)
    infer_graph.replay()
    torch.cuda.synchronize()
    res = {}

    def train():
        nonlocal train_graph
        if train_graph is None:
            st.step(*xb)  # warm-up (allocations)
            train_graph = st.capture(xs, ys)
            train_graph.replay()
            torch.cuda.synchronize()
        return train_graph.replay()

    train_graph = None
    for kind, fn in (("inference", infer_graph.replay), ("training_step", train)):
        if kind == "training_step":
            train()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        e1.synchronize()
        t = e0.elapsed_time(e1) / steps
        res[kind] = {"value": batch / (t / 1e3), "unit": "images/s", "ms_per_batch": t}
    res["workload"] = f"VGG-16 (avg-pool) Tiny-ImageNet 3x64x64, 200 classes, batch {batch}, CUDA graphs"
    return res


def resnet50_inference(dev, batch: int, steps: int, use_graph: bool):
    """ResNet-50 private inference (configs[3]), device-resident dealt input,
    CUDA-event timed per batch with an L2 flush before each; images/s."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import InferenceGraph, TrioNet

    sess = M.TrioSession(seed=11)
    model = M.models.resnet50()
    rng = np.random.default_rng(11)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 3, 224, 224))), rng)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    net = TrioNet(sess)
    run = (lambda g=InferenceGraph(sess, model, params, x): g.replay()) if use_graph else \
        (lambda: net.forward(model, params, x, record=False)[0])
    run()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.mean(ms))
    return {"workload": f"ResNet-50 v1.5 private inference, ImageNet 3x224x224, batch {batch}",
            "value": batch / (t / 1e3), "unit": "images/s", "ms_per_batch": t, "steps": steps,
            "cuda_graph": use_graph, "data": "synthetic (random-init folded-BN weights, U(0,1) images)"}


def resnet50_b1_tp(dev, steps: int = 5):
    """ResNet-50 b=1 private inference with output-channel slabs across all
    ranks (nn.TensorParallel, NCCL all-gather between layers); the result is
    bit-identical to the one-GPU run.  Latency, slowest rank."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import TensorParallel, TPNet

    sess = M.TrioSession(seed=11)
    model = M.models.resnet50()
    rng = np.random.default_rng(11)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (1, 3, 224, 224))), rng)
    net = TPNet(sess, TensorParallel.from_process_group())
    net.forward_tp(model, params, x)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        net.forward_tp(model, params, x)
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": "ResNet-50 v1.5 private inference, batch 1, output channels sharded over all ranks "
                        "(NCCL all-gather per layer), eager",
            "value": 1.0 / (ms / 1e3), "unit": "images/s", "latency_ms": ms, "steps": steps}


def main():
    args = _args()
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_b200(args, ws, rank, local)


if __name__ == "__main__":
    main()
