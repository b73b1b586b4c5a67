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
owner's images and labels H2D from pinned memory, device fx-encoding and
dealing, the step, and the D2H of the opened logits (nn.py:746) inside the
timed region.  `parity`: the first step's opened weights against the REAL
reference's `train_private` on the same batch (SHA-256 digest pinned in
tests/golden/cfg_alexnet_b128.npz); no value is printed on a mismatch.
Multi-GPU (N>1): data parallelism with batch 128 per rank (weak scaling):
batch shards with PRF words drawn at their global offsets, and an NCCL
all-reduce of the weight-gradient cross terms before the replicated
reshare / truncation (nn.DataParallel).

`--impl reference` runs the reference's own CPU implementation (the
unmodified `mpc3` package from baseline/_ref: numpy/OpenBLAS limb GEMMs,
OpenSSL AES, three party threads) through `train_private` at batch 128 on
rank 0 only; see refarm.py.
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
REF_STEPS_CAP = 3  # reference b128 steps take ~25-40 s each on the host: bounded sample
SM_COUNT = 148


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the LeNet / VGG / ResNet-50 side measurements")
    ap.add_argument("--no-graph", action="store_true", help="time eager steps (no CUDA-graph capture)")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _backend() -> str:
    try:
        import torch.distributed as dist

        return dist.get_backend().upper() if dist.is_initialized() else "NCCL"
    except Exception:  # noqa: BLE001 - labelling only
        return "NCCL"


def _config(args, ws):
    return {"workload": "AlexNet-CIFAR private training step (3-party RSS, Z_2^64, t=20)",
            "model": "alexnet_cifar", "global_batch": args.batch * ws, "per_gpu_batch": args.batch,
            "input": "3x32x32", "classes": 10,
            "parallelism": (f"dp{ws} (batch shards, {_backend()} all-reduce of weight-gradient cross terms)"
                            if ws > 1 else "single"),
            "l2": "flushed (256 MiB write) before every timed step, outside its events",
            "inputs": "each step's dealt batch resident in HBM, staged into the graph's static input buffers "
                      "before the L2 flush (outside the events); e2e times the host input path"}


def _synthetic(batch, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, (batch, 3, 32, 32)), rng.integers(0, 10, batch)


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# CPU: the reference's own implementation (refarm.py), or the oracle port


def cpu_alexnet(batch: int, steps: int):
    """(images/s, seconds per step, kind, sample) of the reference's
    AlexNet-CIFAR train_private at `batch`, `steps` iterations in one call,
    after one untimed warm-up iteration at batch 4."""
    import refarm

    imgs, labels = _synthetic(batch, 100)
    mod, src = refarm.load()
    if mod is not None:
        refarm.alexnet_train(4, 1, imgs[:4], labels[:4])  # warm-up: imports, BLAS, code paths
        dt = refarm.alexnet_train(batch, steps, imgs, labels)
        return (batch * steps / dt, dt / steps, "reference",
                f"unmodified reference mpc3 ({os.path.relpath(src, ROOT) if src.startswith(ROOT) else src}): "
                f"run_in_process + nn.train_private(AlexNet-CIFAR, batch {batch}, {steps} iteration(s) in one call, "
                f"incl. weight dealing and the final open, <1%), after 1 untimed warm-up iteration at batch 4")
    # the reference is not importable: the oracle port (oracle/nnmirror.py), same schedule
    from oracle import nnmirror as N
    from oracle import rss as R

    layers, ish = N.alexnet_cifar()
    N.TrainLoop(R.Session(1), layers, ish, 0.01, 4).step(imgs[:4], labels[:4])
    loop = N.TrainLoop(R.Session(0), layers, ish, 0.01, batch)
    t0 = time.perf_counter()
    for _ in range(steps):
        loop.step(imgs, labels)
    dt = time.perf_counter() - t0
    return (batch * steps / dt, dt / steps, "port",
            f"oracle port of the reference (numpy/OpenBLAS float-limb restatement; the reference itself: {src}), "
            f"AlexNet-CIFAR batch {batch}, {steps} step(s), after 1 warm-up step at batch 4")


def run_reference(args, ws, rank):
    if rank != 0:
        return
    import refarm

    steps = max(1, min(args.steps, REF_STEPS_CAP))
    value, per_step, kind, sample = cpu_alexnet(args.batch, steps)
    th = refarm.threads()
    cfg = _config(args, 1)
    cfg["l2"] = "n/a (CPU)"
    cfg["parallelism"] = "3 party threads + OpenBLAS threads on the host"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": 1,
        "requested": {"steps": args.steps, "warmup": args.warmup,
                      "note": f"steps capped at {REF_STEPS_CAP} (each is a full batch-{args.batch} reference step); "
                              f"warm-up = 1 iteration at batch 4"},
        "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64 ring (int)", "data": "synthetic", "config": cfg, "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th["cores"], "kind": kind, "sample": sample,
                         "threads": th},
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


# -- per-launch instrumentation (outside every timed region) ------------------

GEMM_CALLS = ("mpc3_ring_gemm_auto", "mpc3_ring_gemm_auto_z", "mpc3_ring_gemm_t", "mpc3_ring_gemm_t_z")
SIGN_CALLS = ("mpc3_rss_sign", "mpc3_rss_layer_sign", "mpc3_rss_layer_sign_residual", "mpc3_rss_max_tree",
              "mpc3_rss_max_level")
PACK_CALLS = ("mpc3_ring_pack", "mpc3_ring_pack_halves", "mpc3_ring_pack_halves_z", "mpc3_rss_window_gather")


def _category(name: str) -> str:
    if name in GEMM_CALLS:
        return "gemm"
    if name in SIGN_CALLS:
        return "sign"
    if name in PACK_CALLS:
        return "pack"
    if name.startswith("mpc3_ring_"):
        return "local"
    return "protocol"


def _view_numel(view) -> int:
    n = 1
    for d in view._obj.full:
        n *= int(d)
    return n


class Recorder:
    """Wraps the C-ABI entry so that, while `on`, every launch is bracketed
    by CUDA events on its launch stream (torch's current stream: the
    instrumented pass runs with streams serialised) and its algorithmic work
    is recorded: ring-GEMM int8 ops (72 per ring MAC x groups*M*N*2K) and
    sign-circuit AES blocks (23 per ReLU element, 25.5 with a fused layer
    epilogue; max_tree: 23 per pair compared).  While not `on`, it only
    counts launches (gpu_launches)."""

    def __init__(self, capi, engine):
        self.capi, self.engine = capi, engine
        self.orig = capi.call
        self.on = False
        self.count = 0
        self.k = 0
        self.events = []  # (name, category, e0, e1, work, shape)
        self.ms = None  # per-event durations chosen by _instrumented (None: read the events)
        capi.call = self.call
        engine.K.call = self.call

    def restore(self):
        self.capi.call = self.orig
        self.engine.K.call = self.orig

    def call(self, name, *a):
        if name != "mpc3_aes128_expand":
            self.count += 1
        if not self.on:
            return self.orig(name, *a)
        import torch

        if name in ("mpc3_ring_pack", "mpc3_ring_pack_halves", "mpc3_ring_pack_halves_z") and a[3] in (0, 1, 3):
            self.k = int(a[2]._obj.k)  # logical K of the cross-term operand (inner length 2K)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        self.orig(name, *a)
        e1.record()
        work, shape = self._work(name, a)
        self.events.append((name, _category(name), e0, e1, work, shape))

    def _work(self, name, a):
        if name == "mpc3_rss_sign":
            return 23.0 * int(a[9]), (int(a[9]),)
        if name in ("mpc3_rss_layer_sign", "mpc3_rss_layer_sign_residual"):
            n = _view_numel(a[7])
            return 25.5 * n, (n,)
        if name == "mpc3_rss_max_level":
            n = int(a[7]) * (int(a[8]) // 2)
            return 23.0 * n, (n,)
        if name == "mpc3_rss_max_tree":
            rows, m, pairs = int(a[9]), int(a[10]), 0
            while m > 1:
                pairs += rows * (m // 2)
                m = m // 2 + m % 2
            return 23.0 * pairs, (pairs,)
        if name.startswith("mpc3_ring_gemm_t"):
            groups, M, N, kc_half = int(a[11]), int(a[12]), int(a[13]), int(a[14])
            rows = int(a[2]) if int(a[1]) & 1 else (int(a[7]) if a[6] else (self.k or kc_half))
            return 72.0 * groups * M * N * 2 * rows, (groups, M, N, 2 * rows)
        if name.startswith("mpc3_ring_gemm_auto"):
            groups, M, N = int(a[3]), int(a[4]), int(a[5])
            k = self.k if self.k else int(a[6]) // 2
            return 72.0 * groups * M * N * 2 * k, (groups, M, N, 2 * k)
        return 0.0, ()

    def summary(self, step_ms: float) -> dict:
        """Per-category kernel time of the instrumented pass and its share."""
        cats = {}
        for i, (name, cat, e0, e1, work, shape) in enumerate(self.events):
            ms = self.ms[i] if self.ms is not None else e0.elapsed_time(e1)
            c = cats.setdefault(cat, {"ms": 0.0, "launches": 0, "work": 0.0})
            c["ms"] += ms
            c["launches"] += 1
            c["work"] += work
        total = sum(c["ms"] for c in cats.values())
        for c in cats.values():
            c["share_of_kernel_time"] = c["ms"] / total if total else None
            c["share_of_step"] = c["ms"] / step_ms if step_ms else None
        return {"categories": cats, "kernel_ms": total}

    def per_launch(self, cat: str, top: int = 5):
        rows = []
        for i, (name, c, e0, e1, work, shape) in enumerate(self.events):
            if c != cat:
                continue
            us = (self.ms[i] if self.ms is not None else e0.elapsed_time(e1)) * 1e3
            rows.append({"call": name[len("mpc3_"):], "shape": list(shape), "us": round(us, 2),
                         "rate": round(work / (us / 1e6) / (1e12 if cat == "gemm" else 1e9), 2) if us else None})
        rows.sort(key=lambda r: -r["us"])
        return rows[:top]


def lsu_aes_peak(sm_mhz: float) -> float:
    """Hardware ceiling of T-table AES-128 on B200 (G blocks/s): each block
    is 160 table lookups (16 per round x 10); the shared-memory pipe serves
    one conflict-free 32-lane LDS per SM per clock (the tables are laid out
    so lane l always hits bank l) = 32 lookups / clk / SM."""
    return SM_COUNT * sm_mhz * 1e6 * 32 / 160 / 1e9


def roofline_of(rec: Recorder, summ: dict, peaks: dict, sm_mhz: float, traffic: dict) -> dict:
    """The roofline object for the dominant kernel class by share of the
    instrumented pass's kernel time (ring GEMM vs sign circuit), the other
    as `secondary`."""
    cats = summ["categories"]
    # dense int8 = 2x dense bf16 on B200; without MEASURED_PEAKS.json the
    # profiling guide's fallback (1.59 PFLOP/s bf16, burst)
    measured = "bf16_tflops" in peaks
    int8_peak = 2.0 * (peaks["bf16_tflops"] if measured else 1590.0)
    out = {}
    g = cats.get("gemm")
    if g and g["ms"]:
        per = g["work"] / g["launches"] / (g["ms"] / g["launches"] / 1e3) / 1e12
        out["gemm"] = {
            "kernel": "gemm_tc_kernel (tcgen05.mma kind::i8, 8 TMEM diagonal accumulators, TMA)",
            "bound": "tensor", "achieved": per, "peak": int8_peak, "unit": "TFLOP/s", "frac": per / int8_peak,
            "traffic": traffic.get("gemm"), "launches": g["launches"], "kernel_ms_per_step": g["ms"],
            "share_of_kernel_time": g["share_of_kernel_time"], "share_of_step": g["share_of_step"],
            "algorithmic": "72 int8 ops per ring MAC x groups*M*N*2K per launch (TFLOP/s = int8 TOPS)",
            "peak_source": ("2 x MEASURED_PEAKS.json bf16_tflops (of measured)" if measured else
                            "2 x 1.59 PFLOP/s bf16, B200_PROFILING.md fallback: MEASURED_PEAKS.json absent (of fallback)")
                           + "; dense int8 = 2 x dense bf16 on B200",
            "top_launches": rec.per_launch("gemm"),
        }
    s = cats.get("sign")
    if s and s["ms"]:
        rate = s["work"] / (s["ms"] / 1e3) / 1e9
        peak = lsu_aes_peak(sm_mhz)
        out["sign"] = {
            "kernel": "sign circuit (a2b + Kogge-Stone + bit_inject + ReLU mask, AES-128-CTR inline; "
                      "mpc3_rss_sign / mpc3_rss_layer_sign / max_tree)",
            "bound": "aes (shared-memory LSU pipe: 160 T-table lookups per AES block)", "achieved": rate,
            "peak": peak, "unit": "G AES blocks/s", "frac": rate / peak, "traffic": traffic.get("sign"),
            "launches": s["launches"], "kernel_ms_per_step": s["ms"],
            "share_of_kernel_time": s["share_of_kernel_time"], "share_of_step": s["share_of_step"],
            "algorithmic": "23 AES blocks per ReLU element (25.5 with the fused layer reshare + truncation); "
                           "HBM traffic is 48-72 B per element (not the bound)",
            "peak_source": f"{SM_COUNT} SMs x {sm_mhz:.0f} MHz x 32 lookups/clk / 160 lookups per block",
            "top_launches": rec.per_launch("sign"),
        }
    if not out:
        return {}
    dom = max(out, key=lambda k: out[k]["share_of_kernel_time"] or 0)
    r = dict(out[dom])
    r["dominant_by"] = "largest share of the instrumented step's kernel time"
    r["measured"] = ("per-launch CUDA events on the launch stream in one eager pass after the timed region "
                     "(streams serialised, enqueued behind a GPU spin so the events bracket each kernel alone)")
    r["kernel_time_by_category"] = {k: {"ms": round(v["ms"], 4), "share": round(v["share_of_kernel_time"], 4),
                                        "launches": v["launches"]} for k, v in summ["categories"].items()}
    others = [k for k in out if k != dom]
    if others:
        r["secondary"] = out[others[0]]
    return r


def _traffic(workload: str = "alexnet"):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch from the
    committed profiles (tools/traffic.py: one ncu pass over one step of the
    workload), keyed by kernel class."""
    t = {}
    files = (("gemm", "r02_traffic_gemm.json"), ("sign", "r02_traffic_sign.json"), ("gemm", "r01_gemm_traffic.json"))
    if workload == "resnet50_b64":
        files = (("sign", "r02_traffic_r50_sign.json"),)
    for cls, fn in files:
        if cls in t:
            continue
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", fn)))
            t[cls] = tj["traffic_bytes_per_launch"]
        except (OSError, KeyError, ValueError):
            pass
    return t


def _instrumented(fn, rec, torch, passes: int = 2):
    """Eager passes of fn with per-launch events, streams serialised; each
    launch keeps its shortest time over the passes (a host stall while the
    pass is enqueued behind the GPU spin would otherwise stretch one
    launch's events)."""
    from paper_2104_10949_b200 import engine
    from paper_2104_10949_b200 import nn as nn_mod

    saved = (nn_mod.OVERLAP, engine.OVERLAP_PACK)
    nn_mod.OVERLAP, engine.OVERLAP_PACK = False, False
    runs = []
    try:
        for _ in range(passes):
            rec.events.clear()
            rec.on = True
            torch.cuda._sleep(int(2e8))  # ~0.1 s of GPU spin: the host enqueues the whole pass behind it
            fn()
            torch.cuda.synchronize()
            rec.on = False
            runs.append([(ev, ev[2].elapsed_time(ev[3])) for ev in rec.events])
    finally:
        rec.on = False
        nn_mod.OVERLAP, engine.OVERLAP_PACK = saved
    if len(runs) > 1 and all(len(r) == len(runs[0]) for r in runs):
        rec.events = [r[0] for r in runs[0]]
        rec.ms = [min(r[i][1] for r in runs) for i in range(len(runs[0]))]
    else:
        rec.events = [r[0] for r in runs[-1]]
        rec.ms = [r[1] for r in runs[-1]]


def run_b200(args, ws, rank, local):
    import torch

    # one GPU per rank; more ranks than devices (a functional multi-rank run
    # on a one-GPU box, MPC3_DIST_BACKEND=gloo) share them round-robin
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        backend = os.environ.get("MPC3_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import _capi, engine
    from paper_2104_10949_b200.nn import TrainState, one_hot

    b = args.batch
    dev = torch.device("cuda", local)
    # one 3-party session across all ranks (same keys); each rank computes an
    # equal contiguous batch shard; weight-gradient cross terms are summed with
    # NCCL before the replicated reshare/truncation (nn.DataParallel)
    sess = M.TrioSession(seed=0)
    comm = None
    if ws > 1:
        from paper_2104_10949_b200.nn import DataParallel

        sess.dp = DataParallel.nccl()
        comm = {"backend": torch.distributed.get_backend(), "world_size": torch.distributed.get_world_size(),
                "devices": torch.cuda.device_count(),
                "collective": "all_reduce(sum, int64) of weight-gradient cross terms"}
    model = M.alexnet_cifar()
    cfg = M.TrainConfig(0.01, b * ws, args.warmup + args.steps, seed=0)  # global batch b * ws
    st = TrainState(sess, model, cfg)
    # rank r's shard of the global batch; at N=1 exactly the fixture's batch (default_rng(100))
    imgs, labels = _synthetic(b, 100 + rank)
    xe, ye = M.fx_encode(imgs), M.fx_encode(one_hot(labels, 10))

    # device-resident dealt batches (dealing outside the timed region)
    batches = [st.deal_batch(xe, ye) for _ in range(args.warmup + args.steps)]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    rec = Recorder(_capi, engine)

    # parity: the first step (eager) from the dealt initial weights is the
    # reference's train_private iteration 0 on the same batch
    parity = {"status": "not checked"}

    def check_parity():
        # N = 1: the reference's train_private on this batch; N > 1: on the
        # concatenation of the ranks' batches (global batch 128 N)
        if b != BATCH:
            parity["status"] = "not checked (no fixture for this batch)"
            return
        import hashlib

        fixture, key = ("cfg_alexnet_b128.npz", "digest_1") if ws == 1 else ("cfg_alexnet_dp.npz", f"digest_dp{ws}")
        try:
            z = np.load(os.path.join(ROOT, "tests", "golden", fixture))
            fmeta = json.loads(bytes(z["meta"]).decode())
            want = fmeta[key]
        except (OSError, KeyError, ValueError):
            parity["status"] = f"not checked (no fixture for global batch {b * ws})"
            return
        got = hashlib.sha256(b"".join(np.ascontiguousarray(sess.reveal(p), "<u8").tobytes()
                                      for p in st.params)).hexdigest()
        source = fmeta.get(f"{key}_source", "the reference's train_private")
        parity.update({"status": "ok" if got == want else "MISMATCH", "digest": got[:16],
                       "against": f"SHA-256 of the opened weights after step 1 vs {source} at "
                                  f"global batch {b * ws} (tests/golden/{fixture}, make_golden_configs.py)"})

    # a CUDA-graph replay needs the previous replay's counters: eager warm-up
    # steps first (the first one checked), then one graph capture
    n_eager = max(1, args.warmup - 1)
    for i in range(n_eager):
        st.step(*batches[i])
        if i == 0:
            check_parity()
    if parity["status"] == "MISMATCH":
        raise SystemExit(f"[bench] parity check failed: {parity}")
    xs_static = engine.RssTensor(batches[0][0].data.clone())
    ys_static = engine.RssTensor(batches[0][1].data.clone())
    rec.count = 0

    class _Eager:
        def replay(self_inner):
            return st.step(xs_static, ys_static)

    # gloo collectives synchronise with the host and cannot be captured
    if args.no_graph or (ws > 1 and torch.distributed.get_backend() != "nccl"):
        graph = _Eager()
        st.step(xs_static, ys_static)  # counts this step's launches (rec.count)
    else:
        try:
            graph = st.capture(xs_static, ys_static)
        except Exception as e:  # noqa: BLE001 - e.g. a collective that refuses capture: time eagerly
            print(f"[bench] CUDA-graph capture failed ({e!r}); timing eager steps", file=sys.stderr)
            torch.cuda.synchronize()
            graph = _Eager()
    launches_per_step = rec.count
    graph.replay()  # last warm-up step, through the graph
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = Clocks(local)
    switch = sys.getswitchinterval()
    sys.setswitchinterval(1e-4)  # the clock sampler thread runs during the short timed region
    step_ms = []
    for i in range(args.steps):
        xb, yb = batches[min(n_eager + i, len(batches) - 1)]
        # the step's dealt batch, resident in HBM, staged into the graph's
        # static inputs before the timed region (e2e times the whole input path)
        xs_static.data.copy_(xb.data)
        ys_static.data.copy_(yb.data)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    clk = clocks.stop()
    sys.setswitchinterval(switch)
    launches = launches_per_step * args.steps
    total_ms = float(sum(step_ms))
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    value = b * args.steps * ws / (total_ms / 1e3)

    # roofline: one eager instrumented step after the timed region
    peaks = _peaks()
    sm_mhz = float(clk.get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0)
    _instrumented(lambda: st.step(*batches[-1]), rec, torch)
    summ = rec.summary(total_ms / args.steps)
    roofline = roofline_of(rec, summ, peaks, sm_mhz, _traffic())
    rec.events.clear()
    rec.ms = None

    # end-to-end through the public API with host inputs
    e2e = None if args.no_e2e else _e2e(args, ws, dev, sess, st, graph, xs_static, ys_static, imgs, labels, b)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import refarm

        v, per, kind, sample = cpu_alexnet(b, 1)
        cpu = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": kind, "sample": sample,
               "threads": refarm.threads()}

    also = {}
    if not args.no_side:
        also = side_measurements(dev, ws, rank, rec, peaks, sm_mhz, args)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64 ring (int)", "data": "synthetic",
            "config": dict(_config(args, ws), step="eager" if isinstance(graph, _Eager) else "cuda graph replay"),
            "parity": parity, "clocks": clk, "gpu_launches": launches,
            "e2e": e2e, "cpu_baseline": cpu, "comm": comm, "roofline": roofline,
            "step_ms": [round(v, 3) for v in step_ms],
            "also": also,
        }
        print(json.dumps(line), flush=True)
    rec.restore()
    if ws > 1:
        torch.distributed.destroy_process_group()


def _e2e(args, ws, dev, sess, st, graph, xs_static, ys_static, imgs, labels, b):
    """The owner's raw inputs arrive from pinned host memory every step: the
    float64 images (encoded on the device, ring.py:104-115) and the one-hot
    labels; the dealer (PCG64, bit-exact with numpy) runs on the device; the
    step's opened logits (nn.py:746) come back to the host.  Double-buffered:
    two captures of the step (graph k reads static inputs k), so step i's
    host->device copy, encode and deal (into graph i % 2's inputs, on an
    input stream) overlap step i-1's replay, and step i's logits are opened
    and read back on an output stream (the host collects them two steps
    later at the latest).  Every step copies its own inputs in and its own
    result out."""
    import torch

    from paper_2104_10949_b200 import engine
    from paper_2104_10949_b200.nn import one_hot

    nbuf = 2
    pin_img = [torch.empty(imgs.shape, dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    pin_lab = [torch.empty((b, 10), dtype=torch.float64).pin_memory() for _ in range(nbuf)]
    out_host = [torch.empty((b, 10), dtype=torch.int64).pin_memory() for _ in range(nbuf)]
    dev_img = [torch.empty(imgs.shape, dtype=torch.float64, device=dev) for _ in range(nbuf)]
    dev_lab = [torch.empty((b, 10), dtype=torch.float64, device=dev) for _ in range(nbuf)]
    in_stream, out_stream = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    done = [None] * nbuf
    results = []
    bad = torch.zeros(1, dtype=torch.int32, device=dev)
    rng = st.rng
    onehot = one_hot(labels, 10)

    # graph k replays with static inputs k (dealt into directly); an eager
    # step (no graph) or a refused second capture keeps one input buffer and
    # copies each step's dealt shares into it
    graphs, statics = [graph], [(xs_static, ys_static)]
    if hasattr(graph, "xs"):
        try:
            xs2, ys2 = engine.RssTensor(xs_static.data.clone()), engine.RssTensor(ys_static.data.clone())
            graphs.append(st.capture(xs2, ys2))
            statics.append((xs2, ys2))
        except Exception as e:  # noqa: BLE001 - fall back to the copy into one buffer
            print(f"[bench] second e2e capture failed ({e!r}); copying inputs", file=sys.stderr)
            torch.cuda.synchronize()
    double = len(graphs) == nbuf
    held = [None] * nbuf  # single-buffer mode: slot k's dealt shares, alive until the slot comes round again

    def e2e_step(i):
        k = i % nbuf
        if done[k] is not None:  # slot free: step i-2's logits are on the host (its replay has finished)
            done[k].synchronize()
            results.append(out_host[k].numpy().view(np.uint64).copy())
        pin_img[k].numpy()[...] = imgs
        pin_lab[k].numpy()[...] = onehot
        main = torch.cuda.current_stream()
        g = graphs[k if double else 0]
        xs_k, ys_k = statics[k if double else 0]
        # copy in, encode and deal on the input stream, beside the previous
        # step's replay (the dealer's draws are host-ordered: same shares)
        with torch.cuda.stream(in_stream):
            dev_img[k].copy_(pin_img[k], non_blocking=True)
            dev_lab[k].copy_(pin_lab[k], non_blocking=True)
            x_enc = sess.fx_encode_device(dev_img[k], bad)
            y_enc = sess.fx_encode_device(dev_lab[k], bad)
            if double:
                sess.share_device(x_enc, rng, out=xs_k)
                sess.share_device(y_enc, rng, out=ys_k)
            else:
                held[k] = (sess.share_device(x_enc, rng), sess.share_device(y_enc, rng))
            dealt = torch.cuda.Event()
            dealt.record(in_stream)
        main.wait_event(dealt)
        if not double:
            xs_k.data.copy_(held[k][0].data)
            ys_k.data.copy_(held[k][1].data)
        logits = g.replay()
        # open and read back on the output stream
        stepped = torch.cuda.Event()
        stepped.record(main)
        with torch.cuda.stream(out_stream):
            out_stream.wait_event(stepped)
            out_host[k].copy_(engine.reconstruct_device(logits).view(b, 10), non_blocking=True)
            done[k] = torch.cuda.Event()
            done[k].record(out_stream)

    for i in range(2):
        e2e_step(i)
    for k in range(nbuf):
        if done[k] is not None:
            done[k].synchronize()
            done[k] = None
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
    if int(bad.item()):
        raise RuntimeError("input outside the encodable range")
    # the shares the last steps were dealt open to the encoded host inputs
    import paper_2104_10949_b200 as M

    want_x, want_y = M.fx_encode(imgs).reshape(-1), M.fx_encode(onehot).reshape(-1)
    for xs_k, ys_k in statics:
        if not (np.array_equal(engine.to_host(engine.reconstruct_device(xs_k)), want_x)
                and np.array_equal(engine.to_host(engine.reconstruct_device(ys_k)), want_y)):
            raise RuntimeError("e2e: the dealt inputs do not open to the encoded images / labels")
    return {"value": b * args.steps * ws / dt, "unit": UNIT, "inputs_check": "ok (dealt shares open to the inputs)",
            "h2d_bytes_per_step": int(pin_img[0].numel() * 8 + pin_lab[0].numel() * 8),
            "d2h_bytes_per_step": int(out_host[0].numel() * 8),
            "api": "the trio engine API (INTEGRATION.md §2: TrainState + GraphStep) with host-resident inputs; "
                   "the per-party drop-in run_in_process + train_private call is also.dropin_train_private",
            "note": "per step: host images+labels into pinned memory, H2D + device fx-encode + device PCG64 dealer "
                    "(bit-exact with sharing.py:113-118) on an input stream beside the previous step's replay, "
                    + ("straight into the static inputs of one of two captures of the step (alternating), "
                       if double else "into a buffer copied into the graph's static inputs, ")
                    + "graph step, logits opened and copied D2H on an output stream, read on the host; wall clock",
            "graphs": len(graphs)}


# ---------------------------------------------------------------------------
# side measurements (the other BASELINE configs), reported under `also`


def side_measurements(dev, ws, rank, rec, peaks, sm_mhz, args) -> dict:
    import torch

    also = {}
    for key, fn in (("lenet_b64", lambda: lenet_inference(dev)), ("vgg16_ti_b32", lambda: vgg16_ti(dev)),
                    ("resnet50_b64", lambda: resnet50_inference(dev, 64, 3, rec=rec, peaks=peaks, sm_mhz=sm_mhz)),
                    ("resnet50_b1", lambda: resnet50_inference(dev, 1, 10)),
                    ("ring_gemm", lambda: ring_gemm_sweep(dev))):
        try:
            also[key] = fn()
        except Exception as e:  # noqa: BLE001 - reported, not fatal to the headline
            also[key] = {"error": repr(e)[:300]}
    if ws > 1:
        try:
            also["resnet50_b1_tensor_parallel"] = resnet50_b1_tp(dev)
        except Exception as e:  # noqa: BLE001
            also["resnet50_b1_tensor_parallel"] = {"error": repr(e)[:300]}
        # every rank ran the other side workloads as an independent replica:
        # report the aggregate (sum of batches / slowest rank), weak scaling
        for key, rec_ in also.items():
            if key == "resnet50_b1_tensor_parallel" or not isinstance(rec_, dict):
                continue
            for sub in [rec_] + [v for v in rec_.values() if isinstance(v, dict)]:
                if "ms_per_batch" in sub and "value" in sub:
                    t = torch.tensor([sub["ms_per_batch"]], device=dev, dtype=torch.float64)
                    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                    sub["value"] = sub["value"] * sub["ms_per_batch"] / float(t.item()) * ws
                    sub["ms_per_batch"] = float(t.item())
                    sub["scaling"] = f"weak: {ws} independent replicas, slowest rank"
    if rank == 0 and ws == 1:
        try:
            also["dropin_train_private"] = dropin_train_private()
        except Exception as e:  # noqa: BLE001
            also["dropin_train_private"] = {"error": repr(e)[:300]}
        if not args.no_cpu_baseline:
            _side_cpu_baselines(also)
    return also


def ring_gemm_sweep(dev, sizes=(1024, 2048, 4096)) -> dict:
    """The ring GEMM (BASELINE.json's "ring-GEMM TOPS", configs[4]) at M = N = K
    = n on random packed limb planes in the engine's layout (A read MN-major
    from a transposed pack, B K-major: mpc3_ring_gemm_t), L2 flushed before
    each timed launch; 72 int8 ops per ring MAC; cuBLASLt int8
    (torch._int_mm) at the largest n for context."""
    import torch

    from paper_2104_10949_b200 import _capi

    st = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def timed(fn, iters):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return float(np.median(ts))

    out = {"layout": "A MN-major (transposed pack, SWIZZLE_128B), B K-major; L2 flushed per launch", "sizes": []}
    for n in sizes:
        kc = n // 2
        at = torch.randint(0, 256, (8 * kc * 2 * n,), dtype=torch.uint8, device=dev)
        b = torch.randint(0, 256, (8 * n * n,), dtype=torch.uint8, device=dev)
        c = torch.empty(n * n, dtype=torch.int64, device=dev)
        s = timed(lambda: _capi.call("mpc3_ring_gemm_t", at.data_ptr(), 1, kc, 2 * n, n, b.data_ptr(), 0, n, n, 0,
                                     c.data_ptr(), 1, n, n, kc, 0, st), 5)
        out["sizes"].append({"n": n, "ms": s * 1e3, "int8_tops": 72 * n ** 3 / s / 1e12, "ring_tops": 2 * n ** 3 / s / 1e12})
        del at, b, c
    n = sizes[-1]
    try:
        a8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        b8 = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t().contiguous().t()
        s = timed(lambda: torch._int_mm(a8, b8), 5)
        out["cublaslt_int8"] = {"n": n, "tops": 2 * n ** 3 / s / 1e12}
    except Exception as e:  # noqa: BLE001
        out["cublaslt_int8"] = {"error": repr(e)[:200]}
    return out


def _side_cpu_baselines(also):
    """The reference's CPU path for the side configs (refarm.py): LeNet b64
    infer_private; ResNet-50 b1 composed from its per-party protocols (b64
    extrapolated linearly from b1, labelled)."""
    import refarm

    mod, src = refarm.load()
    if mod is None:
        return
    th = refarm.threads()
    try:
        t = refarm.lenet_infer(64)
        also["lenet_b64"]["cpu_baseline"] = {"value": 64 / t, "unit": UNIT, "cores": th["cores"], "kind": "reference",
                                             "sample": "mpc3 infer_private, LeNet batch 64, one pass"}
    except Exception as e:  # noqa: BLE001
        also["lenet_b64"]["cpu_baseline"] = {"error": repr(e)[:200]}
    try:
        t = refarm.resnet50_composed(1)
        base = {"unit": UNIT, "cores": th["cores"], "kind": "reference",
                "sample": "ResNet-50 224x224 batch 1 COMPOSED from mpc3 conv2d_shares + local bias, relu, padded "
                          "avgpool_shares, matmul_shares + bias, residual adds (the reference graph has no "
                          "ResNet layers); one forward pass"}
        also["resnet50_b1"]["cpu_baseline"] = dict(base, value=1 / t, seconds=t)
        also["resnet50_b64"]["cpu_baseline"] = dict(base, value=1 / t, seconds_per_image=t,
                                                    note="extrapolated: b1 per-image time x 64 (linear in batch)")
    except Exception as e:  # noqa: BLE001
        also["resnet50_b1"]["cpu_baseline"] = {"error": repr(e)[:200]}
    if isinstance(also.get("ring_gemm"), dict) and "sizes" in also["ring_gemm"]:
        try:  # the reference's bilinear_exact (ring.py:183-222) at n = 2048 (tests/test_ring.py inputs)
            from mpc3.ring import bilinear_exact, matmul_spec

            n = 2048
            rng = np.random.default_rng(n)
            a = rng.integers(0, 1 << 64, (n, n), dtype=np.uint64)
            b = rng.integers(0, 1 << 64, (n, n), dtype=np.uint64)
            bilinear_exact(a[:64, :64], b[:64, :64], matmul_spec(64, 64, 64))
            t0 = time.perf_counter()
            bilinear_exact(a, b, matmul_spec(n, n, n))
            dt = time.perf_counter() - t0
            also["ring_gemm"]["cpu_baseline"] = {"value": 2 * n ** 3 / dt / 1e12, "unit": "ring-TOPS (2 ops per ring MAC)",
                                                 "cores": th["cores"], "kind": "reference",
                                                 "sample": f"mpc3.ring.bilinear_exact, M = N = K = {n}, one call"}
        except Exception as e:  # noqa: BLE001
            also["ring_gemm"]["cpu_baseline"] = {"error": repr(e)[:200]}


def lenet_inference(dev, batch: int = 64, steps: int = 5):
    """LeNet private inference (configs[0]), MNIST shape, device-resident
    input; the inputs are exactly tests/golden/cfg_lenet_b64.npz's and the
    first replay's logit shares are checked against the reference's."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import InferenceGraph

    sess = M.TrioSession(seed=3)
    model = M.lenet()
    rng = np.random.default_rng(3)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=3)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 1, 28, 28))), rng)
    g = InferenceGraph(sess, model, params, x)
    first = g.replay().data.cpu().numpy().view(np.uint64)
    parity = _fixture_check("lenet_b64", first) if batch == 64 else "not checked"
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / steps
    return {"workload": f"LeNet private inference, MNIST 1x28x28, batch {batch}", "value": batch / (t / 1e3),
            "unit": "images/s", "ms_per_batch": t, "steps": steps, "cuda_graph": True, "parity": parity}


def _fixture_check(name, got) -> str:
    try:
        z = np.load(os.path.join(ROOT, "tests", "golden", f"cfg_{name}.npz"))
    except OSError:
        return "not checked (fixture missing)"
    return "ok (shares == reference)" if np.array_equal(got, z["logits"]) else "MISMATCH"


def vgg16_ti(dev, batch: int = 32, steps: int = 3):
    """VGG-16 (avg-pool variant) on Tiny-ImageNet shape (configs[2]): private
    inference (inputs of tests/golden/cfg_vgg16ti_b32.npz, first replay
    checked) and one private training step (SGD), batch 32, images/s; both
    captured as CUDA graphs like the headline step."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import engine
    from paper_2104_10949_b200.nn import InferenceGraph, TrainState, one_hot

    model = M.models.vgg16()
    sess = M.TrioSession(seed=5)
    rng = np.random.default_rng(5)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=5)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 3, 64, 64))), rng)
    infer_graph = InferenceGraph(sess, model, params, x)
    parity = _fixture_check("vgg16ti_b32", infer_graph.replay().data.cpu().numpy().view(np.uint64)) \
        if batch == 32 else "not checked"
    res = {"inference": None, "training_step": None, "parity_inference": parity}

    tsess = M.TrioSession(seed=5)
    trng = np.random.default_rng(5)
    imgs, labels = trng.uniform(0, 1, (batch, 3, 64, 64)), trng.integers(0, 200, batch)
    st = TrainState(tsess, model, M.TrainConfig(0.01, batch, steps + 4, seed=5))
    xb = st.deal_batch(M.fx_encode(imgs), M.fx_encode(one_hot(labels, 200)))
    xs = engine.RssTensor(xb[0].data.clone())
    ys = engine.RssTensor(xb[1].data.clone())
    st.step(*xb)  # warm-up (allocations)
    train_graph = st.capture(xs, ys)
    train_graph.replay()
    torch.cuda.synchronize()
    for kind, fn in (("inference", infer_graph.replay), ("training_step", train_graph.replay)):
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


def resnet50_inference(dev, batch: int, steps: int, rec=None, peaks=None, sm_mhz=1965.0):
    """ResNet-50 private inference (configs[3]), device-resident dealt input,
    CUDA-graph replays, CUDA-event timed per batch with an L2 flush before
    each; images/s.  At batch 1 the inputs are tests/golden/cfg_resnet50_b1's
    and the first replay is checked against the reference composition.  With
    `rec`, one instrumented eager pass gives the roofline of its dominant
    kernel (the sign circuit, AES-bound)."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import InferenceGraph, TrioNet

    sess = M.TrioSession(seed=11)
    model = M.models.resnet50()
    rng = np.random.default_rng(11)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (batch, 3, 224, 224))), rng)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    g = InferenceGraph(sess, model, params, x)
    first = g.replay().data.cpu().numpy().view(np.uint64)
    parity = _fixture_check(f"resnet50_b{batch}", first) if batch in (1, 64) else "not checked (no fixture)"
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = float(np.mean(ms))
    out = {"workload": f"ResNet-50 v1.5 private inference, ImageNet 3x224x224, batch {batch}",
           "value": batch / (t / 1e3), "unit": "images/s", "ms_per_batch": t, "steps": steps,
           "cuda_graph": True, "parity": parity,
           "data": "synthetic (random-init folded-BN weights, U(0,1) images)"}
    if rec is not None:
        net = TrioNet(sess)
        _instrumented(lambda: net.forward(model, params, x, record=False), rec, torch)
        summ = rec.summary(t)
        rf = roofline_of(rec, summ, peaks or {}, sm_mhz, _traffic("resnet50_b64" if batch == 64 else ""))
        # compact (the whole line must survive the driver's stdout tail): the
        # headline's roofline carries the long-form fields
        keep = ("kernel", "bound", "achieved", "peak", "unit", "frac", "traffic", "launches", "share_of_step",
                "kernel_time_by_category")
        out["roofline"] = {k: rf[k] for k in keep if k in rf}
        out["roofline"]["top_launches"] = rf.get("top_launches", [])[:3]
        if "secondary" in rf:
            out["roofline"]["secondary"] = {k: rf["secondary"][k] for k in ("kernel", "achieved", "unit", "frac")
                                            if k in rf["secondary"]}
        rec.events.clear()
        rec.ms = None
    return out


def resnet50_b1_tp(dev, steps: int = 5):
    """ResNet-50 b=1 private inference with output-channel slabs across all
    ranks (nn.TensorParallel, NCCL all-gather between layers); the result is
    bit-identical to the one-GPU run.  Captured as a CUDA graph with its
    all-gathers (nn.InferenceGraph; eager if the capture is refused).
    Latency, slowest rank."""
    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200.nn import InferenceGraph, TensorParallel, TPNet

    sess = M.TrioSession(seed=11)
    model = M.models.resnet50()
    rng = np.random.default_rng(11)
    params = [sess.share(w, rng) for w in M.init_params(model, seed=11)]
    x = sess.share(M.fx_encode(rng.uniform(0, 1, (1, 3, 224, 224))), rng)
    tp = TensorParallel.from_process_group()
    net = TPNet(sess, tp)
    mode = "CUDA graph"

    def run():
        return net.forward_tp(model, params, x)

    if torch.distributed.get_backend() == "nccl":  # gloo collectives synchronise with the host: no capture
        try:
            run = InferenceGraph(sess, model, params, x,
                                 forward=lambda s, m, p, xx: TPNet(s, tp).forward_tp(m, p, xx)).replay
        except Exception as e:  # noqa: BLE001 - a collective that refuses capture: time eager passes
            print(f"[bench] TP graph capture failed ({e!r}); timing eager passes", file=sys.stderr)
            torch.cuda.synchronize()
            mode = "eager"
    else:
        mode = "eager"
    first = run().data.cpu().numpy().view(np.uint64)
    parity = _fixture_check("resnet50_b1", first)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    return {"workload": "ResNet-50 v1.5 private inference, batch 1, output channels sharded over all ranks "
                        f"({torch.distributed.get_backend()} all-gather per layer), {mode}",
            "value": 1.0 / (ms / 1e3), "unit": "images/s", "latency_ms": ms, "steps": steps, "parity": parity}


def dropin_train_private(batch: int = BATCH, iterations: int = 16):
    """The per-party drop-in path a reference user calls: run_in_process +
    train_private (three party threads rendezvousing on the trio engine),
    host data in, opened weights out; wall clock of the whole call.  A
    2-iteration call is checked against the reference's digest first."""
    import hashlib

    import torch

    import paper_2104_10949_b200 as M
    from paper_2104_10949_b200 import nn as nn_mod

    imgs, labels = _synthetic(batch, 100)

    def run(iters):
        cfg = M.TrainConfig(0.01, batch, iters, 0)
        job = (lambda ctx: M.train_private(ctx, M.alexnet_cifar(), cfg, (imgs, labels) if ctx.party == 0 else None))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = M.run_in_process(job, seed=0)
        torch.cuda.synchronize()
        return res, time.perf_counter() - t0

    res, _ = run(2)  # also the warm-up
    try:
        z = np.load(os.path.join(ROOT, "tests", "golden", "cfg_alexnet_b128.npz"))
        want = json.loads(bytes(z["meta"]).decode())["digest_2"] if batch == BATCH else None
    except (OSError, KeyError, ValueError):
        want = None
    got = hashlib.sha256(b"".join(np.ascontiguousarray(w, "<u8").tobytes() for w in res[0].weights)).hexdigest()
    _, dt = run(iterations)
    return {"workload": f"per-party run_in_process + train_private, AlexNet-CIFAR batch {batch}, "
                        f"{iterations} iterations (setup, weight dealing, per-iteration H2D + device dealing, "
                        f"eager steps (a CUDA graph from {nn_mod.GRAPH_MIN_STEPS} remaining iterations on), "
                        f"opened logits every iteration, opened weights)",
            "value": batch * iterations / dt, "unit": UNIT, "seconds": dt,
            "parity": "not checked" if want is None else ("ok (2-iteration weights digest == reference)"
                                                          if got == want else "MISMATCH")}


def main():
    args = _args()
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_b200(args, ws, rank, local)


if __name__ == "__main__":
    main()
