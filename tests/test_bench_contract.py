"""bench.py's JSON-line contract (the driver parses it).

The reference arm runs here on the CPU (the real `mpc3` from baseline/_ref
or /root/reference; batch 4 to stay quick); the B200 arm needs a GPU.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_reference_arm_line():
    import refarm

    if refarm.load()[0] is None:
        pytest.skip("reference package not importable here")
    line = _run(["--impl", "reference", "--steps", "1", "--warmup", "1", "--batch", "4"], 600)
    assert BASE_KEYS <= set(line)
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["per_gpu_batch"] == 4 and line["steps"] == 1


@pytest.mark.gpu
def test_b200_arm_line():
    line = _run(["--steps", "3", "--warmup", "3", "--no-side", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(line) | {"cpu_baseline"}
    assert line["parity"]["status"] == "ok"
    assert line["gpu_launches"] > 0 and line["clocks"]["sm_mhz"]
    r = line["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] <= 1.05
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    assert line["config"]["step"] == "cuda graph replay"
