"""The data-parallel bench path as real processes (needs a B200).

`bench.py` under torchrun with 2 ranks: one process per rank, batch shards,
the weight-gradient all-reduce through torch.distributed (gloo here: the
test box has one GPU, which both ranks share; NCCL on a multi-GPU node is
the same code path).  The step-1 weights must equal the REFERENCE's
train_private on the concatenated global batch of 256
(tests/golden/cfg_alexnet_dp.npz), which bench.py checks itself.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_two_rank_data_parallel_bench_matches_reference_digest():
    env = dict(os.environ, MPC3_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--no-side", "--no-cpu-baseline", "--no-e2e"]
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert line["parity"]["status"] == "ok", line["parity"]


def test_two_rank_tensor_parallel_resnet50_b1_matches_reference_shares():
    """nn.TPNet output-channel slabs over 2 processes (all-gather per layer):
    the gathered ResNet-50 b1 logits equal the reference composition's shares."""
    env = dict(os.environ, MPC3_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29534", os.path.join(ROOT, "tools", "tp_check.py")]
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    rec = json.loads(p.stdout.strip().splitlines()[-1])
    assert rec["parity"].startswith("ok"), rec
