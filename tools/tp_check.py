"""ResNet-50 batch-1 tensor-parallel inference (nn.TPNet) under torchrun:
prints rank 0's bench record, whose `parity` compares the gathered logits
with the reference composition's shares (tests/golden/cfg_resnet50_b1.npz).

MPC3_DIST_BACKEND=gloo python -m torch.distributed.run --nproc-per-node 2 tools/tp_check.py
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    backend = os.environ.get("MPC3_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    rec = bench.resnet50_b1_tp(torch.device("cuda", local), steps=2)
    if dist.get_rank() == 0:
        print(json.dumps(rec), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
