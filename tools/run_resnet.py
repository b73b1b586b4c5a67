"""One ResNet-50 private inference pass (bench.resnet50_inference) for launch
lists under ncu:  python tools/run_resnet.py [batch] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    print(bench.resnet50_inference(torch.device("cuda", 0), b, steps, use_graph=False))
