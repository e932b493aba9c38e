"""Run only the C5 K3 distance measurement of bench.py (profiling driver)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("FNB_AB_ROOT"):  # A/B: a package copy with another library build
    sys.path.insert(0, os.environ["FNB_AB_ROOT"])
import bench  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(json.dumps(bench.c5_distance(dev, torch.cuda.current_stream(), flush, reps=int(sys.argv[1]) if len(sys.argv) > 1 else 3,
                                   population=sys.argv[2] if len(sys.argv) > 2 else "random")))
