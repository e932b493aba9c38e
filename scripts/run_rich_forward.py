"""The generic forward (rich schema, C2 shapes) alone -- profiling driver."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(bench.rich_schema(dev, torch.cuda.current_stream(), flush, reps=2))
