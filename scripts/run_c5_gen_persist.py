"""run_c5_generation with an L2 set-aside for persisting (evict_last) lines (experiment driver)."""
import ctypes
import glob
import os
import sys

import torch

mb = int(os.environ.get("FNB_L2_PERSIST_MB", "0"))
torch.cuda.init()
torch.zeros(1, device="cuda")
if mb:
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
        glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = ctypes.CDLL(cands[0])
    st = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(mb << 20))  # cudaLimitPersistingL2CacheSize
    val = ctypes.c_size_t(0)
    rt.cudaDeviceGetLimit(ctypes.byref(val), 6)
    print("persist limit", st, val.value, file=sys.stderr)
sys.argv = [sys.argv[0]] + sys.argv[1:]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "run_c5_generation.py")).read())
