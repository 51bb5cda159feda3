import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_10016_b200 import _lib
out = torch.empty(148 * 64, dtype=torch.float64, device="cuda"); st = _lib.stream_handle()
for mode in (0, 1, 2):
    for blocks in (148 * 4, 148 * 8):
        it = 2000
        f = lambda: _lib.call("wq_probe_log", it, blocks, mode, _lib.ptr(out), st)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        s = e0.elapsed_time(e1) * 1e-3
        n = blocks * 256 * it * 4
        print(f"mode {mode} blocks {blocks}: {n / s / 1e9:8.1f} Glog/s  -> {s * 1.965e9 * 148 * 64 / n:5.1f} FP64-lane-slots per log")
