import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_10016_b200 import _lib
U = torch.rand(148 * 16 * 64, 72, dtype=torch.float64, device="cuda")
out = torch.empty(148 * 64, dtype=torch.float64, device="cuda"); st = _lib.stream_handle()
for mode, name in ((0, "as kernel"), (1, "no B loads"), (2, "no A LDS"), (3, "no loads")):
    for cps in (1, 2, 3):
        blocks = 148 * cps; it = 200
        f = lambda: _lib.call("wq_probe_phi", it, blocks, mode, _lib.ptr(U), _lib.ptr(out), st)
        f(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        s = e0.elapsed_time(e1) * 1e-3
        print(f"{name:12s} CTAs/SM {cps}: {blocks * 8 * it * 180 * 512 / s / 1e12:6.2f} TF")
