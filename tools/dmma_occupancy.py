"""DMMA / DFMA throughput vs resident warps per SM (probe kernels are 8 warps per CTA)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_10016_b200 import _lib
out = torch.empty(148 * 64, dtype=torch.float64, device="cuda")
st = _lib.stream_handle()
def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3
for cps in (1, 2, 3, 4):
    blocks = 148 * cps
    it = 4000
    s = t(lambda: _lib.call("wq_dmma_peak", it, blocks, 0, _lib.ptr(out), st))
    f = t(lambda: _lib.call("wq_fp64_peak", it * 4, blocks, _lib.ptr(out), st))
    print(f"warps/SM {8*cps:3d}: dmma {blocks*8*it*8*512/s/1e12:6.2f} TF   dfma {blocks*256*it*4*64*2/f/1e12:6.2f} TF")
