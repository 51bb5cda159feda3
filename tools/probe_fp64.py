"""FP64 pipe probes: DFMA, DMMA, DMMA+DFMA (prints TFLOP/s)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_10016_b200 import _lib

def t(fn):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3

out = torch.empty(148 * 64, dtype=torch.float64, device="cuda")
st = _lib.stream_handle()
for blocks in (148 * 4, 148 * 8):
    it = 4000
    s = t(lambda: _lib.call("wq_fp64_peak", it * 4, blocks, _lib.ptr(out), st))
    print("dfma", blocks, blocks * 256 * it * 4 * 64 * 2 / s / 1e12)
    s = t(lambda: _lib.call("wq_dmma_peak", it, blocks, 0, _lib.ptr(out), st))
    print("dmma", blocks, blocks * 8 * it * 8 * 512 / s / 1e12)
    s = t(lambda: _lib.call("wq_dmma_peak", it, blocks, 1, _lib.ptr(out), st))
    print("dmma+dfma", blocks, "time ratio vs dmma-only flops", (blocks * 8 * it * 8 * 512 + blocks * 256 * it * 32 * 2) / s / 1e12)
