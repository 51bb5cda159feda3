import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
curve, space = bench.workload(32768, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
sm = AS._smooth(disc)
res = {}
for npass in (1, 2, 1, 2):
    _lib.call("wq_set_ik1_passes", npass)
    f = lambda: _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, 0, _lib.ptr(sm["flag"]), _lib.stream_handle())
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); f(); f(); e1.record(); torch.cuda.synchronize()
    res.setdefault(npass, []).append(e0.elapsed_time(e1) / 3)
    if npass == 1: ref = X[:2048].clone()
    else: print(npass, "== mode 1 bits:", bool(torch.equal(ref, X[:2048])))
print(res)
