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
AS._assemble_into(disc, X); torch.cuda.synchronize()
lp, d = AS._logpart_dev(disc); zext = AS._zext_table(disc)
args = (N, 3, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1], lp.zstride,
        _lib.ptr(d["uext"]), _lib.ptr(zext), _lib.ptr(d["s_w"]), 1.0, 0.0)
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print("x2_pairs", t(lambda: _lib.call("wq_x2_pairs", *args, _lib.ptr(X), N, _lib.stream_handle())))
for L in (4, 8, 16, 32):
    runs = AS._to_dev(torch, AS.diag_runs(N, L))
    print("x2_runs L", L, t(lambda: _lib.call("wq_x2_runs", *args, _lib.ptr(runs), runs.shape[0], _lib.ptr(X), N, _lib.stream_handle())))
