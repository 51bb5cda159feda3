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
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
AS._FUSED = False
print("separate", t(lambda: AS._assemble_into(disc, X)))
ref = X[:1024].clone()
AS._FUSED = True
for lead in (296, 1024, 4096, 16384):
    AS._FUSED_LEAD = lead
    print("fused lead", lead, t(lambda: AS._assemble_into(disc, X)), bool(torch.equal(ref, X[:1024])))
