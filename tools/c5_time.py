"""C5 assembly timing + per-entry-point split (tools only)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
if os.environ.get("SEG") == "0": AS._SEG_MIN_N = 1 << 60
curve, space = bench.workload_c5()
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
for _ in range(2): AS._assemble_into(disc, X)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): AS._assemble_into(disc, X)
e1.record(); torch.cuda.synchronize()
orig = _lib.call; split = {}
def timed(name, *a):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(); r = orig(name, *a); s1.record(); torch.cuda.synchronize()
    split[name] = split.get(name, 0.0) + s0.elapsed_time(s1); return r
_lib.call = timed; AS._assemble_into(disc, X); _lib.call = orig
print(json.dumps({"ms": e0.elapsed_time(e1) / 3, "split": {k: round(v, 2) for k, v in sorted(split.items(), key=lambda t: -t[1])}}))
if len(sys.argv) > 1:
    np.save(sys.argv[1], X[::97].cpu().numpy())
