import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 1
curve, space = bench.workload(n_el, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
sm = AS._smooth(disc)
_lib.call("wq_set_ik1_passes", mode)
for _ in range(2):
    _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, 0, _lib.ptr(sm["flag"]), _lib.stream_handle())
torch.cuda.synchronize()
print("ok")
