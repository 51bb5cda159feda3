"""One C4-like assembly for ncu captures of x2_pairs (tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
curve, space = bench.workload(n_el, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
for _ in range(2):
    AS._assemble_v2(disc, X, -1 / (4 * np.pi), chunks=1)
torch.cuda.synchronize()
print("ok")
