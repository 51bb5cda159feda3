"""Run the v2 circulant pipeline a few times (for ncu / nsys-free profiling)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1703_10016_b200 import assembly as AS
import paper_1703_10016_b200 as W

ap = argparse.ArgumentParser()
ap.add_argument("--n-el", type=int, default=4096)
ap.add_argument("--p", type=int, default=3)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
curve, space = bench.workload(a.n_el, a.p)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    AS._assemble_into(disc, X)
torch.cuda.synchronize()
AS._check_flag(AS._smooth(disc))
print("ok", N)
