"""Repeat-run stress of the warp-specialised kernels (tools only): the same assembly many
times, every result compared bit for bit with the first (a hand-over race between warp groups
would show up as a sporadic difference)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS

def run(name, curve, space, reps):
    disc = W.build_discretization(curve, space, 1)
    N = space.dim
    X = torch.empty((N, N), dtype=torch.float64, device="cuda")
    AS._assemble_into(disc, X); torch.cuda.synchronize()
    ref = X.clone()
    bad = 0
    for _ in range(reps):
        X.fill_(float("nan"))
        AS._assemble_into(disc, X); torch.cuda.synchronize()
        bad += int(not torch.equal(X, ref))
    print(f"{name}: N={N} reps={reps} mismatching runs={bad} finite={bool(torch.isfinite(ref).all())}", flush=True)
    return bad

bad = 0
for p, n in ((3, 32768), (2, 8192), (4, 8192), (5, 8192), (3, 2250)):
    c, s = bench.workload(n, p)
    bad += run(f"closed p={p}", c, s, 40 if n < 30000 else 25)
c5 = bench.workload_c5()
bad += run("config 5", c5[0], c5[1], 15)
sys.exit(1 if bad else 0)
