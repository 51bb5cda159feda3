"""C4: ik1 and x2 chunked on two streams (x2 chunk k waits for ik1 chunk k) vs one
stream; CUDA-event times (tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS
curve, space = bench.workload(32768, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
zext = AS._zext_table(disc)
alpha = -1 / (4 * np.pi)
ref = None
for chunks in (1, 2, 4, 8, 16, 32, 1):
    for _ in range(2):
        AS._assemble_v2(disc, X, alpha, zext=zext, chunks=chunks)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        AS._assemble_v2(disc, X, alpha, zext=zext, chunks=chunks)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = X[::97, ::89].clone()
    print(f"chunks {chunks:3d}: {e0.elapsed_time(e1) / 5:.3f} ms  same: {bool(torch.equal(ref, X[::97, ::89]))}", flush=True)
