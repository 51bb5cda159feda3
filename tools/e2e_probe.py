import sys, time
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS
curve, space = bench.workload(32768, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True)
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
AS._assemble_into(disc, X); torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); host.copy_(X); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"plain D2H 8.6 GB: {1e3*(t1-t0):.1f} ms ({8.59/(t1-t0):.1f} GB/s)")
    t0 = time.perf_counter(); AS._assemble_into(disc, X); host.copy_(X, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"assemble + copy: {1e3*(t1-t0):.1f} ms")
    for ch in (1, 8, 32):
        t0 = time.perf_counter(); W.assemble_matrix_to_host(disc, out=host, chunks=ch); torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"to_host chunks={ch}: {1e3*(t1-t0):.1f} ms")
