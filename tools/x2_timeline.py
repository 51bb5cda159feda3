"""Per-CTA phase breakdown of x2_pairs at C4 (clock64 stamps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
curve, space = bench.workload(n_el, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
AS._assemble_into(disc, X); torch.cuda.synchronize()
nb = -(-N // 64); pairs = nb * (nb + 1) // 2
buf = torch.zeros((pairs, 8), dtype=torch.int64, device="cuda")
_lib.call("wq_debug_x2_timing", _lib.ptr(buf))
AS._assemble_v2(disc, X, -1 / (4 * np.pi), chunks=1)
torch.cuda.synchronize()
_lib.call("wq_debug_x2_timing", None)
t = buf.cpu().numpy().astype(np.float64)
d = np.diff(t, axis=1)
names = ["stage0", "phi0", "contract0", "stage1", "phi1", "contract1", "epilogue"]
tot = t[:, 7] - t[:, 0]
print("per-CTA cycles: mean total %.0f" % tot.mean())
for k, nm in enumerate(names):
    print(f"  {nm:10s} mean {d[:, k].mean():8.0f}  ({100 * d[:, k].mean() / tot.mean():5.1f}%)  p10 {np.percentile(d[:, k], 10):8.0f} p90 {np.percentile(d[:, k], 90):8.0f}")

