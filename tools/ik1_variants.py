"""Time ik1_sym variants (wq_set_ik1_passes 1 / 2) at C4 with CUDA events (tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
curve, space = bench.workload(n_el, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
sm = AS._smooth(disc)
ref = None
for mode in (1, 2, 1, 2):
    _lib.call("wq_set_ik1_passes", mode)
    run = lambda: _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, 0,
                            _lib.ptr(sm["flag"]), _lib.stream_handle())
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = X.clone()
    same = bool(torch.equal(ref, X))
    print(f"mode {mode}: {e0.elapsed_time(e1) / 5:.3f} ms  bit-identical to first: {same}", flush=True)
