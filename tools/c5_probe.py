"""Config-5 (graded + double knots, p=4, open slit) assembly on one GPU:
host precompute time, per-phase device times, size-independent checks."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
curve, space = bench.workload_c5(n_el)
t0 = time.perf_counter()
disc = W.build_discretization(curve, space, 1)
t1 = time.perf_counter()
lp = AS._log_part(disc)
t2 = time.perf_counter()
N = space.dim
print(f"C5 n_el={n_el} N={N} nq={disc.nodes.n} build={t1-t0:.2f}s logpart={t2-t1:.2f}s "
      f"graded={lp.graded} max_near={lp.near_cnt.max()} bw={lp.bw}", flush=True)
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    AS._ik1_into(disc, X, accumulate=False)
    ev[1].record()
    AS._ik2_x2_into(disc, X, accumulate=True)
    ev[2].record()
    _lib.call("wq_symmetrize", _lib.ptr(X), N, -1.0 / (4 * np.pi), _lib.stream_handle())
    ev[3].record()
    torch.cuda.synchronize()
    t = [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
    print(f"rep {rep}: ik1 {t[0]:.2f} ms  ik2(x2) {t[1]:.2f} ms  symm {t[2]:.2f} ms  "
          f"total {sum(t):.2f} ms -> {N*N/(sum(t)*1e-3):.3e} entries/s", flush=True)
AS._check_flag(AS._smooth(disc))
A = X
print("finite", bool(torch.isfinite(A).all()), "sym", bool(torch.equal(A, A.T)),
      "diag>0", bool((A.diagonal() > 0).all()), "absmax", float(A.abs().max()))
A2 = AS.assemble_matrix_device(disc)
print("deterministic", bool(torch.equal(A, A2)))
