"""Timing probe (tools only): C4 ik1_sym / x2 / full step in isolation and in sequence."""
import os, sys, json
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
lp, d = AS._logpart_dev(disc); sm = AS._smooth(disc)
zext = AS._zext_table(disc)
alpha = -1 / (4 * np.pi)
def ik1():
    _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, sm["span64"], _lib.ptr(sm["flag"]), _lib.stream_handle())
def x2():
    _lib.call("wq_x2_pairs", N, 3, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1], lp.zstride,
              _lib.ptr(d["uext"]), _lib.ptr(zext), _lib.ptr(d["s_w"]), alpha, float(os.environ.get("W_IK1", "2.0")), _lib.ptr(X), N, _lib.stream_handle())
def step():
    AS._assemble_into(disc, X)
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
res = {"x2": t(x2), "ik1": t(ik1), "ik1+x2": t(lambda: (ik1(), x2())), "step": t(step), "x2_again": t(x2)}
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
