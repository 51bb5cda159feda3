"""Does running ik1_sym and x2_pairs concurrently (two streams, independent
buffers) beat running them back to back?  Prints ms for each mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib

curve, space = bench.workload(32768, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X1 = torch.empty((N, N), dtype=torch.float64, device="cuda")
X2 = torch.empty((N, N), dtype=torch.float64, device="cuda")
sm = AS._smooth(disc); lp, d = AS._logpart_dev(disc)
zext = AS._zext_table(disc)
s1 = torch.cuda.Stream(priority=0); s2 = torch.cuda.Stream(priority=-1)

def ik1(st):
    _lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X1), N, 0, _lib.ptr(sm["flag"]), _lib.stream_handle(st))

def x2(st):
    _lib.call("wq_x2_pairs", N, 3, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1], lp.zstride,
              _lib.ptr(d["uext"]), _lib.ptr(zext), _lib.ptr(d["s_w"]), 1.0, 0.0, _lib.ptr(X2), N, _lib.stream_handle(st))

def timeit(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

cur = torch.cuda.current_stream()
def seq():
    ik1(cur); x2(cur)
def conc():
    s1.wait_stream(cur); s2.wait_stream(cur)
    ik1(s1); x2(s2)
    cur.wait_stream(s1); cur.wait_stream(s2)
print("ik1 alone", timeit(lambda: ik1(cur)))
print("x2 alone", timeit(lambda: x2(cur)))
print("sequential", timeit(seq))
print("concurrent", timeit(conc))
