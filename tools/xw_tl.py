"""x2ws phase clocks of pair 20 of every CTA (tools only; WQB200_LIB = the WQ_X2_TIMELINE build)."""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
curve, space = bench.workload(32768, 3)
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
lp, d = AS._logpart_dev(disc); sm = AS._smooth(disc)
zext = AS._zext_table(disc)
buf = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
lib = _lib.load()
def x2():
    _lib.call("wq_x2_pairs", N, 3, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1], lp.zstride,
              _lib.ptr(d["uext"]), _lib.ptr(zext), _lib.ptr(d["s_w"]), -1 / (4 * np.pi), 2.0, _lib.ptr(X), N,
              _lib.stream_handle())
_lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, sm["span64"], _lib.ptr(sm["flag"]), _lib.stream_handle())
x2(); torch.cuda.synchronize()
assert lib.wq_debug_x2_timeline(ctypes.c_void_p(buf.data_ptr())) == 0
x2(); torch.cuda.synchronize()
lib.wq_debug_x2_timeline(None)
t = buf.view(148, 32).cpu().numpy().astype(np.int64)
base = t[:, 0:1]
rel = (t - base)
names = {0: "P o0 start", 1: "P o0 window", 2: "P o0 dmma done", 3: "P o0 empty ok", 4: "P o0 handed",
         5: "P o1 start", 6: "P o1 window", 7: "P o1 dmma done", 8: "P o1 empty ok", 9: "P o1 handed",
         15: "E top", 16: "E before full0", 17: "E full0", 18: "E S0 done", 19: "E before full1",
         20: "E full1", 21: "E S1 done", 22: "E stores issued"}
for k, n in names.items():
    print(f"{n:18s} mean {rel[:, k].mean():9.0f}  min {rel[:, k].min():7d}  max {rel[:, k].max():7d}")
