"""Phase clocks of the warp-specialised tensor-core Y-stage (tools only; WQB200_LIB = a build
with -DWQ_YS_TIMELINE): the 20th tile of every CTA of the LAST wq_ystage_mma launch of one C5
assembly (the D stage) or, with THETA=1, of the Theta stage."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib
curve, space = bench.workload_c5()
disc = W.build_discretization(curve, space, 1)
N = space.dim
X = torch.empty((N, N), dtype=torch.float64, device="cuda")
AS._assemble_into(disc, X); torch.cuda.synchronize()
lib = _lib.load()
buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
want_theta = os.environ.get("THETA") == "1"
orig = _lib.call
def hook(name, *a):
    if name == "wq_ystage_mma":
        nal = a[3]
        on = (nal == 17) == want_theta
        lib.wq_debug_ys_timeline(ctypes.c_void_p(buf.data_ptr() if on else 0))
    return orig(name, *a)
_lib.call = hook
AS._assemble_into(disc, X); torch.cuda.synchronize()
_lib.call = orig
t = buf.view(148, 64).cpu().numpy().astype(np.int64)
t = t[t[:, 0] > 0]
rel = t - t[:, :1]
names = {}
for b in range(5):
    for k, n in enumerate(["start", "window", "dmma done", "empty ok", "handed"]):
        names[5 * b + k] = f"P b{b} {n}"
names.update({32: "E tile top", 33: "E params", 34: "E Ci/Cv/out init", 35: "E synced", 52: "E tile done"})
for b in range(5):
    names[36 + 3 * b] = f"E b{b} before full"; names[37 + 3 * b] = f"E b{b} full"; names[38 + 3 * b] = f"E b{b} contracted"
for k in sorted(names):
    print(f"{names[k]:22s} mean {rel[:, k].mean():9.0f}  min {rel[:, k].min():8d}  max {rel[:, k].max():8d}")
