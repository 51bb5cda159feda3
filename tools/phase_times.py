"""Per-entry-point device time of one assembly: wraps _lib.call with CUDA
events (host-synchronous per call, so for attribution only)."""
import sys, os, collections
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib

which = sys.argv[1] if len(sys.argv) > 1 else "c5"
n_el = int(sys.argv[2]) if len(sys.argv) > 2 else (16384 if which == "c5" else 32768)
curve, space = bench.workload_c5(n_el) if which == "c5" else bench.workload(n_el, 3)
disc = W.build_discretization(curve, space, 1)
if os.environ.get("WQ_YS_SYM") == "0":
    AS._YS_SYM_D = False
AS._log_part(disc)
A = AS.assemble_matrix_device(disc)   # warm
torch.cuda.synchronize()
orig = _lib.call
acc = collections.defaultdict(float)
cnt = collections.Counter()
calls = collections.defaultdict(list)

def timed(name, *args):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(name, *args)
    e1.record()
    torch.cuda.synchronize()
    acc[name] += e0.elapsed_time(e1)
    cnt[name] += 1
    calls[name].append(e0.elapsed_time(e1))
    return r

_lib.call = timed
AS.assemble_matrix_device(disc, out=A)
torch.cuda.synchronize()
_lib.call = orig
tot = sum(acc.values())
print(f"{which} n_el={n_el} N={space.dim}: total {tot:.2f} ms over {sum(cnt.values())} calls")
for k, v in sorted(acc.items(), key=lambda t: -t[1]):
    extra = "  [" + ", ".join(f"{t:.2f}" for t in calls[k]) + "]" if 1 < cnt[k] <= 4 else ""
    print(f"  {k:24s} {v:9.3f} ms  x{cnt[k]}{extra}")
