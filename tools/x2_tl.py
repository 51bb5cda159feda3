"""x2 per-CTA phase clocks (tools only; needs tools/_build/libwqb200_tl.so from
tools/x2_timeline_build.sh, selected with WQB200_LIB)."""
import ctypes, os, sys, json
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
nb = -(-N // 64); pairs = nb * (nb + 1) // 2
buf = torch.zeros(pairs * 10, dtype=torch.int64, device="cuda")
lib = _lib.load()
def x2():
    _lib.call("wq_x2_pairs", N, 3, lp.da + 1, lp.nApad, lp.s_w.shape[1], lp.uext.shape[1], lp.zstride,
              _lib.ptr(d["uext"]), _lib.ptr(zext), _lib.ptr(d["s_w"]), -1 / (4 * np.pi), float(os.environ.get("W_IK1", "2.0")), _lib.ptr(X), N,
              _lib.stream_handle())
_lib.call("wq_ik1_sym", AS.ctypes_ref(sm["struct"]), _lib.ptr(X), N, sm["span64"], _lib.ptr(sm["flag"]), _lib.stream_handle())
x2(); torch.cuda.synchronize()
assert lib.wq_debug_x2_timeline(ctypes.c_void_p(buf.data_ptr())) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); x2(); e1.record(); torch.cuda.synchronize()
lib.wq_debug_x2_timeline(None)
t = buf.view(pairs, 10).cpu().numpy()
names = ["wait0", "phi0", "S0", "handoff", "wait1", "phi1", "S1", "store"]
ph = np.diff(t[:, :9], axis=1)
out = {"ms": e0.elapsed_time(e1), "cycles_mean": {k: float(v) for k, v in zip(names, ph.mean(0))},
       "total_mean": float((t[:, 8] - t[:, 0]).mean())}
# per-SM occupancy of the DMMA phases (phi + S) by the CTAs resident on it
busy, span = 0, 0
for s in np.unique(t[:, 9])[:16]:
    rows = t[t[:, 9] == s]
    lo, hi = rows[:, 0].min(), rows[:, 8].max()
    grid = np.zeros(int((hi - lo) // 64) + 2, bool)
    for r in rows:
        for a, b in ((1, 3), (5, 7)):        # phi+S of both orientations
            grid[int((r[a] - lo) // 64): int((r[b] - lo) // 64) + 1] = True
    busy += grid.sum(); span += len(grid)
    ctas = len(rows)
out["sm_fraction_in_dmma_phases"] = busy / span
out["ctas_per_sm_sampled"] = ctas
print(json.dumps(out))
