"""Time wq_gen_pair_blocks on one chunk of C5 outer elements: far kernel with
and without the gap table, and with the near kernel skipped."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS, _lib, precompute as PC

curve, space = bench.workload_c5(16384)
disc = W.build_discretization(curve, space, 1)
lp, d = AS._logpart_dev(disc)
n = lp.n_el
nU, nB = lp.u.shape[2], lp.db + 1
w, c = np.unique(lp.elh, return_counts=True)
h0 = float(w[np.argmax(c)])
print("h0", h0, "count exact", c.max(), "within 1e-12:", int(np.sum(np.abs(lp.elh - h0) <= 1e-12 * h0)))
m2u = AS._gap_table(disc, lp, 1.0)
chunk = 128
wt = torch.empty((n, nU, nB, chunk), dtype=torch.float64, device="cuda")
wd = torch.empty_like(wt)
flags = torch.empty((n, -(-chunk // 64)), dtype=torch.int32, device="cuda")
st = _lib.stream_handle()
for e0 in (0, 8000):
    for label, tab, mx in (("table", True, int(lp.near_cnt.max())), ("gauss", False, int(lp.near_cnt.max())),
                           ("table,no-near", True, 0)):
        for rep in range(2):
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            _lib.call("wq_gen_pair_blocks", n, e0, e0 + chunk, lp.da, lp.db, nU - 1, 0, 0.0,
                      _lib.ptr(d["elh"]), _lib.ptr(d["elm"]), _lib.ptr(d["u"]), _lib.ptr(d["v"]),
                      _lib.ptr(d["near_lo"]), _lib.ptr(d["near_cnt"]), mx,
                      _lib.ptr(d["near_unit"]), _lib.ptr(d["touch"]), _lib.ptr(d["gx"]),
                      _lib.ptr(d["gw"]), _lib.ptr(m2u) if tab else None,
                      _lib.ptr(d["ca"]), _lib.ptr(d["cb"]), _lib.ptr(wt), _lib.ptr(wd), chunk, _lib.ptr(flags), st)
            ev1.record()
            torch.cuda.synchronize()
        if label == "table":
            ref = wt.clone()
        if label == "gauss":
            print("   table vs gauss max rel", float((wt - ref).abs().max() / ref.abs().max()))
        print(f"e0={e0} {label:14s} {ev0.elapsed_time(ev1):8.3f} ms  ({chunk * n / ev0.elapsed_time(ev1) / 1e6:.3f} Gpairs/s)")
