"""Small assemblies through every kernel family (a quick all-paths smoke; the
pool has compute-sanitizer disabled): circulant fast path, general uniform
path (open, double knots, nref = 2), graded lattice and block routes,
near-diagonal node pairs, RHS kernels, dense solve."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1703_10016_b200 as W
from paper_1703_10016_b200 import assembly as AS

cases = []
th = 2 * np.pi * np.arange(16) / 16
ell = W.load_curve({"degree": 3, "closed": True, "breakpoints": np.linspace(0, 1, 17).tolist(),
                    "control_points": np.column_stack([2 * np.cos(th), np.sin(th)]).tolist()})
slit = W.load_curve({"degree": 1, "knots": [-1, -1, 1, 1], "control_points": [[-1, 0], [1, 0]]})
cases.append(("circulant p3", ell, W.make_cyclic_basis(3, np.linspace(0, 1, 129)), 1))
cases.append(("open p2", slit, W.make_open_basis(2, np.linspace(-1, 1, 33)), 1))
cases.append(("open p4 double knots", slit,
              W.make_open_basis(4, np.linspace(-1, 1, 25), np.where((np.arange(23) % 3 == 1) & (np.arange(23) < 21), 2, 1)), 1))
cases.append(("closed nref2", ell, W.make_cyclic_basis(3, np.linspace(0, 1, 33)), 2))
c5 = bench.workload_c5(256, growth_elems=20)
cases.append(("graded lattice p4", c5[0], c5[1], 1))
for name, curve, space, nref in cases:
    disc = W.build_discretization(curve, space, nref)
    A = AS.assemble_matrix_device(disc)
    torch.cuda.synchronize()
    print(f"{name}: N={space.dim} finite={bool(torch.isfinite(A).all())}", flush=True)
AS._LATTICE_MAX_OFF = -1   # graded block route
disc = W.build_discretization(c5[0], c5[1], 1)
A = AS.assemble_matrix_device(disc)
b = W.assemble_b1_weighted(disc, lambda s: np.ones_like(s))
x = W.solve_system(A, b)
print("graded blocks + b1w + solve:", bool(np.isfinite(x).all()), flush=True)
b2 = W.assemble_b2(ell, W.make_cyclic_basis(3, np.linspace(0, 1, 17)), lambda s: np.ones_like(s))
print("b2:", bool(np.isfinite(b2).all()), flush=True)
