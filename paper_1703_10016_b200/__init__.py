"""B200-native (sm_100a, FP64) IgA-SGBEM V-matrix assembly.

Drop-in for the assembly entry points of the reference package ``wqbem``
(arXiv 1703.10016): knot vector, degree, geometry in; dense Galerkin matrix
of the 2D Laplace single-layer operator plus right-hand side out.  The
O(N^2) work runs in hand-written CUDA kernels behind the C-ABI in
``include/wqb200.h``; see DESIGN.md.
"""

from .errors import (
    ConstructionError,
    DeviceError,
    DomainError,
    GeometryError,
    MetricError,
    SolverError,
    UsageError,
    WqbemError,
)
from .splines import BasisSpec, RefinedBasis, make_cyclic_basis, make_open_basis, refine_uniform
from .geometry import BoundaryCurve, curve_eval, load_curve, parametric_speed
from .assembly import (
    Discretization,
    NodeVector,
    assemble_b1,
    assemble_b1_weighted,
    assemble_b2,
    assemble_ik1,
    assemble_ik2,
    assemble_matrix_device,
    assemble_matrix_to_host,
    assemble_weighted_matrix,
    build_discretization,
    scale_and_symmetrize,
)
from .solver import condition_number, solve_system

__version__ = "0.1.0"
