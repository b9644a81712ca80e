"""B200-native IMEX-DG hot path of arXiv 2408.08129 (drop-in for orodg).

Host-side input builders (mesh, basis, geometry, cases, partition) mirror
the reference's modules; the operators, the implicit solver and the IMEX
step run in libdg.so (hand-written sm_100a fp64 CUDA) through the C ABI in
include/dg.h.  Importing this package does not touch the GPU; the first
device call loads libdg.so and raises DeviceError if it is missing.
"""

__version__ = "0.1.0"

from .basis import ReferenceBasis, make_basis
from .boundary import BoundaryCondition, wall_everywhere
from .errors import (ConfigurationError, DeviceError, GeometryError, MeshError,
                     OrodgError, PositivityError, SolverError, UsageError)
from .field import StateField, allocate_field, project_initial_data
from .geometry import apply_terrain_mapping, build_geometry
from .mesh import ForestMesh, build_uniform_mesh, refine_region
from .partition import Partition, partition_leaves
from .physics import (CONST, DIMENSIONAL, FlowModel, PhysicalConstants,
                      conserved_to_primitive, gravity_source)


def __getattr__(name):
    # device-facing modules import torch lazily
    if name in ("DGOperators",):
        from .dgops import DGOperators
        return DGOperators
    if name in ("SplitOperators", "ImplicitSolveConfig", "ButcherTableau", "ars222",
                "imex_step", "run_time_loop", "build_helmholtz_action", "StepStats"):
        from . import imex
        return getattr(imex, name)
    if name in ("gmres", "KrylovStats"):
        from . import krylov
        return getattr(krylov, name)
    raise AttributeError(name)
