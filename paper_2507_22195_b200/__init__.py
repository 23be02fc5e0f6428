"""B200-native macro-element HDG operator (arXiv 2507.22195 hot path).

Drop-in for the reference package's Discretization / LinearizedSystem /
solver / time-march API, with every operator evaluated by hand-written
sm_100a CUDA kernels in libmhdg_b200.so (no CPU fallback).
"""

from .assembly import (  # noqa: F401
    Discretization,
    FieldSet,
    FreeStream,
    LinearizedSystem,
    ResidualSet,
    StageContext,
    boundary_trace_operator,
)
from .cases import IsentropicVortex, TaylorGreen  # noqa: F401
from .errors import *  # noqa: F401,F403
from .fluxes import DissipationSpec  # noqa: F401
from .gas import GasModel, ViscousParams  # noqa: F401
from .mesh import build_box_macro_mesh, dof_counts  # noqa: F401

__version__ = "0.1.0"
