"""porodg_b200: B200-native (sm_100a) GMRES slab solver for the porodg
space-time Biot reference (arxiv 1801.04984). See DESIGN.md."""
from ._lib import InvalidArgument, PdgError, SolverError  # noqa: F401
from .problem import ProblemSpec, config0, config1, config3, terzaghi_recorded  # noqa: F401
from .solver import (BlockSolver, FixedStressConfig, GmresOptions, SlabSolver, SolveOptions,  # noqa: F401
                     SpatialOperators, march)

__all__ = ["SpatialOperators", "BlockSolver", "SlabSolver", "SolveOptions", "GmresOptions", "FixedStressConfig",
           "march", "SolverError", "InvalidArgument", "PdgError", "ProblemSpec", "config0", "config1", "config3",
           "terzaghi_recorded"]
