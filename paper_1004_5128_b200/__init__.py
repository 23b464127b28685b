"""B200-native Grünwald–Letnikov fractional reaction–diffusion history stepper.

Drop-in for the hot path of the reference package ``fracgrid`` (arXiv 1004.5128):
``solver.run`` → ``step`` → ``history_sum`` run as one fused sm_100a kernel per
time step over an HBM-resident stencil history.  The
reference-compatible 2D API lives in :mod:`.solver`; 1D/3D, nonlinear reaction
and batched ensembles in :mod:`.problem`.
"""

__version__ = "0.1.0"

from ._engine import DivergenceError, HistoryCapacityError, MemoryBudgetError  # noqa: F401
from ._lib import NativeLibraryError  # noqa: F401
from .coefficients import PsiTable, build_table, build_tables, partial_sum, psi  # noqa: F401
from .grid import Grid2D, HistoryBuffer, stencil  # noqa: F401
from .problem import FieldConfig, FieldResult, LinearDecay, Saturating, run_field  # noqa: F401
from .schedule import (  # noqa: F401
    AdaptiveMemory,
    FullMemory,
    MemorySchedule,
    ShortMemory,
    adaptive_schedule,
    full_schedule,
    short_schedule,
)
from .solver import SimulationConfig, SimulationResult, StabilityWarning, history_sum, run, step  # noqa: F401
