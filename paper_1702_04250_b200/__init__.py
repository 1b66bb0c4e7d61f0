"""B200-native PPPM particle-mesh core (drop-in for the reference ``pppm`` hot path).

Hot path: particle_map -> compute_rho1d/drho1d -> make_rho ->
Poisson (cuFFT + hand-written Green / ik / ad kernel) -> fieldforce_ik /
fieldforce_ad, as sm_100a CUDA kernels behind the C ABI in
``include/pppm_b200.h``.  The Python functions here mirror the reference's
operator API (gridmap.py / kspace.py / stencil.py) and accept its objects.
"""

__version__ = "0.1.0"

from .model import (
    AtomSystem,
    ConfigurationError,
    DiffMode,
    EnergyBreakdown,
    PppmParams,
    SimulationBox,
    SingularityError,
    SUPPORTED_ORDERS,
    wrap,
)
from .stencil import (
    PADDED_LEN,
    StencilTable,
    assignment_weights,
    build_table,
    derivative_weights,
    lookup_weights,
    weight_rows,
)
from .gridmap import (
    ChargeGrid,
    FieldGrids,
    distribute_force_ad,
    distribute_force_ik,
    map_charge,
    particle_map,
)
from .kspace import KSpacePlan, build_plan, kspace_energy, poisson_ad, poisson_ik
from .shortrange import LjParams, build_cell_list, pair_forces, self_energy
from .driver import compute_forces, integrate_nve
from .context import PinnedArray, PppmContext
from ._runtime import get_device, get_precision, set_device, set_precision
from ._native import library_path
from .install import install, uninstall

__all__ = [name for name in dir() if not name.startswith("_")]
