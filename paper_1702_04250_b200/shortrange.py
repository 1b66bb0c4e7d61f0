"""Drop-in short-range pair operators (the "pair" bucket either side of the mesh path).

Mirrors shortrange.py of the reference: ``LjParams`` (shortrange.py:30-46),
``build_cell_list`` (:74-100), ``pair_forces`` (:201-267) and ``self_energy``
(:270-278).  The cell list and the screened-Coulomb (+ truncated LJ) pair loop
run on the device in fp64 (``k_pair.cu`` behind ``pppm_ctx_pair_forces``):
one thread per atom over the distinct cells of its periodic 27-stencil, atoms
inside a cell in index order, so the result is bitwise reproducible;
overlapping atoms raise ``SingularityError`` like the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import _runtime as rt
from .model import ConfigurationError

OVERLAP_DISTANCE = 1e-10


@dataclass(frozen=True)
class LjParams:
    """Truncated, unshifted Lennard-Jones parameters (disabled by default)."""

    epsilon: float = 1.0
    sigma: float = 1.0
    cutoff: float = 2.5
    enabled: bool = False

    def __post_init__(self):
        if self.enabled:
            if self.epsilon < 0.0:
                raise ValueError("LJ epsilon must be non-negative")
            if self.sigma <= 0.0:
                raise ValueError("LJ sigma must be positive")
            if self.cutoff <= 0.0:
                raise ValueError("LJ cutoff must be positive")


@dataclass(frozen=True)
class CellList:
    """Geometry of the periodic cell list (the device builds the atom lists).

    ``dims`` / ``cutoff`` as the reference's CellList (shortrange.py:49-71); the
    per-atom arrays live on the device and are rebuilt by every pair call.
    """

    dims: tuple
    cutoff: float

    @property
    def n_cells(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz


def build_cell_list(system, cutoff: float) -> CellList:
    """Cell-list geometry with the reference's validation (shortrange.py:74-100)."""
    if cutoff <= 0.0:
        raise ConfigurationError("cutoff must be positive")
    lengths = np.asarray(system.box.lengths, dtype=np.float64)
    if cutoff > 0.5 * float(lengths.min()):
        raise ConfigurationError(
            f"cutoff {cutoff} exceeds half the smallest box edge ({0.5 * float(lengths.min())})")
    dims = tuple(max(1, int(L // cutoff)) for L in lengths)
    return CellList(dims=dims, cutoff=float(cutoff))


def lj_array(lj):
    """LJ parameters for the C ABI ({epsilon, sigma, cutoff}) or None when disabled."""
    if lj is None or not getattr(lj, "enabled", False):
        return None
    return np.array([lj.epsilon, lj.sigma, lj.cutoff], dtype=np.float64)


def pair_context(system, coulomb_constant=1.0, dielectric=1.0):
    """A device context for the box (the pair kernels use its box, stream and C)."""
    lengths = np.asarray(system.box.lengths, dtype=np.float64)
    return rt.context((8, 8, 8), lengths, 3, nat.MODE_IK, nat.PREC_FP64, 1.0, coulomb_constant, dielectric)


def pair_forces(system, cells, alpha, cutoff, lj=None, *, coulomb_constant=1.0, dielectric=1.0, workers=1,
                counters=None):
    """Screened real-space forces and energy of all pairs within ``cutoff``.

    Returns ``(forces, pair_energy)``; ``workers`` is accepted for signature
    compatibility (the device sum order does not depend on it).
    """
    if alpha <= 0.0:
        raise ConfigurationError("alpha must be positive")
    if cells is not None and cutoff > cells.cutoff * (1.0 + 1e-12):
        raise ConfigurationError("cell list was built for a smaller cutoff")
    pos, q = rt.atoms_arrays(system)
    n = pos.shape[0]
    ctx = pair_context(system, coulomb_constant, dielectric)
    forces = np.empty((n, 3))
    energy = np.zeros(1)
    cnt = np.zeros(2, dtype=np.int64)
    ljp = lj_array(lj)
    ctx("pppm_ctx_pair_forces", nat.ptr(pos), nat.ptr(q), n, nat.F64, nat.HOST, float(alpha), float(cutoff),
        None if ljp is None else nat.ptr(ljp), nat.ptr(forces), energy.ctypes.data_as(nat._dp), nat.ptr(cnt))
    if counters is not None:
        counters["pair_candidates"] = counters.get("pair_candidates", 0) + int(cnt[0])
        counters["pairs_within_cutoff"] = counters.get("pairs_within_cutoff", 0) + int(cnt[1])
    return forces, float(energy[0])


def self_energy(system, alpha: float, *, coulomb_constant: float = 1.0, dielectric: float = 1.0) -> float:
    """-C alpha / sqrt(pi) sum q_i^2 (shortrange.py:270-278)."""
    if alpha <= 0.0:
        raise ConfigurationError("alpha must be positive")
    scale = coulomb_constant / dielectric
    return -scale * alpha / math.sqrt(math.pi) * float(np.sum(np.asarray(system.charges, dtype=np.float64) ** 2))
