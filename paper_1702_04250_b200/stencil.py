"""Stencil weights (compute_rho1d / compute_drho1d) and lookup tables.

Mirrors the reference's public stencil API (stencil.py:23-151): rows of the
centred cardinal B-spline of order S, zero-padded to length 8, lowest grid
node first, and the nearest-entry table at ``n_points`` bin centres.  The rows
are evaluated on the GPU by the same device function the mapping kernels use
(``bspline_rows`` in csrc/pppm_common.cuh, fp64 without FMA contraction), so
they are bitwise equal to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as nat
from . import _runtime as rt
from .model import SUPPORTED_ORDERS

PADDED_LEN = 8


def _check_order(order):
    if order not in SUPPORTED_ORDERS:
        raise ValueError(f"unsupported stencil order {order}; expected one of {SUPPORTED_ORDERS}")


def _check_offset(t):
    if not np.isfinite(t):
        raise ValueError("fractional offset must be finite")
    if not (-0.5 <= t < 0.5):
        raise ValueError(f"fractional offset {t} outside [-1/2, 1/2)")


def weight_rows(t, order):
    """Assignment and derivative rows at offsets ``t`` (stencil.py:38-77), on the GPU."""
    _check_order(order)
    t = np.asarray(t, dtype=np.float64)
    flat = np.ascontiguousarray(t.reshape(-1))
    a = np.empty((flat.size, PADDED_LEN))
    d = np.empty((flat.size, PADDED_LEN))
    if flat.size:
        nat.require_device(rt.get_device())
        nat.call("pppm_weight_rows", rt.get_device(), int(order), nat.ptr(flat), flat.size,
                 nat.ptr(a), nat.ptr(d))
    return a.reshape(t.shape + (PADDED_LEN,)), d.reshape(t.shape + (PADDED_LEN,))


def assignment_weights(t, order):
    """Length-8 assignment row at offset ``t`` in [-1/2, 1/2) (stencil.py:80-90)."""
    _check_order(order)
    _check_offset(t)
    return weight_rows(float(t), order)[0]


def derivative_weights(t, order):
    """Length-8 derivative row d/dt (stencil.py:93-102)."""
    _check_order(order)
    _check_offset(t)
    return weight_rows(float(t), order)[1]


@dataclass(frozen=True)
class StencilTable:
    """Rows at ``n_points`` bin centres; bin k covers [-1/2 + k/n, -1/2 + (k+1)/n)."""

    order: int
    n_points: int
    assignment: np.ndarray
    derivative: np.ndarray

    @property
    def bin_width(self) -> float:
        return 1.0 / self.n_points

    def bin_index(self, t):
        """Bin of offset ``t`` (stencil.py:123-126).  Host helper for callers; the
        kernels compute the same index on the device (csrc/pppm_common.cuh)."""
        idx = np.floor((np.asarray(t, dtype=float) + 0.5) * self.n_points).astype(np.intp)
        return np.clip(idx, 0, self.n_points - 1)


def build_table(order, n_points=5000) -> StencilTable:
    """Tabulate both weight families at the bin centres, on the GPU (stencil.py:129-139)."""
    _check_order(order)
    n_points = int(n_points)
    if n_points < 2:
        raise ValueError("n_points must be >= 2")
    a = np.empty((n_points, PADDED_LEN))
    d = np.empty((n_points, PADDED_LEN))
    nat.require_device(rt.get_device())
    nat.call("pppm_table_rows", rt.get_device(), int(order), n_points, nat.ptr(a), nat.ptr(d))
    a.flags.writeable = False
    d.flags.writeable = False
    return rt.types().StencilTable(order=order, n_points=n_points, assignment=a, derivative=d)


def lookup_weights(table, t):
    """Rows of the bin containing ``t`` (stencil.py:142-151)."""
    _check_offset(t)
    idx = int(table.bin_index(float(t)))
    return table.assignment[idx], table.derivative[idx]
