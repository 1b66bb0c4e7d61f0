"""Process-wide state of the drop-in: device, default precision, context cache,
and the result types handed back to callers.

The reference binds its operators by import and has no plugin registry
(SURVEY §8b), so the drop-in functions are plain functions that look up a
device context per mesh geometry here.  ``install()`` swaps ``TYPES`` to the
reference's own classes so objects returned into the reference are the types
it checks for (``fields.mode is DiffMode.IK`` in gridmap.py:251).
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np

from . import _native as nat
from . import model

_state_lock = threading.Lock()
_device = int(os.environ.get("PPPM_B200_DEVICE", "0"))
_precision = os.environ.get("PPPM_B200_PRECISION", "fp64")
_contexts: "OrderedDict[tuple, nat.Context]" = OrderedDict()
MAX_CONTEXTS = 16


class _Types:
    def __init__(self):
        self.reset()

    def reset(self):
        from . import gridmap, stencil

        self.DiffMode = model.DiffMode
        self.ChargeGrid = gridmap.ChargeGrid
        self.FieldGrids = gridmap.FieldGrids
        self.StencilTable = stencil.StencilTable
        self.KSpacePlan = None  # None: this package's own plan class
        self.EnergyBreakdown = model.EnergyBreakdown


TYPES = None


def types():
    global TYPES
    if TYPES is None:
        TYPES = _Types()
    return TYPES


def set_device(device: int):
    global _device
    _device = int(device)


def get_device() -> int:
    return _device


def set_precision(precision: str):
    """Default precision of the drop-in calls: "fp64" (parity 1e-10) or "mixed"."""
    global _precision
    if precision == "fp32":
        precision = "mixed"
    if precision not in model.PRECISIONS:
        raise model.ConfigurationError(f"precision must be one of {model.PRECISIONS}")
    _precision = precision


def get_precision() -> str:
    return _precision


def precision_of(params) -> str:
    p = getattr(params, "precision", None) or _precision
    return "mixed" if p == "fp32" else p


def mode_code(mode) -> int:
    value = getattr(mode, "value", mode)
    if value == "ik":
        return nat.MODE_IK
    if value == "ad":
        return nat.MODE_AD
    raise model.ConfigurationError("mode must be a DiffMode")


def prec_code(precision: str) -> int:
    return nat.PREC_FP64 if precision == "fp64" else nat.PREC_MIXED


def context(dims, lengths, order, mode, precision, alpha, coulomb_constant=1.0, dielectric=1.0):
    """Cached device context for one geometry / order / mode / precision."""
    key = (_device, tuple(int(d) for d in dims), tuple(float(v) for v in lengths), int(order),
           int(mode), int(precision), float(alpha), float(coulomb_constant), float(dielectric))
    with _state_lock:
        ctx = _contexts.get(key)
        if ctx is not None:
            _contexts.move_to_end(key)
            return ctx
    ctx = nat.Context(_device, dims, lengths, order, mode, precision, alpha, coulomb_constant,
                      dielectric)
    with _state_lock:
        _contexts[key] = ctx
        while len(_contexts) > MAX_CONTEXTS:
            _, old = _contexts.popitem(last=False)
            old.close()
    return ctx


def clear_contexts():
    with _state_lock:
        while _contexts:
            _, c = _contexts.popitem()
            c.close()


def apply_table(ctx: nat.Context, params, table):
    """Select exact rows or upload the caller's table rows (stencil.py:105-151)."""
    if not params.use_table:
        if ctx.table_key != ("exact",):
            ctx("pppm_ctx_set_table", 0, None, None)
            ctx.table_key = ("exact",)
        return
    if table is None or int(table.order) != int(params.order):
        raise types_config_error("a stencil table matching the order is required")
    a = np.ascontiguousarray(table.assignment, dtype=np.float64)
    d = np.ascontiguousarray(table.derivative, dtype=np.float64)
    key = ("rows", id(table.assignment), a.ctypes.data, id(table.derivative), d.ctypes.data,
           int(table.n_points))
    if ctx.table_key != key:
        ctx("pppm_ctx_set_table", int(table.n_points), nat.ptr(a), nat.ptr(d))
        ctx.table_key = key
        ctx._table_refs = (a, d)  # keep the arrays alive while the key is cached


def types_config_error(msg):
    return nat.ERRORS.config(msg)


def atoms_arrays(system):
    pos = np.ascontiguousarray(system.positions, dtype=np.float64)
    q = np.ascontiguousarray(system.charges, dtype=np.float64)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError("positions must have shape (N, 3)")
    return pos, q


def geometry(system, params):
    """dims and spacing with the reference's dims check (gridmap.py:81-89)."""
    dims = tuple(int(d) for d in params.grid_dims)
    lengths = np.asarray(system.box.lengths, dtype=np.float64)
    spacing = tuple(float(lengths[d]) / dims[d] for d in range(3))
    if any(dims[d] < int(params.order) for d in range(3)):
        raise types_config_error("grid dimensions must be >= the stencil order")
    return dims, spacing, lengths


def count_touch(counters, key, n_atoms, order):
    if counters is not None:
        counters[key] = counters.get(key, 0) + n_atoms * order ** 3
