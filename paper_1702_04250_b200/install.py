"""Rebind the reference package's hot-path names to this package's operators.

The reference has no plugin registry: ``compute_forces`` and the CLI use the
names bound at import time in ``pppm/driver.py:32-33`` and re-exported in
``pppm/__init__.py:32-41``.  ``install(pppm)`` rebinds them in
``pppm``, ``pppm.driver``, ``pppm.gridmap``, ``pppm.kspace`` and
``pppm.stencil``, and makes this package return the reference's own result
types and raise its ConfigurationError.  Call it before modules that do
``from pppm import map_charge`` are imported (e.g. from a pytest plugin).
"""

from __future__ import annotations

from . import _native as nat
from . import _runtime as rt
from . import driver, gridmap, kspace, shortrange, stencil

HOT_PATH = {
    "gridmap": ("map_charge", "distribute_force_ik", "distribute_force_ad"),
    "kspace": ("build_plan", "poisson_ik", "poisson_ad", "kspace_energy"),
    "stencil": ("build_table",),
}
# either side of the mesh path: the pair loop and the force driver
NEXT_PATH = {
    "shortrange": ("pair_forces",),
    "driver": ("compute_forces", "integrate_nve"),
}
_SOURCES = {"gridmap": gridmap, "kspace": kspace, "stencil": stencil, "shortrange": shortrange, "driver": driver}
_saved = {}


def install(pppm_module, force_driver=True):
    """Point the reference's hot-path names at the B200 operators.

    ``force_driver`` also rebinds the pair loop and the force driver
    (compute_forces / integrate_nve) to their device versions."""
    import importlib

    mods = {name: importlib.import_module(f"{pppm_module.__name__}.{name}")
            for name in ("gridmap", "kspace", "stencil", "driver", "model", "shortrange")}
    T = rt.types()
    T.DiffMode = mods["model"].DiffMode
    T.ChargeGrid = mods["gridmap"].ChargeGrid
    T.FieldGrids = mods["gridmap"].FieldGrids
    T.StencilTable = mods["stencil"].StencilTable
    T.KSpacePlan = mods["kspace"].KSpacePlan
    T.EnergyBreakdown = mods["model"].EnergyBreakdown
    nat.ERRORS.config = mods["model"].ConfigurationError
    nat.ERRORS.singular = mods["model"].SingularityError
    # errors raised by this package's own validation are the reference's class,
    # and the stencil orders are the reference's (its tests assert that even
    # orders are rejected, test_stencil.py:150-152; 4 and 6 stay available
    # through this package's own API)
    from . import model as own_model

    for mod in (kspace, shortrange, stencil, gridmap, driver, own_model):
        if hasattr(mod, "ConfigurationError"):
            _swap(mod, "ConfigurationError", mods["model"].ConfigurationError)
    _swap(stencil, "SUPPORTED_ORDERS", tuple(mods["model"].SUPPORTED_ORDERS))
    paths = dict(HOT_PATH, **(NEXT_PATH if force_driver else {}))
    for modname, names in paths.items():
        for name in names:
            new = getattr(_SOURCES[modname], name)
            for target in (pppm_module, mods[modname], mods["driver"]):
                if hasattr(target, name):
                    _saved.setdefault((target.__name__, name), (target, getattr(target, name)))
                    setattr(target, name, new)
    return sorted({name for names in paths.values() for name in names})


def _swap(target, name, value):
    _saved.setdefault((target.__name__, name), (target, getattr(target, name)))
    setattr(target, name, value)


def uninstall():
    """Restore every name ``install`` rebound."""
    for (_, name), (target, old) in list(_saved.items()):
        setattr(target, name, old)
    _saved.clear()
    rt.types().reset()
    from .model import ConfigurationError

    nat.ERRORS.config = ConfigurationError
    nat.ERRORS.singular = None
