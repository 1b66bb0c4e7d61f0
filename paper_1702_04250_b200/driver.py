"""Drop-in force driver: the full force evaluation and NVE integration on the device.

Mirrors ``compute_forces`` (driver.py:232-307) and ``integrate_nve``
(driver.py:310-376) of the reference.  One C-ABI call evaluates the screened
pair forces (``k_pair.cu``), make_rho -> Poisson -> fieldforce (the mesh path)
and the self energy on the device; ``integrate_nve`` keeps positions,
velocities and forces resident for the whole velocity-Verlet trajectory and
reduces the energy / temperature / momentum series on the device (fp64,
fixed-order sums).  Section timing: the reference's three measured sections
(``pair``, ``pppm_fft``, ``pppm_non_fft``, driver.py:1-9) are CUDA-event times
of the device call, so ``make_report`` records (driver.py:383-423) keep their
schema with GPU timings.
"""

from __future__ import annotations

import json
import time

import numpy as np

from . import _native as nat
from . import _runtime as rt
from . import kspace, stencil
from .model import EnergyBreakdown
from .shortrange import lj_array

REPORT_SECTIONS = ("pppm_non_fft", "pppm_fft", "pair", "other")


def _energy_type():
    T = rt.types()
    return getattr(T, "EnergyBreakdown", None) or EnergyBreakdown


def _solver_ctx(system, params, table, plan):
    """Device context of the force evaluation with the caller's table and influence."""
    params.validate_for_box(system.box)
    dims, _, lengths = rt.geometry(system, params)
    prec = rt.prec_code(rt.precision_of(params))
    ctx = rt.context(dims, lengths, params.order, rt.mode_code(params.mode), prec, params.alpha,
                     params.coulomb_constant, params.dielectric)
    if params.use_table and table is None:
        table = stencil.build_table(params.order, params.table_points)
    rt.apply_table(ctx, params, table)
    if plan is None:
        key = ("device", "pme", kspace.DECONV_FLOOR)
        if ctx.green_key != key:
            ctx("pppm_ctx_build_influence", nat.INFLUENCE_PME, kspace.DECONV_FLOOR)
            ctx.green_key = key
    elif isinstance(plan, kspace.KSpacePlan):
        key = ("device", plan.variant, plan.deconv_floor)
        if ctx.green_key != key:
            kind = nat.INFLUENCE_PME if plan.variant == "pme" else nat.INFLUENCE_OPTIMAL
            ctx("pppm_ctx_build_influence", kind, plan.deconv_floor)
            ctx.green_key = key
    else:  # a foreign (reference) plan: upload its influence grid
        g = np.ascontiguousarray(plan.influence, dtype=np.float64)
        key = ("host", id(plan.influence), g.ctypes.data)
        if ctx.green_key != key:
            ctx("pppm_ctx_set_influence", nat.ptr(g))
            ctx.green_key = key
            ctx._green_ref = g
    return ctx


def _count(counters, params, n, cnt):
    if counters is None:
        return
    counters["pair_candidates"] = counters.get("pair_candidates", 0) + int(cnt[0])
    counters["pairs_within_cutoff"] = counters.get("pairs_within_cutoff", 0) + int(cnt[1])
    rt.count_touch(counters, "cells_touched_map", n, int(params.order))
    rt.count_touch(counters, "cells_touched_distribute", n, int(params.order))
    nx, ny, nz = params.grid_dims
    counters["grid_points"] = nx * ny * nz


def compute_forces(system, params, table=None, plan=None, lj=None, *, workers=1, timer=None, counters=None):
    """One full force evaluation: screened pair part plus mesh part.

    Returns ``(forces, EnergyBreakdown, sections)``.
    """
    t0 = time.perf_counter()
    ctx = _solver_ctx(system, params, table, plan)
    pos, q = rt.atoms_arrays(system)
    n = pos.shape[0]
    forces = np.empty((n, 3))
    e = np.zeros(3)
    cnt = np.zeros(2, dtype=np.int64)
    sec = np.zeros(3)
    ljp = lj_array(lj)
    ctx("pppm_ctx_compute_forces", nat.ptr(pos), nat.ptr(q), n, nat.F64, nat.HOST, float(params.cutoff),
        None if ljp is None else nat.ptr(ljp), nat.ptr(forces), nat.ptr(e), nat.ptr(cnt), nat.ptr(sec))
    _count(counters, params, n, cnt)
    sections = {"pppm_non_fft": float(sec[0]), "pppm_fft": float(sec[1]), "pair": float(sec[2])}
    if timer is not None:
        for name, dt in sections.items():
            timer.add(name, dt)
        timer.add("other", max(0.0, time.perf_counter() - t0 - sum(sections.values())))
    energy = _energy_type()(pair=float(e[0]), kspace=float(e[1]), self_energy=float(e[2]))
    return forces, energy, sections


def make_report(*, sections, wall_total, n_atoms, params, steps, workers, counters=None, extra=None):
    """A timing record with the reference's schema (driver.py:383-423)."""
    from . import __version__

    measured = {k: float(sections.get(k, 0.0)) for k in REPORT_SECTIONS if k != "other"}
    record = {
        "sections": {**measured, "other": max(0.0, wall_total - sum(measured.values()))},
        "n_atoms": int(n_atoms),
        "steps": int(steps),
        "workers": int(workers),
        "params": {
            "cutoff": params.cutoff, "accuracy": params.accuracy, "order": params.order,
            "mode": getattr(params.mode, "value", params.mode), "alpha": params.alpha,
            "grid_dims": list(params.grid_dims), "table_points": params.table_points,
            "use_table": params.use_table,
        },
        "counters": dict(counters or {}),
        "build_id": f"paper_1702_04250_b200-{__version__}",
    }
    if extra:
        record.update(extra)
    return record


def validate_report(record) -> None:
    """Raise ValueError unless ``record`` matches the report schema (driver.py:426-441)."""
    if not isinstance(record, dict):
        raise ValueError("report record must be a dict")
    sections = record.get("sections")
    if not isinstance(sections, dict) or set(sections) != set(REPORT_SECTIONS):
        raise ValueError(f"report sections must be exactly {REPORT_SECTIONS}")
    for key, value in sections.items():
        if not isinstance(value, (int, float)) or value < 0:
            raise ValueError(f"section {key} must be a non-negative number")
    for key in ("n_atoms", "steps", "workers", "params", "build_id"):
        if key not in record:
            raise ValueError(f"report record missing {key!r}")
    if not isinstance(record["params"], dict):
        raise ValueError("params echo must be a dict")


def report_line(record) -> str:
    """One JSON line, keys sorted (driver.write_records, fmt json)."""
    return json.dumps(record, sort_keys=True)


def integrate_nve(system, params, dt, steps, lj=None, *, workers=1, timer=None, counters=None):
    """Velocity-Verlet NVE trajectory with a device force evaluation per step.

    Returns ``{"series", "final", "steps", "dt"}`` like driver.py:310-376
    (temperature = sum(m v^2) / (3N), k_B = 1).
    """
    if system.velocities is None:
        raise ValueError("NVE integration needs initial velocities")
    if dt <= 0.0:
        raise ValueError("dt must be positive")
    steps = int(steps)
    ctx = _solver_ctx(system, params, None, None)
    pos, q = rt.atoms_arrays(system)
    n = pos.shape[0]
    vel = np.ascontiguousarray(system.velocities, dtype=np.float64)
    masses = np.ascontiguousarray(system.masses, dtype=np.float64)
    series = np.empty((steps + 1, 7))
    pos_out = np.empty((n, 3))
    vel_out = np.empty((n, 3))
    ljp = lj_array(lj)
    sec = np.zeros(3)
    cnt = np.zeros(2, dtype=np.int64)
    t0 = time.perf_counter()
    ctx("pppm_ctx_integrate_nve", nat.ptr(pos), nat.ptr(vel), nat.ptr(masses), nat.ptr(q), n, float(dt), steps,
        float(params.cutoff), None if ljp is None else nat.ptr(ljp), nat.ptr(series), nat.ptr(pos_out),
        nat.ptr(vel_out), nat.ptr(sec), nat.ptr(cnt))
    wall = time.perf_counter() - t0
    if timer is not None:
        # the reference's sections, accumulated over the steps + 1 force evaluations
        # (CUDA events per evaluation); the rest of the wall time is "other"
        sections = {"pppm_non_fft": float(sec[0]), "pppm_fft": float(sec[1]), "pair": float(sec[2])}
        for name, dt_s in sections.items():
            timer.add(name, dt_s)
        timer.add("other", max(0.0, wall - sum(sections.values())))
    if counters is not None:
        evals = steps + 1
        counters["pair_candidates"] = counters.get("pair_candidates", 0) + int(cnt[0])
        counters["pairs_within_cutoff"] = counters.get("pairs_within_cutoff", 0) + int(cnt[1])
        for _ in range(evals):
            rt.count_touch(counters, "cells_touched_map", n, int(params.order))
            rt.count_touch(counters, "cells_touched_distribute", n, int(params.order))
        nx, ny, nz = params.grid_dims
        counters["grid_points"] = nx * ny * nz
    out = {
        "total_energy": series[:, 0].copy(),
        "kinetic": series[:, 1].copy(),
        "potential": series[:, 2].copy(),
        "temperature": series[:, 3].copy(),
        "momentum": series[:, 4:7].copy(),
    }
    return {"series": out, "final": system.with_positions(pos_out, vel_out), "steps": steps, "dt": dt}
