"""Golden fixtures for the rows either side of the mesh path:
shortrange.pair_forces, driver.compute_forces and driver.integrate_nve of the
REAL reference package.  Build container only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_md.py

Inputs are stored next to the outputs so the GPU tests replay them exactly.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import pppm  # noqa: E402  (the reference)
from pppm import driver as rdrv  # noqa: E402
from pppm import shortrange as rsr  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def pair_case(name, system, alpha, cutoff, lj=None, scale=(1.0, 1.0)):
    counters = {}
    cells = rsr.build_cell_list(system, cutoff)
    f, e = rsr.pair_forces(system, cells, alpha, cutoff, lj, coulomb_constant=scale[0], dielectric=scale[1],
                           counters=counters)
    ljv = np.array([lj.epsilon, lj.sigma, lj.cutoff, float(lj.enabled)]) if lj is not None else np.zeros(4)
    save(name, pos=system.positions, q=system.charges, lengths=system.box.lengths, alpha=np.float64(alpha),
         cutoff=np.float64(cutoff), lj=ljv, cc=np.float64(scale[0]), diel=np.float64(scale[1]), forces=f,
         energy=np.float64(e), cand=np.int64(counters["pair_candidates"]),
         within=np.int64(counters["pairs_within_cutoff"]), cell_dims=np.array(cells.dims),
         self_energy=np.float64(rsr.self_energy(system, alpha, coulomb_constant=scale[0], dielectric=scale[1])))


def params_for(dims, order, mode, alpha, cutoff, use_table=True):
    return pppm.PppmParams(cutoff=cutoff, accuracy=1e-4, order=order, mode=pppm.DiffMode(mode), alpha=alpha,
                           grid_dims=tuple(dims), use_table=use_table)


def forces_case(name, system, params, lj=None):
    counters = {}
    f, e, _ = rdrv.compute_forces(system, params, lj=lj, counters=counters)
    ljv = np.array([lj.epsilon, lj.sigma, lj.cutoff, float(lj.enabled)]) if lj is not None else np.zeros(4)
    save(name, pos=system.positions, q=system.charges, lengths=system.box.lengths, dims=np.array(params.grid_dims),
         order=np.int64(params.order), mode=np.array(params.mode.value), alpha=np.float64(params.alpha),
         cutoff=np.float64(params.cutoff), use_table=np.bool_(params.use_table), lj=ljv, forces=f,
         e_pair=np.float64(e.pair), e_kspace=np.float64(e.kspace), e_self=np.float64(e.self_energy),
         cand=np.int64(counters["pair_candidates"]), within=np.int64(counters["pairs_within_cutoff"]))


def main():
    # random gas, cubic box (>= 3 cells per axis), plain screened Coulomb
    s = rdrv.generate_scenario("random_gas", 600, seed=11)
    pair_case("pair_gas", s, 0.9, 3.0)
    # non-cubic box with 2 cells along x (deduplicated stencil), LJ on, C / eps != 1
    rng = np.random.default_rng(12)
    box = pppm.SimulationBox([6.2, 9.0, 13.0])
    pos = rng.uniform(0, 1, (300, 3)) * box.lengths
    q = np.where(np.arange(300) % 2 == 0, 0.7, -0.7)
    s2 = pppm.AtomSystem(box=box, positions=pos, charges=q)
    pair_case("pair_box_lj", s2, 1.1, 3.0, rsr.LjParams(epsilon=0.3, sigma=0.8, cutoff=2.5, enabled=True),
              scale=(2.0, 1.5))

    # cell counts where Python's int(L // rc) differs from a truncated L / rc
    # (1.0 // 0.1 == 9.0 but 1.0 / 0.1 == 10.0; 3.0 // 0.1 == 29.0)
    rng = np.random.default_rng(15)
    box = pppm.SimulationBox([1.0, 3.0, 2.1])
    pos = rng.uniform(0, 1, (400, 3)) * box.lengths
    q = np.where(np.arange(400) % 2 == 0, 1.0, -1.0)
    pair_case("pair_floordiv", pppm.AtomSystem(box=box, positions=pos, charges=q), 20.0, 0.1)

    # full force evaluation, both modes, table on (the reference's default)
    g = rdrv.generate_scenario("random_gas", 512, seed=13, min_separation=0.8)
    forces_case("forces_gas_ik", g, params_for((16, 16, 16), 5, "ik", 0.8, 3.0))
    forces_case("forces_gas_ad_lj", g, params_for((15, 16, 18), 7, "ad", 0.8, 3.0, use_table=False),
                lj=rsr.LjParams(epsilon=0.2, sigma=0.7, cutoff=2.0, enabled=True))

    # NVE: 128 ions with velocities, unequal masses, 6 steps
    nv = rdrv.generate_scenario("random_gas", 128, seed=14, min_separation=1.0, temperature=0.5)
    m = 1.0 + 0.5 * (np.arange(128) % 3)
    nv = pppm.AtomSystem(box=nv.box, positions=nv.positions, charges=nv.charges, masses=m,
                         velocities=nv.velocities)
    params = params_for((12, 12, 12), 5, "ik", 0.9, 3.0)
    out = rdrv.integrate_nve(nv, params, 2e-3, 6)
    ser = out["series"]
    save("nve_gas", pos=nv.positions, q=nv.charges, masses=nv.masses, vel=nv.velocities, lengths=nv.box.lengths,
         dims=np.array(params.grid_dims), order=np.int64(5), alpha=np.float64(0.9), cutoff=np.float64(3.0),
         dt=np.float64(2e-3), steps=np.int64(6), total=ser["total_energy"], kinetic=ser["kinetic"],
         potential=ser["potential"], temperature=ser["temperature"], momentum=ser["momentum"],
         final_pos=out["final"].positions, final_vel=out["final"].velocities)


if __name__ == "__main__":
    main()
