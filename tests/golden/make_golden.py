"""Generate the golden parity fixtures from the REAL reference package.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` files next to this script.  Every array in them is an
output of the reference's own public/internal functions
(``pppm.stencil``, ``pppm.gridmap``, ``pppm.kspace``) on seeded inputs; the
inputs are stored alongside so the GPU parity tests and the oracle checks
replay exactly the same data.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import pppm  # noqa: E402  (the reference)
from pppm import stencil as rstencil  # noqa: E402
from pppm import gridmap as rgrid  # noqa: E402
from pppm import kspace as rk  # noqa: E402
from paper_1702_04250_b200 import scenarios  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def stencil_fixture():
    rng = np.random.default_rng(100)
    t = np.concatenate([
        [-0.5, np.nextafter(-0.5, 1.0), -0.25, 0.0, 0.25, np.nextafter(0.5, 0.0), 1e-300, -1e-17],
        rng.uniform(-0.5, 0.5, 248),
    ])
    out = {"t": t}
    for order in (3, 5, 7):
        a, d = rstencil.weight_rows(t, order)
        out[f"assign_{order}"] = a
        out[f"deriv_{order}"] = d
    tab = rstencil.build_table(5, 5000)
    idx = rng.integers(0, 5000, 64)
    out["table5_idx"] = idx
    out["table5_assign"] = tab.assignment[idx]
    out["table5_deriv"] = tab.derivative[idx]
    tab3 = rstencil.build_table(3, 4)
    out["table3x4_assign"] = tab3.assignment
    out["table3x4_deriv"] = tab3.derivative
    tb = np.concatenate([[-0.5, -0.25, 0.0, 0.25, np.nextafter(0.5, 0.0), -0.3749999999],
                         rng.uniform(-0.5, 0.5, 58)])
    out["bin_t"] = tb
    out["bin_5000"] = tab.bin_index(tb)
    save("stencil", **out)


def params_for(dims, order, mode, alpha, use_table, cutoff=2.0):
    return pppm.PppmParams(cutoff=cutoff, accuracy=1e-4, order=order,
                           mode=pppm.DiffMode(mode), alpha=alpha,
                           grid_dims=tuple(dims), use_table=use_table)


def pipeline_case(name, pos, q, lengths, dims, order, mode, alpha, use_table,
                  store_green=True, influence="pme"):
    box = pppm.SimulationBox(lengths)
    system = pppm.AtomSystem(box=box, positions=pos, charges=q,
                             allow_net_charge=abs(float(np.sum(q))) > 1e-12 * np.abs(q).sum())
    params = params_for(dims, order, mode, alpha, use_table)
    table = pppm.build_table(order, 5000) if use_table else None
    nodes, arows, drows = rgrid._stencil_rows(system, params, table)
    counters = {}
    rho = pppm.map_charge(system, params, table, counters=counters)
    plan = pppm.build_plan(dims, box, alpha, order, influence=influence)
    energy = pppm.kspace_energy(rho, plan)
    out = dict(
        pos=system.positions, q=system.charges, lengths=np.asarray(lengths, dtype=np.float64),
        dims=np.asarray(dims), order=np.int64(order), mode=np.array(mode), alpha=np.float64(alpha),
        use_table=np.bool_(use_table), nodes=np.stack(nodes), rho=rho.values, energy=np.float64(energy),
        cells_touched_map=np.int64(counters["cells_touched_map"]),
        ax=arows[0], ay=arows[1], az=arows[2],
    )
    if store_green:
        out["green"] = plan.influence
    if mode == "ik":
        fields = pppm.poisson_ik(rho, plan)
        out.update(ex=fields.ex, ey=fields.ey, ez=fields.ez)
        forces = pppm.distribute_force_ik(fields, system, params, table)
    else:
        fields = pppm.poisson_ad(rho, plan)
        out.update(phi=fields.phi)
        forces = pppm.distribute_force_ad(fields, system, params, table)
    out["forces"] = forces
    save(name, **out)


def main():
    stencil_fixture()

    # particle_map edge cases: node == n before wrap, exact half-cell points,
    # values one ulp below L and at 0, plus config-1-like random atoms.
    lengths = np.array([20.0, 20.0, 20.0])
    h = 20.0 / 16
    edge = np.array([
        [19.9, 0.0, 10.0],
        [np.nextafter(20.0, 0.0), 0.625, 1.875],
        [h * 3.5, h * 0.5, h * 15.5],
        [np.nextafter(h * 0.5, 0.0), np.nextafter(h * 0.5, 1.0), 1e-300],
        [5.0, 7.5, 12.5],
        [0.3125 * 3, 19.375, np.nextafter(19.375, 20.0)],
    ])
    gpos, gq, _ = scenarios.random_gas(4096, 1, 20.0)
    pos = np.concatenate([edge, gpos[: 4096 - edge.shape[0]]])
    q = np.where(np.arange(pos.shape[0]) % 2 == 0, 1.0, -1.0)
    pipeline_case("config1_exact", pos, q, lengths, (16, 16, 16), 5, "ik", 0.30, False)
    pipeline_case("config1_table", pos, q, lengths, (16, 16, 16), 5, "ik", 0.30, True)

    # non-cubic box, mixed odd/even dims, every odd order, both modes, both weight modes
    rng = np.random.default_rng(7)
    lengths = np.array([7.0, 8.0, 9.0])
    pos = rng.uniform(0, 1, (200, 3)) * lengths
    q = np.where(np.arange(200) % 2 == 0, 1.0, -1.0)
    pipeline_case("box_s3_ad_table", pos, q, lengths, (12, 14, 15), 3, "ad", 0.9, True)
    pipeline_case("box_s3_ik_exact", pos, q, lengths, (12, 14, 15), 3, "ik", 0.9, False)
    pipeline_case("box_s7_ik_table", pos, q, lengths, (12, 14, 15), 7, "ik", 0.9, True)
    pipeline_case("box_s7_ad_exact", pos, q, lengths, (12, 14, 15), 7, "ad", 0.9, False)
    pipeline_case("box_s5_ad_exact", pos, q, lengths, (13, 14, 16), 5, "ad", 0.9, False)

    # fp32-representable positions (mixed-precision parity input), config-3-like density
    n = 2048
    edge_len = (n / 0.1) ** (1.0 / 3.0)
    gpos, gq, glen = scenarios.random_gas(n, 3, edge_len)
    p32 = scenarios.round_to_f32(gpos, glen).astype(np.float64)
    pipeline_case("mixed_gas_ik", p32, gq, glen, (16, 16, 16), 5, "ik", scenarios.ALPHA_10A, False)
    pipeline_case("mixed_gas_ad", p32, gq, glen, (16, 16, 16), 5, "ad", scenarios.ALPHA_10A, False)

    # water-like molecules (config-2-like geometry, small), ad, non-unit charges
    wpos, wq, wlen = scenarios.water(300, 2, 2)
    pipeline_case("water_s5_ad", wpos, wq, wlen, (20, 20, 20), 5, "ad", 0.5, False)
    pipeline_case("water_s5_ik_table", wpos, wq, wlen, (20, 20, 20), 5, "ik", 0.5, True)

    # optimal (alias-summed) influence variant
    box = pppm.SimulationBox([5.0, 6.0, 7.0])
    plan = pppm.build_plan((10, 12, 9), box, 1.1, 5, influence="optimal")
    pme = pppm.build_plan((10, 12, 9), box, 1.1, 5)
    save("influence", lengths=np.array([5.0, 6.0, 7.0]), dims=np.array([10, 12, 9]),
         alpha=np.float64(1.1), order=np.int64(5), optimal=plan.influence, pme=pme.influence,
         ik_x=pme.ik_x, ik_y=pme.ik_y, ik_z=pme.ik_z)


if __name__ == "__main__":
    main()
