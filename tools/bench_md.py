"""Measure the rows either side of the mesh path on a BASELINE
configuration: the full device force evaluation (driver.compute_forces: pair +
mesh + self, host arrays in and out) and the device-resident velocity-Verlet
step (driver.integrate_nve), fp64 by default.

    python tools/bench_md.py [--config 2] [--calls 10] [--nve-steps 20] [--precision fp64|mixed]
    PYTHONPATH=/root/reference/pkg/src python tools/bench_md.py --reference   # build container only

Prints one JSON line.  Real-space cutoff 10 A (BASELINE configs 2 / 4).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--calls", type=int, default=10)
    ap.add_argument("--nve-steps", type=int, default=20)
    ap.add_argument("--cutoff", type=float, default=10.0)
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--reference", action="store_true", help="time the reference compute_forces (CPU) instead")
    args = ap.parse_args()
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[args.config]
    pos, q, lengths = cfg.build()
    n = pos.shape[0]
    line = {"what": "compute_forces (pair + mesh + self) and NVE step", "config": args.config, "n_atoms": n,
            "mesh": list(cfg.dims), "order": cfg.order, "mode": cfg.mode, "cutoff": args.cutoff,
            "alpha": cfg.alpha}
    if args.reference:
        import pppm

        box = pppm.SimulationBox(lengths)
        s = pppm.AtomSystem(box=box, positions=pos, charges=q, allow_net_charge=True)
        params = pppm.PppmParams(cutoff=args.cutoff, accuracy=1e-4, order=cfg.order, mode=pppm.DiffMode(cfg.mode),
                                 alpha=cfg.alpha, grid_dims=cfg.dims)
        counters = {}
        t0 = time.perf_counter()
        _, e, sections = pppm.compute_forces(s, params, counters=counters)
        dt = time.perf_counter() - t0
        line.update({"impl": "reference (CPU, 1 worker)", "compute_forces_s": dt, "atoms_per_s": n / dt,
                     "sections_s": sections, "pairs_within_cutoff": counters.get("pairs_within_cutoff"),
                     "energy_total": e.total})
        print(json.dumps(line))
        return

    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    box = pb.SimulationBox(lengths)
    s = pb.AtomSystem(box=box, positions=pos, charges=q, allow_net_charge=True)
    params = pb.PppmParams(cutoff=args.cutoff, accuracy=1e-4, order=cfg.order, mode=pb.DiffMode(cfg.mode),
                           alpha=cfg.alpha, grid_dims=cfg.dims, precision=args.precision)
    counters = {}
    f, e, _ = pb.compute_forces(s, params, counters=counters)
    f, e, sections = pb.compute_forces(s, params)
    times = []
    for _ in range(args.calls):
        t0 = time.perf_counter()
        f, e, _ = pb.compute_forces(s, params)
        times.append(time.perf_counter() - t0)
    tf = min(times)
    rng = np.random.default_rng(0)
    vel = rng.normal(scale=0.01, size=(n, 3))
    sv = pb.AtomSystem(box=box, positions=pos, charges=q, velocities=vel, allow_net_charge=True)
    pb.integrate_nve(sv, params, 1e-4, 2)
    t0 = time.perf_counter()
    out = pb.integrate_nve(sv, params, 1e-4, args.nve_steps)
    tn = time.perf_counter() - t0
    drift = float(np.max(np.abs(out["series"]["total_energy"] - out["series"]["total_energy"][0])))
    from paper_1702_04250_b200 import driver

    report = driver.make_report(sections=sections, wall_total=tf, n_atoms=n, params=params, steps=1, workers=1,
                                counters=counters)
    driver.validate_report(report)
    line.update({"impl": f"b200 ({args.precision})", "compute_forces_s": tf, "atoms_per_s": n / tf,
                 "report": report,
                 "pairs_within_cutoff": counters.get("pairs_within_cutoff", 0),
                 "energy_total": e.total, "nve_steps": args.nve_steps, "nve_s_per_step": tn / args.nve_steps,
                 "nve_atom_steps_per_s": n * args.nve_steps / tn, "nve_energy_drift": drift})
    print(json.dumps(line))


if __name__ == "__main__":
    main()
