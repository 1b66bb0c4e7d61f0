"""MD on the resident path (driver.py:310-376): positions
moved every step (update_positions / update_positions_async), atoms that left
their brick take the direct path, the residents are re-sorted automatically
above a mover fraction; the mixed-precision NVE driver keeps the atoms
resident.  Checked against fresh evaluations and the fp64 trajectory."""

import numpy as np
import pytest

from conftest import load_golden, rel_rms

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    yield pb
    pb.set_precision("fp64")


@pytest.mark.parametrize("mode", ["ik", "ad"])
@pytest.mark.parametrize("sync", [True, False])
def test_moving_residents_with_automatic_resort(pb, mode, sync):
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(11)
    n, edge = 60000, 64.0
    pos, q, lengths = scenarios.random_gas(n, 12, edge)
    q32 = q.astype(np.float32)
    ctx = pb.PppmContext((48, 48, 48), lengths, order=5, mode=mode, precision="mixed", alpha=0.3)
    ref = pb.PppmContext((48, 48, 48), lengths, order=5, mode=mode, precision="mixed", alpha=0.3)
    try:
        ctx.set_resort(0.03)
        ctx.load_atoms(scenarios.round_to_f32(pos, lengths), q32)
        cur = pos.copy()
        for step in range(12):
            cur = scenarios.wrap(cur + rng.normal(0.0, 0.35, cur.shape), lengths)
            p32 = scenarios.round_to_f32(cur, lengths)
            if sync:
                ctx.update_positions(p32)
            else:
                ctx.update_positions_async(p32)
            ctx.step()
            ctx.synchronize()
            if step % 4 == 3:
                f, e = ctx.forces(), ctx.energy()
                fr, er = ref.compute(p32, q32)
                assert rel_rms(f, fr) <= 3e-6, step
                assert abs(e - er) <= 3e-6 * abs(er)
        info = ctx.resident_info()
        assert info["resorts"] >= 1
        assert 0 <= info["movers"] < n
    finally:
        ctx.close()
        ref.close()


def test_enqueue_only_loop_still_resorts(pb):
    """A host that only enqueues (device positions, no synchronisation between
    steps) runs ahead of the device: the mover count of an update is consumed
    when its event has completed - a count in flight is kept, not re-recorded -
    so the automatic re-sort still happens, and the forces stay right."""
    import torch

    from paper_1702_04250_b200 import _native as nat
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(5)
    n, edge, steps = 200000, 96.0, 60
    pos, q, lengths = scenarios.random_gas(n, 13, edge)
    q32 = q.astype(np.float32)
    traj = np.empty((steps, n, 3), dtype=np.float32)
    cur = pos.copy()
    for i in range(steps):
        cur = scenarios.wrap(cur + rng.normal(0.0, 0.25, cur.shape), lengths)
        traj[i] = scenarios.round_to_f32(cur, lengths)
    dev = torch.from_numpy(traj).to("cuda:0")
    ctx = pb.PppmContext((64, 64, 64), lengths, order=5, mode="ik", precision="mixed", alpha=0.3)
    ref = pb.PppmContext((64, 64, 64), lengths, order=5, mode="ik", precision="mixed", alpha=0.3)
    try:
        ctx.set_resort(0.02)
        ctx.load_atoms(scenarios.round_to_f32(pos, lengths), q32)
        for i in range(steps):
            ctx.update_positions_async(dev[i].data_ptr(), mem=nat.DEVICE)
            ctx.step()
        ctx.synchronize()
        info = ctx.resident_info()
        assert info["resorts"] >= 1
        f, e = ctx.forces(), ctx.energy()
        fr, er = ref.compute(traj[-1], q32)
        assert rel_rms(f, fr) <= 3e-6
        assert abs(e - er) <= 3e-6 * abs(er)
    finally:
        ctx.close()
        ref.close()


def test_mixed_nve_resident_matches_fp64(pb):
    """integrate_nve in mixed precision (resident mesh path) follows the fp64
    (reference arithmetic) trajectory to fp32 accuracy."""
    g = load_golden("nve_gas")
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"],
                      masses=g["masses"], velocities=g["vel"])
    params64 = pb.PppmParams(cutoff=float(g["cutoff"]), accuracy=1e-4, order=5, mode=pb.DiffMode.IK,
                             alpha=float(g["alpha"]), grid_dims=tuple(int(d) for d in g["dims"]), use_table=False)
    params32 = pb.PppmParams(cutoff=float(g["cutoff"]), accuracy=1e-4, order=5, mode=pb.DiffMode.IK,
                             alpha=float(g["alpha"]), grid_dims=tuple(int(d) for d in g["dims"]), use_table=False,
                             precision="mixed")
    steps, dt = 20, float(g["dt"])
    a = pb.integrate_nve(s, params64, dt, steps)
    b = pb.integrate_nve(s, params32, dt, steps)
    ea, eb = a["series"]["total_energy"], b["series"]["total_energy"]
    assert np.abs(eb - ea).max() <= 1e-5 * np.abs(ea).max()
    assert rel_rms(b["final"].positions, a["final"].positions) <= 1e-6
