"""CPU: the oracle's pair / force-driver / NVE restatement (oracle/pppm_oracle.py)
pinned against the reference's own outputs (tests/golden/make_golden_md.py), and
the host-side validation of the drop-in shortrange / driver mirrors."""

import numpy as np
import pytest

from conftest import load_golden, rel_rms
from oracle import pppm_oracle as orc


def _lj(g):
    v = g["lj"]
    return (float(v[0]), float(v[1]), float(v[2])) if v[3] > 0 else None


@pytest.mark.parametrize("name", ["pair_gas", "pair_box_lj"])
def test_pair_oracle_matches_reference(name):
    g = load_golden(name)
    f, e, within = orc.pair_forces(g["pos"], g["q"], g["lengths"], float(g["alpha"]), float(g["cutoff"]), _lj(g),
                                   float(g["cc"]), float(g["diel"]))
    assert rel_rms(f, g["forces"]) <= 1e-13
    assert abs(e - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
    assert within == int(g["within"])
    assert abs(orc.self_energy(g["q"], float(g["alpha"]), float(g["cc"]), float(g["diel"])) - float(g["self_energy"])) \
        <= 1e-14 * abs(float(g["self_energy"]))


@pytest.mark.parametrize("name", ["forces_gas_ik", "forces_gas_ad_lj"])
def test_compute_forces_oracle_matches_reference(name):
    g = load_golden(name)
    order = int(g["order"])
    table = orc.table_rows(order, 5000) if bool(g["use_table"]) else None
    f, (ep, ek, es) = orc.compute_forces(g["pos"], g["q"], g["lengths"], tuple(g["dims"]), order, float(g["alpha"]),
                                         float(g["cutoff"]), str(g["mode"]), table, _lj(g))
    assert rel_rms(f, g["forces"]) <= 1e-12
    for a, b in ((ep, g["e_pair"]), (ek, g["e_kspace"]), (es, g["e_self"])):
        assert abs(a - float(b)) <= 1e-11 * abs(float(b))


def test_nve_oracle_matches_reference():
    g = load_golden("nve_gas")
    table = orc.table_rows(5, 5000)
    ser, pos, vel = orc.integrate_nve(g["pos"], g["vel"], g["masses"], g["q"], g["lengths"], tuple(g["dims"]), 5,
                                      float(g["alpha"]), float(g["cutoff"]), float(g["dt"]), int(g["steps"]),
                                      "ik", table)
    ref = np.column_stack([g["total"], g["kinetic"], g["potential"], g["temperature"], g["momentum"]])
    scale = np.maximum(np.abs(ref), 1e-12).max(axis=0)
    assert np.max(np.abs(ser - ref) / scale) <= 1e-10
    assert np.max(np.abs(pos - g["final_pos"])) <= 1e-11
    assert rel_rms(vel, g["final_vel"]) <= 1e-10


def test_host_validation_of_pair_mirrors():
    import paper_1702_04250_b200 as pb

    with pytest.raises(ValueError):
        pb.LjParams(epsilon=-1.0, enabled=True)
    with pytest.raises(ValueError):
        pb.LjParams(sigma=0.0, enabled=True)
    box = pb.SimulationBox([6.0, 9.0, 13.0])
    s = pb.AtomSystem(box=box, positions=[[1.0, 1.0, 1.0], [2.0, 2.0, 2.0]], charges=[1.0, -1.0])
    assert pb.build_cell_list(s, 3.0).dims == (2, 3, 4)
    with pytest.raises(pb.ConfigurationError):
        pb.build_cell_list(s, 3.5)
    with pytest.raises(pb.ConfigurationError):
        pb.build_cell_list(s, 0.0)
    assert s.masses.tolist() == [1.0, 1.0] and s.velocities is None
    s2 = s.with_positions([[7.0, 1.0, 1.0], [2.0, 2.0, 2.0]], np.zeros((2, 3)))
    assert s2.positions[0, 0] == pytest.approx(1.0) and s2.velocities.shape == (2, 3)
    e = pb.EnergyBreakdown(pair=1.0, kspace=2.0, self_energy=-0.5)
    assert e.total == 2.5
    err = pb.SingularityError(3, 5, 1e-12)
    assert err.pair == (3, 5) and "overlap" in str(err)
    with pytest.raises(ValueError):
        pb.integrate_nve(s, None, 1e-3, 1)  # no velocities
