"""GPU parity of the rows either side of the mesh path: device pair
forces (shortrange.pair_forces), the full force evaluation
(driver.compute_forces) and the device NVE trajectory (driver.integrate_nve)
through the C ABI, against the reference's golden outputs
(tests/golden/make_golden_md.py) and the CPU oracle.  fp64: 1e-10."""

import numpy as np
import pytest

from conftest import load_golden, rel_rms
from oracle import pppm_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    pb.set_precision("fp64")
    yield pb
    pb.set_precision("fp64")


def _lj(pb, g):
    v = g["lj"]
    return pb.LjParams(epsilon=float(v[0]), sigma=float(v[1]), cutoff=float(v[2]), enabled=bool(v[3] > 0))


def _params(pb, g, precision="fp64"):
    return pb.PppmParams(cutoff=float(g["cutoff"]), accuracy=1e-4, order=int(g["order"]),
                         mode=pb.DiffMode(str(g["mode"])), alpha=float(g["alpha"]), grid_dims=tuple(g["dims"]),
                         use_table=bool(g["use_table"]), precision=precision)


@pytest.mark.parametrize("name", ["pair_gas", "pair_box_lj", "pair_floordiv"])
def test_pair_forces_vs_reference(pb, name):
    g = load_golden(name)
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"])
    cells = pb.build_cell_list(s, float(g["cutoff"]))
    assert cells.dims == tuple(int(v) for v in g["cell_dims"])
    counters = {}
    f, e = pb.pair_forces(s, cells, float(g["alpha"]), float(g["cutoff"]), _lj(pb, g),
                          coulomb_constant=float(g["cc"]), dielectric=float(g["diel"]), counters=counters)
    assert rel_rms(f, g["forces"]) <= 1e-12
    assert abs(e - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
    assert counters["pair_candidates"] == int(g["cand"])
    assert counters["pairs_within_cutoff"] == int(g["within"])
    # Newton's third law holds to rounding
    assert np.abs(f.sum(axis=0)).max() <= 1e-10 * np.abs(f).max()
    # bitwise reproducible
    f2, e2 = pb.pair_forces(s, cells, float(g["alpha"]), float(g["cutoff"]), _lj(pb, g),
                            coulomb_constant=float(g["cc"]), dielectric=float(g["diel"]))
    assert np.array_equal(f, f2) and e == e2


@pytest.mark.parametrize("name", ["forces_gas_ik", "forces_gas_ad_lj"])
def test_compute_forces_vs_reference(pb, name):
    g = load_golden(name)
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"])
    lj = _lj(pb, g) if g["lj"][3] > 0 else None
    counters = {}
    f, e, sections = pb.compute_forces(s, _params(pb, g), lj=lj, counters=counters)
    assert rel_rms(f, g["forces"]) <= 1e-10
    assert abs(e.pair - float(g["e_pair"])) <= 1e-10 * abs(float(g["e_pair"]))
    assert abs(e.kspace - float(g["e_kspace"])) <= 1e-10 * abs(float(g["e_kspace"]))
    assert abs(e.self_energy - float(g["e_self"])) <= 1e-12 * abs(float(g["e_self"]))
    assert e.total == pytest.approx(float(g["e_pair"]) + float(g["e_kspace"]) + float(g["e_self"]), rel=1e-10)
    assert counters["pair_candidates"] == int(g["cand"]) and counters["pairs_within_cutoff"] == int(g["within"])
    assert set(sections) == {"pppm_non_fft", "pppm_fft", "pair"} and min(sections.values()) > 0.0
    from paper_1702_04250_b200 import driver

    rec = driver.make_report(sections=sections, wall_total=sum(sections.values()) * 1.5, n_atoms=len(g["q"]),
                             params=_params(pb, g), steps=1, workers=1, counters=counters)
    driver.validate_report(rec)


def test_compute_forces_mixed_precision(pb):
    g = load_golden("forces_gas_ik")
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"])
    f, e, _ = pb.compute_forces(s, _params(pb, g, precision="mixed"))
    assert rel_rms(f, g["forces"]) <= 1e-5
    assert abs(e.kspace - float(g["e_kspace"])) <= 1e-5 * abs(float(g["e_kspace"]))


def test_integrate_nve_vs_reference(pb):
    g = load_golden("nve_gas")
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"], masses=g["masses"],
                      velocities=g["vel"])
    params = pb.PppmParams(cutoff=float(g["cutoff"]), accuracy=1e-4, order=5, mode=pb.DiffMode.IK,
                           alpha=float(g["alpha"]), grid_dims=tuple(g["dims"]))
    out = pb.integrate_nve(s, params, float(g["dt"]), int(g["steps"]))
    ser = out["series"]
    for key, ref in (("total_energy", g["total"]), ("kinetic", g["kinetic"]), ("potential", g["potential"]),
                     ("temperature", g["temperature"])):
        assert np.max(np.abs(ser[key] - ref)) <= 1e-9 * np.abs(ref).max(), key
    assert np.max(np.abs(ser["momentum"] - g["momentum"])) <= 1e-9 * max(1.0, np.abs(g["momentum"]).max())
    assert np.max(np.abs(out["final"].positions - g["final_pos"])) <= 1e-10
    assert rel_rms(out["final"].velocities, g["final_vel"]) <= 1e-9
    assert out["steps"] == int(g["steps"]) and out["dt"] == float(g["dt"])


def test_pair_forces_vs_oracle_random_boxes(pb):
    rng = np.random.default_rng(5)
    for lengths, rc in (([7.0, 7.5, 20.0], 3.4), ([12.0, 12.0, 12.0], 2.5), ([9.0, 6.5, 8.0], 3.0)):
        n = 400
        pos = rng.uniform(0, 1, (n, 3)) * np.array(lengths)
        q = rng.normal(size=n)
        q -= q.mean()
        s = pb.AtomSystem(box=pb.SimulationBox(lengths), positions=pos, charges=q)
        f, e = pb.pair_forces(s, None, 0.7, rc)
        fo, eo, _ = orc.pair_forces(s.positions, q, np.array(lengths), 0.7, rc)
        assert rel_rms(f, fo) <= 1e-12
        assert abs(e - eo) <= 1e-12 * abs(eo)


def test_pair_singularity_and_validation(pb):
    box = pb.SimulationBox([10.0, 10.0, 10.0])
    s = pb.AtomSystem(box=box, positions=[[1.0, 1.0, 1.0], [5.0, 5.0, 5.0], [1.0, 1.0, 1.0 + 1e-12]],
                      charges=[1.0, -1.0, 0.0], allow_net_charge=True)
    with pytest.raises(pb.SingularityError) as ei:
        pb.pair_forces(s, None, 0.5, 3.0)
    assert ei.value.pair == (0, 2)
    assert ei.value.distance < 1e-10
    with pytest.raises(pb.ConfigurationError):
        pb.pair_forces(s, None, 0.5, 6.0)  # cutoff > L/2
    with pytest.raises(pb.ConfigurationError):
        pb.pair_forces(s, None, 0.0, 3.0)


def test_nve_step_error_prefix(pb):
    box = pb.SimulationBox([10.0, 10.0, 10.0])
    s = pb.AtomSystem(box=box, positions=[[1.0, 1.0, 1.0], [1.0, 1.0, 1.0]], charges=[1.0, -1.0],
                      velocities=np.zeros((2, 3)))
    params = pb.PppmParams(cutoff=3.0, accuracy=1e-4, order=5, mode=pb.DiffMode.IK, alpha=0.5,
                           grid_dims=(8, 8, 8))
    with pytest.raises(pb.SingularityError) as ei:
        pb.integrate_nve(s, params, 1e-3, 2)
    assert str(ei.value).startswith("step 0:")
