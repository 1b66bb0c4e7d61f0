"""Pin the CPU oracle against outputs of the real reference (tests/golden)."""

import numpy as np
import pytest

from conftest import PIPELINE_CASES, load_golden, rel_rms
from oracle import pppm_oracle as orc


def test_stencil_rows_bitwise():
    g = load_golden("stencil")
    for order in (3, 5, 7):
        a, d = orc.bspline_rows(g["t"], order)
        assert np.array_equal(a, g[f"assign_{order}"])
        assert np.array_equal(d, g[f"deriv_{order}"])


def test_table_rows_and_bins_bitwise():
    g = load_golden("stencil")
    ta, td = orc.table_rows(5, 5000)
    assert np.array_equal(ta[g["table5_idx"]], g["table5_assign"])
    assert np.array_equal(td[g["table5_idx"]], g["table5_deriv"])
    a3, d3 = orc.table_rows(3, 4)
    assert np.array_equal(a3, g["table3x4_assign"])
    assert np.array_equal(d3, g["table3x4_deriv"])
    assert np.array_equal(orc.table_bin(g["bin_t"], 5000), g["bin_5000"])


def _table(g):
    return orc.table_rows(int(g["order"]), 5000) if bool(g["use_table"]) else None


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_particle_map_bitwise(case):
    g = load_golden(case)
    nodes, _ = orc.particle_map(g["pos"], g["lengths"], g["dims"], int(g["order"]))
    assert np.array_equal(nodes, g["nodes"])
    _, arows, _ = orc.stencil_weights(g["pos"], g["lengths"], g["dims"], int(g["order"]), _table(g))
    assert np.array_equal(arows[0], g["ax"])
    assert np.array_equal(arows[2], g["az"])


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_pipeline_matches_reference(case):
    g = load_golden(case)
    order = int(g["order"])
    table = _table(g)
    rho = orc.map_charge(g["pos"], g["q"], g["lengths"], g["dims"], order, table)
    # same scatter order as the reference: bitwise
    assert np.array_equal(rho, g["rho"])
    green = orc.influence_pme(g["dims"], g["lengths"], float(g["alpha"]), order)
    assert np.array_equal(green, g["green"])
    e = orc.kspace_energy(rho, green, g["lengths"])
    assert abs(e - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))
    if str(g["mode"]) == "ik":
        fields = orc.poisson_ik(rho, green, orc.ik_vectors(g["dims"], g["lengths"]))
        for f, key in zip(fields, ("ex", "ey", "ez")):
            assert np.array_equal(f, g[key])
        forces = orc.fieldforce_ik(fields, g["pos"], g["q"], g["lengths"], g["dims"], order, table)
    else:
        phi = orc.poisson_ad(rho, green)
        assert np.array_equal(phi, g["phi"])
        forces = orc.fieldforce_ad(phi, g["pos"], g["q"], g["lengths"], g["dims"], order, table)
    assert rel_rms(forces, g["forces"]) <= 1e-14


def test_workers_reduction_close():
    g = load_golden("config1_exact")
    base = orc.map_charge(g["pos"], g["q"], g["lengths"], g["dims"], 5)
    for w in (2, 3, 8):
        split = orc.map_charge(g["pos"], g["q"], g["lengths"], g["dims"], 5, workers=w)
        assert np.abs(split - base).max() <= 1e-12 * max(1.0, np.abs(base).max())


def test_influence_variants():
    g = load_golden("influence")
    pme = orc.influence_pme(g["dims"], g["lengths"], float(g["alpha"]), int(g["order"]))
    assert np.array_equal(pme, g["pme"])
    opt = orc.influence_optimal(g["dims"], g["lengths"], float(g["alpha"]), int(g["order"]))
    assert np.allclose(opt, g["optimal"], rtol=1e-13, atol=0)
    ik = orc.ik_vectors(g["dims"], g["lengths"])
    for v, key in zip(ik, ("ik_x", "ik_y", "ik_z")):
        assert np.array_equal(v, g[key])


def test_even_order_extension_properties():
    """Orders 4/6 (not in the reference): partition of unity, first moment, derivative moment."""
    rng = np.random.default_rng(0)
    lengths = np.array([10.0, 10.0, 10.0])
    dims = (20, 20, 20)
    pos = rng.uniform(0, 10, (500, 3))
    for order in (4, 6):
        nodes, offs = orc.particle_map(pos, lengths, dims, order)
        a, d = orc.bspline_rows(offs[0], order)
        lo = nodes[0] - (order - 1) // 2
        idx = lo[:, None] + np.arange(order)[None, :]
        u = pos[:, 0] / 0.5
        assert np.abs(a[:, :order].sum(1) - 1).max() < 1e-14
        assert np.abs((a[:, :order] * idx).sum(1) - u).max() < 1e-12
        assert np.abs((d[:, :order] * idx).sum(1) - 1).max() < 1e-12
