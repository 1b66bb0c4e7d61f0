"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side validation and error mapping, scenario generators, install()."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "pppm_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pppm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    from paper_1702_04250_b200 import _native

    return _native.load()


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 30
    for name in names:
        assert hasattr(lib, name), name


def test_prototypes_cover_header():
    from paper_1702_04250_b200 import _native

    assert sorted(_native.PROTOTYPES) == _declared()


def test_abi_version_and_no_device(lib):
    from paper_1702_04250_b200 import _native

    assert lib.pppm_abi_version() == 1
    n = ctypes.c_int(-1)
    lib.pppm_device_count(ctypes.byref(n))
    if _native.device_count() == 0:
        # no GPU here: the product path must fail loudly, never fall back to the CPU
        import paper_1702_04250_b200 as pb

        with pytest.raises(RuntimeError, match="no CPU fallback"):
            pb.build_table(5, 100)


def test_status_mapping(lib):
    from paper_1702_04250_b200 import _native
    from paper_1702_04250_b200.model import ConfigurationError

    with pytest.raises(ConfigurationError):
        _native.check(_native.ERR_CONFIG)
    with pytest.raises(ValueError):
        _native.check(_native.ERR_VALUE)
    with pytest.raises(RuntimeError):
        _native.check(_native.ERR_CUDA)
    from paper_1702_04250_b200.model import SingularityError

    with pytest.raises(SingularityError) as ei:
        _native.check(_native.ERR_SINGULAR)
    assert isinstance(ei.value.pair, tuple)
    _native.check(_native.OK)


def test_params_validation():
    from paper_1702_04250_b200 import ConfigurationError, DiffMode, PppmParams

    ok = PppmParams(cutoff=2.0, accuracy=1e-4, order=4, mode=DiffMode.IK, alpha=0.9, grid_dims=(8, 8, 8))
    assert ok.grid_dims == (8, 8, 8) and ok.force_scale == 1.0
    with pytest.raises(ConfigurationError):
        PppmParams(cutoff=2.0, accuracy=1e-4, order=7, mode=DiffMode.IK, alpha=0.9, grid_dims=(6, 16, 16))
    with pytest.raises(ConfigurationError):
        PppmParams(cutoff=2.0, accuracy=1e-4, order=8, mode=DiffMode.IK, alpha=0.9, grid_dims=(16,) * 3)
    with pytest.raises(ConfigurationError):
        PppmParams(cutoff=2.0, accuracy=1e-4, order=5, mode=DiffMode.IK, alpha=0.9, grid_dims=(16,) * 3,
                   precision="fp16")


def test_atom_system_wraps_and_checks_neutrality():
    from paper_1702_04250_b200 import AtomSystem, SimulationBox

    box = SimulationBox([2.0, 2.0, 2.0])
    s = AtomSystem(box=box, positions=[[2.5, -0.5, 1.0], [0.1, 0.2, 0.3]], charges=[1.0, -1.0])
    assert np.allclose(s.positions[0], [0.5, 1.5, 1.0])
    assert not s.positions.flags.writeable
    with pytest.raises(ValueError, match="neutral"):
        AtomSystem(box=box, positions=[[0.1, 0.1, 0.1]], charges=[1.0])


def test_random_gas_matches_reference_generator():
    from paper_1702_04250_b200 import scenarios

    g = load_golden("config1_exact")
    pos, q, _ = scenarios.random_gas(4096, 1, 20.0)
    assert np.array_equal(pos[:4090], g["pos"][6:])


def test_water_geometry():
    from paper_1702_04250_b200 import scenarios

    pos, q, lengths = scenarios.water(200, 2, 3)
    assert pos.shape == (602, 3) and abs(q.sum()) < 1e-12
    assert np.all(pos >= 0) and np.all(pos < lengths)
    o, h1, h2 = pos[0:600:3], pos[1:600:3], pos[2:600:3]

    def mi(d):
        return d - np.round(d / lengths) * lengths

    d1, d2 = mi(h1 - o), mi(h2 - o)
    assert np.allclose(np.linalg.norm(d1, axis=1), 1.0)
    ang = np.degrees(np.arccos(np.sum(d1 * d2, 1) / (np.linalg.norm(d1, axis=1) * np.linalg.norm(d2, axis=1))))
    assert np.allclose(ang, 109.47)
    assert np.isclose((200 / lengths.prod()), scenarios.WATER_DENSITY)


def test_configs_shapes():
    from paper_1702_04250_b200 import scenarios

    c = scenarios.CONFIGS
    assert c[1].n_atoms == 4096 and c[3].n_atoms == 1 << 20 and c[5].n_atoms == 1 << 23
    pos, q, lengths = c[2].build()
    assert pos.shape == (32000, 3) and np.count_nonzero(q) == 31998
    assert abs(c[3].alpha - 0.2731551) < 1e-6
    p32 = scenarios.round_to_f32(np.array([[np.nextafter(10.0, 0.0), 1.0, 2.0]]), np.array([10.0] * 3))
    assert p32.dtype == np.float32 and np.all(p32.astype(np.float64) < 10.0)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present")
def test_install_rebinds_reference_names():
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import pppm
        import pppm.driver
        import paper_1702_04250_b200 as pb

        orig = pppm.driver.map_charge
        names = pb.install(pppm)
        assert "map_charge" in names and "poisson_ik" in names
        assert pppm.map_charge is pb.map_charge
        assert pppm.driver.map_charge is pb.map_charge
        assert pppm.gridmap.distribute_force_ad is pb.distribute_force_ad
        assert pppm.kspace.kspace_energy is pb.kspace_energy
        # the force driver either side of the path
        assert "compute_forces" in names and "pair_forces" in names
        assert pppm.compute_forces is pb.compute_forces
        assert pppm.driver.integrate_nve is pb.integrate_nve
        assert pppm.shortrange.pair_forces is pb.pair_forces
        from paper_1702_04250_b200 import _native, _runtime

        assert _native.ERRORS.singular is pppm.model.SingularityError
        assert _runtime.types().EnergyBreakdown is pppm.model.EnergyBreakdown
        pb.uninstall()
        assert pppm.driver.map_charge is orig
        assert pppm.driver.compute_forces is not pb.compute_forces
        assert _native.ERRORS.singular is None
        mesh_only = pb.install(pppm, force_driver=False)
        assert "compute_forces" not in mesh_only and pppm.driver.compute_forces is not pb.compute_forces
        pb.uninstall()
    finally:
        sys.path.remove("/root/reference/pkg/src")
