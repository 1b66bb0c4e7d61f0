"""GPU checks of drop-in API details beyond the numerics of the hot path:
the plan's transform pair (kspace.py:244), a caller-supplied transform pair
(build_plan(fft=...), kspace.py:207), the measured imag_residue
(kspace.py:264-268), NVE report sections / counters (driver.py:310-376),
graph invalidation when one-shot calls regrow the binning buffers, and the
mixed-precision grid-size limit."""

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


def test_plan_transforms_round_trip(pb):
    """test_kspace.py:105-112 restated: backward(forward(v)) == v, and the device
    pair has numpy's fftn / ifftn semantics."""
    box = pb.SimulationBox([5.0, 5.0, 5.0])
    plan = pb.build_plan((16, 12, 10), box, 1.0, 3)
    rng = np.random.default_rng(1)
    for _ in range(3):
        v = rng.normal(size=(10, 12, 16))
        fw = plan.forward(v)
        assert np.abs(fw - np.fft.fftn(v)).max() <= 1e-12 * np.abs(fw).max()
        back = plan.backward(fw)
        assert np.abs(back - v).max() <= 1e-12 * np.abs(v).max()
        assert np.abs(back - np.fft.ifftn(fw)).max() <= 1e-12 * np.abs(v).max()
    x = rng.normal(size=37) + 1j * rng.normal(size=37)
    assert np.abs(plan.forward(x) - np.fft.fftn(x)).max() <= 1e-12 * np.abs(x).sum()


@pytest.mark.parametrize("case", ["config1_exact", "box_s7_ad_exact"])
def test_custom_transform_pair_is_honoured(pb, case):
    """build_plan(fft=(fwd, bwd)): the solve runs the caller's transforms and
    gives the same fields / energy as the device transforms."""
    g = load_golden(case)
    box = pb.SimulationBox(g["lengths"])
    system = pb.AtomSystem(box=box, positions=g["pos"], charges=g["q"])
    dims = tuple(int(d) for d in g["dims"])
    order, alpha, mode = int(g["order"]), float(g["alpha"]), str(g["mode"])
    params = pb.PppmParams(cutoff=2.0, accuracy=1e-4, order=order, mode=pb.DiffMode(mode), alpha=alpha,
                           grid_dims=dims, use_table=False)
    rho = pb.map_charge(system, params)
    calls = {"fwd": 0, "bwd": 0}

    def fwd(a):
        calls["fwd"] += 1
        return np.fft.fftn(a)

    def bwd(a):
        calls["bwd"] += 1
        return np.fft.ifftn(a)

    dev = pb.build_plan(dims, box, alpha, order)
    cus = pb.build_plan(dims, box, alpha, order, fft=(fwd, bwd))
    assert cus.forward is fwd and cus.backward is bwd
    solve = pb.poisson_ik if mode == "ik" else pb.poisson_ad
    fd, fc = solve(rho, dev), solve(rho, cus)
    names = ("ex", "ey", "ez") if mode == "ik" else ("phi",)
    for name in names:
        assert rel_rms(getattr(fc, name), getattr(fd, name)) <= 1e-12
        assert rel_rms(getattr(fc, name), g[name if name != "phi" else "phi"]) <= 1e-10
    assert calls["fwd"] == 1 and calls["bwd"] == len(names)
    e_d, e_c = pb.kspace_energy(rho, dev), pb.kspace_energy(rho, cus)
    assert abs(e_c - e_d) <= 1e-12 * abs(e_d)
    assert 0.0 <= fc.imag_residue <= 1e-10


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_imag_residue_measured(pb, precision):
    """imag_residue is measured from a complex back transform (kspace.py:264-268):
    rounding-level, bounded as in test_kspace.py:160."""
    g = load_golden("config1_exact")
    box = pb.SimulationBox(g["lengths"])
    system = pb.AtomSystem(box=box, positions=g["pos"], charges=g["q"])
    pb.set_precision(precision)
    try:
        for mode in ("ik", "ad"):
            params = pb.PppmParams(cutoff=2.0, accuracy=1e-4, order=5, mode=pb.DiffMode(mode), alpha=0.3,
                                   grid_dims=(16, 16, 16), use_table=False, precision=precision)
            rho = pb.map_charge(system, params)
            plan = pb.build_plan((16, 16, 16), box, 0.3, 5)
            f = pb.poisson_ik(rho, plan) if mode == "ik" else pb.poisson_ad(rho, plan)
            bound = 1e-10 if precision == "fp64" else 1e-5
            assert 0.0 <= f.imag_residue <= bound
            if precision == "fp64":
                ref = g["ex"] if mode == "ik" else None
                if ref is not None:
                    assert rel_rms(f.ex, ref) <= 1e-10
    finally:
        pb.set_precision("fp64")


class _Timer:
    def __init__(self):
        self.seconds = {}

    def add(self, name, dt):
        self.seconds[name] = self.seconds.get(name, 0.0) + dt


def test_nve_report_sections_and_counters(pb):
    """integrate_nve accumulates the reference's report sections and per-step
    counters (driver.py:310-376), as its compute_forces calls would."""
    g = load_golden("nve_gas")
    s = pb.AtomSystem(box=pb.SimulationBox(g["lengths"]), positions=g["pos"], charges=g["q"],
                      masses=g["masses"], velocities=g["vel"])
    params = pb.PppmParams(cutoff=float(g["cutoff"]), accuracy=1e-4, order=5, mode=pb.DiffMode.IK,
                           alpha=float(g["alpha"]), grid_dims=tuple(int(d) for d in g["dims"]))
    steps = int(g["steps"])
    timer, counters = _Timer(), {}
    out = pb.integrate_nve(s, params, float(g["dt"]), steps, timer=timer, counters=counters)
    assert np.abs(out["series"]["total_energy"] - g["total"]).max() <= 1e-9 * np.abs(g["total"]).max()
    for name in ("pair", "pppm_fft", "pppm_non_fft"):
        assert timer.seconds[name] > 0.0
    assert "other" in timer.seconds and "device" not in timer.seconds
    n = len(g["q"])
    assert counters["cells_touched_map"] == (steps + 1) * n * 125
    assert counters["cells_touched_distribute"] == (steps + 1) * n * 125
    # the pair counters sum over the steps + 1 evaluations: compare with one
    # compute_forces on the initial state times a lower bound
    one = {}
    pb.compute_forces(s, params, counters=one)
    assert counters["pair_candidates"] >= one["pair_candidates"]
    assert counters["pairs_within_cutoff"] > 0


@pytest.mark.parametrize("big_n", [60000, 300000])
def test_one_shot_call_regrowing_bins_keeps_resident_step(pb, big_n):
    """A one-shot compute with more atoms regrows the binning buffers (300,000
    atoms: in two atom groups with their own slots); the resident step's
    captured graphs must be re-captured, not replayed on freed memory."""
    from paper_1702_04250_b200 import scenarios

    pos, q, lengths = scenarios.random_gas(4000, 31, 24.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext((24, 24, 24), lengths, order=5, mode="ik", precision="mixed", alpha=0.4)
    try:
        ctx.load_atoms(p32, q.astype(np.float32))
        for _ in range(3):  # eager, capture, replay
            ctx.step()
        ctx.synchronize()
        f0 = ctx.forces()
        big, qb, _ = scenarios.random_gas(big_n, 32, 24.0)
        ctx.compute(scenarios.round_to_f32(big, lengths), qb.astype(np.float32))
        for _ in range(2):
            ctx.step()
        ctx.synchronize()
        f1 = ctx.forces()
    finally:
        ctx.close()
    assert rel_rms(f1, f0) <= 1e-6
    f_ref, _, _ = orc.pppm_step(p32.astype(np.float64), q, lengths, (24, 24, 24), 5, 0.4, "ik")
    assert rel_rms(f1, f_ref) <= 1e-5


def test_mixed_grid_limit(pb):
    with pytest.raises(pb.ConfigurationError, match="1024"):
        pb.PppmContext((2048, 8, 8), (2048.0, 8.0, 8.0), order=5, mode="ik", precision="mixed", alpha=0.3)


@pytest.mark.parametrize("groups", ["1", "4"])
@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_compute_chunked_h2d_and_fp32_forces(pb, mode, groups, monkeypatch):
    """pppm_compute_ex: host atoms in groups of the caller's order (each binned
    into its own brick slots and spread as it lands, forces copied back group
    by group; 400,006 atoms -> 3 groups with a ragged last one) or, with
    PPPM_B200_GROUPS=1, binned chunk by chunk into one set of slots; forces
    returned as fp64 or fp32; same result as the resident step and the oracle."""
    from paper_1702_04250_b200 import scenarios

    monkeypatch.setenv("PPPM_B200_GROUPS", groups)
    pos, q, lengths = scenarios.random_gas(400006, 41, 160.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    q32 = q.astype(np.float32)
    ctx = pb.PppmContext((64, 64, 64), lengths, order=5, mode=mode, precision="mixed", alpha=0.25)
    try:
        f64, e64 = ctx.compute(p32, q32)
        f32, e32 = ctx.compute(p32, q32, out=np.empty((q.size, 3), dtype=np.float32))
        ctx.load_atoms(p32, q32)
        ctx.step()
        ctx.synchronize()
        fr = ctx.forces()
    finally:
        ctx.close()
    assert f32.dtype == np.float32
    assert rel_rms(f32, f64) <= 1e-6 and abs(e32 - e64) <= 1e-6 * abs(e64)
    assert rel_rms(f64, fr) <= 1e-6
    sub = np.random.default_rng(3).choice(q.size, 4096, replace=False)
    rho_ref = orc.map_charge(p32.astype(np.float64), q, lengths, (64, 64, 64), 5, workers=8)
    g = orc.influence_pme((64, 64, 64), lengths, 0.25, 5)
    if mode == "ik":
        fields = orc.poisson_ik(rho_ref, g, orc.ik_vectors((64, 64, 64), lengths))
        f_ref = orc.fieldforce_ik(fields, p32[sub].astype(np.float64), q[sub], lengths, (64, 64, 64), 5)
    else:
        phi = orc.poisson_ad(rho_ref, g)
        f_ref = orc.fieldforce_ad(phi, p32[sub].astype(np.float64), q[sub], lengths, (64, 64, 64), 5)
    assert rel_rms(f64[sub], f_ref) <= 1e-5


def test_compute_groups_at_config5_size(pb):
    """pppm_compute_ex in four atom groups at BASELINE config 5's size (8,388,608
    atoms, 256^3): same forces and energy as the resident step on the same atoms
    (whose parity against the oracle tests/test_configs_gpu.py checks)."""
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[5]
    pos, q, lengths = cfg.build()
    p32 = scenarios.round_to_f32(pos, lengths)
    q32 = q.astype(np.float32)
    ctx = pb.PppmContext(cfg.dims, lengths, order=cfg.order, mode=cfg.mode, precision="mixed", alpha=cfg.alpha)
    try:
        f, e = ctx.compute(p32, q32, out=np.empty((q.size, 3), dtype=np.float32))
        ctx.load_atoms(p32, q32)
        ctx.step()
        ctx.synchronize()
        fr, er = ctx.forces(), ctx.energy()
    finally:
        ctx.close()
    assert rel_rms(f, fr) <= 2e-6
    assert abs(e - er) <= 2e-6 * abs(er)
