"""GPU parity: the sm_100a path through the C ABI vs the reference golden
vectors (tests/golden, made by the real reference) and the CPU oracle.

Bars (BASELINE.json north_star): particle_map bit-exact; fp64 forces / energy
1e-10 relative RMS; mixed precision 1e-5 relative RMS.
"""

import numpy as np
import pytest

from conftest import PIPELINE_CASES, load_golden, rel_rms
from oracle import pppm_oracle as orc

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10
MIXED_TOL = 1e-5


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    pb.set_precision("fp64")
    yield pb
    pb.set_precision("fp64")


def _system(pb, g):
    box = pb.SimulationBox(g["lengths"])
    net = abs(float(g["q"].sum())) > 1e-12 * np.abs(g["q"]).sum()
    return pb.AtomSystem(box=box, positions=g["pos"], charges=g["q"], allow_net_charge=net)


def _params(pb, g, precision="fp64"):
    return pb.PppmParams(cutoff=2.0, accuracy=1e-4, order=int(g["order"]),
                         mode=pb.DiffMode(str(g["mode"])), alpha=float(g["alpha"]),
                         grid_dims=tuple(int(d) for d in g["dims"]), use_table=bool(g["use_table"]),
                         precision=precision)


# --------------------------------------------------------------------------- stencil


def test_weight_rows_bitwise(pb):
    g = load_golden("stencil")
    for order in (3, 5, 7):
        a, d = pb.weight_rows(g["t"], order)
        assert np.array_equal(a, g[f"assign_{order}"])
        assert np.array_equal(d, g[f"deriv_{order}"])


def test_table_rows_bitwise(pb):
    g = load_golden("stencil")
    tab = pb.build_table(5, 5000)
    assert np.array_equal(tab.assignment[g["table5_idx"]], g["table5_assign"])
    assert np.array_equal(tab.derivative[g["table5_idx"]], g["table5_deriv"])
    t3 = pb.build_table(3, 4)
    assert np.array_equal(t3.assignment, g["table3x4_assign"])
    assert np.array_equal(t3.derivative, g["table3x4_deriv"])
    assert not tab.assignment.flags.writeable


def test_known_rows(pb):
    assert np.array_equal(pb.assignment_weights(0.0, 3), [0.125, 0.75, 0.125, 0, 0, 0, 0, 0])
    assert np.array_equal(pb.derivative_weights(0.0, 3), [-0.5, 0.0, 0.5, 0, 0, 0, 0, 0])
    with pytest.raises(ValueError, match="outside"):
        pb.assignment_weights(0.5, 3)


def test_even_order_rows_match_oracle(pb):
    t = np.random.default_rng(1).uniform(-0.5, 0.5, 500)
    for order in (4, 6):
        a, d = pb.weight_rows(t, order)
        ra, rd = orc.bspline_rows(t, order)
        assert np.array_equal(a, ra)
        assert np.array_equal(d, rd)


# --------------------------------------------------------------------------- particle_map


@pytest.mark.parametrize("case", PIPELINE_CASES)
def test_particle_map_bit_exact(pb, case):
    g = load_golden(case)
    nodes = pb.particle_map(_system(pb, g), _params(pb, g))
    assert nodes.dtype == np.int32
    assert np.array_equal(nodes.astype(np.int64), g["nodes"])


def test_particle_map_node_equals_n_prewrap(pb):
    g = load_golden("config1_exact")
    nodes = pb.particle_map(_system(pb, g), _params(pb, g))
    assert nodes.max() == 16  # x = 19.9 on a 16-mesh of a 20 A box maps to node 16 before wrap


def test_particle_map_mixed_rounds_to_fp32(pb):
    g = load_golden("mixed_gas_ik")
    params = _params(pb, g, "mixed")
    nodes = pb.particle_map(_system(pb, g), params)
    assert np.array_equal(nodes.astype(np.int64), g["nodes"])


# --------------------------------------------------------------------------- full pipeline fp64


def _run(pb, g, precision="fp64"):
    pb.set_precision(precision)
    try:
        system, params = _system(pb, g), _params(pb, g, precision)
        table = pb.build_table(params.order, 5000) if params.use_table else None
        rho = pb.map_charge(system, params, table)
        plan = pb.build_plan(params.grid_dims, system.box, params.alpha, params.order)
        energy = pb.kspace_energy(rho, plan)
        if params.mode is pb.DiffMode.IK:
            fields = pb.poisson_ik(rho, plan)
            forces = pb.distribute_force_ik(fields, system, params, table)
        else:
            fields = pb.poisson_ad(rho, plan)
            forces = pb.distribute_force_ad(fields, system, params, table)
    finally:
        pb.set_precision("fp64")
    return rho, fields, energy, forces, plan


FP64_CASES = [c for c in PIPELINE_CASES if not c.startswith("mixed")]


@pytest.mark.parametrize("case", FP64_CASES)
def test_pipeline_fp64_vs_reference(pb, case):
    g = load_golden(case)
    rho, fields, energy, forces, plan = _run(pb, g)
    assert rel_rms(rho.values, g["rho"]) <= 1e-12
    assert abs(energy - float(g["energy"])) <= FP64_TOL * abs(float(g["energy"]))
    keys = ("ex", "ey", "ez") if str(g["mode"]) == "ik" else ("phi",)
    for k in keys:
        assert rel_rms(getattr(fields, k), g[k]) <= FP64_TOL
    assert rel_rms(forces, g["forces"]) <= FP64_TOL
    assert not rho.values.flags.writeable
    assert forces.flags.writeable


@pytest.mark.parametrize("case", ["config1_exact", "box_s7_ad_exact"])
def test_poisson_from_reference_rho(pb, case):
    """Poisson alone, fed the reference's own charge grid."""
    g = load_golden(case)
    dims = tuple(int(d) for d in g["dims"])
    h = tuple(float(g["lengths"][d]) / dims[d] for d in range(3))
    rho = pb.ChargeGrid(dims=dims, spacing=h, values=g["rho"])
    plan = pb.build_plan(dims, pb.SimulationBox(g["lengths"]), float(g["alpha"]), int(g["order"]))
    assert rel_rms(plan.influence, g["green"]) <= 1e-14
    if str(g["mode"]) == "ik":
        f = pb.poisson_ik(rho, plan)
        for k in ("ex", "ey", "ez"):
            assert rel_rms(getattr(f, k), g[k]) <= 1e-12
    else:
        f = pb.poisson_ad(rho, plan)
        assert rel_rms(f.phi, g["phi"]) <= 1e-12
    assert abs(pb.kspace_energy(rho, plan) - float(g["energy"])) <= 1e-12 * abs(float(g["energy"]))


def test_influence_optimal_and_ik(pb):
    g = load_golden("influence")
    box = pb.SimulationBox(g["lengths"])
    dims = tuple(int(d) for d in g["dims"])
    opt = pb.build_plan(dims, box, float(g["alpha"]), int(g["order"]), influence="optimal")
    # alias sums partially cancel: compare against the grid's scale
    assert np.abs(opt.influence - g["optimal"]).max() <= 1e-12 * np.abs(g["optimal"]).max()
    pme = pb.build_plan(dims, box, float(g["alpha"]), int(g["order"]))
    assert np.allclose(pme.influence, g["pme"], rtol=1e-13, atol=0)
    for k in ("ik_x", "ik_y", "ik_z"):
        assert np.allclose(getattr(pme, k), g[k], rtol=1e-15, atol=0)


def test_determinism_bitwise(pb):
    g = load_golden("config1_table")
    a = _run(pb, g)
    b = _run(pb, g)
    assert np.array_equal(a[0].values, b[0].values)
    assert np.array_equal(a[3], b[3])
    assert a[2] == b[2]


# --------------------------------------------------------------------------- mixed precision


@pytest.mark.parametrize("case", ["mixed_gas_ik", "mixed_gas_ad"])
def test_pipeline_mixed_vs_reference(pb, case):
    g = load_golden(case)
    rho, fields, energy, forces, _ = _run(pb, g, "mixed")
    assert rel_rms(rho.values, g["rho"]) <= MIXED_TOL
    assert abs(energy - float(g["energy"])) <= MIXED_TOL * abs(float(g["energy"]))
    assert rel_rms(forces, g["forces"]) <= MIXED_TOL


@pytest.mark.parametrize("case", ["water_s5_ik_table", "box_s7_ik_table", "box_s3_ad_table"])
def test_pipeline_mixed_table_and_orders(pb, case):
    g = load_golden(case)
    _, _, energy, forces, _ = _run(pb, g, "mixed")
    # the golden positions are fp64; compare against the oracle on fp32-rounded inputs
    from paper_1702_04250_b200.scenarios import round_to_f32

    p32 = round_to_f32(g["pos"], g["lengths"]).astype(np.float64)
    table = orc.table_rows(int(g["order"]), 5000) if bool(g["use_table"]) else None
    f_ref, e_ref, _ = orc.pppm_step(p32, g["q"], g["lengths"], g["dims"], int(g["order"]),
                                    float(g["alpha"]), str(g["mode"]), table)
    assert rel_rms(forces, f_ref) <= MIXED_TOL
    assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref)


# --------------------------------------------------------------------------- even orders (extension)


@pytest.mark.parametrize("order", [4, 6])
@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_even_orders_vs_oracle(pb, order, mode):
    from paper_1702_04250_b200 import scenarios

    pos, q, lengths = scenarios.water(400, 1, 40 + order)
    dims = (20, 20, 20)
    g = dict(pos=pos, q=q, lengths=lengths, dims=np.array(dims), order=order, mode=np.array(mode),
             alpha=0.5, use_table=False)
    _, _, energy, forces, _ = _run(pb, g)
    f_ref, e_ref, _ = orc.pppm_step(pos, q, lengths, dims, order, 0.5, mode)
    assert rel_rms(forces, f_ref) <= FP64_TOL
    assert abs(energy - e_ref) <= FP64_TOL * abs(e_ref)


# --------------------------------------------------------------------------- known answers & invariants


def _mk(pb, order=7, dims=(16, 16, 16), mode="ik", use_table=True, alpha=0.9, precision="fp64"):
    return pb.PppmParams(cutoff=2.0, accuracy=1e-4, order=order, mode=pb.DiffMode(mode), alpha=alpha,
                         grid_dims=dims, use_table=use_table, precision=precision)


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_atom_on_node_order3(pb, precision):
    box = pb.SimulationBox([8.0] * 3)
    s = pb.AtomSystem(box=box, positions=[[2.0, 2.0, 2.0]], charges=[1.0], allow_net_charge=True)
    grid = pb.map_charge(s, _mk(pb, order=3, dims=(8, 8, 8), use_table=False, precision=precision))
    tol = 1e-12 if precision == "fp64" else 1e-6
    assert abs(grid.values[2, 2, 2] - 0.75 ** 3 / grid.cell_volume) <= tol * 0.75 ** 3
    assert np.count_nonzero(grid.values) == 27
    assert abs(grid.total_charge - 1.0) <= tol


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_coincident_opposite_charges_cancel(pb, precision):
    box = pb.SimulationBox([8.0] * 3)
    s = pb.AtomSystem(box=box, positions=[[1.3, 2.7, 3.1]] * 2, charges=[1.0, -1.0])
    tab = pb.build_table(5, 5000)
    grid = pb.map_charge(s, _mk(pb, order=5, precision=precision), tab)
    assert np.all(grid.values == 0.0)


def test_charge_conservation_and_counters(pb):
    rng = np.random.default_rng(0)
    params = _mk(pb, order=7, dims=(12, 12, 12))
    tab = pb.build_table(7, 5000)
    for _ in range(20):
        n = int(rng.integers(1, 30)) * 2
        edge = (n / 0.3) ** (1 / 3)
        s = pb.AtomSystem(box=pb.SimulationBox([edge] * 3), positions=rng.uniform(0, edge, (n, 3)),
                          charges=np.where(np.arange(n) % 2 == 0, 1.0, -1.0))
        counters = {}
        grid = pb.map_charge(s, params, tab, counters=counters)
        assert abs(grid.total_charge - s.net_charge) <= 1e-12 * n
        assert counters["cells_touched_map"] == n * 343


def test_linearity(pb):
    rng = np.random.default_rng(1)
    box = pb.SimulationBox([6.0] * 3)
    params = _mk(pb, order=5, dims=(12, 12, 12))
    tab = pb.build_table(5, 5000)
    pos = rng.uniform(0, 6, (40, 3))
    q1, q2 = rng.normal(size=40), rng.normal(size=40)

    def grid_for(q):
        s = pb.AtomSystem(box=box, positions=pos, charges=q, allow_net_charge=True)
        return pb.map_charge(s, params, tab).values

    assert np.abs(grid_for(q1 + q2) - (grid_for(q1) + grid_for(q2))).max() <= 1e-12


def test_translation_equivariance_bitwise(pb):
    box = pb.SimulationBox([8.0] * 3)
    params = _mk(pb, order=5, dims=(16, 16, 16))
    tab = pb.build_table(5, 5000)
    rng = np.random.default_rng(2)
    pos = rng.integers(0, 8 * (1 << 20), (30, 3)).astype(float) / (1 << 20)
    q = np.where(np.arange(30) % 2 == 0, 1.0, -1.0)
    shifted = pos.copy()
    shifted[:, 0] += 0.5
    g0 = pb.map_charge(pb.AtomSystem(box=box, positions=pos, charges=q), params, tab).values
    g1 = pb.map_charge(pb.AtomSystem(box=box, positions=shifted, charges=q), params, tab).values
    assert np.array_equal(g1, np.roll(g0, 1, axis=2))


@pytest.mark.parametrize("precision", ["fp64", "mixed"])
def test_constant_field_gives_qc(pb, precision):
    box = pb.SimulationBox([8.0] * 3)
    rng = np.random.default_rng(7)
    q = np.where(np.arange(20) % 2 == 0, 1.0, -1.0)
    s = pb.AtomSystem(box=box, positions=rng.uniform(0, 8, (20, 3)), charges=q)
    for order in (3, 4, 5, 6, 7):
        params = _mk(pb, order=order, precision=precision, use_table=False)
        grid = np.full((16, 16, 16), 2.5)
        fields = pb.FieldGrids(mode=pb.DiffMode.IK, dims=(16, 16, 16), spacing=(0.5,) * 3,
                               ex=grid, ey=grid, ez=grid)
        forces = pb.distribute_force_ik(fields, s, params)
        tol = 1e-12 if precision == "fp64" else 1e-5
        assert np.abs(forces - 2.5 * q[:, None]).max() <= tol


def test_ad_constant_and_ramp(pb):
    box = pb.SimulationBox([8.0] * 3)
    rng = np.random.default_rng(11)
    q = np.where(np.arange(20) % 2 == 0, 1.0, -1.0)
    s = pb.AtomSystem(box=box, positions=rng.uniform(0, 8, (20, 3)), charges=q)
    params = _mk(pb, order=7, mode="ad")
    tab = pb.build_table(7, 5000)
    f = pb.distribute_force_ad(pb.FieldGrids(mode=pb.DiffMode.AD, dims=(16, 16, 16), spacing=(0.5,) * 3,
                                             phi=np.full((16, 16, 16), 3.7)), s, params, tab)
    assert np.abs(f).max() <= 1e-12
    dims, h, slope = (32, 32, 32), 0.25, 0.75
    phi = np.tile(slope * np.arange(32) * h, (32, 32, 1))
    s2 = pb.AtomSystem(box=box, positions=rng.uniform(2.0, 6.0, (20, 3)), charges=q)
    params = _mk(pb, order=5, dims=dims, mode="ad")
    f = pb.distribute_force_ad(pb.FieldGrids(mode=pb.DiffMode.AD, dims=dims, spacing=(h,) * 3, phi=phi),
                               s2, params, pb.build_table(5, 5000))
    assert np.abs(f[:, 0] + q * slope).max() <= 1e-10
    assert np.abs(f[:, 1:]).max() <= 1e-10


def test_ik_momentum_conservation(pb):
    for seed in range(3):
        n = 96
        rng = np.random.default_rng(seed)
        edge = (n / 1.0) ** (1 / 3)
        s = pb.AtomSystem(box=pb.SimulationBox([edge] * 3), positions=rng.uniform(0, edge, (n, 3)),
                          charges=np.where(np.arange(n) % 2 == 0, 1.0, -1.0))
        params = _mk(pb, order=7, dims=(18, 18, 18), alpha=1.1)
        tab = pb.build_table(7, 5000)
        rho = pb.map_charge(s, params, tab)
        plan = pb.build_plan(params.grid_dims, s.box, params.alpha, params.order)
        f = pb.distribute_force_ik(pb.poisson_ik(rho, plan), s, params, tab)
        assert np.abs(f.sum(axis=0)).max() <= 1e-9 * np.mean(np.linalg.norm(f, axis=1))


# --------------------------------------------------------------------------- errors


def test_error_behaviour(pb):
    box = pb.SimulationBox([8.0] * 3)
    s = pb.AtomSystem(box=box, positions=[[1.0, 2.0, 3.0], [4.0, 5.0, 6.0]], charges=[1.0, -1.0])
    params = _mk(pb, order=5)
    grid = np.zeros((16, 16, 16))
    ad = pb.FieldGrids(mode=pb.DiffMode.AD, dims=(16, 16, 16), spacing=(0.5,) * 3, phi=grid)
    ik = pb.FieldGrids(mode=pb.DiffMode.IK, dims=(16, 16, 16), spacing=(0.5,) * 3, ex=grid, ey=grid, ez=grid)
    with pytest.raises(ValueError, match="IK"):
        pb.distribute_force_ik(ad, s, params, pb.build_table(5, 100))
    with pytest.raises(ValueError, match="AD"):
        pb.distribute_force_ad(ik, s, params, pb.build_table(5, 100))
    with pytest.raises(pb.ConfigurationError):
        pb.map_charge(s, params, None)  # table required
    with pytest.raises(pb.ConfigurationError):
        pb.map_charge(s, params, pb.build_table(3, 100))  # wrong order
    small = pb.ChargeGrid(dims=(12, 12, 12), spacing=(1.0,) * 3, values=np.zeros((12, 12, 12)))
    with pytest.raises(ValueError, match="dims"):
        pb.poisson_ik(small, pb.build_plan((16, 16, 16), box, 0.9, 5))

    class Raw:  # an unwrapped system (bypasses AtomSystem's wrap)
        box = pb.SimulationBox([8.0] * 3)
        positions = np.array([[8.5, 1.0, 1.0], [1.0, 1.0, 1.0]])
        charges = np.array([1.0, -1.0])

    with pytest.raises(RuntimeError, match="wrapped"):
        pb.map_charge(Raw(), _mk(pb, order=5, use_table=False))
    with pytest.raises(RuntimeError, match="wrapped"):
        pb.distribute_force_ik(ik, Raw(), _mk(pb, order=5, use_table=False))


# --------------------------------------------------------------------------- BASELINE configs


def test_config2_water_ad_fp64_vs_oracle(pb):
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[2]
    pos, q, lengths = cfg.build()
    g = dict(pos=pos, q=q, lengths=lengths, dims=np.array(cfg.dims), order=cfg.order,
             mode=np.array(cfg.mode), alpha=cfg.alpha, use_table=False)
    _, _, energy, forces, _ = _run(pb, g)
    f_ref, e_ref, _ = orc.pppm_step(pos, q, lengths, cfg.dims, cfg.order, cfg.alpha, cfg.mode)
    assert rel_rms(forces, f_ref) <= FP64_TOL
    assert abs(energy - e_ref) <= FP64_TOL * abs(e_ref)


@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_config3_full_size_mixed(pb, mode):
    """1,048,576 atoms / 128^3 (BASELINE config 3): full-size parity on an atom
    subset, plus the size-independent invariants (charge conservation, ik momentum)."""
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[3]
    p32, q, lengths = cfg.build()
    ctx = pb.PppmContext(cfg.dims, lengths, order=cfg.order, mode=mode, precision="mixed", alpha=cfg.alpha)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    forces, energy, rho = ctx.forces(), ctx.energy(), ctx.rho()
    ctx.close()
    h = lengths / np.array(cfg.dims)
    assert abs(rho.sum() * np.prod(h)) <= 1e-5 * np.sqrt(q.size)
    pos = p32.astype(np.float64)
    rho_ref = orc.map_charge(pos, q, lengths, cfg.dims, cfg.order)
    assert rel_rms(rho, rho_ref) <= MIXED_TOL
    g = orc.influence_pme(cfg.dims, lengths, cfg.alpha, cfg.order)
    e_ref = orc.kspace_energy(rho_ref, g, lengths)
    assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref)
    sub = np.random.default_rng(5).choice(q.size, 4096, replace=False)
    if mode == "ik":
        fields = orc.poisson_ik(rho_ref, g, orc.ik_vectors(cfg.dims, lengths))
        f_ref = orc.fieldforce_ik(fields, pos[sub], q[sub], lengths, cfg.dims, cfg.order)
        fnorm = np.mean(np.linalg.norm(forces, axis=1))
        assert np.abs(forces.sum(axis=0)).max() <= 1e-4 * fnorm * np.sqrt(q.size)
    else:
        phi = orc.poisson_ad(rho_ref, g)
        f_ref = orc.fieldforce_ad(phi, pos[sub], q[sub], lengths, cfg.dims, cfg.order)
    assert rel_rms(forces[sub], f_ref) <= MIXED_TOL


# --------------------------------------------------------------------------- fp32 path edge cases


@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_mixed_overflow_buckets(pb, mode):
    """A dense cluster overfills its brick buckets: the overflow records take
    the global-atomic / direct-gather path (extra CTAs) and must agree too."""
    from paper_1702_04250_b200.scenarios import round_to_f32

    rng = np.random.default_rng(21)
    lengths = np.array([32.0, 32.0, 32.0])
    n = 6000
    pos = np.concatenate([rng.uniform(0, 32, (n // 2, 3)), 5.0 + rng.uniform(0, 1.5, (n // 2, 3))])
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    p32 = round_to_f32(pos, lengths)
    dims = (32, 32, 32)
    ctx = pb.PppmContext(dims, lengths, order=5, mode=mode, precision="mixed", alpha=0.4)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    forces, energy, rho = ctx.forces(), ctx.energy(), ctx.rho()
    ctx.close()
    f_ref, e_ref, rho_ref = orc.pppm_step(p32.astype(np.float64), q, lengths, dims, 5, 0.4, mode)
    assert rel_rms(rho, rho_ref) <= MIXED_TOL
    assert rel_rms(forces, f_ref) <= MIXED_TOL
    assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref)


@pytest.mark.parametrize("order,dims", [(7, (7, 7, 7)), (3, (3, 4, 5)), (6, (9, 6, 11)), (4, (8, 8, 4))])
def test_mixed_tiny_meshes(pb, order, dims):
    """Meshes smaller than the brick tile (TMA boxes partly outside the padded mesh)."""
    from paper_1702_04250_b200.scenarios import round_to_f32

    rng = np.random.default_rng(order)
    lengths = np.array(dims, dtype=np.float64) * 1.3
    n = 200
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    p32 = round_to_f32(pos, lengths)
    for mode in ("ik", "ad"):
        ctx = pb.PppmContext(dims, lengths, order=order, mode=mode, precision="mixed", alpha=0.8)
        ctx.load_atoms(p32, q.astype(np.float32))
        ctx.step()
        ctx.synchronize()
        forces, energy = ctx.forces(), ctx.energy()
        ctx.close()
        f_ref, e_ref, _ = orc.pppm_step(p32.astype(np.float64), q, lengths, dims, order, 0.8, mode)
        assert rel_rms(forces, f_ref) <= MIXED_TOL
        assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref)


def test_resident_graph_replay_is_stable(pb):
    """CUDA-graph replays of the resident step give the same forces as the first (eager) run."""
    from paper_1702_04250_b200 import scenarios

    pos, q, lengths = scenarios.random_gas(20000, 4, 45.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext((32, 32, 32), lengths, order=5, mode="ik", precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    f0 = ctx.forces()
    for _ in range(3):  # eager, capture, replay
        ctx.step()
    ctx.synchronize()
    f3 = ctx.forces()
    ctx.close()
    assert rel_rms(f3, f0) <= 1e-6


@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_kernel_variants_agree(pb, mode):
    """Every make_rho / fieldforce variant of the fp32 path (A/B switches of
    pppm_ctx_set_variant) gives the same charge mesh and forces to 1e-5 (the
    brick tiles meet in the halo through fp32 TMA reduce-adds, whose order is
    not fixed)."""
    from paper_1702_04250_b200 import _native as nat
    from paper_1702_04250_b200 import scenarios

    pos, q, lengths = scenarios.random_gas(30000, 8, 50.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext((32, 32, 32), lengths, order=5, mode=mode, precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    rho0, f0 = ctx.rho(), ctx.forces()
    tried = 0
    for kernel, variant in ((0, 3), (1, 4), (1, 5), (1, 1), (1, 2), (1, 0), (0, 0)):
        try:
            ctx.ctx("pppm_ctx_set_variant", kernel, variant)
        except ValueError as exc:  # A/B variants are compiled only with -DPPPM_AB_VARIANTS
            assert "not built" in str(exc)
            continue
        tried += 1
        ctx.step()
        ctx.synchronize()
        rho, f = ctx.rho(), ctx.forces()
        assert rel_rms(rho, rho0) <= 1e-5
        assert rel_rms(f, f0) <= 1e-5
    ctx.close()
    assert tried >= 2


@pytest.mark.parametrize("mode", ["ik", "ad"])
def test_resident_direct_movers_and_overflow(pb, mode):
    """Brick-ordered residents (make_rho maps positions itself, no binning
    pass): same forces / energy as the one-shot binned path, after moving
    atoms across bricks with update_positions (direct path for movers) and
    with a dense cluster that overflows its bucket at load."""
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(21)
    n, edge = 40000, 50.0
    pos, q, lengths = scenarios.random_gas(n, 9, edge)
    pos[:3000] = 20.0 + rng.uniform(0, 2.0, (3000, 3))      # one overfull brick
    p32 = scenarios.round_to_f32(pos, lengths)
    q32 = q.astype(np.float32)
    ctx = pb.PppmContext((32, 32, 32), lengths, order=5, mode=mode, precision="mixed", alpha=0.3)
    ref = pb.PppmContext((32, 32, 32), lengths, order=5, mode=mode, precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q32)
    for trial in range(3):
        for _ in range(2):  # eager, then graph replay
            ctx.step()
        ctx.synchronize()
        f, e = ctx.forces(), ctx.energy()
        fr, er = ref.compute(p32, q32)
        # movers take the direct fp32 path in the resident step, their brick
        # tile's fixed point in the binned one: rounding-level differences
        assert rel_rms(f, fr) <= 3e-6
        assert abs(e - er) <= 3e-6 * abs(er)
        # move every atom by up to ~1.5 mesh cells: many leave their brick
        p32 = scenarios.round_to_f32(np.mod(p32.astype(np.float64) + rng.uniform(-2.3, 2.3, p32.shape), edge),
                                     lengths)
        ctx.update_positions(p32)
    ctx.close()
    ref.close()


@pytest.mark.parametrize("order,n", [(5, 120000), (7, 120000), (5, 1 << 20)])
def test_fp64_tile_make_rho_bitwise(pb, order, n, monkeypatch):
    """fp64 make_rho on brick-ordered residents accumulates per-brick shared tiles of
    three 32-bit limbs (k_spread_fix64_tile): the same 64-bit fixed-point contributions
    as the direct kernel, so the mesh must be bitwise the same - with a brick that
    overflows its bucket at load and after moving atoms across bricks - and match the
    oracle at the fp64 bar."""
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(8)
    # (from 2^20 atoms on the tiles hold two limbs per cell instead of three)
    dims = (64, 64, 32) if n < (1 << 20) else (128, 128, 64)
    lengths = np.array([96.0, 96.0, 48.0]) * (dims[0] // 64)
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    pos[:2500] = np.array([40.0, 50.0, 20.0]) + rng.uniform(0, 3.0, (2500, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0) * rng.uniform(0.5, 1.5, n)
    q -= q.mean()
    moved = np.mod(pos + rng.uniform(-2.0, 2.0, pos.shape), lengths)
    out = {}
    for tiles in ("1", "0"):
        monkeypatch.setenv("PPPM_B200_FIX64_TILES", tiles)
        ctx = pb.PppmContext(dims, lengths, order=order, mode="ik", precision="fp64", alpha=0.3)
        ctx.load_atoms(pos, q)
        ctx.step()
        ctx.synchronize()
        r0 = ctx.rho().copy()
        ctx.set_resort(1.0)
        ctx.update_positions(moved)
        for _ in range(2):
            ctx.step()
        ctx.synchronize()
        out[tiles] = (r0, ctx.rho().copy(), ctx.forces().copy())
        ctx.close()
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1])
    assert np.array_equal(out["1"][2], out["0"][2])
    rho_ref = orc.map_charge(moved, q, lengths, dims, order)
    assert rel_rms(out["1"][1], rho_ref) <= 1e-11  # 64-bit fixed point with the global scale 2^(62 - log2(N max|q|))


@pytest.mark.parametrize("mode,order,table,nx", [("ik", 5, 0, 128), ("ad", 5, 0, 128), ("ik", 3, 5000, 128),
                                                 ("ad", 4, 0, 128), ("ik", 7, 0, 128), ("ik", 5, 0, 136),
                                                 ("ad", 5, 0, 136)])
def test_resident_pipelined_movers_holes_overflow(pb, mode, order, table, nx):
    """The pipelined resident make_rho (several bricks per CTA: 128 x 128 x 64 mesh) and
    the ranked record hand-off to fieldforce, on their rare paths: a cell so full that
    its bank bucket overflows (atoms take the direct path, their fieldforce slots stay
    reserved as holes), a brick so full that it overflows at load, and atoms moved
    across bricks with update_positions - against the one-shot binned path."""
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(33)
    # (nx = 136: an odd number of bricks along x - one-brick make_rho items and fieldforce stages
    # on the pipelined path, no brick pairs)
    dims, n = (nx, 128, 64), 500000
    lengths = np.array([1.5 * nx, 192.0, 96.0])
    pos, q, _ = scenarios.random_gas(n, 11, 192.0)
    pos[:, 0] *= nx / 128.0
    pos[:, 2] *= 0.5
    pos[:300] = np.array([50.2, 60.3, 40.4]) + rng.uniform(0, 0.8, (300, 3))       # one cell: one bank bucket
    pos[300:3300] = np.array([120.0, 30.0, 20.0]) + rng.uniform(0, 6.0, (3000, 3))  # bricks beyond the slot capacity
    p32 = scenarios.round_to_f32(np.mod(pos, lengths), lengths)
    q32 = q.astype(np.float32)
    # (orders 3-5: two-brick make_rho items and fieldforce stages, exact and table weights;
    # order 7: two-brick make_rho items, per-brick ranked fieldforce stages)
    ctx = pb.PppmContext(dims, lengths, order=order, mode=mode, precision="mixed", alpha=0.3, table_points=table)
    ref = pb.PppmContext(dims, lengths, order=order, mode=mode, precision="mixed", alpha=0.3, table_points=table)
    ctx.load_atoms(p32, q32)
    for trial in range(3):
        for _ in range(2):  # eager, then graph replay
            ctx.step()
        ctx.synchronize()
        f, e = ctx.forces(), ctx.energy()
        fr, er = ref.compute(p32, q32)
        assert rel_rms(f, fr) <= 3e-6
        assert abs(e - er) <= 3e-6 * abs(er)
        # ~1 cell rms displacement: a good fraction of the atoms leaves its brick
        p32 = scenarios.round_to_f32(np.mod(p32.astype(np.float64) + rng.uniform(-1.5, 1.5, p32.shape), lengths),
                                     lengths)
        ctx.set_resort(1.0)  # keep the movers on the direct path (no automatic re-sort)
        ctx.update_positions(p32)
    ctx.close()
    ref.close()


@pytest.mark.parametrize("order", [4, 5])
def test_resident_map_on_cell_boundaries(pb, order):
    """The resident make_rho maps positions itself in fp32 arithmetic with an exact
    fp64 fallback near rounding boundaries (particle_map_f32): atoms placed on the
    node-rounding boundaries of their order (half-cell points for odd, cell edges for
    even orders), a few fp32 ulps either side, must land in the reference's cells -
    one wrong node shifts a whole stencil and breaks the mesh at the 1e-2 level.
    128^3 so that the pipelined kernel (several bricks per CTA) is the one running."""
    from paper_1702_04250_b200 import scenarios

    rng = np.random.default_rng(77)
    dims, edge, n = (128, 128, 128), 96.0, 300000
    lengths = np.array([edge, edge * 1.03125, edge * 0.96875])
    h = lengths / np.array(dims)
    cells = rng.integers(0, 128, (n, 3))
    frac = np.where(order & 1, 0.5, 0.0)
    pos = (cells + frac) * h
    # two thirds of the coordinates sit on a boundary (+- 0..3 ulps), the rest anywhere
    free = rng.random((n, 3)) < 1.0 / 3.0
    pos = np.where(free, rng.uniform(0, 1, (n, 3)) * lengths, pos)
    p32 = scenarios.round_to_f32(np.mod(pos, lengths), lengths)
    for _ in range(3):
        step = rng.integers(-1, 2, p32.shape)
        p32 = np.where(step > 0, np.nextafter(p32, np.float32(np.inf)),
                       np.where(step < 0, np.nextafter(p32, np.float32(-np.inf)), p32)).astype(np.float32)
    p32 = scenarios.round_to_f32(np.mod(p32.astype(np.float64), lengths), lengths)
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    ctx = pb.PppmContext(dims, lengths, order=order, mode="ik", precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q.astype(np.float32))
    for _ in range(2):
        ctx.step()
    ctx.synchronize()
    rho, forces = ctx.rho(), ctx.forces()
    ctx.close()
    pos64 = p32.astype(np.float64)
    rho_ref = orc.map_charge(pos64, q, lengths, dims, order)
    assert rel_rms(rho, rho_ref) <= MIXED_TOL
    g = orc.influence_pme(dims, lengths, 0.3, order)
    fields = orc.poisson_ik(rho_ref, g, orc.ik_vectors(dims, lengths))
    sub = rng.choice(n, 4096, replace=False)
    f_ref = orc.fieldforce_ik(fields, pos64[sub], q[sub], lengths, dims, order)
    assert rel_rms(forces[sub], f_ref) <= MIXED_TOL


@pytest.mark.parametrize("dims,order", [((64, 32, 16), 5), ((16, 128, 32), 3), ((128, 16, 64), 7),
                                        ((32, 32, 256), 4), ((48, 64, 32), 5)])
def test_mixed_fused_poisson_shapes(pb, dims, order):
    """The fused Poisson path on non-cubic power-of-two meshes (own plane FFT
    kernels for nx != ny, the z kernel at several nz, the cuFFT 2D fallback for
    nx = 48) against the oracle: rho, fields-driven forces and energy."""
    from paper_1702_04250_b200.scenarios import round_to_f32

    rng = np.random.default_rng(sum(dims))
    lengths = np.array(dims, dtype=np.float64) * 0.7
    n = 3000
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    p32 = round_to_f32(pos, lengths)
    for mode in ("ik", "ad"):
        ctx = pb.PppmContext(dims, lengths, order=order, mode=mode, precision="mixed", alpha=0.5)
        ctx.load_atoms(p32, q.astype(np.float32))
        ctx.step()
        ctx.synchronize()
        forces, energy = ctx.forces(), ctx.energy()
        ctx.close()
        f_ref, e_ref, _ = orc.pppm_step(p32.astype(np.float64), q, lengths, dims, order, 0.5, mode)
        assert rel_rms(forces, f_ref) <= MIXED_TOL, (dims, order, mode)
        assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref), (dims, order, mode)
