"""z-slab decomposition on one GPU (loopback exchanges between P slab
contexts): the decomposed make_rho -> distributed FFT -> fieldforce must match
the CPU oracle (mixed precision, 1e-5) and the one-GPU path."""

import numpy as np
import pytest

from conftest import rel_rms
from oracle import pppm_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    return pb


@pytest.mark.parametrize("P", [1, 2, 4])
@pytest.mark.parametrize("mode", ["ik", "ad"])
@pytest.mark.parametrize("order", [5, 4, 7])
def test_loopback_slabs_vs_oracle(pb, P, mode, order):
    from paper_1702_04250_b200 import scenarios
    from paper_1702_04250_b200.slab import LoopbackSlabs

    dims = (32, 24, 32)
    n = 12000
    lengths = np.array([40.0, 30.0, 40.0])
    rng = np.random.default_rng(100 + P)
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    alpha = 0.35
    lb = LoopbackSlabs(dims, lengths, order, mode, alpha, P)
    try:
        lb.load_atoms(p32, q.astype(np.float32))
        assert sum(len(i) for i in lb.index) == n
        lb.step()
        forces, energy = lb.forces(n), lb.energy()
    finally:
        lb.close()
    f_ref, e_ref, _ = orc.pppm_step(p32.astype(np.float64), q, lengths, dims, order, alpha, mode)
    assert rel_rms(forces, f_ref) <= 1e-5
    assert abs(energy - e_ref) <= 1e-5 * abs(e_ref)


def test_loopback_matches_single_gpu(pb):
    from paper_1702_04250_b200 import scenarios
    from paper_1702_04250_b200.slab import LoopbackSlabs

    dims, n = (32, 32, 32), 16000
    pos, q, lengths = scenarios.random_gas(n, 9, 40.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext(dims, lengths, order=5, mode="ik", precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    f1, e1 = ctx.forces(), ctx.energy()
    ctx.close()
    lb = LoopbackSlabs(dims, lengths, 5, "ik", 0.3, 4)
    try:
        lb.load_atoms(p32, q.astype(np.float32))
        lb.step()
        f4, e4 = lb.forces(n), lb.energy()
    finally:
        lb.close()
    assert rel_rms(f4, f1) <= 2e-6
    assert abs(e4 - e1) <= 1e-6 * abs(e1)


@pytest.mark.parametrize("mode,order", [("ik", 5), ("ad", 7), ("ik", 4)])
def test_native_nccl_one_slab(pb, mode, order):
    """The whole slab step inside the library (NCCL send/recv / all-to-all /
    all-reduce on the context stream, CUDA graphs) with one slab: NCCL to
    itself exercises every exchange of the multi-GPU code path on one GPU."""
    from paper_1702_04250_b200 import scenarios
    from paper_1702_04250_b200.slab import SlabContext, nccl_unique_id

    dims, n = (32, 32, 32), 20000
    pos, q, lengths = scenarios.random_gas(n, 17, 42.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext(dims, lengths, order=order, mode=mode, precision="mixed", alpha=0.3)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    f1, e1 = ctx.forces(), ctx.energy()
    ctx.close()
    slab = SlabContext(dims, lengths, order, mode, 0.3, 1, 0)
    try:
        slab.load_atoms(p32, q.astype(np.float32))
        slab.attach_nccl(nccl_unique_id())
        for _ in range(3):  # eager, capture, replay
            slab.step()
        slab.synchronize()
        fs, es = slab.forces(), slab.energy()
        ms = slab.time_steps(3, 1)
    finally:
        slab.close()
    assert rel_rms(fs, f1) <= 2e-6
    assert abs(es - e1) <= 1e-6 * abs(e1)
    assert ms["spread"] > 0 and ms["poisson"] > 0 and ms["gather"] > 0
    f_ref, e_ref, _ = orc.pppm_step(p32.astype(np.float64), q, lengths, dims, order, 0.3, mode)
    assert rel_rms(fs, f_ref) <= 1e-5


def test_slab_update_positions_reports_atoms_leaving_the_slab(pb):
    from paper_1702_04250_b200 import scenarios
    from paper_1702_04250_b200.slab import LoopbackSlabs

    dims, n = (32, 32, 32), 8000
    pos, q, lengths = scenarios.random_gas(n, 5, 40.0)
    p32 = scenarios.round_to_f32(pos, lengths)
    lb = LoopbackSlabs(dims, lengths, 5, "ik", 0.3, 2)
    try:
        lb.load_atoms(p32, q.astype(np.float32))
        s0 = lb.slabs[0]
        mine = p32[lb.index[0]].copy()
        s0.update_positions(mine)            # unchanged: fine
        mine[0, 2] = np.float32(lengths[2] * 0.75)   # into slab 1's half of the box
        with pytest.raises(RuntimeError, match="left their z-slab"):
            s0.update_positions(mine)
    finally:
        lb.close()


def test_loopback_p8_config5_shape(pb):
    """BASELINE config 5's shape (8,388,608 atoms, 256^3, order 5, ik) over 8
    loopback slabs of 32 planes: same forces / energy as the one-GPU mesh."""
    from paper_1702_04250_b200 import scenarios
    from paper_1702_04250_b200.slab import LoopbackSlabs

    cfg = scenarios.CONFIGS[5]
    p32, q, lengths = cfg.build()
    ctx = pb.PppmContext(cfg.dims, lengths, order=cfg.order, mode="ik", precision="mixed", alpha=cfg.alpha)
    ctx.load_atoms(p32, q.astype(np.float32))
    ctx.step()
    ctx.synchronize()
    f1, e1 = ctx.forces(), ctx.energy()
    ctx.close()
    lb = LoopbackSlabs(cfg.dims, lengths, cfg.order, "ik", cfg.alpha, 8)
    try:
        lb.load_atoms(p32, q.astype(np.float32))
        assert [s.nzl for s in lb.slabs] == [32] * 8
        lb.step()
        f8, e8 = lb.forces(q.size), lb.energy()
    finally:
        lb.close()
    assert rel_rms(f8, f1) <= 2e-6
    assert abs(e8 - e1) <= 1e-6 * abs(e1)
