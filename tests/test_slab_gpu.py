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
