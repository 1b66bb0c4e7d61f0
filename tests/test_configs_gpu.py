"""GPU parity at the BASELINE.json configurations' full named shapes.

* config 4: 262,144 water-like atoms (87,381 rigid 3-site molecules + 1
  zero-charge pad) on 64^3, interpolation orders 3..7 x {ik, ad}, fp32 mesh.
  Orders 4 and 6 are this repo's extension (the reference rejects them,
  model.py:18): parity unpinned by the reference, checked against the
  oracle's extension registration.
* config 5: 8,388,608 point charges on 256^3, order 5, ik, fp32 mesh, on one
  GPU (the multi-GPU slab path is checked on this shape in test_slab_gpu.py).
  The oracle scatter runs in 64Ki-atom chunks over private replicas summed in
  order (gridmap.py:186-207; BASELINE.md §3's chunked reference run).

Each case checks, against the CPU oracle (oracle/pppm_oracle.py) on the same
fp32-rounded positions: the full charge mesh and the k-space energy to 1e-5
relative RMS / relative error, and the forces of 8,192 sampled atoms to 1e-5
relative RMS (north_star's mixed-precision bar), plus charge conservation.
"""

import dataclasses
import os

import numpy as np
import pytest

from conftest import rel_rms
from oracle import pppm_oracle as orc

pytestmark = pytest.mark.gpu

MIXED_TOL = 1e-5
N_SAMPLE = 8192
WORKERS = max(1, min(16, len(os.sched_getaffinity(0))))


@pytest.fixture(scope="module")
def pb():
    import __graft_entry__

    __graft_entry__.build()
    import paper_1702_04250_b200 as pb

    return pb


def _device_step(pb, cfg, p32, q, lengths, mode):
    ctx = pb.PppmContext(cfg.dims, lengths, order=cfg.order, mode=mode, precision="mixed", alpha=cfg.alpha)
    try:
        ctx.load_atoms(p32, q.astype(np.float32))
        ctx.step()
        ctx.synchronize()
        return ctx.forces(), ctx.energy(), ctx.rho()
    finally:
        ctx.close()


def _check(cfg, p32, q, lengths, mode, forces, energy, rho):
    dims, order = cfg.dims, cfg.order
    h = lengths / np.array(dims)
    # charge conservation to fp32 rounding of the deposits (~1e-7 per atom, random sign)
    assert abs(rho.sum() * np.prod(h) - q.sum()) <= 1e-6 * np.sum(np.abs(q))
    pos = p32.astype(np.float64)
    rho_ref = orc.map_charge(pos, q, lengths, dims, order, workers=WORKERS)
    assert rel_rms(rho, rho_ref) <= MIXED_TOL
    g = orc.influence_pme(dims, lengths, cfg.alpha, order)
    e_ref = orc.kspace_energy(rho_ref, g, lengths)
    assert abs(energy - e_ref) <= MIXED_TOL * abs(e_ref)
    sub = np.random.default_rng(cfg.index * 10 + order).choice(q.size, N_SAMPLE, replace=False)
    if mode == "ik":
        fields = orc.poisson_ik(rho_ref, g, orc.ik_vectors(dims, lengths))
        f_ref = orc.fieldforce_ik(fields, pos[sub], q[sub], lengths, dims, order)
    else:
        phi = orc.poisson_ad(rho_ref, g)
        f_ref = orc.fieldforce_ad(phi, pos[sub], q[sub], lengths, dims, order)
    err = rel_rms(forces[sub], f_ref)
    assert err <= MIXED_TOL, err
    return err


@pytest.fixture(scope="module")
def config4():
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[4]
    pos, q, lengths = cfg.build()
    assert pos.shape == (262144, 3) and cfg.dims == (64, 64, 64)
    assert np.count_nonzero(q == 0.0) == 1 and abs(q.sum()) < 1e-9
    return cfg, pos, q, lengths


@pytest.mark.parametrize("mode", ["ik", "ad"])
@pytest.mark.parametrize("order", [3, 4, 5, 6, 7])
def test_config4_water_order_sweep(pb, config4, order, mode):
    cfg, p32, q, lengths = config4
    cfg = dataclasses.replace(cfg, order=order)
    forces, energy, rho = _device_step(pb, cfg, p32, q, lengths, mode)
    _check(cfg, p32, q, lengths, mode, forces, energy, rho)


def test_config5_full_shape_ik(pb):
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[5]
    p32, q, lengths = cfg.build()
    assert p32.shape == (1 << 23, 3) and cfg.dims == (256, 256, 256)
    forces, energy, rho = _device_step(pb, cfg, p32, q, lengths, "ik")
    # size-independent invariant: ik forces sum to ~0 (momentum, test_gridmap.py:236-251)
    fnorm = np.mean(np.linalg.norm(forces, axis=1))
    assert np.abs(forces.sum(axis=0)).max() <= 1e-4 * fnorm * np.sqrt(q.size)
    _check(cfg, p32, q, lengths, "ik", forces, energy, rho)
