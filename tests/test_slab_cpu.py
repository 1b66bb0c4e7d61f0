"""The multi-GPU exchange schedule (paper_1702_04250_b200.slab.SlabStep over
torch.distributed) on CPU: world size 2 with gloo, each rank a numpy model of
its slab's device steps (tests/slab_model.py); the assembled forces and energy
must equal the single-process oracle."""

import os
import socket
import sys

import numpy as np
import pytest

from conftest import ROOT, rel_rms

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, order, out_dir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pppm_oracle as orc
    from paper_1702_04250_b200.slab import SlabStep, TorchComm, owner_of_nodes
    from slab_model import NumpySlab

    dims, lengths, alpha = (16, 12, 16), np.array([20.0, 15.0, 20.0]), 0.45
    rng = np.random.default_rng(3)
    n = 600
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    nodes, _ = orc.particle_map(pos, lengths, dims, order)
    owner = owner_of_nodes(nodes[2], dims[2], world)
    mine = np.nonzero(owner == rank)[0]
    slab = NumpySlab(dims, lengths, order, mode, alpha, world, rank)
    slab.load_atoms(pos[mine], q[mine])
    SlabStep(slab, TorchComm())()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), idx=mine, forces=slab.forces, energy=slab.energy_buf[0])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode,order", [("ik", 5), ("ad", 5), ("ik", 4), ("ad", 7)])
def test_two_rank_gloo_schedule(tmp_path, mode, order):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), mode, order, str(tmp_path)), nprocs=world, join=True)
    from oracle import pppm_oracle as orc

    dims, lengths, alpha = (16, 12, 16), np.array([20.0, 15.0, 20.0]), 0.45
    rng = np.random.default_rng(3)
    n = 600
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    forces = np.full((n, 3), np.nan)
    energies = []
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        forces[d["idx"]] = d["forces"]
        energies.append(float(d["energy"]))
    assert not np.isnan(forces).any()
    f_ref, e_ref, _ = orc.pppm_step(pos, q, lengths, dims, order, alpha, mode)
    assert rel_rms(forces, f_ref) <= 1e-10
    for e in energies:  # all-reduced on every rank
        assert abs(e - e_ref) <= 1e-10 * abs(e_ref)


def test_owner_partition():
    from paper_1702_04250_b200.slab import owner_of_nodes

    nodes_z = np.array([0, 7, 8, 15, 16, 31, 32])  # 32 planes, 4 slabs; node 32 wraps to 0
    assert list(owner_of_nodes(nodes_z, 32, 4)) == [0, 0, 1, 1, 2, 3, 0]


def _migrate_worker(rank, world, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pppm_oracle as orc
    from paper_1702_04250_b200.slab import migrate_atoms, owner_of_nodes

    dims, lengths = (16, 12, 16), np.array([20.0, 15.0, 20.0])
    rng = np.random.default_rng(8)
    n = 3000
    pos = rng.uniform(0, 1, (n, 3)) * lengths
    gid = np.arange(n, dtype=np.int64)
    nodes, _ = orc.particle_map(pos, lengths, dims, 5)
    mine = owner_of_nodes(nodes[2], dims[2], world) == rank
    my_pos, my_gid = pos[mine], gid[mine]
    # move every atom; many cross into another slab
    moved = orc.wrap(my_pos + rng.uniform(-4.0, 4.0, my_pos.shape), lengths)
    nodes2, _ = orc.particle_map(moved, lengths, dims, 5)
    new_pos, new_gid = migrate_atoms(owner_of_nodes(nodes2[2], dims[2], world), [moved, my_gid])
    np.savez(os.path.join(out_dir, f"mig{rank}.npz"), pos=new_pos, gid=new_gid)
    dist.barrier()
    dist.destroy_process_group()


def test_four_rank_atom_migration(tmp_path):
    """migrate_atoms (all-to-all-v over gloo): after a move every atom lives on
    the slab owning its new node_z, nothing is lost or duplicated."""
    world = 4
    mp.spawn(_migrate_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle import pppm_oracle as orc
    from paper_1702_04250_b200.slab import owner_of_nodes

    dims, lengths = (16, 12, 16), np.array([20.0, 15.0, 20.0])
    seen = []
    for r in range(world):
        z = np.load(tmp_path / f"mig{r}.npz")
        nodes, _ = orc.particle_map(z["pos"], lengths, dims, 5)
        assert np.all(owner_of_nodes(nodes[2], dims[2], world) == r)
        seen.append(z["gid"])
    allg = np.sort(np.concatenate(seen))
    assert np.array_equal(allg, np.arange(3000))
