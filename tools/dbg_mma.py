"""Debug helper: constant-field fieldforce_ik (mixed) at one order, max error vs q*E."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1702_04250_b200 as pb  # noqa: E402

order = int(sys.argv[1])
natoms = int(sys.argv[2]) if len(sys.argv) > 2 else 20
box = pb.SimulationBox([8.0] * 3)
rng = np.random.default_rng(7)
q = np.where(np.arange(natoms) % 2 == 0, 1.0, -1.0)
s = pb.AtomSystem(box=box, positions=rng.uniform(0, 8, (natoms, 3)), charges=q)
params = pb.PppmParams(cutoff=2.0, accuracy=1e-4, order=order, mode=pb.DiffMode("ik"), alpha=0.9,
                       grid_dims=(16, 16, 16), use_table=False, precision="mixed")
grid = np.full((16, 16, 16), 2.5)
fields = pb.FieldGrids(mode=pb.DiffMode.IK, dims=(16, 16, 16), spacing=(0.5,) * 3, ex=grid, ey=grid, ez=grid)
forces = pb.distribute_force_ik(fields, s, params)
print("order", order, "n", natoms, "maxerr", np.abs(forces - 2.5 * q[:, None]).max())
