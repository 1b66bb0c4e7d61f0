"""make_rho / fieldforce time vs atoms per brick on the config-3 mesh (128^3,
order 5, ik, mixed): separates per-brick from per-atom cost."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_04250_b200 as pb  # noqa: E402
from paper_1702_04250_b200 import scenarios  # noqa: E402

edge = (1 << 20) / 0.1
edge = edge ** (1 / 3)
for n in (1 << 18, 1 << 19, 1 << 20, 1 << 21, 3 << 20):
    pos, q, lengths = scenarios.random_gas(n, 3, edge)
    p32 = scenarios.round_to_f32(pos, lengths)
    ctx = pb.PppmContext((128, 128, 128), lengths, order=5, mode="ik", precision="mixed", alpha=0.2731)
    ctx.load_atoms(p32, q.astype(np.float32))
    ms = ctx.time_steps(20, 5, flush_l2=True)
    ctx.close()
    print(json.dumps({"n": n, "atoms_per_brick": n / 4096, "spread_us": ms["spread"] / 20 * 1e3,
                      "gather_us": ms["gather"] / 20 * 1e3, "poisson_us": ms["poisson"] / 20 * 1e3}), flush=True)
