"""One resident config-3-mesh step at N atoms (ncu target): python tools/density_one.py N"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_04250_b200 as pb  # noqa: E402
from paper_1702_04250_b200 import scenarios  # noqa: E402

n = int(sys.argv[1])
edge = ((1 << 20) / 0.1) ** (1 / 3)
pos, q, lengths = scenarios.random_gas(n, 3, edge)
p32 = scenarios.round_to_f32(pos, lengths)
ctx = pb.PppmContext((128, 128, 128), lengths, order=5, mode="ik", precision="mixed", alpha=0.2731)
ctx.load_atoms(p32, q.astype(np.float32))
ms = ctx.time_steps(4, 2, flush_l2=True)
print(ms)
ctx.close()
