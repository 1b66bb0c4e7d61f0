"""Small end-to-end cases for compute-sanitizer (racecheck / synccheck /
memcheck) over the warp-specialized / TMA / mbarrier kernels: resident steps
(k_spread_tma, k_gather_ws ik + ad), the one-shot binned path (k_bin_fixed,
binned k_spread_tma / k_gather_ws), the fused Poisson kernels, orders 5 and 7
(S = 7: k_gather_tma), and a slab step over NCCL (one slab)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1702_04250_b200 as pb  # noqa: E402
from paper_1702_04250_b200 import scenarios  # noqa: E402
from paper_1702_04250_b200.slab import SlabContext, nccl_unique_id  # noqa: E402

pos, q, lengths = scenarios.random_gas(6000, 3, 30.0)
p32 = scenarios.round_to_f32(pos, lengths)
q32 = q.astype(np.float32)
for order in (5, 7):
    for mode in ("ik", "ad"):
        ctx = pb.PppmContext((24, 24, 24), lengths, order=order, mode=mode, precision="mixed", alpha=0.4)
        ctx.load_atoms(p32, q32)
        for _ in range(3):
            ctx.step()
        ctx.synchronize()
        ctx.compute(p32, q32)
        ctx.close()
        print("ok", order, mode, flush=True)
slab = SlabContext((24, 24, 24), lengths, 5, "ik", 0.4, 1, 0)
slab.load_atoms(p32, q32)
slab.attach_nccl(nccl_unique_id())
slab.step()
slab.synchronize()
slab.close()
print("ok slab", flush=True)
