"""Steady-state cost of the MD step (update_positions_async + make_rho + Poisson +
fieldforce on moving resident atoms) against the re-sort threshold, BASELINE
config 3 (1,048,576 point charges, 128^3, order 5, ik, mixed).

Positions random-walk on the device (sigma A rms per step, wrapped, rounded to
fp32 inside [0, L)); the loop runs long enough for several re-sorts, which are
inside the timed region.  `--sync` waits for every step's forces on the host (an
integrator on the host); without it the host only enqueues (device-resident MD).

    python tools/md_resort_sweep.py [--steps 300] [--sigma 0.1] [--fractions 0.003,0.006,...] [--sync]

One JSON line per threshold."""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--sigma", type=float, default=0.1)
    ap.add_argument("--fractions", default="-1,0.003,0.006,0.01,0.02,0.05,0")  # -1: the random walk alone
    ap.add_argument("--sync", action="store_true")
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()

    import torch

    import paper_1702_04250_b200 as pb
    from paper_1702_04250_b200 import _native as nat
    from paper_1702_04250_b200 import scenarios

    cfg = scenarios.CONFIGS[args.config]
    pos, q, lengths = cfg.build()
    n = pos.shape[0]
    dev = "cuda:0"
    L = torch.tensor(np.asarray(lengths, dtype=np.float64), device=dev)
    L32 = L.to(torch.float32)

    for frac in [float(f) for f in args.fractions.split(",")]:
        ctx = pb.PppmContext(cfg.dims, lengths, order=cfg.order, mode=cfg.mode, precision="mixed", alpha=cfg.alpha,
                             device=0)
        ctx.load_atoms(pos.astype(np.float32), q.astype(np.float32))
        ctx.set_resort(frac)
        sp = ctypes.c_void_p()
        ctx.ctx("pppm_ctx_stream", ctypes.byref(sp))
        stream = torch.cuda.ExternalStream(sp.value, device=0)
        gen = torch.Generator(device=dev)
        gen.manual_seed(7)
        cur = torch.from_numpy(pos.astype(np.float64)).to(dev)
        p32 = torch.empty((n, 3), dtype=torch.float32, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        movers = []
        t0 = 0.0
        with torch.cuda.stream(stream):
            for i in range(args.steps + args.warmup):
                if i == args.warmup:
                    ctx.synchronize()
                    r0 = ctx.resident_info()["resorts"]
                    t0 = time.perf_counter()
                    e0.record(stream)
                cur += torch.randn(cur.shape, generator=gen, device=dev, dtype=torch.float64) * (args.sigma / 3 ** 0.5)
                cur -= torch.floor(cur / L) * L
                p32.copy_(cur)
                p32.masked_fill_(p32 >= L32, 0.0)
                p32.masked_fill_(p32 < 0, 0.0)
                if frac < 0:
                    continue
                ctx.update_positions_async(p32.data_ptr(), mem=nat.DEVICE)
                ctx.step(nat.PHASE_ALL)
                if args.sync:
                    ctx.synchronize()
                    movers.append(ctx.resident_info()["movers"])
            e1.record(stream)
        ctx.synchronize()
        wall = time.perf_counter() - t0
        info = ctx.resident_info()
        ms = e0.elapsed_time(e1) / args.steps
        print(json.dumps({"resort_fraction": frac, "sigma_A": args.sigma, "steps": args.steps, "sync": args.sync,
                          "ms_per_step_incl_random_walk": ms, "wall_ms_per_step": wall / args.steps * 1e3,
                          "resorts": info["resorts"] - r0, "movers_last": info["movers"],
                          "movers_mean": float(np.mean(movers)) if movers else None, "n_atoms": n}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
