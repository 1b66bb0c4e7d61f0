"""Rewrite the measured numbers quoted in README.md from profiles/r02_bench.json and
profiles/r02_sweep.jsonl (run after tools/refresh_profiles.py)."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d = json.loads(open(os.path.join(ROOT, "profiles", "r02_bench.json")).read())
sweep = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "r02_sweep.jsonl"))]


def pick(cfg, mode):
    for r in sweep:
        if r["config"]["workload"].startswith(f"config{cfg}:") and r["config"]["mode"] == mode:
            return r
    return None


ad3, ik5 = pick(3, "ad"), pick(5, "ik")
text = (f"  kernels behind the C ABI in `include/pppm_b200.h`. Config 3 (1M atoms, 128³,\n"
        f"  order 5, ik, mixed) on one B200: **{d['value'] / 1e9:.2f}e9 atom-steps/s** for make_rho +\n"
        f"  fieldforce ({d['ms_make_rho_fieldforce'] * 1e3:.0f} µs), {d['whole_step_atom_steps_per_s'] / 1e9:.2f}e9 for the whole PPPM step; ad: "
        f"{ad3['value'] / 1e9:.2f}e9; config 5\n"
        f"  (8.4M atoms, 256³): {ik5['value'] / 1e9:.2f}e9; fp64 (the reference's arithmetic, config 3): "
        f"{d['value_fp64'] / 1e9:.2f}e9; MD step with\n"
        f"  moving atoms: {d['value_md'] / 1e9:.2f}e9; end to end from pinned host arrays through the C ABI: "
        f"{d['e2e']['value'] / 1e9:.2f}e9\n  (`profiles/README.md`, `profiles/r02_sweep.md`).\n")
p = os.path.join(ROOT, "README.md")
s = open(p).read()
a = s.index("  kernels behind the C ABI in `include/pppm_b200.h`. Config 3")
b = s.index("- **Measured experiments kept as A/B variants**")
open(p, "w").write(s[:a] + text + s[b:])
print(text)
