"""Seeded synthetic inputs for the BASELINE.json configurations.

The paper's SPC/E water benchmark input is not available; these generators
stand in for it with the geometry, charges and density BASELINE.json names.

* ``random_gas`` reproduces the reference generator's point-charge gas
  (driver.py:106-115 / generate_scenario "random_gas"): uniform positions in
  [0, L)^3 from ``np.random.default_rng(seed)`` and alternating +1/-1 charges.
* ``water`` builds rigid 3-site water-like molecules (O-H 1.0 A, H-O-H
  109.47 deg, O -0.8476 / H +0.4238) with uniform random centres and uniform
  random orientations, plus zero-charge padding atoms.
* ``round_to_f32`` produces the fp32-representable positions used by the
  mixed / fp32 configurations; the oracle is fed the same values upcast.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

WATER_DENSITY = 0.0334          # molecules / A^3 (BASELINE configs 2 and 4)
GAS_DENSITY_LARGE = 0.1         # atoms / A^3 (configs 3 and 5)
OH_LENGTH = 1.0
HOH_ANGLE_DEG = 109.47
Q_H = 0.4238
Q_O = -2.0 * Q_H                # -0.8476, exact per-molecule neutrality


def select_alpha(cutoff: float, accuracy: float) -> float:
    """alpha = (1.35 - 0.15 ln eps) / r_c (reference tuner.py:58-64)."""
    return (1.35 - 0.15 * math.log(accuracy)) / cutoff


def random_gas(n: int, seed: int, edge: float):
    """Uniform point charges with alternating signs; returns (pos (n,3), q (n,), lengths)."""
    if n < 2 or n % 2:
        raise ValueError("random_gas needs an even atom count >= 2")
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.0, edge, (n, 3))
    q = np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    return pos, q, np.array([edge, edge, edge], dtype=np.float64)


def _random_rotations(rng, m):
    """Uniform random rotation matrices from normalised Gaussian quaternions."""
    quat = rng.normal(size=(m, 4))
    quat /= np.linalg.norm(quat, axis=1, keepdims=True)
    w, x, y, z = quat.T
    rot = np.empty((m, 3, 3))
    rot[:, 0, 0] = 1 - 2 * (y * y + z * z)
    rot[:, 0, 1] = 2 * (x * y - z * w)
    rot[:, 0, 2] = 2 * (x * z + y * w)
    rot[:, 1, 0] = 2 * (x * y + z * w)
    rot[:, 1, 1] = 1 - 2 * (x * x + z * z)
    rot[:, 1, 2] = 2 * (y * z - x * w)
    rot[:, 2, 0] = 2 * (x * z - y * w)
    rot[:, 2, 1] = 2 * (y * z + x * w)
    rot[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return rot


def water(n_molecules: int, n_pad: int, seed: int, density: float = WATER_DENSITY):
    """Rigid 3-site water-like molecules in a periodic cube at ``density``.

    Atom order is O, H, H per molecule followed by ``n_pad`` zero-charge
    atoms.  Positions are wrapped into [0, L).  Returns (pos, q, lengths).
    """
    edge = (n_molecules / density) ** (1.0 / 3.0)
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, edge, (n_molecules, 3))
    half = math.radians(HOH_ANGLE_DEG) / 2.0
    local = np.array([
        [0.0, 0.0, 0.0],
        [OH_LENGTH * math.sin(half), OH_LENGTH * math.cos(half), 0.0],
        [-OH_LENGTH * math.sin(half), OH_LENGTH * math.cos(half), 0.0],
    ])
    rot = _random_rotations(rng, n_molecules)
    sites = centres[:, None, :] + np.einsum("mij,sj->msi", rot, local)
    pos = sites.reshape(-1, 3)
    q = np.tile(np.array([Q_O, Q_H, Q_H]), n_molecules)
    if n_pad:
        pos = np.concatenate([pos, rng.uniform(0.0, edge, (n_pad, 3))])
        q = np.concatenate([q, np.zeros(n_pad)])
    lengths = np.array([edge, edge, edge], dtype=np.float64)
    return wrap(pos, lengths), q, lengths


def wrap(pos, lengths):
    """Fold positions into [0, L) per dimension (reference model.py:81-95 semantics)."""
    pos = np.asarray(pos, dtype=np.float64)
    lengths = np.asarray(lengths, dtype=np.float64)
    out = pos - np.floor(pos / lengths) * lengths
    out = np.where(out >= lengths, out - lengths, out)
    out = np.where(out < 0.0, out + lengths, out)
    return out


def round_to_f32(pos, lengths):
    """fp32-representable positions inside [0, L): round, then fold any L to 0."""
    p32 = np.asarray(pos, dtype=np.float32).copy()
    lim = np.asarray(lengths, dtype=np.float64)
    bad = p32.astype(np.float64) >= lim
    p32[bad] = 0.0
    return p32


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (index 1-5)."""

    index: int
    name: str
    n_atoms: int
    dims: tuple
    order: int
    mode: str
    precision: str         # "fp64" or "mixed" ("fp32" configs run as mixed)
    alpha: float

    def build(self, seed=None):
        seed = self.index if seed is None else seed
        if self.name == "gas":
            edge = 20.0 if self.index == 1 else (self.n_atoms / GAS_DENSITY_LARGE) ** (1.0 / 3.0)
            pos, q, lengths = random_gas(self.n_atoms, seed, edge)
        else:
            n_mol = (self.n_atoms) // 3
            pad = self.n_atoms - 3 * n_mol
            if self.index == 2:     # 10,667 x 3 > 32,000: use 10,666 + 2 pad
                n_mol, pad = 10666, 2
            pos, q, lengths = water(n_mol, pad, seed)
        if self.precision != "fp64":
            pos = round_to_f32(pos, lengths)
        return pos, q, lengths


ALPHA_10A = select_alpha(10.0, 1e-4)

CONFIGS = {
    1: Config(1, "gas", 4096, (16, 16, 16), 5, "ik", "fp64", 0.30),
    2: Config(2, "water", 32000, (40, 40, 40), 5, "ad", "fp64", ALPHA_10A),
    3: Config(3, "gas", 1 << 20, (128, 128, 128), 5, "ik", "mixed", ALPHA_10A),
    4: Config(4, "water", 262144, (64, 64, 64), 5, "ik", "mixed", ALPHA_10A),
    5: Config(5, "gas", 1 << 23, (256, 256, 256), 5, "ik", "mixed", ALPHA_10A),
}
