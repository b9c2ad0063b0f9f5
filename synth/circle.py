"""The paper's synthetic ablation dataset (sec. IV-B-1) and the
seeded per-point train/validation split ("90% ... 10% reserved").

Generator only -- no arithmetic of the method: 5000 occupied points uniform in angle on the circle
of radius 4 m centred in an 8 m x 8 m region, 5000 empty points uniform inside that disk.
"""
from __future__ import annotations

import numpy as np

BOUNDS = (0.0, 0.0, 8.0, 8.0)
CENTRE = (4.0, 4.0)
RADIUS = 4.0


def gen_circle_dataset(seed: int = 0, n_occ: int = 5000, n_emp: int = 5000):
    """(xy float32 [n, 2], labels uint8 [n]): occupied points first, then empty points."""
    rng = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(4242,)))
    a = rng.uniform(0.0, 2 * np.pi, n_occ)
    occ = np.stack([CENTRE[0] + RADIUS * np.cos(a), CENTRE[1] + RADIUS * np.sin(a)], axis=1)
    r = RADIUS * np.sqrt(rng.uniform(0.0, 1.0, n_emp))          # uniform over the disk area
    b = rng.uniform(0.0, 2 * np.pi, n_emp)
    emp = np.stack([CENTRE[0] + r * np.cos(b), CENTRE[1] + r * np.sin(b)], axis=1)
    xy = np.concatenate([occ, emp]).astype(np.float32)
    lab = np.concatenate([np.ones(n_occ, np.uint8), np.zeros(n_emp, np.uint8)])
    return np.ascontiguousarray(xy), lab


def split_train_val(n: int, fraction: float = 0.9, seed: int = 0):
    """Per-point seeded shuffle -> (train indices, validation indices)."""
    if not 0.0 < fraction < 1.0:
        raise ValueError("fraction must be in (0, 1)")
    perm = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(777,))).permutation(n)
    k = int(round(fraction * n))
    return np.sort(perm[:k]), np.sort(perm[k:])
