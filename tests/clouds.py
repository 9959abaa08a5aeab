"""Seeded synthetic clouds with the shapes BASELINE.json names (no public
dataset exists for this path). Shared by tests, the
golden generator and bench.py."""
from __future__ import annotations

import numpy as np


def disk_cloud(n: int, rng: np.random.Generator, diameter: float = 1.0) -> np.ndarray:
    """i.i.d. uniform in a disk of the given diameter: r = (d/2) sqrt(U), theta = 2 pi U."""
    r = 0.5 * diameter * np.sqrt(rng.random(n))
    th = 2.0 * np.pi * rng.random(n)
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1)


def square_cloud(n: int, rng: np.random.Generator, side: float = 1.0) -> np.ndarray:
    return rng.random((n, 2)) * side


def star_curve_cloud(n: int, rng: np.random.Generator, jitter: float = 0.1) -> np.ndarray:
    """r(theta) = 0.4 (1 + 0.2 cos 5 theta) at theta_j = (j + u_j) 2 pi / n,
    u_j ~ U(-jitter, jitter) (SURVEY.md section 8d 'Jitter' convention)."""
    j = np.arange(n)
    th = (j + rng.uniform(-jitter, jitter, n)) * 2.0 * np.pi / n
    r = 0.4 * (1.0 + 0.2 * np.cos(5.0 * th))
    return np.stack([r * np.cos(th), r * np.sin(th)], axis=1)


def star_interior_cloud(n: int, rng: np.random.Generator) -> np.ndarray:
    """Uniform inside the star curve (rejection sampling)."""
    out = []
    while sum(len(o) for o in out) < n:
        p = rng.uniform(-0.48, 0.48, (2 * n, 2))
        th = np.arctan2(p[:, 1], p[:, 0])
        r = np.hypot(p[:, 0], p[:, 1])
        out.append(p[r <= 0.4 * (1.0 + 0.2 * np.cos(5.0 * th))])
    return np.concatenate(out)[:n]
