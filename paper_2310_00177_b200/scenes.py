"""Synthetic cell-type grids for the benchmark configurations.

Conventions follow the reference rasteriser: x fastest, index (z*ny + y)*nx + x
(discretization.hpp:38); "up" is +y (scene.cpp:162); cells are tested at their
centres against half-open boxes / strict-interior spheres (scene.cpp:70-96);
compositing is last-wins in the listed order (scene.cpp:95-96): air
background -> fluid regions -> solid obstacles -> 1-cell solid shell.
Cell types: 0 fluid, 1 air, 2 solid (scene.hpp:11).
"""
from __future__ import annotations

import numpy as np

FLUID, AIR, SOLID = 0, 1, 2


def _centres(n: int):
    c = np.arange(n, dtype=np.float64) + 0.5
    z, y, x = np.meshgrid(c, c, c, indexing="ij")
    return x, y, z


def _box(x, y, z, x0, x1, y0, y1, z0, z1):
    return (x >= x0) & (x < x1) & (y >= y0) & (y < y1) & (z >= z0) & (z < z1)


def _shell(t: np.ndarray) -> np.ndarray:
    t[0, :, :] = SOLID
    t[-1, :, :] = SOLID
    t[:, 0, :] = SOLID
    t[:, -1, :] = SOLID
    t[:, :, 0] = SOLID
    t[:, :, -1] = SOLID
    return t


def closed_box_half(n: int) -> np.ndarray:
    """C1: solid shell; interior fluid if y < n/2, air above."""
    x, y, z = _centres(n)
    t = np.full((n, n, n), AIR, np.uint8)
    t[y < 0.5 * n] = FLUID
    return _shell(t)


def dam_break(n: int) -> np.ndarray:
    """C2: fluid column x < 0.4n, y < 0.8n plus a floor layer y < 0.1n; solid
    obstacle box x in [0.55n, 0.65n), y in [0, 0.5n), z in [0.35n, 0.65n)."""
    x, y, z = _centres(n)
    t = np.full((n, n, n), AIR, np.uint8)
    t[((x < 0.4 * n) & (y < 0.8 * n)) | (y < 0.1 * n)] = FLUID
    t[_box(x, y, z, 0.55 * n, 0.65 * n, 0.0, 0.5 * n, 0.35 * n, 0.65 * n)] = SOLID
    return _shell(t)


def droplet_pool(n: int, yc: float = 0.75) -> np.ndarray:
    """C3: pool y < 0.4n plus a fluid sphere centre (0.5, yc, 0.5)n, radius 0.1n."""
    x, y, z = _centres(n)
    t = np.full((n, n, n), AIR, np.uint8)
    t[y < 0.4 * n] = FLUID
    r = 0.1 * n
    t[(x - 0.5 * n) ** 2 + (y - yc * n) ** 2 + (z - 0.5 * n) ** 2 < r * r] = FLUID
    return _shell(t)


def droplet_frames(n: int = 128, frames: int = 32):
    """C4: droplet centre y_f = (0.85 - 0.3 f/31) n, f = 0..frames-1."""
    for f in range(frames):
        yield droplet_pool(n, 0.85 - 0.3 * f / max(frames - 1, 1))


def dam_break_pillars(n: int) -> np.ndarray:
    """C5: C2 plus four solid pillars 0.05n wide, 0.5n tall, centred at x, z in {0.25n, 0.75n}."""
    x, y, z = _centres(n)
    t = np.full((n, n, n), AIR, np.uint8)
    t[((x < 0.4 * n) & (y < 0.8 * n)) | (y < 0.1 * n)] = FLUID
    t[_box(x, y, z, 0.55 * n, 0.65 * n, 0.0, 0.5 * n, 0.35 * n, 0.65 * n)] = SOLID
    w = 0.025 * n
    for cx in (0.25 * n, 0.75 * n):
        for cz in (0.25 * n, 0.75 * n):
            t[_box(x, y, z, cx - w, cx + w, 0.0, 0.5 * n, cz - w, cz + w)] = SOLID
    return _shell(t)


DESCRIPTION = {
    "C1": "closed box, fluid lower half",
    "C2": "dam break with obstacle",
    "C3": "droplet-in-pool",
    "C4": "droplet-in-pool sequence",
    "C5": "dam break with obstacle and four pillars",
}

CONFIGS = {
    "C1": (64, closed_box_half, 1234),
    "C2": (128, dam_break, 1235),
    "C3": (256, droplet_pool, 1236),
    "C5": (512, dam_break_pillars, 1237),
}


def config(name: str, n: int | None = None) -> tuple[np.ndarray, int]:
    """(cell types, RHS seed) of a named configuration, optionally at another size."""
    size, fn, seed = CONFIGS[name]
    return fn(n or size), seed


def random_types(shape, seed: int, p=(0.55, 0.3, 0.15), blobs: int = 3) -> np.ndarray:
    """Seeded random mixed grid for parity tests: noise plus a few boxes."""
    rng = np.random.default_rng(seed)
    t = rng.choice(3, size=shape, p=list(p)).astype(np.uint8)
    for _ in range(blobs):
        lo = [int(rng.integers(0, s)) for s in shape]
        hi = [min(s, l + int(rng.integers(1, max(2, s // 2)))) for l, s in zip(lo, shape)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        t[sl] = rng.integers(0, 3)
    return t


def full_rhs(types: np.ndarray, seed: int, normal=None) -> np.ndarray:
    """b_full = Rng(seed).normal() over the full grid, zero at non-fluid cells
    (test_solvers.cpp:30-35 pattern, then restrict). ``normal(seed, n)`` must be
    the reference Rng stream (paper_2310_00177_b200.rhs_normal)."""
    if normal is None:
        from . import rhs_normal as normal
    b = normal(seed, types.size)
    b[types.reshape(-1) != FLUID] = 0.0
    return b
