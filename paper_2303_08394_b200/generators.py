"""Seeded synthetic point clouds (SPEC.md:694-729 `generators`).

Portable counter-based splitmix64 streams (not numpy's Generator, whose output
is not part of any spec), so the same (kind, n, seed) gives the same bits on
every machine.  `fp32=True` rounds positions and charges to float32-
representable values so an fp32 GPU run and the fp64 oracle see identical
inputs (SURVEY 8c parity protocol).
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform(seed: int, stream: int, n: int) -> np.ndarray:
    """n doubles in [0, 1) from the (seed, stream) splitmix64 sequence (53-bit mantissa)."""
    with np.errstate(over="ignore"):
        key = _mix(np.array([np.uint64(seed & 0xFFFFFFFFFFFFFFFF)], dtype=np.uint64))[0] ^ \
            (np.uint64(stream) * _GOLDEN)
        ctr = (np.arange(1, n + 1, dtype=np.uint64) * _GOLDEN) + key
    z = _mix(ctr)
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def gaussian(seed: int, stream: int, n: int) -> np.ndarray:
    """n standard normals (Box-Muller on two uniform streams)."""
    u1 = uniform(seed, 2 * stream + 101, n)
    u2 = uniform(seed, 2 * stream + 102, n)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def sample(kind: str, n: int, seed: int = 0, charges: str = "unit", fp32: bool = False):
    """Particle set (positions n x 3, charges n).

    kind: 'uniform-cube' ([0,1)^3), 'sphere-surface' (unit sphere, normalised
    Gaussians), 'two-cluster' (a dense and a sparse cube; exercises W/X lists).
    charges: 'unit', 'uniform' U[0,1), 'signed' U[-1,1).
    """
    if n < 1:
        from .errors import InvalidArgument
        raise InvalidArgument("sample: n must be >= 1")
    if kind == "uniform-cube":
        pos = np.stack([uniform(seed, d, n) for d in range(3)], axis=1)
    elif kind == "sphere-surface":
        g = np.stack([gaussian(seed, d, n) for d in range(3)], axis=1)
        pos = g / np.linalg.norm(g, axis=1)[:, None]
    elif kind == "two-cluster":
        u = np.stack([uniform(seed, d, n) for d in range(3)], axis=1)
        pick = uniform(seed, 7, n) < 0.5
        pos = np.where(pick[:, None], 0.1 + 0.05 * u, 0.5 + 0.45 * u)
    else:
        from .errors import InvalidArgument
        raise InvalidArgument(f"sample: unknown distribution {kind!r}")
    if charges == "unit":
        q = np.ones(n)
    elif charges == "uniform":
        q = uniform(seed, 11, n)
    elif charges == "signed":
        q = 2.0 * uniform(seed, 11, n) - 1.0
    else:
        from .errors import InvalidArgument
        raise InvalidArgument(f"sample: unknown charge law {charges!r}")
    if fp32:
        pos = pos.astype(np.float32).astype(np.float64)
        q = q.astype(np.float32).astype(np.float64)
    return np.ascontiguousarray(pos), np.ascontiguousarray(q)


# BASELINE.json configs (index 0..4): (kind, n, charges, precision, p, n_crit, gradient)
CONFIGS = {
    1: dict(kind="uniform-cube", n=10_000, charges="uniform", precision=32, p=5, n_crit=64, gradient=False),
    2: dict(kind="uniform-cube", n=1_000_000, charges="uniform", precision=32, p=6, n_crit=150, gradient=True),
    3: dict(kind="sphere-surface", n=1_000_000, charges="signed", precision=32, p=6, n_crit=150, gradient=False),
    4: dict(kind="uniform-cube", n=8_000_000, charges="uniform", precision=64, p=7, n_crit=150, gradient=False),
    5: dict(kind="uniform-cube", n=32_000_000, charges="uniform", precision=32, p=6, n_crit=128, gradient=False),
}


def config_sample(cfg: int, seed: int = 0, n: int | None = None):
    c = CONFIGS[cfg]
    return sample(c["kind"], n or c["n"], seed=seed, charges=c["charges"], fp32=c["precision"] == 32)
