"""Seeded synthetic inputs for the BASELINE.json configurations.

Every draw is the reference's counter-hash RNG ``uniform01(seed, counter)``
(``core/include/blfmm/common.hpp:45-55``), vectorised in numpy, so the same
(seed, counter) gives the same double as the reference and the oracle.
Counter layout: coordinate k of point i -> counter d*i + k;
lambda_j -> counter j under a separate seed; normals -> Box-Muller on counters
(2q, 2q+1). Seeds: points 1000+cfg, weights 2000+cfg, blob centres 3000+cfg.
The domain is always [0,1]^d and is passed explicitly.

No public dataset is involved: BASELINE names none, so these seeded inputs
stand in for the configurations' shapes, sizes and value distributions.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def hash64(x: np.ndarray) -> np.ndarray:
    """common.hpp:45-50 (splitmix64 finaliser), uint64 wrap-around."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def uniform01(seed: int, counter) -> np.ndarray:
    """common.hpp:52-55: 53 mantissa bits of hash64(seed ^ hash64(counter))."""
    c = np.asarray(counter, dtype=np.uint64)
    z = hash64(np.uint64(seed) ^ hash64(c))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normals(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Box-Muller on counter pairs (2q, 2q+1); q = offset .. offset+count-1."""
    q = np.arange(offset, offset + count, dtype=np.uint64)
    u1 = 1.0 - uniform01(seed, np.uint64(2) * q)  # (0, 1]
    u2 = uniform01(seed, np.uint64(2) * q + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


def uniform_points(n: int, d: int, seed: int) -> np.ndarray:
    ctr = np.arange(n * d, dtype=np.uint64)
    return uniform01(seed, ctr).reshape(n, d)


def uniform_weights(n: int, seed: int, nrhs: int = 1) -> np.ndarray:
    """lambda = 2 u - 1 in [-1, 1); rhs r uses counters r*n + j."""
    ctr = np.arange(n * nrhs, dtype=np.uint64)
    w = 2.0 * uniform01(seed, ctr) - 1.0
    return w.reshape(nrhs, n) if nrhs > 1 else w


def generate_quasiuniform(n: int, d: int, seed: int, jitter: float,
                          lo=(0.0, 0.0), hi=(1.0, 1.0)) -> np.ndarray:
    """geometry.cpp:114-144 (d in {1,2}): jittered cell-centred lattice."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if d not in (1, 2):
        raise ValueError("d must be 1 or 2")
    if not (0.0 <= jitter < 1.0):
        raise ValueError("jitter must be in [0,1)")
    if d == 1:
        spacing = (hi[0] - lo[0]) / n
        i = np.arange(n)
        u = 2.0 * uniform01(seed, i.astype(np.uint64)) - 1.0
        return (lo[0] + (i + 0.5 + 0.5 * jitter * u) * spacing).reshape(n, 1)
    k = int(math.ceil(math.sqrt(float(n))))
    sx, sy = (hi[0] - lo[0]) / k, (hi[1] - lo[1]) / k
    idx = np.arange(n)
    i, j = idx // k, idx % k
    u = 2.0 * uniform01(seed, (2 * idx).astype(np.uint64)) - 1.0
    v = 2.0 * uniform01(seed, (2 * idx + 1).astype(np.uint64)) - 1.0
    x = lo[0] + (i + 0.5 + 0.5 * jitter * u) * sx
    y = lo[1] + (j + 0.5 + 0.5 * jitter * v) * sy
    return np.stack([x, y], axis=1)


def blob_points(n: int, seed_pts: int, seed_centres: int, blobs: int = 16,
                sigma_b: float = 0.05) -> np.ndarray:
    """16 equal-weight isotropic Gaussian blobs in [0,1]^3, clipped.

    Point i belongs to blob i % blobs; centres are U[0,1)^3 (counters 3c+k);
    offsets are sigma_b * N(0,1) per axis (Box-Muller pairs 3i+k)."""
    centres = uniform01(seed_centres, np.arange(blobs * 3, dtype=np.uint64)).reshape(blobs, 3)
    z = normals(seed_pts, 3 * n).reshape(n, 3)
    pts = centres[np.arange(n) % blobs] + sigma_b * z
    return np.clip(pts, 0.0, 1.0)


def jittered_lattice(nx: int, ny: int, nz: int, seed: int) -> np.ndarray:
    """x = (i + 0.5 + u)/nx etc., u in U[-1/4, 1/4) per axis (row-major i,j,k)."""
    n = nx * ny * nz
    idx = np.arange(n)
    i, j, k = idx // (ny * nz), (idx // nz) % ny, idx % nz
    u = uniform01(seed, np.arange(3 * n, dtype=np.uint64)).reshape(n, 3) * 0.5 - 0.25
    return np.stack([(i + 0.5 + u[:, 0]) / nx, (j + 0.5 + u[:, 1]) / ny,
                     (k + 0.5 + u[:, 2]) / nz], axis=1)


@dataclass
class Workload:
    """One BASELINE.json configuration with its pinned FMM parameters."""
    name: str
    d: int
    kernel: str
    n: int
    sigma: float
    m: int
    leaf: int
    nrhs: int = 1
    points: str = "uniform"
    weights: str = "uniform"
    cfg: int = 0
    extra: dict = field(default_factory=dict)

    def make(self, n: int | None = None):
        """(points [n,d], weights [n] or [nrhs,n]) for this workload."""
        n = self.n if n is None else n
        sp, sw, sc = 1000 + self.cfg, 2000 + self.cfg, 3000 + self.cfg
        if self.points == "uniform":
            x = uniform_points(n, self.d, sp)
        elif self.points == "blobs":
            x = blob_points(n, sp, sc)
        elif self.points == "lattice":
            nx, ny, nz = self.extra.get("lattice", (64, 64, 128))
            if n != nx * ny * nz:
                # keep the lattice aspect for reduced parity sizes
                s = round((n / (nx * ny * nz)) ** (1.0 / 3.0) * 1e6) / 1e6
                nx, ny, nz = max(1, int(nx * s)), max(1, int(ny * s)), max(1, int(nz * s))
            x = jittered_lattice(nx, ny, nz, sp)
            n = x.shape[0]
        else:
            raise ValueError(self.points)
        if self.weights == "uniform":
            w = uniform_weights(n, sw, self.nrhs)
        else:
            w = normals(sw, n * self.nrhs).reshape(self.nrhs, n)
            if self.nrhs == 1:
                w = w[0]
        return np.ascontiguousarray(x), np.ascontiguousarray(w)


PI = math.pi

# SURVEY.md §8(d) parameter pins.
WORKLOADS = {
    "P1": Workload("P1", 2, "gaussian:c=16", 4096, PI, 64, 3, cfg=1),
    "P1b": Workload("P1b", 2, "gaussian:c=16", 4096, 51.4, 44, 3, cfg=1),
    "P2": Workload("P2", 3, "gaussian:c=64", 262144, 101.8, 58, 4, cfg=2),
    "P2p": Workload("P2p", 3, "gaussian:c=64", 262144, PI, 16, 4, cfg=2),
    "P3": Workload("P3", 3, "imq:c=0.1", 1048576, PI, 16, 6, points="blobs", cfg=3),
    "P4": Workload("P4", 2, "mq:c=0.05", 4194304, PI, 16, 8, weights="normal", cfg=4),
    "P5": Workload("P5", 3, "gaussian:c=64", 524288, PI, 16, 4, nrhs=32,
                   points="lattice", cfg=5, extra={"lattice": (64, 64, 128)}),
}
