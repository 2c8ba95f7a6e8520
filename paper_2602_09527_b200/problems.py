"""Seeded synthetic problems for the BASELINE.json configurations (host side).

The reference ships no generator for BASELINE's phantom / noise laws
(SURVEY.md Appendix C.1-C.4), so this module fixes them and DESIGN.md states
the choices:

* grid convention of pkg/src/proxtomo/phantoms.py:65-67 (``_unit_coords``):
  c_i = (i - (n-1)/2) * 2/n, meshgrid(ij) -> (y, x);
* 2D phantom: K ellipses, drawn per ellipse in the order
  (cx, cy, a, b, phi, value) from ``default_rng(seed)``:
  centre U[-0.7, 0.7]^2, semi-axes U[0.05, 0.4]^2, phi U[0, pi),
  value U[0.1, 1], added inside ((x'/a)^2 + (y'/b)^2 <= 1) with the rotation of
  phantoms.py:104-109;
* 3D phantom: ellipsoids drawn as (cx, cy, cz, a, b, c, phi, theta, psi,
  value), ZYZ Euler rotation;
* noise: b = A x + sigma N(0,1) with sigma = level * max|Ax| (the reference's
  ``level * clean.max()``, phantoms.py:135, for nonnegative phantoms); the
  config-2 "Poisson-like" law is a per-ray std 0.01|Ax| + 1e-3 max|Ax|;
* alpha = 0.01 max|A^T b| / n_pixels; L by ``operator_norm_sq`` (50
  iterations, seed 0); gamma by the reference's ``default_gamma``.
Seeds: phantom 0, noise 1, power 0, solver 0.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    size: int
    n_angles: int
    n_bins: int
    n_ellipses: int
    n_subsets: int
    estimator: str
    p: float
    fgp_inner: int
    epochs: int
    noise: str = "gaussian"     # or "poisson-like"
    depth: int = 1              # > 1: slice-stacked 3D
    phantom_seed: int = 0
    noise_seed: int = 1
    power_seed: int = 0
    power_iterations: int = 50
    solver_seed: int = 0

    @property
    def max_data_passes(self) -> float:
        """epochs -> reference data passes: an SVRG epoch is one snapshot plus N
        steps = 3 passes; SAGA / SGD 1 pass; full 1 pass."""
        return 3.0 * self.epochs if self.estimator in ("svrg", "lsvrg") else float(self.epochs)

    @property
    def n_pixels(self) -> int:
        return self.size * self.size * self.depth


CONFIGS = {
    "c0": BaselineConfig("c0", 128, 180, 192, 10, 10, "svrg", 0.1, 50, 50),
    "c1": BaselineConfig("c1", 512, 720, 768, 30, 20, "saga", 0.05, 100, 100),
    "c2": BaselineConfig("c2", 2048, 1800, 2900, 60, 60, "svrg", 0.05, 100, 30,
                         noise="poisson-like"),
    "c3": BaselineConfig("c3", 256, 360, 384, 40, 40, "svrg", 0.1, 100, 20, depth=256),
    "c4": BaselineConfig("c4", 512, 720, 768, 30, 20, "svrg", 0.05, 100, 100),
}


# L = ||A||^2 by the reference's power method (projector.py:170-197), 50
# iterations from seed 0, per configuration: c0 / c1 are the reference's own
# values (tests/golden/reference_c{0,1}.npz), c2 / c3 the device's (the
# reference cannot build those operators; tests/test_gpu_solver.py checks the
# device method reproduces all four to 1e-5).  Both bench arms derive gamma
# from these so they solve the identical problem.
POWER_L = {
    "c0": 22246.197324964247,
    "c1": 355946.43688261765,
    "c2": 3559457.2673338386,
    "c3": 88986.3085571524,
    "c4": 355946.43688261765,
}


def unit_coords(size: int):
    """phantoms.py:65-67."""
    c = (np.arange(size) - (size - 1) / 2.0) * (2.0 / size)
    return c


def ellipse_phantom(size: int, n_ellipses: int, seed: int = 0) -> np.ndarray:
    """Additive random ellipses on a size x size grid (float64)."""
    rng = np.random.default_rng(seed)
    c = unit_coords(size)
    img = np.zeros((size, size))
    for _ in range(n_ellipses):
        cx, cy = rng.uniform(-0.7, 0.7, size=2)
        a, b = rng.uniform(0.05, 0.4, size=2)
        phi = rng.uniform(0.0, math.pi)
        value = rng.uniform(0.1, 1.0)
        r = max(a, b)
        # bounding box in index space (the test below is exact)
        lo_y, hi_y = np.searchsorted(c, cy - r - 1e-9), np.searchsorted(c, cy + r + 1e-9, "right")
        lo_x, hi_x = np.searchsorted(c, cx - r - 1e-9), np.searchsorted(c, cx + r + 1e-9, "right")
        if lo_y >= hi_y or lo_x >= hi_x:
            continue
        yy, xx = np.meshgrid(c[lo_y:hi_y], c[lo_x:hi_x], indexing="ij")
        cp, sp = math.cos(phi), math.sin(phi)
        xr = (xx - cx) * cp + (yy - cy) * sp
        yr = -(xx - cx) * sp + (yy - cy) * cp
        inside = (xr / a) ** 2 + (yr / b) ** 2 <= 1.0
        img[lo_y:hi_y, lo_x:hi_x] += value * inside
    return img


def _zyz(phi, theta, psi):
    c1, s1 = math.cos(phi), math.sin(phi)
    c2, s2 = math.cos(theta), math.sin(theta)
    c3, s3 = math.cos(psi), math.sin(psi)
    rz1 = np.array([[c1, -s1, 0], [s1, c1, 0], [0, 0, 1]])
    ry = np.array([[c2, 0, s2], [0, 1, 0], [-s2, 0, c2]])
    rz2 = np.array([[c3, -s3, 0], [s3, c3, 0], [0, 0, 1]])
    return rz1 @ ry @ rz2


def ellipsoid_phantom(size: int, n_ellipsoids: int, seed: int = 0) -> np.ndarray:
    """Additive random ellipsoids on a size^3 grid, (z, y, x) layout (float32)."""
    rng = np.random.default_rng(seed)
    c = unit_coords(size)
    vol = np.zeros((size, size, size), dtype=np.float32)
    for _ in range(n_ellipsoids):
        cx, cy, cz = rng.uniform(-0.7, 0.7, size=3)
        axes = rng.uniform(0.05, 0.4, size=3)
        phi, theta, psi = rng.uniform(0.0, math.pi, size=3)
        value = rng.uniform(0.1, 1.0)
        rot = _zyz(phi, theta, psi)
        r = float(axes.max())
        sl = []
        for ctr in (cz, cy, cx):
            lo = np.searchsorted(c, ctr - r - 1e-9)
            hi = np.searchsorted(c, ctr + r + 1e-9, "right")
            sl.append((lo, hi))
        if any(lo >= hi for lo, hi in sl):
            continue
        zz, yy, xx = np.meshgrid(c[sl[0][0]:sl[0][1]], c[sl[1][0]:sl[1][1]],
                                 c[sl[2][0]:sl[2][1]], indexing="ij")
        d = np.stack([xx - cx, yy - cy, zz - cz], axis=-1)
        loc = d @ rot  # coordinates in the ellipsoid frame
        q = ((loc / axes) ** 2).sum(axis=-1)
        vol[sl[0][0]:sl[0][1], sl[1][0]:sl[1][1], sl[2][0]:sl[2][1]] += np.float32(value) * (q <= 1.0)
    return vol


def add_noise(clean: np.ndarray, law: str, seed: int, level: float = 0.01) -> np.ndarray:
    """b = Ax + noise (float64 host arithmetic)."""
    rng = np.random.default_rng(seed)
    clean = np.asarray(clean, dtype=np.float64)
    peak = float(np.abs(clean).max())
    if law == "gaussian":
        return clean + level * peak * rng.standard_normal(clean.shape)
    if law == "poisson-like":
        std = 0.01 * np.abs(clean) + 1e-3 * peak
        return clean + std * rng.standard_normal(clean.shape)
    raise ValueError(f"unknown noise law {law!r}")


def phantom_for(cfg: BaselineConfig) -> np.ndarray:
    if cfg.depth > 1:
        return ellipsoid_phantom(cfg.size, cfg.n_ellipses, cfg.phantom_seed)
    return ellipse_phantom(cfg.size, cfg.n_ellipses, cfg.phantom_seed)


def alpha_from_backprojection(atb_absmax: float, n_pixels: int) -> float:
    """alpha = 0.01 max|A^T b| / n (BASELINE.json configs; n = pixel count)."""
    return 0.01 * atb_absmax / n_pixels
