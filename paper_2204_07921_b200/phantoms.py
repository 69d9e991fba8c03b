"""Deterministic analytic phantoms for the CLI harness (reference
``curvemg.image.phantom``, /root/reference/pkg/src/curvemg/image.py:199-281).

The rasterisation must reproduce the reference's pixels exactly (the CLI's
noisy/restored files and report are compared byte for byte), so the pixel
centres, rotations and inclusion tests follow the reference's formulas and
evaluation order; the code is this package's own.  Host-side NumPy: input
generation, not on the GPU path.
"""

from __future__ import annotations

import math

import numpy as np

from .image import Image

__all__ = ["phantom", "PHANTOM_KINDS"]

# modified Shepp-Logan table (intensity stays inside [0, 1]):
# (added value, semi-axis a, semi-axis b, centre x, centre y, rotation in degrees)
_ELLIPSES = (
    (1.00, 0.6900, 0.9200, 0.00, 0.0000, 0.0),
    (-0.80, 0.6624, 0.8740, 0.00, -0.0184, 0.0),
    (-0.20, 0.1100, 0.3100, 0.22, 0.0000, -18.0),
    (-0.20, 0.1600, 0.4100, -0.22, 0.0000, 18.0),
    (0.10, 0.2100, 0.2500, 0.00, 0.3500, 0.0),
    (0.10, 0.0460, 0.0460, 0.00, 0.1000, 0.0),
    (0.10, 0.0460, 0.0460, 0.00, -0.1000, 0.0),
    (0.10, 0.0460, 0.0230, -0.08, -0.6050, 0.0),
    (0.10, 0.0230, 0.0230, 0.00, -0.6050, 0.0),
    (0.10, 0.0230, 0.0460, 0.06, -0.6050, 0.0),
)


def _unit_grid(size: int):
    """Pixel coordinates on [0, 1): X varies along columns, Y along rows."""
    t = np.arange(size, dtype=np.float64) / size
    return np.meshgrid(t, t)


def _shepp_logan(size: int) -> np.ndarray:
    # pixel centres on [-1, 1], y pointing up
    centres = (2.0 * np.arange(size) + 1.0) / size
    X, Y = np.meshgrid(-1.0 + centres, 1.0 - centres)
    img = np.zeros((size, size))
    for value, a, b, x0, y0, deg in _ELLIPSES:
        c, s = math.cos(math.radians(deg)), math.sin(math.radians(deg))
        dx, dy = X - x0, Y - y0
        xr = dx * c + dy * s
        yr = -dx * s + dy * c
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += value
    return np.clip(img, 0.0, 1.0)


def _side(X, Y, p, q):
    """Signed side of the directed edge p -> q (2-D cross product)."""
    return (X - p[0]) * (q[1] - p[1]) - (Y - p[1]) * (q[0] - p[0])


def _triangle(size: int) -> np.ndarray:
    X, Y = _unit_grid(size)
    img = np.full((size, size), 60.0)
    a, b, c = (0.50, 0.12), (0.88, 0.80), (0.12, 0.72)
    e0, e1, e2 = _side(X, Y, a, b), _side(X, Y, b, c), _side(X, Y, c, a)
    inside = ((e0 >= 0) & (e1 >= 0) & (e2 >= 0)) | ((e0 <= 0) & (e1 <= 0) & (e2 <= 0))
    img[inside] = 200.0
    img[(Y >= 0.06) & (Y <= 0.22) & (X >= 0.06) & (X <= 0.30)] = 140.0
    return img


def _shapes(size: int) -> np.ndarray:
    X, Y = _unit_grid(size)
    img = np.full((size, size), 40.0)
    img[(Y >= 0.10) & (Y <= 0.45) & (X >= 0.08) & (X <= 0.40)] = 120.0
    img[np.abs(X - 0.68) + np.abs(Y - 0.30) <= 0.18] = 220.0
    img[(Y >= 0.60) & (Y <= 0.90) & (X >= 0.15) & (X <= 0.85) & (np.abs(X - Y) <= 0.22)] = 180.0
    img[(Y >= 0.70) & (Y <= 0.78) & (X >= 0.55) & (X <= 0.92)] = 90.0
    return img


PHANTOM_KINDS = {"shepp_logan": (_shepp_logan, 1.0), "triangle": (_triangle, 255.0), "shapes": (_shapes, 255.0)}


def phantom(kind: str, size: int) -> Image:
    """Rasterise phantom ``kind`` at ``size`` x ``size`` (image.py:267-281)."""
    if kind not in PHANTOM_KINDS:
        raise ValueError(f"unknown phantom kind {kind!r}; choose from {sorted(PHANTOM_KINDS)}")
    if size < 32:
        raise ValueError("phantom size must be at least 32")
    fn, peak = PHANTOM_KINDS[kind]
    return Image(fn(size), peak)
