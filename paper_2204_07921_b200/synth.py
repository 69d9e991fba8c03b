"""Seeded synthetic inputs standing in for the paper's photographs.

The paper measures on real test images that are not available here
(PAPER.md:491, :795).  BASELINE.json defines a seeded piecewise-smooth
generator instead; this module implements it with the normative draw order of
SURVEY.md section 8(d).  Noise uses the reference's own recipe
(``add_gaussian_noise``, image.py:124-134) with seed ``seed + 1_000_003``.

The five BASELINE configurations are exposed by :func:`config_input`.
"""

from __future__ import annotations

import math

import numpy as np

from .image import Image, NoiseSpec, add_gaussian_noise

__all__ = ["clean", "noisy", "config_input", "CONFIGS"]


def clean(size: int, n_shapes: int, seed: int, r_range=(10.0, 60.0), texture: bool = False) -> np.ndarray:
    """Clean piecewise-smooth image in [0, 1] (float64, size x size)."""
    rng = np.random.default_rng(seed)
    big = size > 4096
    if not big:
        y, x = np.mgrid[0:size, 0:size]
    theta = rng.uniform(0, 2 * math.pi)
    if big:
        xs = np.arange(size, dtype=np.float64)
        g = math.cos(theta) * xs[None, :] + math.sin(theta) * xs[:, None]
    else:
        g = math.cos(theta) * x + math.sin(theta) * y
    g = (g - g.min()) / (g.max() - g.min())
    img = 0.2 + 0.3 * g
    del g
    for _ in range(n_shapes):
        kind = rng.integers(2)
        cy, cx = rng.uniform(0, size, 2)
        a, b = rng.uniform(*r_range, 2)
        v = rng.uniform()
        # evaluate the mask only on the shape's clipped bounding box (identical result)
        if kind == 0:
            r0, r1 = max(0, int(math.floor(cy - a)) - 1), min(size, int(math.ceil(cy + a)) + 2)
            c0, c1 = max(0, int(math.floor(cx - a)) - 1), min(size, int(math.ceil(cx + a)) + 2)
            yy = np.arange(r0, r1)[:, None]
            xx = np.arange(c0, c1)[None, :]
            mask = (yy - cy) ** 2 + (xx - cx) ** 2 <= a * a
        else:
            r0, r1 = max(0, int(math.floor(cy - a)) - 1), min(size, int(math.ceil(cy + a)) + 2)
            c0, c1 = max(0, int(math.floor(cx - b)) - 1), min(size, int(math.ceil(cx + b)) + 2)
            yy = np.arange(r0, r1)[:, None]
            xx = np.arange(c0, c1)[None, :]
            mask = (np.abs(yy - cy) <= a) & (np.abs(xx - cx) <= b)
        if r1 > r0 and c1 > c0:
            img[r0:r1, c0:c1][mask] = v
    by, bx = rng.uniform(0, size, 2)
    if big:
        xs = np.arange(size, dtype=np.float64)
        ey = np.exp(-((xs - by) ** 2) / (2 * 40.0 ** 2))
        ex = np.exp(-((xs - bx) ** 2) / (2 * 40.0 ** 2))
        rows = np.nonzero(ey > 0)[0]
        cols = np.nonzero(ex > 0)[0]
        r0, r1, c0, c1 = rows[0], rows[-1] + 1, cols[0], cols[-1] + 1
        yy = xs[r0:r1, None]
        xx = xs[None, c0:c1]
        img[r0:r1, c0:c1] += 0.3 * np.exp(-((yy - by) ** 2 + (xx - bx) ** 2) / (2 * 40.0 ** 2))
    else:
        img += 0.3 * np.exp(-((y - by) ** 2 + (x - bx) ** 2) / (2 * 40.0 ** 2))
    if texture:
        h = size // 4
        ty, tx = rng.uniform(0, size - h, 2)
        ty, tx = int(ty), int(tx)
        xcols = np.arange(tx, tx + h, dtype=np.float64)[None, :]
        img[ty:ty + h, tx:tx + h] += 0.1 * np.sin(2 * math.pi * np.broadcast_to(xcols, (h, h)) / 64)
    np.clip(img, 0, 1, out=img)
    return img


def noisy(clean_img: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Reference noise recipe with seed ``seed + 1_000_003`` (unclipped)."""
    if clean_img.shape[0] > 4096:
        rng = np.random.default_rng(seed + 1_000_003)
        out = clean_img + rng.normal(0.0, sigma, size=clean_img.shape)
        return out
    return add_gaussian_noise(Image(clean_img, 1.0), NoiseSpec(sigma, seed + 1_000_003)).data


CONFIGS = {
    1: dict(size=256, n_shapes=8, sigma=20 / 255, seed=0, mode="mean", layers=6, cycles=10, dtype="f64"),
    2: dict(size=512, n_shapes=16, sigma=15 / 255, seed=1, mode="gaussian", layers=6, cycles=50, eps=1e-6,
            dtype="f64"),
    3: dict(size=1024, n_shapes=32, sigma=25 / 255, seed=2, texture=True, mode="mean", layers=3, cycles=500,
            eps=1e-6, dtype="f64"),
    4: dict(size=512, n_shapes=16, batch=64, seed=1000, mode="mean", layers=3, cycles=20, dtype="f32"),
    5: dict(size=16384, n_shapes=512, r_range=(20.0, 800.0), sigma=20 / 255, seed=5, mode="mean", layers=3,
            cycles=10, dtype="f32"),
}


def config_input(cfg: int, index: int = 0, fp32: bool | None = None):
    """(noisy, clean) float64 arrays for a BASELINE config (image ``index`` for config 4).

    fp32 configs are rounded to float32 first and returned as the float64
    values of those float32 numbers (the CPU reference sees the same
    fp32-representable input).
    """
    c = CONFIGS[cfg]
    if cfg == 4:
        sig = np.random.default_rng(4000).uniform(10, 30, 64)[index] / 255
        seed = c["seed"] + index
        cl = clean(c["size"], c["n_shapes"], seed)
        f = noisy(cl, sig, seed)
    else:
        cl = clean(c["size"], c["n_shapes"], c["seed"], c.get("r_range", (10.0, 60.0)), c.get("texture", False))
        f = noisy(cl, c["sigma"], c["seed"])
    if fp32 is None:
        fp32 = c["dtype"] == "f32"
    if fp32:
        f = f.astype(np.float32).astype(np.float64)
    return f, cl
