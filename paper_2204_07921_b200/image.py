"""Boundary value type and harness helpers of the denoising path.

Mirrors the reference ``curvemg.image`` names the solver boundary uses
(/root/reference/pkg/src/curvemg/image.py):

* ``Image``              image.py:34-75   immutable read-only float64 grid + peak
* ``NoiseSpec``          image.py:78-87
* ``add_gaussian_noise`` image.py:124-134 (default_rng(seed).normal, unclipped)
* ``psnr``               image.py:140-149

SSIM runs on the GPU (``metrics.ssim``, bit-identical to image.py:152-192).
Everything here is host-side NumPy; none of it is on the timed GPU path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["Image", "NoiseSpec", "add_gaussian_noise", "psnr"]


@dataclass(frozen=True)
class Image:
    """Dense 2-D scalar field with a declared intensity range (image.py:34-75).

    ``data`` becomes a read-only, C-contiguous float64 copy; ``peak`` is the
    declared dynamic range (255 for denoising work on [0,255], 1.0 for [0,1]).
    """

    data: np.ndarray
    peak: float = 255.0

    def __post_init__(self):
        arr = np.asarray(self.data, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError(f"image data must be 2-D, got shape {arr.shape}")
        if arr.size == 0:
            raise ValueError("image must contain at least one pixel")
        if not np.all(np.isfinite(arr)):
            raise ValueError("image intensities must be finite")
        if self.peak <= 0:
            raise ValueError("peak must be positive")
        arr = np.ascontiguousarray(arr)
        if arr.flags.writeable:
            arr = arr.copy()
            arr.flags.writeable = False
        object.__setattr__(self, "data", arr)

    @classmethod
    def _from_solver(cls, arr: np.ndarray, peak: float) -> "Image":
        """Wrap a freshly allocated solver output without re-validating or
        copying it (the solver raises on non-finite corrections, so the
        values are finite; the array is owned by the new Image)."""
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        arr.flags.writeable = False
        obj = object.__new__(cls)
        object.__setattr__(obj, "data", arr)
        object.__setattr__(obj, "peak", float(peak))
        return obj

    @property
    def height(self) -> int:
        return self.data.shape[0]

    @property
    def width(self) -> int:
        return self.data.shape[1]

    @property
    def shape(self) -> tuple[int, int]:
        return self.data.shape


@dataclass(frozen=True)
class NoiseSpec:
    """Additive white Gaussian noise: std deviation + PRNG seed (image.py:78-87)."""

    sigma: float
    seed: int = 0

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError("sigma must be non-negative")


def add_gaussian_noise(img: Image, spec: NoiseSpec) -> Image:
    """Zero-mean white Gaussian noise, deterministic per seed, not clipped (image.py:124-134)."""
    if spec.sigma == 0.0:
        return img
    rng = np.random.default_rng(spec.seed)
    return Image(img.data + rng.normal(0.0, spec.sigma, size=img.data.shape), img.peak)


def psnr(a: Image, b: Image) -> float:
    """Peak signal-to-noise ratio in dB; ``inf`` for identical images (image.py:140-149)."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if a.peak != b.peak:
        raise ValueError(f"peak mismatch: {a.peak} vs {b.peak}")
    mse = float(np.mean((a.data - b.data) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(a.peak * a.peak / mse)
