"""On-device image metrics: SSIM on the GPU.

``ssim(a, b)`` is a drop-in for ``curvemg.image.ssim`` (image.py:152-192):
same checks, same errors, and the same value bit for bit -- the kernel
(csrc/cmg_metrics.cuh) restates the separable 11x11 filter term by term and
np.mean's pairwise summation.  ``ssim_batch`` scores many image pairs in one
call (the batched denoising path).  The Gaussian window and the constants
are computed here with NumPy exactly as the reference computes them, so the
kernel receives identical inputs.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .image import Image

__all__ = ["ssim", "ssim_batch", "ssim_window"]

_WINDOW, _SIGMA, _K1, _K2 = 11, 1.5, 0.01, 0.03


def ssim_window(size: int = _WINDOW, sigma: float = _SIGMA) -> np.ndarray:
    """_gaussian_window (image.py:157-160)."""
    x = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return g / g.sum()


def ssim_batch(a: np.ndarray, b: np.ndarray, peak: float) -> np.ndarray:
    """Mean SSIM of each pair a[i], b[i] (arrays of shape (batch, m, n), float64
    or float32; float32 values are taken exactly as float64)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim == 2:
        a, b = a[None], b[None]
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape[1:]} vs {b.shape[1:]}")
    if a.ndim != 3:
        raise ValueError("expected (batch, m, n) arrays")
    if min(a.shape[1:]) < _WINDOW:
        raise ValueError(f"image smaller than the {_WINDOW}x{_WINDOW} SSIM window")
    dt = np.float32 if (a.dtype == np.float32 and b.dtype == np.float32) else np.float64
    a = np.ascontiguousarray(a, dtype=dt)
    b = np.ascontiguousarray(b, dtype=dt)
    w = ssim_window()
    c1 = (_K1 * peak) ** 2
    c2 = (_K2 * peak) ** 2
    out = np.zeros(a.shape[0])
    rc = N.lib().cmg_ssim_batch(a.shape[0], a.shape[1], a.shape[2], N.DTYPE["float32" if dt == np.float32 else "float64"],
                                N.ptr(a), N.ptr(b), N.dptr(w), c1, c2, N.dptr(out))
    if rc != N.CMG_OK:
        raise (ValueError if rc == N.CMG_EINVAL else RuntimeError)(N.last_error())
    return out


def ssim(a: Image, b: Image) -> float:
    """Mean structural similarity over 11x11 Gaussian windows (image.py:152-192):
    window sigma 1.5, K1 = 0.01, K2 = 0.03, L = a.peak."""
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {a.shape} vs {b.shape}")
    if min(a.shape) < _WINDOW:
        raise ValueError(f"image smaller than the {_WINDOW}x{_WINDOW} SSIM window")
    return float(ssim_batch(a.data, b.data, a.peak)[0])
