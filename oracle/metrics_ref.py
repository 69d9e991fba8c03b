"""CPU restatement of the reference's image metrics -- TEST INFRASTRUCTURE ONLY
(the checker for the GPU SSIM in paper_2204_07921_b200/metrics.py; never on a
product path).  Follows /root/reference/pkg/src/curvemg/image.py:

* psnr  image.py:140-149
* ssim  image.py:152-192 (_gaussian_window :157-160, _filter_valid :163-167)

Pinned against tests/golden/metrics.json (values produced by the reference).
"""

from __future__ import annotations

import math

import numpy as np


def gaussian_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    x = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    g = np.exp(-(x * x) / (2.0 * sigma * sigma))
    return g / g.sum()


def filter_valid(arr: np.ndarray, w: np.ndarray) -> np.ndarray:
    k = w.size
    rows = sum(w[i] * arr[i: arr.shape[0] - k + 1 + i, :] for i in range(k))
    return sum(w[i] * rows[:, i: arr.shape[1] - k + 1 + i] for i in range(k))


def ssim(x: np.ndarray, y: np.ndarray, peak: float) -> float:
    w = gaussian_window()
    mx, my = filter_valid(x, w), filter_valid(y, w)
    vx = filter_valid(x * x, w) - mx * mx
    vy = filter_valid(y * y, w) - my * my
    cxy = filter_valid(x * y, w) - mx * my
    c1 = (0.01 * peak) ** 2
    c2 = (0.03 * peak) ** 2
    num = (2.0 * mx * my + c1) * (2.0 * cxy + c2)
    den = (mx * mx + my * my + c1) * (vx + vy + c2)
    return float(np.mean(num / den))


def psnr(x: np.ndarray, y: np.ndarray, peak: float) -> float:
    mse = float(np.mean((x - y) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)
