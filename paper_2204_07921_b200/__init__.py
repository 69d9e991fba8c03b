"""paper_2204_07921_b200 -- B200-native multigrid curvature-energy denoising.

Drop-in for the solver entry points of the reference package ``curvemg``
(arXiv 2204.07921; /root/reference/pkg/src/curvemg/__init__.py:3-26): the
same ``denoise(f, config, reference=None) -> (Image, ConvergenceTrace)`` call,
backed by hand-written sm_100a CUDA kernels in ``libcmg.so`` (C ABI:
include/cmg.h).  There is no CPU fallback.
"""

from .driver import (
    MAX_LAYER,
    ConvergenceTrace,
    SolverConfig,
    SolverDivergence,
    TraceRecord,
    denoise,
    denoise_batch,
    energy,
    rel_err_energy,
    rel_err_u,
)
from .image import Image, NoiseSpec, add_gaussian_noise, psnr
from .metrics import ssim, ssim_batch
from .phantoms import phantom
from .planes import planes as plane_table

__all__ = [
    "MAX_LAYER",
    "ConvergenceTrace",
    "SolverConfig",
    "SolverDivergence",
    "TraceRecord",
    "denoise",
    "denoise_batch",
    "energy",
    "rel_err_energy",
    "rel_err_u",
    "Image",
    "NoiseSpec",
    "add_gaussian_noise",
    "psnr",
    "ssim",
    "ssim_batch",
    "plane_table",
    "phantom",
]

__version__ = "0.1.0"
