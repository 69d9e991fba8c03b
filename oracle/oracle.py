"""ctypes wrapper around the C oracle (``oracle/cmg_oracle.c``).

TEST INFRASTRUCTURE ONLY -- imported by tests/, ``__graft_entry__.smoke()``
and bench.py's CPU-baseline / ``--impl reference`` legs as the checker.  The
product package never imports this module.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "build" / "libcmg_oracle.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < (_HERE / "cmg_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.orc_sweep_layer.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.orc_sweep_layer.restype = ctypes.c_int
        L.orc_energy.argtypes = [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int]
        L.orc_energy.restype = ctypes.c_double
        L.orc_curvature_sum.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        L.orc_curvature_sum.restype = ctypes.c_double
        L.orc_pad_odd.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, _dp]
        L.orc_pad_odd.restype = None
        L.orc_plane_table.argtypes = [ctypes.c_int, _ip, _dp]
        L.orc_plane_table.restype = ctypes.c_int
        L.orc_pairwise_sum.argtypes = [_dp, ctypes.c_long]
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_denoise.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                  ctypes.c_double, ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _ip]
        L.orc_denoise.restype = ctypes.c_int
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _c(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


MODES = {"mean": 0, "gaussian": 1}


def sweep_layer(u: np.ndarray, f: np.ndarray, layer: int, mode: str = "mean", inner_iters: int = 1,
                alpha: float = 0.06, threads: int = 1) -> np.ndarray:
    """driver.sweep_layer (driver.py:225-251) on a copy of ``u``; returns the new u."""
    u = _f64(u).copy()
    f = _f64(f)
    m, n = u.shape
    rc = lib().orc_sweep_layer(_c(u), _c(f), m, n, layer, MODES[mode], inner_iters, alpha, threads)
    if rc == 1:
        raise ValueError("corrections must be finite")
    if rc != 0:
        raise ValueError("bad arguments")
    return u


def energy(u, f, alpha: float = 0.06, mode: str = "mean") -> float:
    """tangent.energy (tangent.py:328-341)."""
    u, f = _f64(u), _f64(f)
    m, n = u.shape
    return lib().orc_energy(_c(u), _c(f), m, n, alpha, MODES[mode])


def curvature_field(u, mode: str = "mean") -> np.ndarray:
    u = _f64(u)
    m, n = u.shape
    out = np.empty((m, n))
    lib().orc_curvature_sum(_c(u), m, n, MODES[mode], _c(out))
    return out


def pad_odd(a, widths) -> np.ndarray:
    """np.pad(a, widths, mode='reflect', reflect_type='odd') restated."""
    a = _f64(a)
    (t, b), (l, r) = widths
    m, n = a.shape
    out = np.empty((m + t + b, n + l + r))
    lib().orc_pad_odd(_c(a), m, n, t, b, l, r, _c(out))
    return out


def plane_table(layer: int):
    offs = np.zeros((256, 6), dtype=np.int32)
    ds2 = np.zeros(256)
    k = lib().orc_plane_table(layer, offs.ctypes.data_as(_ip), _c(ds2))
    return offs[:k].copy(), ds2[:k].copy()


def denoise(f, alpha: float = 0.06, mode: str = "mean", layers: int = 3, epsilon: float = 1e-6,
            max_outer: int = 500, inner_iters: int = 1, stop_rule: str = "rel_energy",
            full_vcycle: bool = False, reference=None, peak: float = 1.0, threads: int = 1) -> dict:
    """driver.denoise (driver.py:261-314) restated; returns u and the trace arrays."""
    f = _f64(f)
    m, n = f.shape
    u = np.empty_like(f)
    cap = max_outer + 1
    en = np.full(cap, np.nan)
    re = np.full(cap, np.nan)
    ru = np.full(cap, np.nan)
    ps = np.full(cap, np.nan)
    it = ctypes.c_int(0)
    ref = _f64(reference) if reference is not None else None
    status = lib().orc_denoise(_c(f), m, n, alpha, MODES[mode], layers, epsilon, max_outer, inner_iters,
                               0 if stop_rule == "rel_energy" else 1, int(full_vcycle),
                               _c(ref) if ref is not None else None, peak, threads, _c(u), _c(en), _c(re),
                               _c(ru), _c(ps), ctypes.byref(it))
    k = it.value
    return {
        "u": u,
        "status": status,
        "converged": status == 0,
        "iterations": k,
        "energies": en[: k + 1].copy(),
        "rel_energy": re[: k + 1].copy(),
        "rel_u": ru[: k + 1].copy(),
        "psnr": ps[: k + 1].copy() if ref is not None else None,
    }


def max_threads() -> int:
    return int(lib().orc_max_threads())
