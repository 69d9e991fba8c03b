"""ctypes binding of libcmg.so (the sm_100a solver, C ABI in include/cmg.h).

There is deliberately NO fallback: if the shared library is missing or no
CUDA device is usable, every solver call raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("CMG_LIBRARY", _PKG / "libcmg.so"))

CMG_OK, CMG_EINVAL, CMG_NOT_CONVERGED, CMG_DIVERGED, CMG_ECUDA, CMG_ENONFINITE = 0, 1, 2, 3, 4, 5
MODE = {"mean": 0, "gaussian": 1}
DTYPE = {"float64": 0, "float32": 1}
PREC = {"exact": 0, "fast": 1}
STOP = {"rel_energy": 0, "rel_u": 1}

# every symbol declared in include/cmg.h
SYMBOLS = (
    "cmg_version", "cmg_last_error", "cmg_device_count", "cmg_plan_create", "cmg_plan_destroy", "cmg_solve",
    "cmg_solve_device", "cmg_sweep_layer", "cmg_energy", "cmg_plane_table", "cmg_plan_stats", "cmg_time_sweep",
    "cmg_host_alloc", "cmg_host_free", "cmg_plan_buffer", "cmg_buffer_upload", "cmg_buffer_download",
    "cmg_level_step", "cmg_energy_partials", "cmg_ssim_batch", "cmg_plan_ssim", "cmg_l2_read_bandwidth",
    "cmg_selftest_exact", "cmg_fp64_probe",
    "cmg_plan_stream", "cmg_strip_begin", "cmg_level_step_async", "cmg_strip_partials_async", "cmg_strip_read",
    "cmg_mplan_create", "cmg_mplan_destroy", "cmg_mplan_solve",
    "cmg_radon_create", "cmg_radon_destroy", "cmg_radon_forward", "cmg_radon_adjoint", "cmg_recon_chalf",
    "cmg_recon_prolong", "cmg_recon_block_sums", "cmg_recon_curvature_partials",
)


class NativeUnavailable(RuntimeError):
    """libcmg.so is missing or could not be loaded (no CPU fallback exists)."""


_lib = None

_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_i = ctypes.c_int
_d = ctypes.c_double


def _declare(L):
    L.cmg_version.restype = _i
    L.cmg_version.argtypes = []
    L.cmg_last_error.restype = ctypes.c_char_p
    L.cmg_last_error.argtypes = []
    L.cmg_device_count.restype = _i
    L.cmg_device_count.argtypes = [_ip]
    L.cmg_plan_create.restype = _i
    L.cmg_plan_create.argtypes = [ctypes.POINTER(_vp), _i, _i, _i, _i, _i, _i, _i, _i]
    L.cmg_plan_destroy.restype = _i
    L.cmg_plan_destroy.argtypes = [_vp]
    solve_args = [_vp, _vp, _vp, _vp, _d, _d, _i, _i, _i, _i, _d, _dp, _dp, _dp, _dp, _dp, _ip, _ip]
    L.cmg_solve.restype = _i
    L.cmg_solve.argtypes = solve_args
    L.cmg_solve_device.restype = _i
    L.cmg_solve_device.argtypes = solve_args
    L.cmg_sweep_layer.restype = _i
    L.cmg_sweep_layer.argtypes = [_vp, _vp, _vp, _i, _d, _i]
    L.cmg_energy.restype = _i
    L.cmg_energy.argtypes = [_vp, _vp, _vp, _d, _dp]
    L.cmg_plane_table.restype = _i
    L.cmg_plane_table.argtypes = [_i, _ip, _dp]
    L.cmg_plan_stats.restype = _i
    L.cmg_plan_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_longlong), _ip, _dp]
    L.cmg_time_sweep.restype = _i
    L.cmg_time_sweep.argtypes = [_vp, _i, _i, _i, _dp]
    L.cmg_host_alloc.restype = _vp
    L.cmg_host_alloc.argtypes = [ctypes.c_ulonglong]
    L.cmg_radon_create.restype = _i
    L.cmg_radon_create.argtypes = [ctypes.POINTER(_vp), _i, _i, _i, _i, _d, _ip, _dp, _i]
    L.cmg_radon_destroy.restype = _i
    L.cmg_radon_destroy.argtypes = [_vp]
    for nm in ("cmg_radon_forward", "cmg_radon_adjoint"):
        getattr(L, nm).restype = _i
        getattr(L, nm).argtypes = [_vp, _vp, _vp, _vp]
    L.cmg_recon_chalf.restype = _i
    L.cmg_recon_chalf.argtypes = [_vp, _i, _i, _i, _i, _i, _vp, _vp]
    L.cmg_recon_prolong.restype = _i
    L.cmg_recon_prolong.argtypes = [_vp, _vp, _i, _i, _i, _i, _i, _vp]
    L.cmg_recon_block_sums.restype = _i
    L.cmg_recon_block_sums.argtypes = [_vp, _i, _i, _i, _i, _i, _vp, _vp]
    L.cmg_recon_curvature_partials.restype = _i
    L.cmg_recon_curvature_partials.argtypes = [_vp, _i, _i, _vp, _i, _vp]
    L.cmg_mplan_create.restype = _i
    L.cmg_mplan_create.argtypes = [ctypes.POINTER(_vp), _i, _i, _i, _i, _i, _i, _i, _ip, _i]
    L.cmg_mplan_destroy.restype = _i
    L.cmg_mplan_destroy.argtypes = [_vp]
    L.cmg_mplan_solve.restype = _i
    L.cmg_mplan_solve.argtypes = solve_args
    L.cmg_plan_stream.restype = _i
    L.cmg_plan_stream.argtypes = [_vp, ctypes.POINTER(_vp)]
    L.cmg_strip_begin.restype = _i
    L.cmg_strip_begin.argtypes = [_vp, _d, _i]
    L.cmg_level_step_async.restype = _i
    L.cmg_level_step_async.argtypes = [_vp, _i, _i, _i]
    L.cmg_strip_partials_async.restype = _i
    L.cmg_strip_partials_async.argtypes = [_vp, _i, _i, _i, _i, _i]
    L.cmg_strip_read.restype = _i
    L.cmg_strip_read.argtypes = [_vp, _dp]
    L.cmg_l2_read_bandwidth.restype = _i
    L.cmg_l2_read_bandwidth.argtypes = [_i, ctypes.c_longlong, _i, _dp]
    L.cmg_fp64_probe.restype = _i
    L.cmg_fp64_probe.argtypes = [_i, _dp, _dp, _dp]
    L.cmg_selftest_exact.restype = _i
    L.cmg_selftest_exact.argtypes = [_i, _dp, _dp, ctypes.c_longlong, ctypes.POINTER(ctypes.c_ulonglong)]
    L.cmg_host_free.restype = _i
    L.cmg_host_free.argtypes = [_vp]
    L.cmg_plan_buffer.restype = _i
    L.cmg_plan_buffer.argtypes = [_vp, _i, ctypes.POINTER(_vp)]
    L.cmg_buffer_upload.restype = _i
    L.cmg_buffer_upload.argtypes = [_vp, _i, _vp]
    L.cmg_buffer_download.restype = _i
    L.cmg_buffer_download.argtypes = [_vp, _i, _vp]
    L.cmg_level_step.restype = _i
    L.cmg_level_step.argtypes = [_vp, _i, _i, _i, _d, _i]
    L.cmg_energy_partials.restype = _i
    L.cmg_energy_partials.argtypes = [_vp, _i, _i, _i, _i, _i, _dp]
    L.cmg_ssim_batch.restype = _i
    L.cmg_ssim_batch.argtypes = [_i, _i, _i, _i, _vp, _vp, _dp, _d, _d, _dp]
    L.cmg_plan_ssim.restype = _i
    L.cmg_plan_ssim.argtypes = [_vp, _i, _i, _dp, _d, _d, _dp]


def lib():
    """Load libcmg.so (raises NativeUnavailable if it is absent)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeUnavailable(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_2204_07921_b200/csrc)")
        try:
            L = ctypes.CDLL(str(LIB_PATH))
        except OSError as e:  # pragma: no cover
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
        _declare(L)
        _lib = L
    return _lib


def last_error() -> str:
    return lib().cmg_last_error().decode(errors="replace")


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = lib().cmg_device_count(ctypes.byref(c))
    return c.value if rc == CMG_OK else 0


def ptr(a) -> ctypes.c_void_p:
    """Host pointer of a C-contiguous numpy array (or None)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


def dptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def iptr(a):
    return None if a is None else a.ctypes.data_as(_ip)


class Plan:
    """Owns one cmg_plan (device buffers + graphs) for a fixed problem shape."""

    def __init__(self, m: int, n: int, batch: int, layers: int, mode: str, dtype: str, precision: str,
                 device: int = 0):
        L = lib()
        h = _vp()
        rc = L.cmg_plan_create(ctypes.byref(h), m, n, batch, layers, MODE[mode], DTYPE[dtype], PREC[precision],
                               device)
        if rc != CMG_OK:
            msg = last_error()
            if rc == CMG_EINVAL:
                raise ValueError(msg)
            raise RuntimeError(f"cmg_plan_create failed ({rc}): {msg}")
        self.handle = h
        self.shape = (batch, m, n)
        self.layers, self.mode, self.dtype, self.precision, self.device = layers, mode, dtype, precision, device

    def close(self):
        if getattr(self, "handle", None):
            lib().cmg_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def stats(self):
        ln = ctypes.c_longlong(0)
        cy = ctypes.c_int(0)
        ms = ctypes.c_double(0)
        lib().cmg_plan_stats(self.handle, ctypes.byref(ln), ctypes.byref(cy), ctypes.byref(ms))
        return {"kernel_launches": ln.value, "cycles_run": cy.value, "device_ms": ms.value}

    def time_sweep(self, layer: int, color: int = -1, reps: int = 20) -> float:
        ms = ctypes.c_double(0)
        rc = lib().cmg_time_sweep(self.handle, layer, color, reps, ctypes.byref(ms))
        if rc != CMG_OK:
            raise RuntimeError(f"cmg_time_sweep failed ({rc}): {last_error()}")
        return ms.value


def l2_read_bandwidth(device: int = 0, nbytes: int = 32 << 20, reps: int = 50) -> float:
    """Measured L2 read bandwidth in GB/s (cmg_l2_read_bandwidth)."""
    out = ctypes.c_double(0.0)
    rc = lib().cmg_l2_read_bandwidth(device, nbytes, reps, ctypes.byref(out))
    if rc != CMG_OK:
        raise RuntimeError(last_error())
    return out.value


def fp64_probe(device: int = 0) -> dict:
    """cmg_fp64_probe: sustained DFMA rate (per clock and SM, and as TFLOP/s) and the
    dependent-chain latency of the device's FP64 pipe."""
    r, lat, tf = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_double(0)
    rc = lib().cmg_fp64_probe(device, ctypes.byref(r), ctypes.byref(lat), ctypes.byref(tf))
    if rc != CMG_OK:
        raise RuntimeError(last_error())
    return {"dfma_per_clk_per_sm": r.value, "dep_latency_cycles": lat.value, "tflops": tf.value}


def selftest_exact(a, b, device: int = 0):
    """cmg_selftest_exact: (sqrt mismatches, div mismatches, sqrt out-of-range, div out-of-range) of the
    branch-free correctly rounded sqrt(a) and a / b against the device library."""
    import numpy as np

    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape and a.ndim == 1
    out = (ctypes.c_ulonglong * 4)()
    rc = lib().cmg_selftest_exact(device, a.ctypes.data_as(_dp), b.ctypes.data_as(_dp), a.size, out)
    if rc != CMG_OK:
        raise RuntimeError(f"cmg_selftest_exact failed ({rc})")
    return tuple(int(x) for x in out)


class MPlan:
    """cmg_mplan: one batch sharded over several devices (ids may repeat)."""

    def __init__(self, m: int, n: int, batch: int, layers: int, mode: str, dtype: str, precision: str, devices):
        devs = (ctypes.c_int * len(devices))(*devices)
        h = _vp()
        rc = lib().cmg_mplan_create(ctypes.byref(h), m, n, batch, layers, MODE[mode], DTYPE[dtype], PREC[precision],
                                    devs, len(devices))
        if rc != CMG_OK:
            msg = last_error()
            if rc == CMG_EINVAL:
                raise ValueError(msg)
            raise RuntimeError(f"cmg_mplan_create failed ({rc}): {msg}")
        self.handle = h
        self.devices = tuple(devices)
        self.shape = (batch, m, n)

    def close(self):
        if getattr(self, "handle", None):
            lib().cmg_mplan_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

