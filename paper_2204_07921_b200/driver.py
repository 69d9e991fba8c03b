"""Drop-in solver API: the reference ``curvemg.driver`` names on the B200 path.

Mirrors /root/reference/pkg/src/curvemg/driver.py:

* ``SolverConfig``      driver.py:42-80  (same fields, defaults and validation;
                                          plus ``dtype``, ``precision``, ``device``)
* ``TraceRecord``       driver.py:83-91
* ``ConvergenceTrace``  driver.py:97-143 (same CSV schema ``curvemg-trace-1``)
* ``SolverDivergence``  driver.py:38-39
* ``rel_err_energy``    driver.py:146-150
* ``rel_err_u``         driver.py:153-158
* ``denoise``           driver.py:261-314 -> libcmg.so ``cmg_solve``
* ``denoise_batch``     (new) B images of one shape in one launch sequence

The whole outer loop runs on the GPU (one CUDA graph with a device-side WHILE
node); this module only validates, copies and builds the trace.
"""

from __future__ import annotations

import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .image import Image

__all__ = [
    "SolverConfig",
    "TraceRecord",
    "ConvergenceTrace",
    "SolverDivergence",
    "denoise",
    "denoise_batch",
    "energy",
    "rel_err_energy",
    "rel_err_u",
    "MAX_LAYER",
]

MAX_LAYER = 6  # tangent.py:43
COLOR_ORDER = ((0, 0), (0, 1), (1, 0), (1, 1))  # driver.py:35


class SolverDivergence(RuntimeError):
    """Raised when the objective stops being finite (driver.py:38-39)."""


@dataclass(frozen=True)
class SolverConfig:
    """Knobs of the multi-grid solver (driver.py:42-80).

    Extra B200 fields (not in the reference):
      dtype      "float64" (reference arithmetic) or "float32" (fast storage)
      precision  "exact" (NumPy operation order; bit-identical in float64) or
                 "fast" (closed-form pair distances + rsqrt, mean mode only)
      device     CUDA device ordinal
    """

    alpha: float = 0.06
    mode: str = "mean"
    layers: int = 3
    epsilon: float = 1e-6
    max_outer: int = 500
    inner_iters: int = 1
    stop_rule: str = "rel_energy"
    full_vcycle: bool = False
    threads: int | None = None
    dtype: str = "float64"
    precision: str = "exact"
    device: int = 0

    def __post_init__(self):
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")
        if self.mode not in ("mean", "gaussian"):
            raise ValueError(f"mode must be 'mean' or 'gaussian', got {self.mode!r}")
        if not 1 <= self.layers <= MAX_LAYER:
            raise ValueError(f"layers must be in [1, {MAX_LAYER}]")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.max_outer < 1:
            raise ValueError("max_outer must be at least 1")
        if not 1 <= self.inner_iters <= 15:
            raise ValueError("inner_iters must be in [1, 15]")
        if self.stop_rule not in ("rel_energy", "rel_u"):
            raise ValueError(f"stop_rule must be 'rel_energy' or 'rel_u', got {self.stop_rule!r}")
        if self.threads is not None and self.threads < 1:
            raise ValueError("threads must be positive")
        if self.dtype not in ("float64", "float32"):
            raise ValueError(f"dtype must be 'float64' or 'float32', got {self.dtype!r}")
        if self.precision not in ("exact", "fast"):
            raise ValueError(f"precision must be 'exact' or 'fast', got {self.precision!r}")

    def resolved_threads(self) -> int:
        """Kept for API parity (driver.py:74-80); the GPU path does not use host threads."""
        if self.threads is not None:
            return self.threads
        env = os.environ.get("CURVEMG_THREADS")
        if env:
            return max(1, int(env))
        return os.cpu_count() or 1


def _coerce_config(config) -> SolverConfig:
    """Accept our SolverConfig or any object with the reference's fields."""
    if isinstance(config, SolverConfig):
        return config
    kw = {k: getattr(config, k) for k in ("alpha", "mode", "layers", "epsilon", "max_outer", "inner_iters",
                                          "stop_rule", "full_vcycle", "threads") if hasattr(config, k)}
    for k in ("dtype", "precision", "device"):
        if hasattr(config, k):
            kw[k] = getattr(config, k)
    return SolverConfig(**kw)


@dataclass(frozen=True)
class TraceRecord:
    iteration: int
    energy: float
    rel_energy: float
    rel_u: float
    seconds: float
    psnr: float | None = None


_TRACE_SCHEMA = "curvemg-trace-1"


@dataclass
class ConvergenceTrace:
    """Per-outer-iteration convergence log (driver.py:97-143)."""

    records: list[TraceRecord] = field(default_factory=list)
    converged: bool = False

    @property
    def iterations(self) -> int:
        return self.records[-1].iteration if self.records else 0

    @property
    def final_energy(self) -> float:
        return self.records[-1].energy

    def energies(self) -> np.ndarray:
        return np.array([r.energy for r in self.records])

    def to_csv(self, path) -> None:
        lines = [f"# schema={_TRACE_SCHEMA}", "iter,energy,rel_energy,rel_u,seconds,psnr"]
        for r in self.records:
            psnr_s = "" if r.psnr is None else repr(r.psnr)
            rel_e = "" if math.isnan(r.rel_energy) else repr(r.rel_energy)
            rel_u = "" if math.isnan(r.rel_u) else repr(r.rel_u)
            lines.append(f"{r.iteration},{r.energy!r},{rel_e},{rel_u},{r.seconds!r},{psnr_s}")
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")

    @classmethod
    def from_csv(cls, path) -> "ConvergenceTrace":
        with open(path) as fh:
            lines = [ln.strip() for ln in fh if ln.strip()]
        if not lines or lines[0] != f"# schema={_TRACE_SCHEMA}":
            raise ValueError(f"unrecognized trace schema in {path}")
        records = []
        for ln in lines[2:]:
            it, en, re_, ru, sec, ps = ln.split(",")
            records.append(TraceRecord(iteration=int(it), energy=float(en),
                                       rel_energy=float(re_) if re_ else math.nan,
                                       rel_u=float(ru) if ru else math.nan, seconds=float(sec),
                                       psnr=float(ps) if ps else None))
        return cls(records)


def rel_err_energy(f_new: float, f_old: float) -> float:
    """Relative change of the objective; |f_old| when f_new is 0 (driver.py:146-150)."""
    if f_new == 0.0:
        return abs(f_old)
    return abs(f_new - f_old) / abs(f_new)


def rel_err_u(u_new: np.ndarray, u_old: np.ndarray) -> float:
    """L1 relative change of the iterate (driver.py:153-158)."""
    denom = float(np.abs(u_new).sum())
    if denom == 0.0:
        raise ValueError("rel_err_u undefined for an all-zero iterate")
    return float(np.abs(np.asarray(u_new) - np.asarray(u_old)).sum()) / denom


# ---------------------------------------------------------------------------
# plan cache (device buffers and CUDA graphs are reused across calls)
# ---------------------------------------------------------------------------
_tls = threading.local()
_PLAN_CAP = 16


def get_plan(m: int, n: int, batch: int, cfg: SolverConfig) -> N.Plan:
    """Per-thread plan cache: a plan (device buffers, stream, graph) is only
    ever used and evicted by the thread that created it, so one thread's
    eviction can never free a plan another thread is solving with."""
    plans = getattr(_tls, "plans", None)
    if plans is None:
        plans = _tls.plans = {}
    key = (m, n, batch, cfg.layers, cfg.mode, cfg.dtype, cfg.precision, cfg.device)
    p = plans.get(key)
    if p is None:
        if len(plans) >= _PLAN_CAP:
            for k in list(plans)[: _PLAN_CAP // 2]:
                plans.pop(k).close()
        p = N.Plan(m, n, batch, cfg.layers, cfg.mode, cfg.dtype, cfg.precision, cfg.device)
        plans[key] = p
    return p


def _as_image(x, what: str) -> Image:
    """Duck-typed Image: ours, the reference's ``curvemg.image.Image`` or any
    object with a 2-D ``.data`` and a ``.peak`` (image.py:34-75)."""
    if isinstance(x, Image):
        return x
    if hasattr(x, "data") and hasattr(x, "peak"):
        return Image(np.asarray(x.data), float(x.peak))
    raise TypeError(f"{what} must be an Image")


def _np_dtype(cfg: SolverConfig):
    return np.float64 if cfg.dtype == "float64" else np.float32


def _raise_for(rc: int):
    msg = N.last_error()
    if rc == N.CMG_EINVAL:
        raise ValueError(msg)
    if rc == N.CMG_ENONFINITE:
        raise ValueError("corrections must be finite")
    if rc == N.CMG_ECUDA:
        raise RuntimeError(f"CUDA failure in libcmg: {msg}")


def get_mplan(m: int, n: int, batch: int, cfg: SolverConfig, devices) -> N.MPlan:
    """Per-thread cache of multi-device batch plans (cmg_mplan)."""
    plans = getattr(_tls, "mplans", None)
    if plans is None:
        plans = _tls.mplans = {}
    key = (m, n, batch, cfg.layers, cfg.mode, cfg.dtype, cfg.precision, tuple(devices))
    p = plans.get(key)
    if p is None:
        if len(plans) >= _PLAN_CAP:
            for k in list(plans)[: _PLAN_CAP // 2]:
                plans.pop(k).close()
        p = N.MPlan(m, n, batch, cfg.layers, cfg.mode, cfg.dtype, cfg.precision, list(devices))
        plans[key] = p
    return p


def _solve(fs: np.ndarray, refs, cfg: SolverConfig, peak: float, devices=None):
    """Run cmg_solve (or cmg_mplan_solve over ``devices``) on a (B, m, n) host
    stack; returns (u, traces, statuses, plan)."""
    B, m, n = fs.shape
    multi = devices is not None and len(devices) > 0
    plan = get_mplan(m, n, B, cfg, devices) if multi else get_plan(m, n, B, cfg)
    solve = N.lib().cmg_mplan_solve if multi else N.lib().cmg_solve
    dt = _np_dtype(cfg)
    f_in = np.ascontiguousarray(fs, dtype=dt)
    r_in = None if refs is None else np.ascontiguousarray(refs, dtype=dt)
    u = np.empty_like(f_in)
    cap = cfg.max_outer + 1
    tr = {k: np.full((B, cap), np.nan) for k in ("energy", "rel_e", "rel_u", "psnr", "sec")}
    its = np.zeros(B, dtype=np.int32)
    sts = np.zeros(B, dtype=np.int32)
    rc = solve(plan.handle, N.ptr(f_in), N.ptr(r_in), N.ptr(u), cfg.alpha, cfg.epsilon,
                           cfg.max_outer, cfg.inner_iters, N.STOP[cfg.stop_rule], int(cfg.full_vcycle), peak,
                           N.dptr(tr["energy"]), N.dptr(tr["rel_e"]), N.dptr(tr["rel_u"]), N.dptr(tr["psnr"]),
                           N.dptr(tr["sec"]), N.iptr(its), N.iptr(sts))
    if rc in (N.CMG_EINVAL, N.CMG_ECUDA):
        _raise_for(rc)
    traces = []
    for b in range(B):
        k = int(its[b])
        recs = []
        for i in range(k + 1):
            ps = None if r_in is None else float(tr["psnr"][b, i])
            recs.append(TraceRecord(i, float(tr["energy"][b, i]), float(tr["rel_e"][b, i]),
                                    float(tr["rel_u"][b, i]), float(tr["sec"][b, i]), ps))
        traces.append(ConvergenceTrace(recs, converged=bool(sts[b] == N.CMG_OK)))
    return u, traces, sts, plan


def denoise(f: Image, config, reference: Image | None = None) -> tuple[Image, ConvergenceTrace]:
    """Minimize the curvature energy of ``f`` on the GPU (driver.py:261-314).

    Same contract as the reference: starts from u = f, sweeps levels
    fine-to-coarse each outer iteration (half V-cycle; full with
    ``full_vcycle``) and stops when rel_energy (or rel_u) <= epsilon.
    Raises ValueError for invalid input / non-finite corrections and
    SolverDivergence when the objective becomes non-finite.
    """
    cfg = _coerce_config(config)
    f = _as_image(f, "f")
    if reference is not None:
        reference = _as_image(reference, "reference")
    if reference is not None and reference.shape != f.shape:
        raise ValueError(f"shape mismatch: {f.shape} vs {reference.shape}")
    m, n = f.shape
    refs = None if reference is None else reference.data[None]
    u, traces, sts, _ = _solve(f.data[None], refs, cfg, f.peak)
    st = int(sts[0])
    if st == N.CMG_DIVERGED:
        raise SolverDivergence(f"objective became non-finite at outer iteration {traces[0].iterations + 1}")
    if st == N.CMG_ENONFINITE:
        raise ValueError("corrections must be finite")
    return Image._from_solver(u[0], f.peak), traces[0]


def denoise_batch(fs, config, references=None, peak: float | None = None, devices=None):
    """Denoise B same-shape images in one launch sequence (per-image stopping).

    ``fs`` is a list of Images or a (B, m, n) array; returns a list of
    (Image, ConvergenceTrace).  Divergent images raise like ``denoise``.
    ``devices`` (list of CUDA ordinals, may repeat) shards the batch
    data-parallel over those GPUs (cmg_mplan: contiguous image slices, one
    host thread per shard, no collective); results are identical to one plan.
    """
    cfg = _coerce_config(config)
    if isinstance(fs, np.ndarray):
        stack = fs
        pk = 255.0 if peak is None else peak
    else:
        fs = list(fs)
        stack = np.stack([x.data for x in fs])
        pk = fs[0].peak if peak is None else peak
    if stack.ndim != 3:
        raise ValueError("expected a (B, m, n) stack")
    refs = None
    if references is not None:
        refs = references if isinstance(references, np.ndarray) else np.stack([r.data for r in references])
    u, traces, sts, _ = _solve(stack, refs, cfg, pk, devices)
    for b, st in enumerate(sts):
        if st == N.CMG_DIVERGED:
            raise SolverDivergence(f"image {b}: objective became non-finite")
        if st == N.CMG_ENONFINITE:
            raise ValueError(f"image {b}: corrections must be finite")
    return [(Image._from_solver(u[b], pk), traces[b]) for b in range(stack.shape[0])]


def energy(u, f, alpha: float, mode: str = "mean", device: int = 0) -> float:
    """Total discrete energy on the GPU (tangent.energy, tangent.py:325-341):
    level-1 curvature magnitude sum + alpha/2 ||u - f||^2, float64 (libcmg
    cmg_energy; within 1e-12 relative of the reference's pairwise NumPy sum)."""
    ua = np.ascontiguousarray(getattr(u, "data", u), dtype=np.float64)
    fa = np.ascontiguousarray(getattr(f, "data", f), dtype=np.float64)
    if ua.shape != fa.shape:
        raise ValueError(f"shape mismatch: {ua.shape} vs {fa.shape}")
    if alpha <= 0:
        raise ValueError("alpha must be positive")
    if mode not in ("mean", "gaussian"):
        raise ValueError(f"mode must be 'mean' or 'gaussian', got {mode!r}")
    if ua.ndim != 2:
        raise ValueError("energy expects 2-D images")
    plan = get_plan(ua.shape[0], ua.shape[1], 1, SolverConfig(layers=1, mode=mode, device=device))
    out = np.zeros(1)
    rc = N.lib().cmg_energy(plan.handle, N.ptr(ua), N.ptr(fa), float(alpha), N.dptr(out))
    if rc != N.CMG_OK:
        _raise_for(rc)
    return float(out[0])
