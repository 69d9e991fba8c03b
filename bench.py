"""Benchmark: the BASELINE metric on the B200 hot path.

Workload (BASELINE.json configs[2], the metric's "1024^2 time-to-tolerance"):
mean-curvature denoising of the seeded 1024x1024 synthetic image (32 shapes +
texture, sigma 25/255), J=3 levels, alpha=0.06, epsilon=1e-6 (40 V-cycles, as
the reference).  One STEP = one complete denoise to tolerance.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype float64|float32] [--precision exact|fast] [--config 3]

Prints one JSON line (rank 0).  Under torchrun (N>1) every rank solves its own
replica (the image does not shard: "replicas only", weak scaling); value is
the total over ranks divided by the max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

HBM_FALLBACK = 6650.0


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_sample(f, layers, cycles, threads):
    """Oracle (port of the reference algorithm) on a bounded sample; returns Mpx-sweeps/s."""
    from oracle import oracle as O

    t = time.perf_counter()
    r = O.denoise(f, mode="mean", layers=layers, max_outer=cycles, epsilon=1e-300, threads=threads)
    dt = time.perf_counter() - t
    m, n = f.shape
    return cycles * layers * m * n / dt / 1e6, dt, r


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2204_07921_b200 import synth

    f, _ = synth.config_input(args.config, 0, fp32=(args.dtype == "float32"))
    layers = synth.CONFIGS[args.config]["layers"]
    threads = O.max_threads()
    cycles = args.ref_cycles
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_sample(f, layers, 1, threads)
    vals, times = [], []
    for _ in range(args.steps):
        v, dt, _ = cpu_sample(f, layers, cycles, threads)
        vals.append(v)
        times.append(dt)
    value = float(np.mean(vals))
    m, n = f.shape
    line = {
        "impl": "reference",
        "metric": "Mpixel-sweeps/s (1024^2 MC denoise, J=3)",
        "value": value,
        "unit": "Mpixel-sweeps/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE seeded generator, SURVEY 8d)",
        "config": {"workload": f"config{args.config}: {m}x{n} mean-curvature denoise, J={layers}, alpha=0.06",
                   "sample": f"{cycles} V-cycles per step"},
        "cpu_baseline": {"value": value, "unit": "Mpixel-sweeps/s", "cores": threads, "kind": "port",
                         "sample": f"{cycles} V-cycles of config {args.config} per step (oracle/cmg_oracle.c, "
                                   f"OpenMP over patches, {threads} threads)"},
        "e2e": {"value": value, "unit": "Mpixel-sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import ctypes

    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2204_07921_b200 import _native as N
    from paper_2204_07921_b200 import synth

    c = synth.CONFIGS[args.config]
    f, clean = synth.config_input(args.config, 0, fp32=(args.dtype == "float32"))
    m, n = f.shape
    layers = c["layers"]
    eps = c.get("eps", 1e-300)
    max_outer = c["cycles"]
    prec = args.precision
    plan = N.Plan(m, n, 1, layers, c["mode"], args.dtype, prec, device=local)
    L = N.lib()
    dt = np.float64 if args.dtype == "float64" else np.float32
    esz = np.dtype(dt).itemsize
    nbytes = m * n * esz
    # pinned host buffers for the end-to-end leg
    hp_f = L.cmg_host_alloc(nbytes)
    hp_u = L.cmg_host_alloc(nbytes)
    f_h = np.frombuffer((ctypes.c_char * nbytes).from_address(hp_f), dtype=dt).reshape(m, n)
    u_h = np.frombuffer((ctypes.c_char * nbytes).from_address(hp_u), dtype=dt).reshape(m, n)
    f_h[...] = f.astype(dt)
    cap = max_outer + 1
    en = np.zeros(cap)
    its = np.zeros(1, dtype=np.int32)
    sts = np.zeros(1, dtype=np.int32)

    def solve_host():
        rc = L.cmg_solve(plan.handle, N.ptr(f_h), None, N.ptr(u_h), 0.06, eps, max_outer, 1, 0, 0, 1.0,
                         N.dptr(en), None, None, None, None, N.iptr(its), N.iptr(sts))
        assert rc in (0, 2), N.last_error()

    def solve_dev():
        rc = L.cmg_solve_device(plan.handle, None, None, None, 0.06, eps, max_outer, 1, 0, 0, 1.0,
                                N.dptr(en), None, None, None, None, N.iptr(its), N.iptr(sts))
        assert rc in (0, 2), N.last_error()

    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def l2_flush():
        flush.random_(0, 255)
        torch.cuda.synchronize()

    solve_host()  # uploads f and builds the graph
    for _ in range(max(args.warmup, 3)):
        solve_dev()
    cycles = int(its[0])
    # ---- device-resident timed region (CUDA events inside libcmg around each solve) ----
    sampler = ClockSampler(local)
    sampler.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    dev_ms = []
    launches = 0
    for _ in range(args.steps):
        l2_flush()
        solve_dev()
        st = plan.stats()
        dev_ms.append(st["device_ms"])
        launches += st["kernel_launches"]
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    ms_step = float(np.mean(dev_ms))
    # ---- end-to-end through the C ABI with pinned host buffers ----
    e2e_t = []
    for _ in range(args.steps):
        l2_flush()
        t0 = time.perf_counter()
        solve_host()
        e2e_t.append(time.perf_counter() - t0)
    e2e_ms = 1e3 * float(np.mean(e2e_t))
    # ---- roofline: level-1 four-colour sweep, CUDA events on the plan's stream ----
    l1_ms = plan.time_sweep(1, -1, reps=50)
    lvl_ms = {j: plan.time_sweep(j, -1, reps=20) for j in range(2, layers + 1)}
    px_sweeps = cycles * layers * m * n
    if ws > 1:
        tt = torch.tensor([ms_step, e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms_step, e2e_ms = float(tt[0]), float(tt[1])
    value = ws * px_sweeps / (ms_step * 1e-3) / 1e6
    e2e_value = ws * px_sweeps / (e2e_ms * 1e-3) / 1e6
    peak, peak_src = measured_peaks()
    alg_bytes = 3 * esz * m * n  # read u, read f, write u per pixel-sweep
    achieved = alg_bytes / (l1_ms * 1e-3) / 1e9
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from oracle import oracle as O

        thr = O.max_threads()
        v, dtc, _ = cpu_sample(f, layers, args.ref_cycles, thr)
        cpu = {"value": v, "unit": "Mpixel-sweeps/s", "cores": thr, "kind": "port",
               "sample": f"{args.ref_cycles} V-cycles of config {args.config} ({dtc:.1f} s, oracle/cmg_oracle.c, "
                         f"OpenMP {thr} threads)"}
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(f"{args.dtype}_{prec}_l1")
        except Exception:
            traffic = None
    line = {
        "metric": "Mpixel-sweeps/s (1024^2 MC denoise to tolerance, J=3)",
        "value": value,
        "unit": "Mpixel-sweeps/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64" if args.dtype == "float64" else "f32",
        "data": "synthetic (BASELINE seeded generator, SURVEY 8d)",
        "config": {"workload": f"config{args.config}: {m}x{n} mean-curvature denoise, J={layers}, alpha=0.06, "
                               f"eps={eps:g}, precision={prec}",
                   "cycles_to_tolerance": cycles, "time_to_tolerance_ms": ms_step,
                   "l2": "flushed (512 MiB write) before every timed step; working set is L2-resident within a solve",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "level_sweep_ms": {"1": l1_ms, **{str(k): v for k, v in lvl_ms.items()}}},
        "e2e": {"value": e2e_value, "unit": "Mpixel-sweeps/s", "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": nbytes + 8 * cap, "ms_per_step": e2e_ms},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": "k_sweep_tpp level 1 (4 colour launches)",
                     "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src},
        "clocks": clocks,
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    L.cmg_host_free(hp_f)
    L.cmg_host_free(hp_u)
    plan.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--dtype", choices=["float64", "float32"], default="float64")
    ap.add_argument("--precision", choices=["exact", "fast"], default="exact")
    ap.add_argument("--ref-cycles", type=int, default=6)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
