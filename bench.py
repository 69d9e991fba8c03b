"""Benchmark: the BASELINE metric on the B200 hot path.

Default workload (BASELINE.json configs[2] -- the metric's "1024^2
time-to-tolerance"): mean-curvature denoising of the seeded 1024x1024 image
(32 shapes + texture, sigma 25/255), J=3, alpha=0.06, epsilon=1e-6 (40 V-cycles,
as the reference), float64 with the exact (bit-identical) arithmetic.  One STEP
= one complete denoise to tolerance.  Metric: pixel-sweeps per second (a
pixel-sweep = one pixel relaxed by one level's four-colour pass).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3|4|5] [--dtype float64|float32] [--precision exact|fast]

Multi-GPU (torchrun, one rank per GPU):
  config 3  one image does not shard -> replicas (weak scaling);
  config 4  64 x 512^2 fp32 images, 20 cycles, images sharded over ranks;
  config 5  16384^2 fp32, 10 cycles, horizontal strips with NCCL ghost-row
            exchange after every level (paper_2204_07921_b200.strips).
"""

from __future__ import annotations

import argparse
import ctypes
import json
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
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons sampled (NVML, every 5 ms) during the timed
    region; falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.reasons = set()
        self.smax = None
        self.stop_ev = threading.Event()
        self.nvml = None

    def _sample(self):
        nv = self.nvml
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        mask = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        for nm, bit in self.REASONS.items():
            if mask & bit:
                self.reasons.add(nm)

    def _loop(self):
        while not self.stop_ev.is_set():
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            self.nvml = nv
            self.h = None
            try:  # NVML ignores CUDA_VISIBLE_DEVICES: find the CUDA device by PCI address
                import torch

                pr = torch.cuda.get_device_properties(self.gpu)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = None
            if self.h is None:
                self.h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None

    def stop(self):
        if self.nvml is None:
            return self._smi_once()
        try:
            self._sample()  # at least one sample, taken at the end of the timed region
        except Exception:
            pass
        self.stop_ev.set()
        self.t.join(timeout=1)
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml 5 ms"}

    def _smi_once(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True, timeout=10).stdout.strip()
            parts = [x.strip() for x in out.split(",")]
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            reasons = [nm for nm, v in zip(names, parts[2:6]) if v.lower().startswith("active")]
            return {"sm_mhz": float(parts[0]), "sm_max_mhz": float(parts[1]), "reasons": reasons, "samples": 1,
                    "source": "nvidia-smi after the timed region"}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock query unavailable"], "samples": 0}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(cfgid: int, dtype: str, prec: str):
    from paper_2204_07921_b200 import synth

    c = synth.CONFIGS[cfgid]
    size, layers = c["size"], c["layers"]
    eps = c.get("eps", 1e-300)
    batch = c.get("batch", 1)
    desc = {1: "256^2 MC, J=6, 10 cycles", 2: "512^2 GC, J=6, eps 1e-6 / 50 cycles",
            3: "1024^2 MC to eps 1e-6, J=3", 4: "64 x 512^2 MC, J=3, 20 cycles",
            5: "16384^2 MC, J=3, 10 cycles"}[cfgid]
    return c, size, layers, eps, batch, f"config{cfgid}: {desc}, alpha=0.06, {dtype}, precision={prec}"


def config_dict(cfgid: int, desc: str, images: int, cycles: int, parallelism: str) -> dict:
    """The `config` object both arms print (same keys -> same_config)."""
    return {"workload": desc, "images": images, "cycles": cycles, "parallelism": parallelism,
            "l2": "flushed (512 MiB write) before every timed step; a 1024^2 solve is L2-resident after its "
                  "first sweep" if cfgid != 5 else "flushed before every step; the 16384^2 image (1 GiB per "
                  "buffer) is far larger than L2"}


WORKLOAD_IMAGES = {1: 1, 2: 1, 3: 1, 4: 64, 5: 1}
WORKLOAD_CYCLES = {1: 10, 2: 50, 3: 40, 4: 20, 5: 10}  # config 2 stops at its tolerance (<= 50)


def cpu_workload(cfgid: int, fp32: bool):
    """The bounded CPU sample of a config: the config's own solve (same
    stopping rule and cycle cap) on image 0, except config 5 whose 16384^2
    image is cut to a 1024-row band (10 cycles of it is ~13 s on 16 threads)."""
    from paper_2204_07921_b200 import synth

    c = synth.CONFIGS[cfgid]
    f, _ = synth.config_input(cfgid, 0, fp32=fp32)
    if cfgid == 5:
        f = f[:1024]
    return f, c["layers"], c["cycles"], c.get("eps", 1e-300), c["mode"]


def cpu_sample(f, layers, cycles, eps, threads, mode="mean", min_seconds=10.0):
    """The oracle (C port of the reference algorithm, fp64) on a bounded
    sample: whole solves of `f` repeated until at least `min_seconds` of CPU
    work.  Returns (Mpixel-sweeps/s, seconds per solve, solves, cycles)."""
    from oracle import oracle as O

    m, n = f.shape
    t_all, solves, px = 0.0, 0, 0
    while True:
        t = time.perf_counter()
        r = O.denoise(f, mode=mode, layers=layers, max_outer=cycles, epsilon=eps, threads=threads)
        t_all += time.perf_counter() - t
        solves += 1
        px += r["iterations"] * layers * m * n
        if t_all >= min_seconds:
            break
    return px / t_all / 1e6, t_all / solves, solves, r["iterations"]


def run_reference(args):
    """Reference arm: the reference algorithm on the host cores (oracle port,
    all threads), same workload / metric / unit, bounded sample per step."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    c, size, layers, eps, batch, desc = workload(args.config, args.dtype, args.precision)
    f, layers, cycles, eps, mode = cpu_workload(args.config, args.dtype == "float32")
    threads = O.max_threads()
    O.denoise(f, mode=mode, layers=layers, max_outer=1, epsilon=1e-300, threads=threads)  # warm-up
    vals, times, its = [], [], 0
    for _ in range(args.steps):
        v, dt, _, its = cpu_sample(f, layers, cycles, eps, threads, mode, min_seconds=0.0)
        vals.append(v)
        times.append(dt)
    value = float(np.mean(vals))
    sample = (f"one solve per step of {f.shape[0]}x{f.shape[1]} ({desc}; {its} cycles); oracle/cmg_oracle.c "
              f"(C restatement of the reference NumPy algorithm, fp64), OpenMP over patches, {threads} threads")
    par = {3: "replicas", 4: "dp (images sharded)", 5: "strips"}.get(args.config, "replicas")
    par = f"{par} x{ws}" if ws > 1 else ("single GPU, batch 64" if args.config == 4 else "single GPU")
    line = {
        "impl": "reference",
        "metric": "Mpixel-sweeps/s",
        "value": value,
        "unit": "Mpixel-sweeps/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True,
        "scaling": "weak" if args.config != 5 else "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE seeded generator, SURVEY 8d)",
        "config": config_dict(args.config, desc, WORKLOAD_IMAGES[args.config], its, par),
        "cpu_baseline": {"value": value, "unit": "Mpixel-sweeps/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Mpixel-sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class Pinned:
    """Pinned host array (cmg_host_alloc) for the end-to-end leg."""

    def __init__(self, shape, dtype):
        from paper_2204_07921_b200 import _native as N

        self.N = N
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        self.p = N.lib().cmg_host_alloc(self.nbytes)
        self.a = np.frombuffer((ctypes.c_char * self.nbytes).from_address(self.p), dtype=dtype).reshape(shape)

    def free(self):
        self.N.lib().cmg_host_free(self.p)


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2204_07921_b200 import _native as N
    from paper_2204_07921_b200 import synth

    c, size, layers, eps, batch, desc = workload(args.config, args.dtype, args.precision)
    max_outer = c["cycles"]
    dt = np.float64 if args.dtype == "float64" else np.float32
    esz = np.dtype(dt).itemsize
    L = N.lib()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def l2_flush():
        flush.random_(0, 255)
        torch.cuda.synchronize()

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(*vals):
        if ws == 1:
            return vals
        t = torch.tensor(vals, device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return tuple(float(x) for x in t)

    extra = {}
    if args.config == 5 and ws > 1:
        value_ms, e2e_ms, cycles, launches, clocks, nbytes_in, nbytes_out, l1_ms, m_loc = run_strips(
            args, c, layers, dt, ws, rank, local, l2_flush, barrier, max_over_ranks)
        m, n = size, size
        px_sweeps = cycles * layers * m * n
        imgs_total = 1
        parallelism = f"strips x{ws} (NCCL ghost rows after every level)"
        plan = None
    else:
        # images handled by this rank
        if args.config == 4:
            per = batch // ws
            idx = list(range(rank * per, (rank + 1) * per))
            parallelism = f"dp{ws} (images sharded, no collective)" if ws > 1 else "single GPU, batch 64"
        else:
            idx = [0]
            parallelism = f"replicas x{ws}" if ws > 1 else "single GPU"
        fs = np.stack([synth.config_input(args.config, i, fp32=(args.dtype == "float32"))[0] for i in idx])
        B, m, n = fs.shape
        plan = N.Plan(m, n, B, layers, c["mode"], args.dtype, args.precision, device=local)
        nbytes = B * m * n * esz
        f_h = Pinned((B, m, n), dt)
        u_h = Pinned((B, m, n), dt)
        f_h.a[...] = fs.astype(dt)
        cap = max_outer + 1
        en = np.zeros(B * cap)
        its = np.zeros(B, dtype=np.int32)
        sts = np.zeros(B, dtype=np.int32)

        def solve_host():
            rc = L.cmg_solve(plan.handle, N.ptr(f_h.a), None, N.ptr(u_h.a), 0.06, eps, max_outer, 1, 0, 0, 1.0,
                             N.dptr(en), None, None, None, None, N.iptr(its), N.iptr(sts))
            assert rc in (0, 2), N.last_error()

        def solve_dev():
            rc = L.cmg_solve_device(plan.handle, None, None, None, 0.06, eps, max_outer, 1, 0, 0, 1.0,
                                    N.dptr(en), None, None, None, None, N.iptr(its), N.iptr(sts))
            assert rc in (0, 2), N.last_error()

        solve_host()  # uploads f, builds the graph
        for _ in range(max(args.warmup, 3)):
            solve_dev()
        cycles = int(its.max())
        sampler = ClockSampler(local)
        sampler.start()
        barrier()
        dev_ms, launches = [], 0
        for _ in range(args.steps):
            l2_flush()
            solve_dev()  # CUDA events on the plan's stream bracket the whole solve
            st = plan.stats()
            dev_ms.append(st["device_ms"])
            launches += st["kernel_launches"]
        barrier()
        clocks = sampler.stop()
        e2e_t = []
        for _ in range(args.steps):
            l2_flush()
            barrier()
            t0 = time.perf_counter()
            solve_host()  # H2D of f from pinned memory, solve, D2H of u + trace
            e2e_t.append(time.perf_counter() - t0)
        value_ms = float(np.mean(dev_ms))
        e2e_ms = 1e3 * float(np.mean(e2e_t))
        value_ms, e2e_ms = max_over_ranks(value_ms, e2e_ms)
        l1_ms = plan.time_sweep(1, -1, reps=50)
        extra["level_sweep_ms"] = {"1": l1_ms, **{str(j): plan.time_sweep(j, -1, reps=20)
                                                  for j in range(2, layers + 1)}}
        px_sweeps = cycles * layers * m * n * B * ws
        imgs_total = B * ws
        nbytes_in, nbytes_out = nbytes, nbytes + 8 * cap * B
        m_loc = m
        f_h.free()
        u_h.free()
    value = px_sweeps / (value_ms * 1e-3) / 1e6
    e2e_value = px_sweeps / (e2e_ms * 1e-3) / 1e6
    peak, peak_src = measured_peaks()
    # dominant kernel: the level-1 sweep (fused four-colour tile kernel);
    # algorithmic bytes = 3*sizeof(T) per pixel (read u, read f, write u)
    alg_bytes = 3 * esz * m_loc * n * (1 if args.config != 4 else len(idx))
    achieved = alg_bytes / (l1_ms * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(f"config{args.config}_{args.dtype}_{args.precision}_l1")
        except Exception:
            traffic = None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        from oracle import oracle as O

        thr = O.max_threads()
        fc, lc, cc, ec, mc = cpu_workload(args.config, args.dtype == "float32")
        v, dtc, nsol, itc = cpu_sample(fc, lc, cc, ec, thr, mc)
        cpu = {"value": v, "unit": "Mpixel-sweeps/s", "cores": thr, "kind": "port",
               "sample": f"{nsol} solve(s) of {fc.shape[0]}x{fc.shape[1]} (config {args.config}, {itc} cycles, "
                         f"{dtc:.2f} s each); oracle/cmg_oracle.c (fp64), OpenMP {thr} threads"}
    line = {
        "metric": "Mpixel-sweeps/s",
        "value": value,
        "unit": "Mpixel-sweeps/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": value_ms,
        "higher_is_better": True,
        "scaling": "weak" if args.config != 5 else "strong",
        "vs_baseline": None,
        "dtype": "f64" if args.dtype == "float64" else "f32",
        "data": "synthetic (BASELINE seeded generator, SURVEY 8d)",
        "config": config_dict(args.config, desc, imgs_total, cycles, parallelism),
        "detail": {"time_to_tolerance_ms": value_ms, **extra},
        "e2e": {"value": e2e_value, "unit": "Mpixel-sweeps/s", "h2d_bytes_per_step": int(nbytes_in),
                "d2h_bytes_per_step": int(nbytes_out), "ms_per_step": e2e_ms,
                "path": "cmg_solve (C ABI) with pinned host buffers"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": l1_kernel_name(args.dtype, args.precision, m_loc, n),
                     "algorithmic_bytes_per_launch": int(alg_bytes), "launch_ms": l1_ms, "peak_source": peak_src},
        "clocks": clocks,
    }
    # L2-resident working set (u, f, the rotation buffers of a <= ~32 MB job):
    # the level-1 sweep is measured against the L2 read bandwidth of this GPU,
    # measured live (cmg_l2_read_bandwidth: 32 MiB streamed 50 times)
    if 4 * esz * m_loc * n * (len(idx) if args.config == 4 else 1) <= (64 << 20):
        l2 = N.l2_read_bandwidth(local, 32 << 20, 50)
        line["roofline"].update({"bound": "l2", "peak": l2, "frac": achieved / l2,
                                 "peak_source": "measured live: cmg_l2_read_bandwidth (32 MiB x 50 reads, CUDA "
                                                "events)", "hbm_peak": peak, "hbm_frac": achieved / peak})
        pipes = ROOT / "profiles" / "pipes.json"
        if pipes.exists():
            key = f"config{args.config}_{args.dtype}_{args.precision}_l1"
            pd = json.loads(pipes.read_text()).get(key)
            if pd:
                line["roofline"]["compute"] = pd
        if args.dtype == "float64" and "compute" in line["roofline"]:
            # the compute roof, measured live: sustained DFMA rate and dependent-chain
            # latency of the FP64 pipe (cmg_fp64_probe)
            pr = N.fp64_probe(local)
            cp = line["roofline"]["compute"]
            cp["fp64_probe"] = pr
            if cp.get("fp64_thread_instr_per_launch") and cp.get("ncu_cold_us"):
                import torch

                props = torch.cuda.get_device_properties(local)
                rate = cp["fp64_thread_instr_per_launch"] / (cp["ncu_cold_us"] * 1e-6) / (
                    clocks.get("sm_mhz", 1965.0) * 1e6) / props.multi_processor_count
                cp["fp64_instr_per_clk_per_sm"] = rate  # energy-fused kernel, ncu (cold) duration
                cp["fp64_frac_of_probe"] = rate / pr["dfma_per_clk_per_sm"]
    if args.config == 3 and args.dtype == "float64" and args.precision == "exact":
        line["roofline"]["note"] = ("1024^2 fp64 exact: u and f (16 MiB) stay in the 126 MB L2; the level-1 "
                                    "kernel is FP64-pipe / latency bound (8 correctly rounded sqrt + 10 div per "
                                    "pixel: roofline.compute from ncu), far below the L2 bandwidth; the HBM "
                                    "roofline binds at 16384^2: roofline_fine_level")
    if rank == 0 and ws == 1 and not args.no_fine and args.config != 5:
        line["roofline_fine_level"] = fine_level_roofline(local, peak)
    if rank == 0 and ws == 1 and args.config == 3 and not args.no_fine:
        line["detail"]["other_precisions"] = other_precisions(local, args.steps)
    if rank == 0 and ws == 1 and args.config in (1, 2, 3):
        line["e2e_dropin"] = dropin_e2e(args, c, eps, max_outer, px_sweeps)
    if rank == 0 and ws == 1 and args.config == 3 and not args.no_cpu:
        nb = numpy_reference_leg()
        if nb:
            line["cpu_baseline_numpy"] = nb
    if cpu:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if plan is not None:
        plan.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def dropin_e2e(args, c, eps, max_outer, px_sweeps) -> dict:
    """The drop-in call itself, end to end: paper_2204_07921_b200.denoise(Image,
    SolverConfig) on a pageable numpy image (validation, H2D, solve, D2H,
    trace objects), as a reference user calls curvemg.denoise."""
    import paper_2204_07921_b200 as cmg
    from paper_2204_07921_b200 import synth

    f, _ = synth.config_input(args.config, 0, fp32=(args.dtype == "float32"))
    cfg = cmg.SolverConfig(alpha=0.06, mode=c["mode"], layers=c["layers"], epsilon=eps, max_outer=max_outer,
                           dtype=args.dtype, precision=args.precision)
    img = cmg.Image(f, 1.0)
    for _ in range(2):
        cmg.denoise(img, cfg)
    ts = []
    for _ in range(max(args.steps, 3)):
        t0 = time.perf_counter()
        cmg.denoise(img, cfg)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(ts))
    return {"value": px_sweeps / (ms * 1e-3) / 1e6, "unit": "Mpixel-sweeps/s", "ms_per_step": ms,
            "path": "paper_2204_07921_b200.denoise(Image, SolverConfig), pageable numpy in/out"}


def numpy_reference_leg() -> dict | None:
    """The reference's own NumPy solver (curvemg.denoise, installed offline into
    the git-ignored baseline/_ref) on config 3, threads=1 and threads=None, on
    this host: BASELINE.md section 3's CPU reference numbers, recorded beside the
    oracle-port baseline.  None when baseline/_ref is absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "curvemg").exists():
        return None
    sys.path.insert(0, str(ref))
    try:
        import curvemg
    except Exception:
        return None
    finally:
        sys.path.pop(0)
    from paper_2204_07921_b200 import synth

    f, cl = synth.config_input(3, 0)
    out = {"unit": "Mpixel-sweeps/s", "workload": "config 3 (1024^2 MC, eps 1e-6, J=3), one solve per leg",
           "numpy": np.__version__, "cpu_model": _cpu_model(), "host_cores": os.cpu_count()}
    for thr in (1, None):
        cfg = curvemg.SolverConfig(alpha=0.06, mode="mean", layers=3, epsilon=1e-6, threads=thr)
        t0 = time.perf_counter()
        _, tr = curvemg.denoise(curvemg.Image(f, 1.0), cfg)
        dt = time.perf_counter() - t0
        key = "threads_1" if thr == 1 else "threads_none"
        out[key] = {"seconds_per_solve": dt, "cycles": tr.iterations,
                    "value": tr.iterations * 3 * f.size / dt / 1e6,
                    "threads": cfg.resolved_threads()}
    return out


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def l1_kernel_name(dtype: str, prec: str, m: int, n: int) -> str:
    """The level-1 kernel the plan dispatches (cmg.cu plan heuristics)."""
    if dtype == "float32" and prec == "fast":
        tile = "56, 120" if m * n >= (4 << 20) and n >= 240 else "56, 56"
        fsrc = ", f from L2" if tile == "56, 120" else ""
        return f"k_l1_x2<{tile}{fsrc}> (level-1 sweep, four colours in one launch, packed f32x2)"
    t = "double" if dtype == "float64" else "float"
    return f"k_l1_tile<{t}, {prec}> (level-1 sweep, four colours in one launch)"


def other_precisions(local: int, steps: int) -> dict:
    """Config 3 in the other modes, device-timed like the headline: fp64 with the
    closed-form curvature (north_star fp64 bar: energy 1e-9 rel, image 1e-8
    max-abs; tests/test_gpu_parity.py) and fp32 (energy 1e-4 rel, PSNR 0.05 dB)."""
    from paper_2204_07921_b200 import _native as N
    from paper_2204_07921_b200 import synth

    out = {}
    for dt, prec in (("float64", "fast"), ("float32", "fast")):
        f, _ = synth.config_input(3, 0, fp32=(dt == "float32"))
        p = N.Plan(1024, 1024, 1, 3, "mean", dt, prec, device=local)
        fh = np.ascontiguousarray(f[None].astype(dt))
        assert N.lib().cmg_buffer_upload(p.handle, 3, N.ptr(fh)) == 0
        en = np.zeros(64)
        its = np.zeros(1, dtype=np.int32)
        sts = np.zeros(1, dtype=np.int32)

        def solve():
            rc = N.lib().cmg_solve_device(p.handle, None, None, None, 0.06, 1e-6, 60, 1, 0, 0, 1.0, N.dptr(en),
                                          None, None, None, None, N.iptr(its), N.iptr(sts))
            assert rc in (0, 2), N.last_error()
            return p.stats()["device_ms"]

        for _ in range(3):
            solve()
        ms = float(np.mean([solve() for _ in range(max(steps, 3))]))
        out[f"{dt}_{prec}"] = {"time_to_tolerance_ms": ms, "cycles": int(its[0]),
                               "Mpixel_sweeps_per_s": int(its[0]) * 3 * 1024 * 1024 / (ms * 1e-3) / 1e6}
        p.close()
    return out


def fine_level_roofline(local: int, peak: float) -> dict:
    """Level-1 sweep (the fine-level relaxation: all four colours, one launch)
    at config 5's size, 16384^2 fp32 fast: 3 GiB of u/f, far beyond L2, so the
    sweep streams HBM.  Algorithmic bytes = 12 per pixel (read u, read f,
    write u).  Timed with CUDA events on the plan's stream (cmg_time_sweep)."""
    import torch
    from paper_2204_07921_b200 import _native as N
    from paper_2204_07921_b200.strips import _DevView

    size = 16384
    p = N.Plan(size, size, 1, 3, "mean", "float32", "fast", device=local)
    g = torch.Generator(device="cuda").manual_seed(5)
    src = torch.rand((size, size), device="cuda", dtype=torch.float32, generator=g)
    for i in range(4):
        ptr = ctypes.c_void_p()
        assert N.lib().cmg_plan_buffer(p.handle, i, ctypes.byref(ptr)) == 0
        torch.as_tensor(_DevView(ptr.value, (size, size), "<f4"), device="cuda").copy_(src)
    del src
    torch.cuda.synchronize()
    en = np.zeros(2)
    its = np.zeros(1, dtype=np.int32)
    sts = np.zeros(1, dtype=np.int32)
    rc = N.lib().cmg_solve_device(p.handle, None, None, None, 0.06, 1e-300, 1, 1, 0, 0, 1.0, N.dptr(en), None, None,
                                  None, None, N.iptr(its), N.iptr(sts))
    assert rc in (0, 2), N.last_error()
    p.time_sweep(1, -1, reps=20)  # warm
    ms = p.time_sweep(1, -1, reps=50)
    p.close()
    alg = 12 * size * size
    ach = alg / (ms * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get("config5_float32_fast_l1")
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
            "kernel": l1_kernel_name("float32", "fast", size, size),
            "workload": "16384^2 fp32 (config 5 size), image far larger than L2",
            "algorithmic_bytes_per_launch": alg, "launch_ms": ms}


def run_strips(args, c, layers, dt, ws, rank, local, l2_flush, barrier, max_over_ranks):
    """config 5: one image, horizontal strips (one per rank)."""
    import torch

    from paper_2204_07921_b200 import strips as S
    from paper_2204_07921_b200 import synth
    from paper_2204_07921_b200.driver import SolverConfig

    f, _ = synth.config_input(5, 0, fp32=True)
    m, n = f.shape
    cfg = SolverConfig(mode="mean", layers=layers, max_outer=c["cycles"], epsilon=1e-300, dtype=args.dtype,
                       precision=args.precision, device=local)
    G = S.ghost_rows(layers)
    geoms = [S.StripGeometry(m, n, g0, g1, G) for g0, g1 in S.partition_rows(m, ws, layers)]
    g = geoms[rank]
    st = S.CudaStrip(g, cfg, local)
    win = np.ascontiguousarray(f[g.w0:g.w1].astype(dt))
    st.upload(3, win)
    if ws > 1:
        ex = S.DistExchange(st, geoms, rank)
    else:
        ex = S.LocalExchange([st])

    def solve():
        st.upload(0, win)
        return S.solve_strips([st], ex, cfg, m * n)

    for _ in range(max(args.warmup, 3)):
        solve()
    sampler = ClockSampler(local)
    sampler.start()
    times = []
    cycles = 0
    for _ in range(args.steps):
        l2_flush()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, tr = solve()
        e1.record()
        barrier()
        times.append(e0.elapsed_time(e1))
        cycles = tr.iterations
    clocks = sampler.stop()
    ms = float(np.mean(times))
    e2e = []
    for _ in range(args.steps):
        barrier()
        t0 = time.perf_counter()
        st.upload(0, win)
        cur, tr = S.solve_strips([st], ex, cfg, m * n)
        own = st.download(cur)[g.local(g.g0):g.local(g.g1)]
        barrier()
        e2e.append(time.perf_counter() - t0)
    e2e_ms = 1e3 * float(np.mean(e2e))
    ms, e2e_ms = max_over_ranks(ms, e2e_ms)
    l1_ms = st.plan.time_sweep(1, -1, reps=5)
    esz = np.dtype(dt).itemsize
    st.close()
    launches = cycles * (layers + 1) + 1
    return (ms, e2e_ms, cycles, launches, clocks, win.nbytes * ws, own.nbytes * ws, l1_ms, g.rows)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--dtype", choices=["float64", "float32"], default=None)
    ap.add_argument("--precision", choices=["exact", "fast"], default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fine", action="store_true", help="skip the 16384^2 fine-level roofline leg")
    args = ap.parse_args()
    if args.dtype is None:
        args.dtype = "float32" if args.config in (4, 5) else "float64"
    if args.precision is None:
        args.precision = "fast" if args.dtype == "float32" else "exact"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
