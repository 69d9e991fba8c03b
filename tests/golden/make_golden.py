"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where the read-only reference is mounted):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --configs  # BASELINE config trajectories (~2 min)

It imports ``curvemg`` from /root/reference/pkg/src (pure Python + NumPy) and
records its outputs; the reference itself never travels to the GPU box, only
these fixtures do.  Every fixture is produced with ``threads=1``.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

import curvemg  # noqa: E402
from curvemg import driver, hierarchy, tangent  # noqa: E402

from paper_2204_07921_b200 import synth  # noqa: E402


def planes_fixture():
    out = {}
    for j in range(1, 7):
        out[str(j)] = [[*p.x, *p.y, *p.z, p.ds2] for p in tangent.plane_set(j).planes]
    (HERE / "planes.json").write_text(json.dumps(out))


PAD_CASES = [((1, 1), ((1, 1), (1, 1))), ((1, 7), ((1, 6), (1, 3))), ((2, 3), ((1, 20), (1, 33))),
             ((3, 2), ((1, 5), (1, 6))), ((5, 7), ((1, 62), (1, 1))), ((4, 4), ((1, 4), (1, 4))),
             ((37, 53), ((1, 6), (1, 4))), ((9, 2), ((1, 30), (1, 30)))]

SWEEP_SIZES = [(37, 53), (20, 9), (64, 48), (5, 7), (3, 3), (1, 9), (9, 1), (70, 130), (31, 31), (2, 2)]


def sweeps_fixture():
    rng = np.random.default_rng(20260101)
    arrays = {}
    meta = []
    for ci, (shape, widths) in enumerate(PAD_CASES):
        a = rng.standard_normal(shape)
        arrays[f"pad{ci}_in"] = a
        arrays[f"pad{ci}_out"] = np.pad(a, widths, mode="reflect", reflect_type="odd")
    k = 0
    for (m, n) in SWEEP_SIZES:
        for mode in ("mean", "gaussian"):
            for layer in range(1, 7):
                if m * n > 1000 and layer in (2, 4, 5):
                    continue
                if m * n > 3000 and layer == 6:
                    continue
                for it in ((1, 3) if (layer <= 2 and m * n <= 3000) else (1,)):
                    u = rng.random((m, n))
                    f = np.clip(u + 0.1 * rng.standard_normal((m, n)), -0.5, 1.5)
                    cfg = curvemg.SolverConfig(mode=mode, layers=6, inner_iters=it, threads=1, alpha=0.06)
                    part = hierarchy.Partition(layer, (m, n))
                    mp, npd = part.padded_shape
                    fpad = tangent.solver_pad(f, ((1, 1 + mp - m), (1, 1 + npd - n)))
                    uo = u.copy()
                    driver.sweep_layer(uo, fpad, part, cfg, None)
                    arrays[f"s{k}_u"] = u
                    arrays[f"s{k}_f"] = f
                    arrays[f"s{k}_out"] = uo
                    meta.append(dict(key=f"s{k}", m=m, n=n, mode=mode, layer=layer, inner_iters=it, alpha=0.06))
                    k += 1
    # energies of random fields
    emeta = []
    for e, (m, n) in enumerate([(37, 53), (1, 1), (2, 5), (64, 64), (1, 17)]):
        for mode in ("mean", "gaussian"):
            u = rng.random((m, n))
            f = u + 0.1 * rng.standard_normal((m, n))
            arrays[f"e{e}{mode[0]}_u"] = u
            arrays[f"e{e}{mode[0]}_f"] = f
            emeta.append(dict(key=f"e{e}{mode[0]}", mode=mode, energy=tangent.energy(u, f, 0.06, mode),
                              curv=tangent.curvature_field(u, mode).tolist() if m * n < 20 else None))
    np.savez_compressed(HERE / "sweeps.npz", **arrays)
    (HERE / "sweeps.json").write_text(json.dumps(dict(pads=[[list(s), [list(w) for w in ws]]
                                                            for s, ws in PAD_CASES],
                                                      sweeps=meta, energies=emeta), indent=0))


DENOISE_CASES = [
    dict(m=37, n=53, layers=3, mode="mean", inner_iters=1, full_vcycle=False, stop_rule="rel_energy", max_outer=8),
    dict(m=64, n=48, layers=6, mode="gaussian", inner_iters=1, full_vcycle=False, stop_rule="rel_energy",
         max_outer=6),
    dict(m=30, n=31, layers=4, mode="gaussian", inner_iters=3, full_vcycle=True, stop_rule="rel_u", max_outer=4),
    dict(m=5, n=7, layers=3, mode="mean", inner_iters=1, full_vcycle=False, stop_rule="rel_energy", max_outer=3),
    dict(m=96, n=96, layers=3, mode="gaussian", inner_iters=1, full_vcycle=False, stop_rule="rel_energy",
         max_outer=20),
    dict(m=80, n=72, layers=2, mode="mean", inner_iters=2, full_vcycle=True, stop_rule="rel_energy",
         max_outer=200, epsilon=1e-5),
    dict(m=1, n=40, layers=2, mode="mean", inner_iters=1, full_vcycle=False, stop_rule="rel_energy", max_outer=5),
    dict(m=129, n=67, layers=5, mode="mean", inner_iters=1, full_vcycle=False, stop_rule="rel_u", max_outer=6,
         epsilon=1e-3),
]


def denoise_fixture():
    rng = np.random.default_rng(7)
    arrays = {}
    meta = []
    for k, c in enumerate(DENOISE_CASES):
        m, n = c["m"], c["n"]
        clean = np.clip(rng.random() * 0.5 + 0.25 + 0.2 * np.sin(np.arange(m)[:, None] / 5.0)
                        * np.cos(np.arange(n)[None, :] / 7.0), 0, 1)
        f = clean + 0.08 * rng.standard_normal((m, n))
        cfg = curvemg.SolverConfig(alpha=0.06, mode=c["mode"], layers=c["layers"], epsilon=c.get("epsilon", 1e-6),
                                   max_outer=c["max_outer"], inner_iters=c["inner_iters"],
                                   stop_rule=c["stop_rule"], full_vcycle=c["full_vcycle"], threads=1)
        img, tr = curvemg.denoise(curvemg.Image(f, 1.0), cfg, curvemg.Image(clean, 1.0))
        arrays[f"d{k}_f"] = f
        arrays[f"d{k}_clean"] = clean
        arrays[f"d{k}_u"] = img.data
        meta.append(dict(key=f"d{k}", **c, epsilon_used=cfg.epsilon, iterations=tr.iterations,
                         converged=tr.converged, energies=tr.energies().tolist(),
                         rel_energy=[r.rel_energy for r in tr.records], rel_u=[r.rel_u for r in tr.records],
                         psnr=[r.psnr for r in tr.records]))
    np.savez_compressed(HERE / "denoise_small.npz", **arrays)
    (HERE / "denoise_small.json").write_text(json.dumps(meta, indent=0))


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def configs_fixture():
    runs = [
        ("c1_J6", 1, dict(layers=6, max_outer=10, epsilon=1e-300, mode="mean"), False),
        ("c1_J3", 1, dict(layers=3, max_outer=10, epsilon=1e-300, mode="mean"), False),
        ("c2_J3", 2, dict(layers=3, max_outer=50, epsilon=1e-6, mode="gaussian"), False),
        ("c2_J6", 2, dict(layers=6, max_outer=50, epsilon=1e-6, mode="gaussian"), False),
        ("c3_f64", 3, dict(layers=3, max_outer=500, epsilon=1e-6, mode="mean"), False),
        ("c3_f32in", 3, dict(layers=3, max_outer=500, epsilon=1e-6, mode="mean"), True),
        ("c4_img0", 4, dict(layers=3, max_outer=20, epsilon=1e-300, mode="mean"), True),
    ]
    out = {}
    for name, cfgid, kw, fp32 in runs:
        f, cl = synth.config_input(cfgid, 0, fp32=fp32)
        cfg = curvemg.SolverConfig(alpha=0.06, threads=1, **kw)
        t = time.perf_counter()
        img, tr = curvemg.denoise(curvemg.Image(f, 1.0), cfg, curvemg.Image(cl, 1.0))
        dt = time.perf_counter() - t
        out[name] = dict(config=cfgid, fp32_input=fp32, **kw, seconds=dt, iterations=tr.iterations,
                         converged=tr.converged, energies=tr.energies().tolist(),
                         psnr=[r.psnr for r in tr.records], rel_u=[r.rel_u for r in tr.records],
                         f_sha256=_sha(f), u_sha256=_sha(img.data), u_sum=float(img.data.sum()),
                         u_min=float(img.data.min()), u_max=float(img.data.max()))
        print(name, f"{dt:.1f}s", tr.iterations, tr.energies()[-1], flush=True)
    (HERE / "configs.json").write_text(json.dumps(out, indent=1))


def metrics_io_fixture():
    """SSIM / PSNR of seeded image pairs (curvemg.image, image.py:140-192) and the
    reference's own PGM (8/16-bit) and CSV+JSON files of one small image
    (image.py:289-335), read back by the reference."""
    from curvemg import image as I

    rng = np.random.default_rng(77)
    cases, arrays = [], {}
    for k, (m, n, peak, dt) in enumerate([(11, 11, 1.0, "f8"), (11, 40, 1.0, "f8"), (37, 53, 255.0, "f8"),
                                          (128, 128, 1.0, "f8"), (200, 256, 1.0, "f4"), (64, 96, 255.0, "f4")]):
        x = rng.uniform(0, peak, (m, n))
        y = np.clip(x + rng.normal(0, 0.1 * peak, (m, n)), 0, peak)
        x, y = x.astype(dt).astype(np.float64), y.astype(dt).astype(np.float64)
        a, b = I.Image(x, peak), I.Image(y, peak)
        arrays[f"x{k}"], arrays[f"y{k}"] = x, y
        cases.append(dict(shape=[m, n], peak=peak, dtype=dt, ssim=I.ssim(a, b), psnr=I.psnr(a, b),
                          ssim_self=I.ssim(a, a)))
    np.savez_compressed(HERE / "metrics.npz", **arrays)
    (HERE / "metrics.json").write_text(json.dumps(cases, indent=1))
    io_dir = HERE / "io"
    io_dir.mkdir(exist_ok=True)
    img = I.Image(np.clip(rng.normal(120, 60, (17, 23)), -10, 300), 255.0)
    np.save(io_dir / "image.npy", img.data)
    I.write_pgm(img, io_dir / "img8.pgm", bits=8)
    I.write_pgm(img, io_dir / "img16.pgm", bits=16)
    I.write_csv(img, io_dir / "img.csv")
    back = {name: I.read_pgm(io_dir / name) for name in ("img8.pgm", "img16.pgm")}
    np.savez_compressed(io_dir / "read_back.npz", img8=back["img8.pgm"].data, img16=back["img16.pgm"].data,
                        csv=I.read_csv(io_dir / "img.csv").data)
    (io_dir / "read_back.json").write_text(json.dumps({k: v.peak for k, v in back.items()}))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", action="store_true")
    a = ap.parse_args()
    if a.configs:
        configs_fixture()
    else:
        planes_fixture()
        sweeps_fixture()
        denoise_fixture()
        metrics_io_fixture()
