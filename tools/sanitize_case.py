"""Small solves through every production kernel family, for compute-sanitizer
(tools/sanitize.sh): fp64 exact MC/GC (k_l1_tile, k_rowpair, k_sweep_bpp,
k_energy), fp64 fast, and a 2048^2 fp32 fast large job (k_l1_x2,
k_rowpair_bulk, k_energy_bulk, k_patch_fsum, per-colour k_sweep_team)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg  # noqa: E402
from paper_2204_07921_b200 import synth  # noqa: E402

rng = np.random.default_rng(0)
small = np.clip(0.5 + 0.05 * rng.standard_normal((67, 45)), 0, 1)
f1, _ = synth.config_input(1)
f2, _ = synth.config_input(2)
cases = [
    (small, dict(mode="mean", layers=3, max_outer=2)),
    (small, dict(mode="gaussian", layers=6, max_outer=2)),
    (f1, dict(mode="mean", layers=6, max_outer=2)),
    (f1, dict(mode="mean", layers=3, max_outer=2, precision="fast")),
    (f2, dict(mode="gaussian", layers=3, max_outer=1)),
    (np.tile(f1, (8, 8)), dict(mode="mean", layers=3, max_outer=1, dtype="float32", precision="fast")),
]
for f, kw in cases:
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cmg.SolverConfig(epsilon=1e-300, **kw))
    print(f.shape, kw, tr.iterations, tr.final_energy, flush=True)
print("sanitize case ok")
