"""One level-step of each level on a large synthetic image (for ncu)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200.driver import get_plan
size = int(sys.argv[1]); dtype = sys.argv[2]; prec = sys.argv[3]
rng = np.random.default_rng(0)
x = np.linspace(0, 1, size)
f = (0.5 + 0.3 * np.sin(6 * x)[:, None] * np.cos(5 * x)[None, :]) + rng.standard_normal((size, size)) * 0.08
cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=1, epsilon=1e-300, dtype=dtype, precision=prec)
img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
print("ok", tr.energies())
