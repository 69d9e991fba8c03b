"""Run a few solves of a BASELINE config (for ncu launch lists / captures)."""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg  # noqa: E402
from paper_2204_07921_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--precision", default="exact")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--cycles", type=int, default=0)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
f, cl = synth.config_input(a.config, 0, fp32=(a.dtype == "float32"))
cfg = cmg.SolverConfig(mode=c["mode"], layers=c["layers"], epsilon=c.get("eps", 1e-300),
                       max_outer=a.cycles or c["cycles"], dtype=a.dtype, precision=a.precision)
for _ in range(a.reps):
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
print("iterations", tr.iterations, "energy", tr.final_energy)
