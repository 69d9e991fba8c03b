"""Time single sweep kernels (cmg_time_sweep) on config 3 after one solve."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import synth
from paper_2204_07921_b200.driver import get_plan
prec = sys.argv[1] if len(sys.argv) > 1 else "exact"
f, _ = synth.config_input(3)
cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=2, epsilon=1e-300, precision=prec)
cmg.denoise(cmg.Image(f, 1.0), cfg)
p = get_plan(1024, 1024, 1, cfg)
out = {}
for layer in (1, 2, 3):
    out[layer] = [round(p.time_sweep(layer, c, reps=200) * 1000, 2) for c in range(4)]
print(os.environ.get("CMG_DBG", "0"), prec, out)
