"""ncu capture driver: one profiled V-cycle of config 3 (1024^2 fp64 exact) and
one of a config-5-sized image (16384^2 fp32 fast), each after a warm-up solve.
Run under `ncu --profile-from-start off` with CMG_NO_GRAPH=1 (ncu cannot
profile kernel nodes of graphs that hold conditional nodes)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg  # noqa: E402
from paper_2204_07921_b200 import synth  # noqa: E402


def run(f, dtype, prec, layers=3):
    for cycles, prof in ((2, False), (2, True)):
        cfg = cmg.SolverConfig(mode="mean", layers=layers, max_outer=cycles, epsilon=1e-300, dtype=dtype,
                               precision=prec)
        if prof:
            torch.cuda.profiler.start()
        img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
        if prof:
            torch.cuda.profiler.stop()
    print(dtype, prec, f.shape, "energies", tr.energies())


torch.cuda.init()
which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("both", "c3"):
    f3, _ = synth.config_input(3, 0)
    run(f3, "float64", "exact")
if which in ("both", "c5"):
    rng = np.random.default_rng(0)
    f3, _ = synth.config_input(3, 0, fp32=True)
    big = np.tile(f3, (16, 16)).astype(np.float32)  # 16384^2, config-3 texture repeated
    run(big, "float32", "fast")
