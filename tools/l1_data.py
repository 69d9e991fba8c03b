"""Is the level-1 sweep time data dependent?  config-5 input vs tiled config-3."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_07921_b200 import _native as N
def prime(p, B):
    # one solve cycle on the resident f: sets the plan's solve parameters (alpha, backward constants)
    en = np.zeros(2 * B); its = np.zeros(B, dtype=np.int32); sts = np.zeros(B, dtype=np.int32)
    rc = N.lib().cmg_solve_device(p.handle, None, None, None, 0.06, 1e-300, 1, 1, 0, 0, 1.0, N.dptr(en), None, None,
                                  None, None, N.iptr(its), N.iptr(sts))
    assert rc in (0, 2), N.last_error()
from paper_2204_07921_b200 import synth

size = 16384
p = N.Plan(size, size, 1, 3, "mean", "float32", "fast")
f5, _ = synth.config_input(5, 0, fp32=True)
f3, _ = synth.config_input(3, 0, fp32=True)
tiled = np.ascontiguousarray(np.tile(f3, (16, 16)))
rnd = np.random.default_rng(0).random((size, size), dtype=np.float32)
for name, img in (("config5", f5), ("tiled3", tiled), ("uniform", rnd), ("config5", f5)):
    img = np.ascontiguousarray(img, dtype=np.float32)  # keep alive across the calls
    for i in range(4):
        assert N.lib().cmg_buffer_upload(p.handle, i, N.ptr(img)) == 0
    prime(p, 1)
    t0 = time.time()
    while time.time() - t0 < 0.5:
        p.time_sweep(1, -1, reps=5)
    print(name, {l: round(p.time_sweep(l, -1, reps=10) * 1e3, 1) for l in (1, 2, 3, 0)}, flush=True)
