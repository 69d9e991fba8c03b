"""Run the energy kernel (cmg_time_sweep layer 0) on one plan: m n B dtype reps."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_07921_b200 import _native as N  # noqa: E402

m, n, B, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
p = N.Plan(m, n, B, 3, "mean", dt, "fast" if dt == "float32" else "exact")
u = np.random.default_rng(0).random((B, m, n)).astype(dt)
for i in range(4):
    assert N.lib().cmg_buffer_upload(p.handle, i, N.ptr(u)) == 0
prime(p, B)
print("energy us", p.time_sweep(0, -1, reps=reps) * 1e3)
