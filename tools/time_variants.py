"""Compare kernel variants fairly: one plan per env setting in ONE process,
levels timed round-robin (cmg_time_sweep), median over rounds.
usage: time_variants.py SIZE DTYPE PREC BATCH LEVELS '[{env}, ...]'"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2204_07921_b200 import _native as N  # noqa: E402
from paper_2204_07921_b200 import synth  # noqa: E402

size, dt, prec, B = int(sys.argv[1]), sys.argv[2], sys.argv[3], int(sys.argv[4])
levels = [int(x) for x in sys.argv[5].split(",")]
envs = json.loads(sys.argv[6])
f3, _ = synth.config_input(3, 0, fp32=(dt == "float32"))
rep = max(1, size // 1024)
img = np.ascontiguousarray(np.broadcast_to(np.tile(f3, (rep, rep))[:size, :size].astype(dt), (B, size, size)))
plans = []
keys = set(k for e in envs for k in e)
for e in envs:
    for k in keys:
        os.environ.pop(k, None)
    os.environ.update(e)
    p = N.Plan(size, size, B, 3, "mean", dt, prec)
    for i in range(4):
        assert N.lib().cmg_buffer_upload(p.handle, i, N.ptr(img)) == 0
    en = np.zeros(2 * B)
    its = np.zeros(B, dtype=np.int32)
    sts = np.zeros(B, dtype=np.int32)
    rc = N.lib().cmg_solve_device(p.handle, None, None, None, 0.06, 1e-300, 1, 1, 0, 0, 1.0, N.dptr(en), None, None,
                                  None, None, N.iptr(its), N.iptr(sts))
    assert rc in (0, 2), N.last_error()
    plans.append(p)
t0 = time.time()
while time.time() - t0 < 1.0:
    plans[0].time_sweep(levels[0], -1, reps=5)
res = {(i, l): [] for i in range(len(plans)) for l in levels}
for rnd in range(5):
    for i, p in enumerate(plans):
        for l in levels:
            res[(i, l)].append(p.time_sweep(l, -1, reps=10) * 1e3)
for i, e in enumerate(envs):
    print(f"{size}x{B} {dt} {prec} {json.dumps(e):36s}", {l: round(statistics.median(res[(i, l)]), 1) for l in levels})
