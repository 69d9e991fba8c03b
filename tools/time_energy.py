"""Time the energy + finalize kernel (cmg_time_sweep layer 0) for a few plans
and CTA counts; run in a subprocess per env setting."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r)
from paper_2204_07921_b200 import _native as N
def prime(p, B):
    # one solve cycle on the resident f: sets the plan's solve parameters (alpha, backward constants)
    en = np.zeros(2 * B); its = np.zeros(B, dtype=np.int32); sts = np.zeros(B, dtype=np.int32)
    rc = N.lib().cmg_solve_device(p.handle, None, None, None, 0.06, 1e-300, 1, 1, 0, 0, 1.0, N.dptr(en), None, None,
                                  None, None, N.iptr(its), N.iptr(sts))
    assert rc in (0, 2), N.last_error()
m, n, B, dt = %(m)d, %(n)d, %(B)d, %(dt)r
p = N.Plan(m, n, B, 3, "mean", dt, "fast" if dt == "float32" else "exact")
rng = np.random.default_rng(0)
u = rng.random((B, m, n)).astype(dt)
for i in range(4):
    assert N.lib().cmg_buffer_upload(p.handle, i, N.ptr(u)) == 0
prime(p, B)
print(p.time_sweep(0, -1, reps=20) * 1e3)
"""
cases = [(1024, 1024, 1, "float64"), (1024, 1024, 1, "float32"), (512, 512, 64, "float32"), (16384, 16384, 1, "float32")]
envs = [{"CMG_EBULK": "0"}, {"CMG_EBULK": "1"}, {"CMG_EBULK": "1", "CMG_EBULK_NS": "2"}, {"CMG_EBULK": "1", "CMG_EBULK_NS": "6"},
        {"CMG_ENERGY_CTAS": "1184"}]
for m, n, B, dt in cases:
    for e in envs:
        env = dict(os.environ, CMG_VERBOSE="1", **e)
        r = subprocess.run([sys.executable, "-c", CODE % dict(root=str(ROOT), m=m, n=n, B=B, dt=dt)], env=env,
                           capture_output=True, text=True)
        info = [l for l in r.stderr.splitlines() if "energy CTAs" in l]
        print(f"{m}x{n}x{B} {dt:8s} {json.dumps(e):32s} {r.stdout.strip():>10s} us  {info[-1] if info else r.stderr[-300:]}")
