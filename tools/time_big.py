"""Per-level sweep times (cmg_time_sweep, all colours) and the energy pass on
a large image, for several kernel-selection environments (one subprocess each).
usage: time_big.py SIZE DTYPE PREC [BATCH]"""
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
from paper_2204_07921_b200 import synth
size, dt, prec, B = %(size)d, %(dt)r, %(prec)r, %(B)d
f3, _ = synth.config_input(3, 0, fp32=(dt == "float32"))
rep = max(1, size // 1024)
img = np.tile(f3, (rep, rep))[:size, :size].astype(dt)
u = np.ascontiguousarray(np.broadcast_to(img, (B, size, size)))
p = N.Plan(size, size, B, 3, "mean", dt, prec)
for i in range(4):
    assert N.lib().cmg_buffer_upload(p.handle, i, N.ptr(u)) == 0
prime(p, B)
import time
t0 = time.time()
while time.time() - t0 < 1.0:  # clocks up before timing
    p.time_sweep(1, -1, reps=5)
r = {l: round(p.time_sweep(l, -1, reps=10) * 1e3, 1) for l in (1, 2, 3, 0)}
print(r)
"""
size, dt, prec = int(sys.argv[1]), sys.argv[2], sys.argv[3]
B = int(sys.argv[4]) if len(sys.argv) > 4 else 1
envs = json.loads(sys.argv[5]) if len(sys.argv) > 5 else [{}]
for e in envs:
    env = dict(os.environ, CMG_VERBOSE="1", **e)
    r = subprocess.run([sys.executable, "-c", CODE % dict(root=str(ROOT), size=size, dt=dt, prec=prec, B=B)], env=env,
                       capture_output=True, text=True)
    info = [l for l in r.stderr.splitlines() if "cmg plan" in l]
    print(f"{size}x{B} {dt} {prec} {json.dumps(e):40s} us {r.stdout.strip()}  {info[-1][-40:] if info else r.stderr[-400:]}")
