"""One level-1 sweep (cmg_sweep_layer, fp32 fast) under several kernel variants; pairwise differences."""
import os, subprocess, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r)
from paper_2204_07921_b200 import _native as N
m, n = %(m)d, %(n)d
rng = np.random.default_rng(1)
u = (0.5 + 0.2 * rng.standard_normal((m, n))).astype(np.float32)
f = (0.5 + 0.2 * rng.standard_normal((m, n))).astype(np.float32)
p = N.Plan(m, n, 1, 3, "mean", "float32", "fast")
assert N.lib().cmg_sweep_layer(p.handle, N.ptr(u), N.ptr(f), 1, 0.06, 1) == 0, N.last_error()
np.save(%(path)r, u)
"""
m, n = int(sys.argv[1]), int(sys.argv[2])
variants = {"fast": {}, "generic": {"CMG_L1X2": "3"}, "newton_diag": {"CMG_L1X2": "2"}, "per_colour": {"CMG_FUSED": "0"}}
res = {}
for tag, env in variants.items():
    path = f"/tmp/l1_{tag}.npy"
    r = subprocess.run([sys.executable, "-c", CODE % dict(root=str(ROOT), m=m, n=n, path=path)],
                       env=dict(os.environ, **env), capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    res[tag] = np.load(path)
tags = list(res)
for i in range(len(tags)):
    for j in range(i + 1, len(tags)):
        a, b = res[tags[i]], res[tags[j]]
        print(f"{tags[i]:12s} vs {tags[j]:12s}: {int((a != b).sum()):7d} differ, max {float(np.abs(a.astype(np.float64) - b).max()):.3g}")
