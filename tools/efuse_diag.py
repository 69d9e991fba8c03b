"""Compare the energy-fused cycle (default) with CMG_EFUSE=0 on small cases."""
import os, subprocess, sys, json
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
code = r'''
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import synth
out = {}
f1, cl1 = synth.config_input(1)
for name, f, kw, B in [("c1_J3", f1[:96, :80], dict(mode="mean", layers=3, max_outer=5), 1),
                       ("c1_J1", f1[:96, :80], dict(mode="mean", layers=1, max_outer=3), 1),
                       ("c1_J2", f1[:96, :80], dict(mode="mean", layers=2, max_outer=3), 1),
                       ("b2", f1[:64, :64], dict(mode="mean", layers=3, max_outer=4), 2)]:
    cfg = cmg.SolverConfig(epsilon=1e-300, **kw)
    if B == 1:
        img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
        out[name] = dict(e=tr.energies().tolist(), ru=[r.rel_u for r in tr.records], s=float(img.data.sum()))
    else:
        res = cmg.denoise_batch([cmg.Image(f, 1.0), cmg.Image(f[::-1].copy(), 1.0)], cfg)
        out[name] = [dict(e=t.energies().tolist(), s=float(u.data.sum())) for u, t in res]
print(json.dumps(out))
''' % str(ROOT)
res = {}
for tag, env in (("efuse", {}), ("plain", {"CMG_EFUSE": "0"})):
    e = dict(os.environ); e.update(env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
    if r.returncode:
        print(tag, "FAILED", r.stderr[-2000:]); continue
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1])
for k in res.get("plain", {}):
    print(k)
    print("  efuse", res["efuse"][k])
    print("  plain", res["plain"][k])
