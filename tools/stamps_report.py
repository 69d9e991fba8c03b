"""Run config-3 solves with CMG_STAMPS=1 and report per-node device time."""
import os, sys, collections
from pathlib import Path
os.environ["CMG_STAMPS"] = "1"
os.environ.setdefault("CMG_STAMPS_FILE", "/tmp/cmg_stamps.txt")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import synth
prec = sys.argv[1] if len(sys.argv) > 1 else "exact"
dtype = sys.argv[2] if len(sys.argv) > 2 else "float64"
f, _ = synth.config_input(3, fp32=(dtype == "float32"))
cfg = cmg.SolverConfig(mode="mean", layers=3, epsilon=1e-6, dtype=dtype, precision=prec)
for _ in range(2):
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
rows = [tuple(map(int, ln.split())) for ln in open(os.environ["CMG_STAMPS_FILE"])]
agg = collections.defaultdict(list)
for (t0, a), (t1, b) in zip(rows, rows[1:]):
    agg[t1].append((b - a) / 1000.0)
tot = (rows[-1][1] - rows[0][1]) / 1000.0
print(f"{prec} {dtype}: cycles {tr.iterations}, stamped span {tot:.1f} us, per cycle {tot / tr.iterations:.1f} us")
names = {90: "energy", 91: "finalize", 99: "cond", 101: "L1 fused", 102: "L2 fused", 103: "L3 fused"}
for tag in sorted(agg):
    v = agg[tag]
    nm = names.get(tag, f"L{tag // 10} colour {tag % 10}")
    print(f"  {nm:14s} n={len(v):4d} mean {sum(v)/len(v):7.2f} us")
