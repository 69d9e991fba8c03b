"""Per-kernel summary of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launch_summary.py profiles/r02/ncu/launches_c3.csv.gz > profiles/r02/ncu/launches_c3_summary.md
"""
import collections
import csv
import gzip
import io
import sys

txt = gzip.open(sys.argv[1], "rt").read()
start = txt.index('"ID"')
rows = list(csv.DictReader(io.StringIO(txt[start:])))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    v = v / 1000.0 if r["Metric Unit"] in ("ns", "nsecond") else v
    name = r["Kernel Name"].split("(")[0]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print("# Launch list, bench.py config 3 (CMG_NO_GRAPH=1, --steps 2 --warmup 3 --no-cpu --no-fine), "
      "ncu gpu__time_duration.sum --clock-control none\n")
print("Cold-cache, serialised per-launch times of every launch of the run (warm-up, timed, e2e, drop-in and "
      "time_sweep legs). `k_l1_tile<..., true>` is the energy-fused level-1 kernel with the branch-free pixel code "
      "(it also sums and finalizes the energy of its input; the bench's `level_sweep_ms` times the plain level-1 "
      "sweep); the torch kernel is bench.py's L2 flush.\n")
print("| kernel | launches | total_us | mean_us | share |\n|---|---|---|---|---|")
for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name[:90]}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
print(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | | |")
