"""Per-level sweep timings on a large image (config-5 scale) -> achieved GB/s."""
import sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200.driver import get_plan

size = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
dtype = sys.argv[2] if len(sys.argv) > 2 else "float32"
prec = sys.argv[3] if len(sys.argv) > 3 else "fast"
rng = np.random.default_rng(0)
x = np.linspace(0, 1, size)
f = (0.5 + 0.3 * np.sin(6 * x)[:, None] * np.cos(5 * x)[None, :]).astype(np.float32)
f += (rng.standard_normal((size, size), dtype=np.float32) * np.float32(0.08))
cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=2, epsilon=1e-300, dtype=dtype, precision=prec)
t = time.time()
img, tr = cmg.denoise(cmg.Image(f.astype(np.float64), 1.0), cfg)
p = get_plan(size, size, 1, cfg)
st = p.stats()
esz = 4 if dtype == "float32" else 8
print(f"size {size} {dtype} {prec}: solve 2 cycles device {st['device_ms']:.2f} ms, energies {tr.energies()}")
for layer in (1, 2, 3):
    ms = p.time_sweep(layer, -1, reps=10)
    gbs = 3 * esz * size * size / (ms * 1e-3) / 1e9
    print(f"  level {layer}: {ms:.3f} ms per 4-colour pass -> {gbs:.0f} GB/s algorithmic ({gbs/6488:.2%} of 6488)")
