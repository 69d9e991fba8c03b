"""Large-job dispatch on narrow, ragged images (batches of fp32 images whose
rows are far shorter than the bulk row-parity window): the one-tile-per-row
level-2 kernel and the vectorised per-patch f sums against the oracle, and
against the same solve with the narrow-image tile switched off."""

import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2204_07921_b200 as cmg
from oracle import oracle as O
rng = np.random.default_rng(7)
out = {}
for (m, n, B) in ((300, 404, 36), (257, 512, 34), (190, 96, 240)):
    yy, xx = np.mgrid[0:m, 0:n]
    base = 0.5 + 0.3 * np.sin(yy / 9.0) * np.cos(xx / 6.0)
    fs = [(base + 0.06 * rng.standard_normal((m, n))).astype(np.float32).astype(np.float64) for _ in range(B)]
    cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=3, epsilon=1e-300, dtype="float32", precision="fast")
    res = cmg.denoise_batch([cmg.Image(f, 1.0) for f in fs], cfg)
    for b in (0, B // 2, B - 1):
        ref = O.denoise(fs[b], mode="mean", layers=3, max_outer=3, epsilon=1e-300)
        e, er = res[b][1].energies(), ref["energies"]
        assert np.all(np.abs(e - er) <= 1e-4 * np.abs(er)), (m, n, b, e, er)
        assert np.max(np.abs(res[b][0].data - ref["u"])) < 1e-3, (m, n, b)
    out[f"{m}x{n}"] = np.stack([r[0].data for r in res])
np.savez(%(out)r, **out)
"""


def _run(env_extra, path):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": str(ROOT), "out": str(path)}], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(path)


def test_narrow_image_batches(tmp_path):
    a = _run({}, tmp_path / "default.npz")
    b = _run({"CMG_RP_NT2": "0"}, tmp_path / "three_tiles.npz")
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k  # the tile width does not change any value
