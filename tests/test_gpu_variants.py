"""Every kernel variant of the solver reproduces the reference bit for bit.

The production path picks kernels by problem size (fused SMEM tiles with TMA
staging for large images, per-colour team kernels for small ones, packed
fp32x2 level 1, ...).  Small golden cases would only ever exercise one of
them, so each variant is forced through its environment switch in a fresh
process and checked against the reference fixtures (fp64, exact arithmetic).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

VARIANTS = {
    "fused_all_tma": {"CMG_FUSE_MASK": "7"},
    "fused_all_no_tma": {"CMG_FUSE_MASK": "7", "CMG_TMA": "0"},
    "per_colour_only": {"CMG_FUSED": "0"},
    "host_chunked_graph": {"CMG_NO_WHILE": "1"},
    "plain_stream_launches": {"CMG_NO_GRAPH": "1"},
    "separate_finalize": {"CMG_FUSED_FINALIZE": "0"},
    "energy_bulk_copies": {"CMG_EBULK": "1"},
    "energy_bulk_copies_2_stages": {"CMG_EBULK": "1", "CMG_EBULK_NS": "2"},
    "team_sizes_8_32": {"CMG_FUSE_MASK": "1", "CMG_TS2": "8", "CMG_TS3": "32"},
    "row_parity_levels_2_3": {"CMG_ROWPAIR": "3"},
    "row_parity_team_sizes_8_8": {"CMG_ROWPAIR": "3", "CMG_RP_TS2": "8", "CMG_TS3": "8"},
    "row_parity_off": {"CMG_ROWPAIR": "0"},
    "row_parity_level2_256_threads": {"CMG_RP_TNT": "256"},
    "row_parity_ldg_staging": {"CMG_ROWPAIR": "3", "CMG_RP_TMA": "0"},
    "row_parity_ldg_staging_8_8": {"CMG_ROWPAIR": "3", "CMG_RP_TMA": "0", "CMG_RP_TS2": "8", "CMG_TS3": "8"},
    "no_programmatic_launch": {"CMG_PDL": "0"},
    "level1_wide_tiles": {"CMG_L1_WIDE": "1"},
    "level1_library_sqrt_div": {"CMG_L1_LOOP": "0"},
    "level1_branch_free_wide_tiles": {"CMG_L1_WIDE": "1", "CMG_L1_TH": "0"},
    "level1_branch_free_28_row_tiles": {"CMG_L1_TH": "28"},
    "level1_library_sqrt_div_28_row_tiles": {"CMG_L1_LOOP": "0", "CMG_L1_TH": "28"},
    "energy_256_threads": {"CMG_ENERGY_NT": "256"},
    "energy_separate_pass": {"CMG_EFUSE": "0"},
    "energy_separate_pass_per_colour": {"CMG_EFUSE": "0", "CMG_ROWPAIR": "0"},
}

SCRIPT = r"""
import json, sys, hashlib
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import _native as N
from paper_2204_07921_b200 import synth
g = %(golden)r
meta = json.load(open(g + "/denoise_small.json"))
arr = np.load(g + "/denoise_small.npz")
bad = []
for c in meta:
    k = c["key"]
    cfg = cmg.SolverConfig(alpha=0.06, mode=c["mode"], layers=c["layers"], epsilon=c["epsilon_used"],
                           max_outer=c["max_outer"], inner_iters=c["inner_iters"], stop_rule=c["stop_rule"],
                           full_vcycle=c["full_vcycle"])
    img, tr = cmg.denoise(cmg.Image(arr[k + "_f"], 1.0), cfg, cmg.Image(arr[k + "_clean"], 1.0))
    if tr.iterations != c["iterations"] or not np.array_equal(img.data, arr[k + "_u"]):
        bad.append(k)
smeta = json.load(open(g + "/sweeps.json"))
sarr = np.load(g + "/sweeps.npz")
plans = {}
for c in smeta["sweeps"]:
    k = c["key"]
    key = (c["m"], c["n"], c["mode"])
    if key not in plans:
        plans[key] = N.Plan(c["m"], c["n"], 1, 6, c["mode"], "float64", "exact")
    u = np.ascontiguousarray(sarr[k + "_u"]).copy()
    f = np.ascontiguousarray(sarr[k + "_f"])  # keep alive across the call
    rc = N.lib().cmg_sweep_layer(plans[key].handle, N.ptr(u), N.ptr(f), c["layer"], c["alpha"], c["inner_iters"])
    if rc != 0 or not np.array_equal(u, sarr[k + "_out"]):
        bad.append(k)
cfgs = json.load(open(g + "/configs.json"))
for name in ("c1_J3", "c2_J3"):
    gc = cfgs[name]
    f, cl = synth.config_input(gc["config"], 0, fp32=gc["fp32_input"])
    cfg = cmg.SolverConfig(alpha=0.06, mode=gc["mode"], layers=gc["layers"], epsilon=gc["epsilon"],
                           max_outer=gc["max_outer"])
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
    sha = hashlib.sha256(np.ascontiguousarray(img.data).tobytes()).hexdigest()
    if sha != gc["u_sha256"] or tr.iterations != gc["iterations"]:
        bad.append(name)
print(json.dumps(bad))
"""


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_bitexact(name):
    env = dict(os.environ)
    env.update(VARIANTS[name])
    code = SCRIPT % {"root": str(ROOT), "golden": str(ROOT / "tests" / "golden")}
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    bad = json.loads(out.stdout.strip().splitlines()[-1])
    assert bad == [], f"{name}: mismatching cases {bad}"


SCRIPT32 = r"""
import sys
import numpy as np
sys.path.insert(0, %(root)r)
import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import synth
f, _ = synth.config_input(1)
f = np.tile(f, (3, 3))[:704, :640]
cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=5, epsilon=1e-300, dtype="float32", precision="fast")
img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg)
np.save(%(out)r, img.data)
"""

# same kernels, different code paths / schedules: bit-identical images
VARIANTS32_EXACT = {
    "l1_generic_loop": {"CMG_L1X2": "3"},
    "l1_tiles_56x120": {"CMG_L1X2": "4"},
    "l1_tiles_120x56": {"CMG_L1X2": "8"},
    "l1_tiles_88x88_192_threads": {"CMG_L1X2": "5"},
    "l1_f_from_global_56x120": {"CMG_L1X2": "11"},
    "l1_f_from_global_56x56": {"CMG_L1X2": "12"},
    "energy_bulk_copies": {"CMG_EBULK": "1"},
    "host_chunked_graph": {"CMG_NO_WHILE": "1"},
}
# other kernel families (fused coarse tiles, per-colour kernels) evaluate the
# fp32 fast closed forms with different reduction orders: equal to fp32 rounding
VARIANTS32_CLOSE = {
    "fused_all": {"CMG_FUSE_MASK": "7"},
    "per_colour_only": {"CMG_FUSED": "0"},
    "per_colour_f_pixels": {"CMG_FUSED": "0", "CMG_FSUM": "0"},
    # the large-job row-parity kernels (one thread per patch) forced on this small image
    "row_parity_bulk_1_stage": {"CMG_ROWPAIR": "3", "CMG_RP1": "3"},
    "row_parity_bulk_2_stages_128": {"CMG_ROWPAIR": "3", "CMG_RP1": "3", "CMG_RP_STAGES": "2", "CMG_RP_NT": "128"},
    "row_parity_bulk_32_threads": {"CMG_ROWPAIR": "3", "CMG_RP1": "3", "CMG_RP_NT": "32"},
    "row_parity_one_thread_ldg": {"CMG_ROWPAIR": "3", "CMG_RP1": "3", "CMG_RP_BULK": "0"},
}


def _run32(env_extra, tmp_path, tag):
    env = dict(os.environ)
    env.update(env_extra)
    out = tmp_path / f"{tag}.npy"
    r = subprocess.run([sys.executable, "-c", SCRIPT32 % {"root": str(ROOT), "out": str(out)}], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.mark.parametrize("name", sorted(VARIANTS32_EXACT))
def test_fp32_variant_same_image(name, tmp_path):
    """fp32 fast: these variants reproduce the default path's image bit for bit."""
    assert np.array_equal(_run32(VARIANTS32_EXACT[name], tmp_path, name), _run32({}, tmp_path, "default"))


@pytest.mark.parametrize("name", sorted(VARIANTS32_CLOSE))
def test_fp32_variant_close_image(name, tmp_path):
    a = _run32(VARIANTS32_CLOSE[name], tmp_path, name)
    b = _run32({}, tmp_path, "default")
    assert np.abs(a.astype(np.float64) - b).max() <= 1e-5

