"""Host-side logic: config validation, trace I/O, generator, C-ABI exports.

No compute call reaches the GPU here.
"""

import ctypes
import json
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import _native as N
from paper_2204_07921_b200 import synth
from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]


def test_solver_config_validation_mirrors_reference():
    # driver.py:55-72
    cmg.SolverConfig()
    for kw in (dict(alpha=0), dict(mode="x"), dict(layers=0), dict(layers=7), dict(epsilon=0), dict(max_outer=0),
               dict(inner_iters=0), dict(inner_iters=16), dict(stop_rule="x"), dict(threads=0), dict(dtype="f16"),
               dict(precision="approx")):
        with pytest.raises(ValueError):
            cmg.SolverConfig(**kw)
    c = cmg.SolverConfig()
    assert (c.alpha, c.mode, c.layers, c.epsilon, c.max_outer, c.inner_iters, c.stop_rule, c.full_vcycle) == \
        (0.06, "mean", 3, 1e-6, 500, 1, "rel_energy", False)


def test_config_coercion_from_foreign_object():
    class Ref:  # duck-typed reference SolverConfig
        alpha, mode, layers, epsilon, max_outer, inner_iters = 0.1, "gaussian", 4, 1e-5, 7, 2
        stop_rule, full_vcycle, threads = "rel_u", True, None

    from paper_2204_07921_b200.driver import _coerce_config
    c = _coerce_config(Ref())
    assert c.mode == "gaussian" and c.layers == 4 and c.full_vcycle and c.stop_rule == "rel_u"


def test_rel_err_known_answers():
    # SPEC known answer: rel_err_energy(2.3158, 2.4117) = 0.041411...
    assert abs(cmg.rel_err_energy(2.3158, 2.4117) - 0.0414111754) < 1e-9
    assert cmg.rel_err_energy(0.0, -3.0) == 3.0
    a = np.array([[1.0, 2.0]])
    assert cmg.rel_err_u(a, a) == 0.0
    with pytest.raises(ValueError):
        cmg.rel_err_u(np.zeros((2, 2)), np.ones((2, 2)))


def test_trace_csv_roundtrip(tmp_path):
    tr = cmg.ConvergenceTrace([cmg.TraceRecord(0, 5.0, math.nan, math.nan, 0.0, 20.0),
                               cmg.TraceRecord(1, 4.0, 0.25, 0.1, 0.5, 21.5)], converged=True)
    p = tmp_path / "t.csv"
    tr.to_csv(p)
    assert p.read_text().splitlines()[0] == "# schema=curvemg-trace-1"
    back = cmg.ConvergenceTrace.from_csv(p)
    assert back.iterations == 1 and back.final_energy == 4.0
    assert back.records[1] == tr.records[1]
    assert math.isnan(back.records[0].rel_energy)


def test_image_validation():
    with pytest.raises(ValueError):
        cmg.Image(np.zeros(3))
    with pytest.raises(ValueError):
        cmg.Image(np.array([[np.nan]]))
    im = cmg.Image(np.ones((2, 2)), 1.0)
    assert not im.data.flags.writeable
    # image.py:140-149 known answer: constant diff 5, peak 255 -> 34.1514 dB
    a = cmg.Image(np.full((4, 4), 10.0), 255.0)
    b = cmg.Image(np.full((4, 4), 15.0), 255.0)
    assert abs(cmg.psnr(a, b) - 34.1514) < 1e-4


def test_generator_matches_survey_numbers():
    f, cl = synth.config_input(1)
    assert f.shape == (256, 256) and cl.min() >= 0 and cl.max() <= 1
    # E0 = 3673.5929 for config 1
    assert abs(O.energy(f, f, 0.06, "mean") - 3673.5929) < 1e-3
    f4, _ = synth.config_input(4, 3)
    assert np.array_equal(f4, f4.astype(np.float32).astype(np.float64))


def test_plane_table_generated_header_matches_python():
    txt = (ROOT / "paper_2204_07921_b200" / "csrc" / "planes_table.h").read_text()
    rows = re.findall(r"\{(-?\d+),(-?\d+),(-?\d+),(-?\d+),(-?\d+),(-?\d+)\}", txt)
    assert len(rows) == 256
    ref = [(*p.x, *p.y, *p.z) for p in cmg.plane_table(6)]
    assert [tuple(int(v) for v in r) for r in rows] == ref


def _header_symbols():
    txt = (ROOT / "include" / "cmg.h").read_text()
    return sorted(set(re.findall(r"\b(cmg_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert sorted(N.SYMBOLS) == _header_symbols()


libexists = pytest.mark.skipif(not N.LIB_PATH.exists(), reason="libcmg.so not built (run __graft_entry__.build())")


@libexists
def test_capi_library_exports_every_symbol():
    L = ctypes.CDLL(str(N.LIB_PATH))
    for s in _header_symbols():
        assert hasattr(L, s), s
    assert N.lib().cmg_version() >= 100


@libexists
def test_capi_plane_table_matches_reference(golden_dir):
    g = json.loads((golden_dir / "planes.json").read_text())
    for j in range(1, 7):
        offs = np.zeros(256 * 6, dtype=np.int32)
        ds2 = np.zeros(256)
        k = N.lib().cmg_plane_table(j, N.iptr(offs), N.dptr(ds2))
        ref = np.array(g[str(j)])
        assert k == len(ref)
        assert np.array_equal(offs[: 6 * k].reshape(k, 6), ref[:, :6].astype(np.int32))
        assert np.array_equal(ds2[:k], ref[:, 6])


@libexists
def test_capi_rejects_bad_plans_without_gpu():
    h = ctypes.c_void_p()
    assert N.lib().cmg_plan_create(ctypes.byref(h), 0, 5, 1, 3, 0, 0, 0, 0) == N.CMG_EINVAL
    assert N.lib().cmg_plan_create(ctypes.byref(h), 5, 5, 1, 7, 0, 0, 0, 0) == N.CMG_EINVAL
    assert "layers" in N.last_error()


@libexists
def test_no_cpu_fallback_when_no_device():
    if N.device_count() > 0:
        pytest.skip("a GPU is present")
    f = cmg.Image(np.random.default_rng(0).random((8, 8)), 1.0)
    with pytest.raises(RuntimeError):
        cmg.denoise(f, cmg.SolverConfig(max_outer=1))
