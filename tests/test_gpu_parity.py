"""GPU parity: libcmg.so (through its C ABI) against the reference's golden
fixtures and the pinned CPU oracle.

Bars (BASELINE north_star):
  * exact fp64 path: bit-identical u to the reference (both modes), energies
    within 1e-12 relative (the device energy uses the closed-form level-1
    curvature and a tree sum; NumPy uses a pairwise sum);
  * fast fp64 MC: per-cycle energy 1e-9 relative, final image 1e-8 max-abs;
  * fp32 MC: final energy 1e-4 relative and |dPSNR| <= 0.05 dB vs fp64 reference.
"""

import hashlib
import json

import numpy as np
import pytest

import paper_2204_07921_b200 as cmg
from paper_2204_07921_b200 import _native as N
from paper_2204_07921_b200 import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ENERGY_RTOL_EXACT = 1e-12
ENERGY_RTOL_FP64 = 1e-9
U_ATOL_FP64 = 1e-8
ENERGY_RTOL_FP32 = 1e-4
PSNR_ATOL_FP32 = 0.05


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if N.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu tests must run on a B200")


@pytest.fixture(scope="module")
def sweeps(golden_dir):
    return json.loads((golden_dir / "sweeps.json").read_text()), np.load(golden_dir / "sweeps.npz")


def _plan(m, n, mode, layers=6, dtype="float64", precision="exact", batch=1):
    return N.Plan(m, n, batch, layers, mode, dtype, precision)


def test_sweep_layer_bitexact_vs_reference(sweeps):
    meta, arr = sweeps
    plans = {}
    bad = []
    for c in meta["sweeps"]:
        k = c["key"]
        key = (c["m"], c["n"], c["mode"])
        if key not in plans:
            plans[key] = _plan(c["m"], c["n"], c["mode"])
        u = np.ascontiguousarray(arr[f"{k}_u"]).copy()
        f = np.ascontiguousarray(arr[f"{k}_f"])
        rc = N.lib().cmg_sweep_layer(plans[key].handle, N.ptr(u), N.ptr(f), c["layer"], c["alpha"],
                                     c["inner_iters"])
        assert rc == 0, N.last_error()
        if not np.array_equal(u, arr[f"{k}_out"]):
            bad.append((c, float(np.abs(u - arr[f"{k}_out"]).max())))
    assert not bad, bad[:5]


def test_energy_vs_reference(sweeps):
    meta, arr = sweeps
    for c in meta["energies"]:
        k = c["key"]
        u, f = np.ascontiguousarray(arr[f"{k}_u"]), np.ascontiguousarray(arr[f"{k}_f"])
        p = _plan(u.shape[0], u.shape[1], c["mode"], layers=1)
        out = np.zeros(1)
        rc = N.lib().cmg_energy(p.handle, N.ptr(u), N.ptr(f), 0.06, N.dptr(out))
        assert rc == 0, N.last_error()
        assert abs(out[0] - c["energy"]) <= ENERGY_RTOL_EXACT * abs(c["energy"]), (c, out[0])


def test_denoise_small_bitexact_vs_reference(golden_dir):
    meta = json.loads((golden_dir / "denoise_small.json").read_text())
    arr = np.load(golden_dir / "denoise_small.npz")
    for c in meta:
        k = c["key"]
        cfg = cmg.SolverConfig(alpha=0.06, mode=c["mode"], layers=c["layers"], epsilon=c["epsilon_used"],
                               max_outer=c["max_outer"], inner_iters=c["inner_iters"], stop_rule=c["stop_rule"],
                               full_vcycle=c["full_vcycle"])
        img, tr = cmg.denoise(cmg.Image(arr[f"{k}_f"], 1.0), cfg, cmg.Image(arr[f"{k}_clean"], 1.0))
        assert tr.iterations == c["iterations"], k
        assert tr.converged == c["converged"], k
        assert np.array_equal(img.data, arr[f"{k}_u"]), (k, float(np.abs(img.data - arr[f"{k}_u"]).max()))
        e = tr.energies()
        ref = np.array(c["energies"])
        assert np.all(np.abs(e - ref) <= ENERGY_RTOL_EXACT * np.abs(ref)), k
        ps = np.array([r.psnr for r in tr.records])
        assert np.allclose(ps, np.array(c["psnr"]), rtol=1e-12, atol=1e-12), k


@pytest.mark.parametrize("name", ["c1_J6", "c1_J3", "c2_J3", "c2_J6", "c3_f64", "c4_img0"])
def test_baseline_configs_exact_fp64(golden_dir, name):
    g = json.loads((golden_dir / "configs.json").read_text())[name]
    f, cl = synth.config_input(g["config"], 0, fp32=g["fp32_input"])
    cfg = cmg.SolverConfig(alpha=0.06, mode=g["mode"], layers=g["layers"], epsilon=g["epsilon"],
                           max_outer=g["max_outer"])
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg, cmg.Image(cl, 1.0))
    assert tr.iterations == g["iterations"]
    ref = np.array(g["energies"])
    assert np.all(np.abs(tr.energies() - ref) <= ENERGY_RTOL_EXACT * np.abs(ref))
    # the trajectory is bit-identical to the reference (GC is ulp-chaotic: SURVEY 0.2)
    assert _sha(img.data) == g["u_sha256"]


def test_config3_fast_fp64_within_tolerance(golden_dir):
    g = json.loads((golden_dir / "configs.json").read_text())["c3_f64"]
    f, cl = synth.config_input(3)
    cfg = cmg.SolverConfig(mode="mean", layers=3, epsilon=1e-6, precision="fast")
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg, cmg.Image(cl, 1.0))
    ref = np.array(g["energies"])
    assert tr.iterations == g["iterations"]
    assert np.all(np.abs(tr.energies() - ref) <= ENERGY_RTOL_FP64 * np.abs(ref))
    r = O.denoise(f, layers=3, epsilon=1e-6, threads=O.max_threads())
    assert np.abs(img.data - r["u"]).max() <= U_ATOL_FP64


@pytest.mark.parametrize("name", ["c3_f32in", "c4_img0"])
def test_fp32_mode_within_tolerance(golden_dir, name):
    g = json.loads((golden_dir / "configs.json").read_text())[name]
    f, cl = synth.config_input(g["config"], 0, fp32=True)
    cfg = cmg.SolverConfig(mode="mean", layers=3, epsilon=g["epsilon"], max_outer=g["max_outer"], dtype="float32",
                           precision="fast")
    img, tr = cmg.denoise(cmg.Image(f, 1.0), cfg, cmg.Image(cl, 1.0))
    e_ref = g["energies"][-1]
    assert abs(tr.final_energy - e_ref) <= ENERGY_RTOL_FP32 * abs(e_ref)
    assert abs(tr.records[-1].psnr - g["psnr"][-1]) <= PSNR_ATOL_FP32


def test_batch_equals_single_images():
    imgs = [synth.config_input(4, i)[0][:200, :180] for i in range(3)]
    cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=6, epsilon=1e-300)
    out = cmg.denoise_batch([cmg.Image(x, 1.0) for x in imgs], cfg)
    for x, (u, tr) in zip(imgs, out):
        u1, tr1 = cmg.denoise(cmg.Image(x, 1.0), cfg)
        assert np.array_equal(u.data, u1.data)
        assert np.allclose(tr.energies(), tr1.energies(), rtol=1e-13, atol=0)


def test_batch_per_image_stopping():
    a = synth.config_input(4, 0)[0][:64, :64]
    b = np.full((64, 64), 0.5)  # constant image: fixed point, converges at cycle 1
    cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=30, epsilon=1e-6)
    out = cmg.denoise_batch([cmg.Image(a, 1.0), cmg.Image(b, 1.0)], cfg)
    (ua, ta), (ub, tb) = out
    r = O.denoise(a, layers=3, max_outer=30, epsilon=1e-6)
    assert ta.iterations == r["iterations"]
    assert np.array_equal(ua.data, r["u"])
    assert tb.iterations == 1 and tb.converged and np.array_equal(ub.data, b)


def test_nonfinite_corrections_raise_valueerror():
    rng = np.random.default_rng(0)
    f = rng.random((16, 16)) * 1e308
    with pytest.raises(ValueError):
        cmg.denoise(cmg.Image(f, 1.0), cmg.SolverConfig(max_outer=2))
    r = O.denoise(f, max_outer=2)
    assert r["status"] == 1


def test_gaussian_fp32_runs_and_decreases_energy():
    f, cl = synth.config_input(2)
    cfg = cmg.SolverConfig(mode="gaussian", layers=3, max_outer=10, epsilon=1e-300, dtype="float32")
    img, tr = cmg.denoise(cmg.Image(f[:256, :256], 1.0), cfg)
    assert tr.energies()[5] < tr.energies()[0]


def test_launch_stats_reported():
    f, _ = synth.config_input(1)
    cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=4, epsilon=1e-300)
    cmg.denoise(cmg.Image(f, 1.0), cfg)
    from paper_2204_07921_b200.driver import get_plan
    st = get_plan(256, 256, 1, cfg).stats()
    # fused levels: >= J fused launches + energy + finalize per cycle (or 1 persistent launch)
    assert st["cycles_run"] == 4 and st["kernel_launches"] >= 1


@pytest.mark.parametrize("parts,mode,dtype", [(2, "mean", "float64"), (3, "gaussian", "float64"),
                                              (4, "mean", "float32")])
def test_virtual_strips_equal_single_gpu_solve(parts, mode, dtype):
    """Strip decomposition on one GPU (virtual strips, D2D ghost exchange) ==
    the single-plan solve, bit for bit."""
    from paper_2204_07921_b200.strips import denoise_strips

    f, cl = synth.config_input(1)
    f = f[:, :200]
    cl = cl[:, :200]
    cfg = cmg.SolverConfig(mode=mode, layers=3, max_outer=6, epsilon=1e-300, dtype=dtype,
                           precision="fast" if dtype == "float32" else "exact")
    u1, t1 = cmg.denoise(cmg.Image(f, 1.0), cfg, cmg.Image(cl, 1.0))
    u2, t2 = denoise_strips(cmg.Image(f, 1.0), cfg, parts=parts, reference=cmg.Image(cl, 1.0))
    assert np.array_equal(u1.data, u2.data)
    assert t1.iterations == t2.iterations
    rtol = 1e-12 if dtype == "float64" else 1e-9
    assert np.allclose(t1.energies(), t2.energies(), rtol=rtol, atol=0)


def test_nonfinite_energy_raises_solver_divergence():
    """f ~ U[0,1) * 1e306: the level-1 curvature sum overflows, the
    corrections stay finite (their plane normals overflow to inf, so the
    distances are 0), and the energy after cycle 1 is inf -> the reference
    raises SolverDivergence("objective became non-finite at outer iteration 1")
    (driver.py:300-303; checked against curvemg in the build container)."""
    rng = np.random.default_rng(0)
    f = rng.random((32, 32)) * 1e306
    r = O.denoise(f, max_outer=3)
    assert r["status"] == 3 and r["iterations"] == 1
    with pytest.raises(cmg.SolverDivergence, match="outer iteration 1"):
        cmg.denoise(cmg.Image(f, 1.0), cmg.SolverConfig(max_outer=3))
    out = None
    with pytest.raises(cmg.SolverDivergence):
        out = cmg.denoise_batch([cmg.Image(f, 1.0), cmg.Image(np.full((32, 32), 0.5), 1.0)],
                                cmg.SolverConfig(max_outer=3))
    assert out is None


def test_batch_sharded_over_devices_equals_one_plan():
    """denoise_batch(devices=[...]) (cmg_mplan: contiguous image slices, one
    host thread per shard) == one plan, bit for bit.  One GPU here: the same
    device id twice gives two independent plans/streams on it."""
    imgs = [synth.config_input(4, i)[0][:160, :144] for i in range(5)]
    cfg = cmg.SolverConfig(mode="mean", layers=3, max_outer=8, epsilon=1e-5)
    one = cmg.denoise_batch([cmg.Image(x, 1.0) for x in imgs], cfg)
    two = cmg.denoise_batch([cmg.Image(x, 1.0) for x in imgs], cfg, devices=[0, 0])
    three = cmg.denoise_batch([cmg.Image(x, 1.0) for x in imgs], cfg, devices=[0, 0, 0])
    for (u1, t1), (u2, t2), (u3, t3) in zip(one, two, three):
        assert np.array_equal(u1.data, u2.data) and np.array_equal(u1.data, u3.data)
        assert t1.iterations == t2.iterations == t3.iterations
        assert np.array_equal(t1.energies(), t2.energies()) and np.array_equal(t1.energies(), t3.energies())
