"""CLI / report harness on the GPU backend against the reference's own CLI
outputs (tests/golden/cli, made by tests/golden/make_golden_cli.py running
curvemg.cli; reference cli.py:47-275, image.py:90-107, :199-281)."""

import hashlib
import json
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2204_07921_b200 import cli
from paper_2204_07921_b200.phantoms import phantom

GOLD = Path(__file__).resolve().parent / "golden" / "cli"
CASES = ["denoise_triangle", "denoise_shepp_gc_rel_u", "bench_sizes", "mri_radial"]

# the reference CLI invocations (make_golden_cli.CASES)
ARGS = {
    "denoise_triangle": ["denoise", "--phantom", "triangle", "--size", "64", "--sigma", "12", "--seed", "3",
                         "--max-outer", "8", "--threads", "1"],
    "denoise_shepp_gc_rel_u": ["denoise", "--phantom", "shepp_logan", "--size", "48", "--sigma", "0.05",
                               "--mode", "gaussian", "--stop", "u", "--epsilon", "1e-3", "--layers", "4",
                               "--max-outer", "30", "--threads", "1", "--clip"],
    "bench_sizes": ["bench", "--sizes", "64,96", "--bench-iters", "4", "--threads", "1"],
    "mri_radial": ["mri", "--phantom", "shepp_logan", "--size", "48", "--sigma", "4", "--rate", "0.3",
                   "--layers", "2", "--max-outer", "4", "--epsilon", "1e-300", "--threads", "1"],
}


def _manifest(path: Path) -> dict:
    d = json.loads(path.read_text())
    d.pop("output_dir")
    return d


def test_phantoms_match_reference():
    ref = json.loads((GOLD / "phantoms.json").read_text())
    for key, r in ref.items():
        kind, size = key.rsplit("_", 1)
        img = phantom(kind, int(size))
        assert img.peak == r["peak"]
        assert hashlib.sha256(img.data.tobytes()).hexdigest() == r["sha256"], key


@pytest.mark.parametrize("case", CASES)
def test_manifest_from_args_matches_reference(case, tmp_path):
    m = cli.manifest_from_args(ARGS[case] + ["--output-dir", str(tmp_path)])
    ours = json.loads(m.to_json())
    ours.pop("output_dir")
    assert ours == _manifest(GOLD / case / "manifest.json")
    # JSON round trip (cli.py:73-88), including the B200-only keys
    m2 = cli.RunManifest.from_json(m.to_json())
    assert m2 == m
    m.dtype, m.precision = "float32", "fast"
    assert cli.RunManifest.from_json(m.to_json()) == m
    with pytest.raises(ValueError, match="unknown manifest keys"):
        cli.RunManifest.from_json('{"bogus": 1}')


def _text_no_dir(path: Path) -> str:
    """The file's exact text with the output_dir value blanked (byte comparison)."""
    return re.sub(r'"output_dir": "[^"]*"', '"output_dir": "X"', path.read_text())


def _trace(path: Path):
    lines = path.read_text().splitlines()
    assert lines[0] == "# schema=curvemg-trace-1"
    rows = [ln.split(",") for ln in lines[2:]]
    return lines[1], rows


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_cli_outputs_match_reference(case, tmp_path):
    g = GOLD / case
    code = cli.run(cli.manifest_from_args(ARGS[case] + ["--output-dir", str(tmp_path)]))
    assert code == int((g / "exit_code").read_text())
    assert _manifest(tmp_path / "manifest.json") == _manifest(g / "manifest.json")
    assert _text_no_dir(tmp_path / "manifest.json") == _text_no_dir(g / "manifest.json")
    if case.startswith("bench"):
        ref = [ln.split(",") for ln in (g / "bench.csv").read_text().splitlines()]
        ours = [ln.split(",") for ln in (tmp_path / "bench.csv").read_text().splitlines()]
        assert ours[:2] == ref[:2]  # schema + header
        for a, b in zip(ours[2:], ref[2:]):
            assert a[:3] == b[:3]  # size, pixels, iterations (seconds / ratios are timings)
        return
    recon = case.startswith("mri")
    if recon:  # reconstruction: inner products / FFT sum in another order -> rounding-level agreement
        assert (tmp_path / "mask.pgm").read_bytes() == (g / "mask.pgm").read_bytes()
        for f in ("kspace.csv", "restored.csv"):
            a, b = np.loadtxt(tmp_path / f, delimiter=","), np.loadtxt(g / f, delimiter=",")
            assert np.abs(a - b).max() <= 1e-7 * max(1.0, np.abs(b).max()), f
    else:
        # images: byte-identical files (fp64 exact path is bit-identical to the reference)
        for f in sorted(p.name for p in g.iterdir() if p.name.startswith(("noisy", "restored"))):
            assert (tmp_path / f).read_bytes() == (g / f).read_bytes(), f
    # trace: same rows; energies within the device-sum tolerance, seconds differ
    h1, r1 = _trace(tmp_path / "trace.csv")
    h2, r2 = _trace(g / "trace.csv")
    assert h1 == h2 and len(r1) == len(r2)
    for a, b in zip(r1, r2):
        assert a[0] == b[0]
        assert abs(float(a[1]) - float(b[1])) <= (1e-8 if recon else 1e-12) * abs(float(b[1]))
        for k in (2, 3):  # rel_energy, rel_u (empty at iteration 0)
            assert (a[k] == "") == (b[k] == "")
            if b[k]:
                tol = 1e-6 if recon else 1e-9
                assert abs(float(a[k]) - float(b[k])) <= tol * abs(float(b[k])) + 1e-12
        assert abs(float(a[5]) - float(b[5])) <= (1e-7 if recon else 1e-9)
    # report.json: identical except the wall time and the GPU energy sum order
    ro = json.loads((tmp_path / "report.json").read_text())
    rr = json.loads((g / "report.json").read_text())
    for k in ("command", "converged", "iterations"):
        assert ro[k] == rr[k], k
    for k in ("psnr", "ssim"):
        assert ro[k] == rr[k] if not recon else abs(ro[k] - rr[k]) <= 1e-7, k
    assert abs(ro["energy"] - rr["energy"]) <= (1e-8 if recon else 1e-12) * abs(rr["energy"])
    ro["config"].pop("output_dir"), rr["config"].pop("output_dir")
    assert ro["config"] == rr["config"]
    assert set(ro) == set(rr)


@pytest.mark.gpu
def test_cli_ct_runs_on_gpu(tmp_path):
    """The reference's `ct` command raises TypeError (it passes value_range= to
    reconstruct); here it runs the intended reconstruction."""
    code = cli.run(cli.manifest_from_args(["ct", "--phantom", "shepp_logan", "--size", "48", "--projections", "16",
                                           "--layers", "2", "--max-outer", "3", "--epsilon", "1e-300",
                                           "--output-dir", str(tmp_path)]))
    assert code == cli.EXIT_NOT_CONVERGED
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["iterations"] == 3 and np.isfinite(rep["energy"]) and rep["psnr"] > 10
    for f in ("sinogram.csv", "sinogram.csv.json", "restored.csv", "trace.csv", "manifest.json"):
        assert (tmp_path / f).exists(), f
