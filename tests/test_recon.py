"""Reconstruction on the GPU against the reference's own outputs
(tests/golden/recon.*, made by tests/golden/make_golden_recon.py running
curvemg.reconstruction; reference reconstruction.py:97-442).

Bars: the Radon forward/adjoint and the masks are bit-identical; the power
estimate, the trajectories and the reconstructed images agree to rounding
(inner products and the FFT sum in a different order on the GPU).
"""

import json

import numpy as np
import pytest

from paper_2204_07921_b200 import recon as R
from paper_2204_07921_b200.driver import SolverConfig
from paper_2204_07921_b200.image import Image


@pytest.fixture(scope="module")
def gold(golden_dir):
    return json.loads((golden_dir / "recon.json").read_text()), np.load(golden_dir / "recon.npz")


def test_masks_match_reference(gold):
    meta, arr = gold
    assert np.array_equal(R.radial_mask((48, 48), 0.3).mask, arr["mask_radial"])
    assert np.array_equal(R.cartesian_mask((48, 48), 0.3, seed=2).mask, arr["mask_cartesian"])
    assert R.RadonGeometry.for_image((48, 48), 16).detector_count == meta["ct"]["detector_count"]
    with pytest.raises(ValueError):
        R.radial_mask((8, 8), 0.0)


def test_measurement_io_roundtrip(tmp_path, gold):
    meta, arr = gold
    geom = R.RadonGeometry.for_image((48, 48), 16)
    R.save_sinogram(arr["ct_sino"], geom, tmp_path / "s.csv")
    s, g = R.load_sinogram(tmp_path / "s.csv")
    assert np.array_equal(s, arr["ct_sino"]) and g == geom
    mask = R.SamplingMask("radial", arr["mask_radial"])
    R.save_kspace(arr["mri_radial_k"], mask, tmp_path / "k.csv")
    assert np.array_equal(R.load_kspace(tmp_path / "k.csv"), arr["mri_radial_k"])
    R.mask_to_pgm(mask, tmp_path / "m.pgm")
    assert np.array_equal(R.mask_from_pgm(tmp_path / "m.pgm").mask, mask.mask)


@pytest.mark.gpu
def test_radon_operator_bitexact(gold):
    meta, arr = gold
    A = R.RadonTransform((48, 48), R.RadonGeometry.for_image((48, 48), 16))
    assert np.array_equal(A.forward(arr["x"]).cpu().numpy(), arr["ct_fwd_x"])
    assert np.array_equal(A.adjoint(arr["ct_y"]).cpu().numpy(), arr["ct_adj_y"])
    assert abs(R.power_norm_estimate(A) - meta["ct"]["power"]) <= 1e-12 * meta["ct"]["power"]


def _check_run(tr, u, g, u_ref):
    e, er = tr.energies(), np.array(g["energies"])
    assert tr.iterations == g["iterations"]
    assert np.all(np.abs(e - er) <= 1e-8 * np.abs(er)), (e, er)
    assert np.allclose([r.psnr for r in tr.records], g["psnr"], rtol=0, atol=1e-7)
    assert np.abs(u - u_ref).max() <= 1e-7 * max(1.0, np.abs(u_ref).max())


@pytest.mark.gpu
def test_ct_reconstruction_matches_reference(gold):
    meta, arr = gold
    A = R.RadonTransform((48, 48), R.RadonGeometry.for_image((48, 48), 16))
    cfg = SolverConfig(alpha=0.06, mode="mean", layers=2, max_outer=4, epsilon=1e-300)
    img, tr = R.reconstruct(arr["ct_sino"], A, cfg, reference=Image(arr["clean"], 1.0), peak=1.0)
    _check_run(tr, img.data, meta["ct"], arr["ct_u"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["radial", "cartesian"])
def test_mri_reconstruction_matches_reference(gold, kind):
    meta, arr = gold
    F = R.MaskedFourier(R.SamplingMask(kind, arr[f"mask_{kind}"]))
    assert abs(R.power_norm_estimate(F) - meta[f"mri_{kind}"]["power"]) <= 1e-12
    cfg = SolverConfig(alpha=0.06, mode="mean", layers=2, max_outer=4, epsilon=1e-300)
    img, tr = R.reconstruct(arr[f"mri_{kind}_k"], F, cfg, reference=Image(arr["clean"], 1.0), peak=1.0)
    _check_run(tr, img.data, meta[f"mri_{kind}"], arr[f"mri_{kind}_u"])


@pytest.mark.gpu
def test_reconstruct_rejects_gaussian_prior(gold):
    meta, arr = gold
    A = R.RadonTransform((48, 48), R.RadonGeometry.for_image((48, 48), 16))
    with pytest.raises(ValueError, match="mean-curvature"):
        R.reconstruct(arr["ct_sino"], A, SolverConfig(mode="gaussian"))
