"""Golden outputs of the REFERENCE reconstruction path (curvemg.reconstruction,
/root/reference/pkg/src/curvemg/reconstruction.py) for tests/test_recon.py.

    python tests/golden/make_golden_recon.py

CT: 48x48 Shepp-Logan, 16 angles, noisy sinogram; MRI: 48x48 Shepp-Logan,
golden-angle radial mask (rate 0.3) and a Cartesian mask, noisy k-space.
Records the operator outputs on a random image (bit-exactness of the Radon
splat/gather), the masks, the power-norm estimates and the reconstruction
trajectories (layers 2, 4 cycles).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from curvemg import SolverConfig  # noqa: E402
from curvemg import reconstruction as R  # noqa: E402
from curvemg.image import phantom  # noqa: E402


def main():
    arr, meta = {}, {}
    clean = phantom("shepp_logan", 48)
    arr["clean"] = clean.data
    rng = np.random.default_rng(7)
    x = rng.random((48, 48))
    arr["x"] = x
    # CT
    geom = R.RadonGeometry.for_image((48, 48), 16)
    A = R.RadonTransform((48, 48), geom)
    arr["ct_fwd_x"] = A.forward(x)
    y = rng.standard_normal(A.measurement_shape)
    arr["ct_y"] = y
    arr["ct_adj_y"] = A.adjoint(y)
    sino = A.forward(clean.data)
    sino = sino + np.random.default_rng(3).normal(0.0, 0.01 * np.abs(sino).max(), sino.shape)
    arr["ct_sino"] = sino
    meta["ct"] = dict(n_angles=16, detector_count=geom.detector_count, power=R.power_norm_estimate(A))
    cfg = SolverConfig(alpha=0.06, mode="mean", layers=2, max_outer=4, epsilon=1e-300, threads=1)
    img, tr = R.reconstruct(sino, A, cfg, reference=clean, peak=1.0)
    arr["ct_u"] = img.data
    meta["ct"].update(energies=tr.energies().tolist(), psnr=[r.psnr for r in tr.records], iterations=tr.iterations,
                      energy_final=R.reconstruction_energy(img.data, sino, A, 0.06))
    # MRI
    for kind in ("radial", "cartesian"):
        mask = R.radial_mask((48, 48), 0.3) if kind == "radial" else R.cartesian_mask((48, 48), 0.3, seed=2)
        arr[f"mask_{kind}"] = mask.mask
        F = R.MaskedFourier(mask)
        k = F.forward(clean.data)
        noise = np.random.default_rng(5).normal(0.0, 0.02 / np.sqrt(2.0), (k.size, 2))
        k = k + noise[:, 0] + 1j * noise[:, 1]
        arr[f"mri_{kind}_k"] = k
        img, tr = R.reconstruct(k, F, cfg, reference=clean, peak=1.0)
        arr[f"mri_{kind}_u"] = img.data
        meta[f"mri_{kind}"] = dict(rate=mask.rate, power=R.power_norm_estimate(F), energies=tr.energies().tolist(),
                                   psnr=[r.psnr for r in tr.records], iterations=tr.iterations)
    np.savez_compressed(HERE / "recon.npz", **arr)
    (HERE / "recon.json").write_text(json.dumps(meta, indent=1))
    print(json.dumps(meta)[:400])


if __name__ == "__main__":
    main()
