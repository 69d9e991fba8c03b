"""on-device SSIM (bit-identical to curvemg.image.ssim) and the
reference's PGM / CSV file formats, checked against fixtures the reference
produced (tests/golden/make_golden.py: metrics_io_fixture)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import metrics_ref as MR  # noqa: E402
from paper_2204_07921_b200 import Image, imageio  # noqa: E402

G = ROOT / "tests" / "golden"


def _cases():
    meta = json.loads((G / "metrics.json").read_text())
    arr = np.load(G / "metrics.npz")
    return [(c, arr[f"x{k}"], arr[f"y{k}"]) for k, c in enumerate(meta)]


def test_metric_oracle_pinned_to_reference():
    for c, x, y in _cases():
        assert MR.ssim(x, y, c["peak"]) == c["ssim"]
        assert MR.psnr(x, y, c["peak"]) == c["psnr"]
        assert MR.ssim(x, x, c["peak"]) == c["ssim_self"]


def test_file_formats_byte_identical_to_reference(tmp_path):
    d = G / "io"
    img = Image(np.load(d / "image.npy"), 255.0)
    imageio.write_pgm(img, tmp_path / "a8.pgm", bits=8)
    imageio.write_pgm(img, tmp_path / "a16.pgm", bits=16)
    imageio.write_csv(img, tmp_path / "a.csv")
    assert (tmp_path / "a8.pgm").read_bytes() == (d / "img8.pgm").read_bytes()
    assert (tmp_path / "a16.pgm").read_bytes() == (d / "img16.pgm").read_bytes()
    assert (tmp_path / "a.csv").read_bytes() == (d / "img.csv").read_bytes()
    assert json.loads((tmp_path / "a.csv.json").read_text()) == json.loads((d / "img.csv.json").read_text())


def test_file_formats_read_like_reference():
    d = G / "io"
    back = np.load(d / "read_back.npz")
    peaks = json.loads((d / "read_back.json").read_text())
    for name, key in (("img8.pgm", "img8"), ("img16.pgm", "img16")):
        im = imageio.read_pgm(d / name)
        assert np.array_equal(im.data, back[key]) and im.peak == peaks[name]
    im = imageio.read_csv(d / "img.csv")
    assert np.array_equal(im.data, back["csv"]) and im.peak == 255.0


def test_file_format_errors(tmp_path):
    img = Image(np.zeros((3, 4)), 1.0)
    with pytest.raises(ValueError):
        imageio.write_pgm(img, tmp_path / "x.pgm", bits=12)
    (tmp_path / "p2.pgm").write_bytes(b"P2\n2 2\n255\n0 0 0 0\n")
    with pytest.raises(ValueError):
        imageio.read_pgm(tmp_path / "p2.pgm")
    (tmp_path / "short.pgm").write_bytes(b"P5\n# comment\n2 2\n")
    with pytest.raises(ValueError):
        imageio.read_pgm(tmp_path / "short.pgm")
    # comments between header fields are accepted
    (tmp_path / "c.pgm").write_bytes(b"P5\n# made by hand\n2 1\n# max\n255\n" + bytes([7, 200]))
    assert np.array_equal(imageio.read_pgm(tmp_path / "c.pgm").data, [[7.0, 200.0]])
    imageio.write_csv(img, tmp_path / "nosidecar.csv")
    (tmp_path / "nosidecar.csv.json").unlink()
    assert imageio.read_csv(tmp_path / "nosidecar.csv").peak == 255.0


def test_ssim_argument_errors_before_any_device_work():
    from paper_2204_07921_b200 import ssim

    with pytest.raises(ValueError, match="shape mismatch"):
        ssim(Image(np.zeros((12, 12)), 1.0), Image(np.zeros((12, 13)), 1.0))
    with pytest.raises(ValueError, match="SSIM window"):
        ssim(Image(np.zeros((10, 30)), 1.0), Image(np.zeros((10, 30)), 1.0))


@pytest.mark.gpu
def test_gpu_ssim_bit_identical_to_reference():
    from paper_2204_07921_b200 import ssim

    for c, x, y in _cases():
        a, b = Image(x, c["peak"]), Image(y, c["peak"])
        assert ssim(a, b) == c["ssim"], c["shape"]
        assert ssim(a, a) == c["ssim_self"]


@pytest.mark.gpu
def test_gpu_ssim_batch_matches_single_and_fp32_input():
    from paper_2204_07921_b200 import ssim_batch

    cases = [(c, x, y) for c, x, y in _cases() if c["shape"] == [200, 256]]
    c, x, y = cases[0]
    xs = np.stack([x, y, x]).astype(np.float32)
    ys = np.stack([y, x, x]).astype(np.float32)
    out = ssim_batch(xs, ys, c["peak"])
    assert out[0] == c["ssim"]  # fixture values are fp32-representable
    assert out[1] == MR.ssim(y, x, c["peak"])
    assert out[2] == 1.0
