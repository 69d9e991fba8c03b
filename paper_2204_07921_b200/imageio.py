"""Image files for the denoising path: binary PGM (P5,
8/16-bit) and float64 CSV with a JSON sidecar.  Behaviour (byte layout,
value mapping, peaks, errors) follows /root/reference/pkg/src/curvemg/
image.py:289-335 so files round-trip between the two packages; checked
against files the reference wrote (tests/golden/io).  Host-side I/O only.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .image import Image

__all__ = ["write_pgm", "read_pgm", "write_csv", "read_csv"]


def write_pgm(img: Image, path, bits: int = 8) -> None:
    """P5 file; intensities scaled by maxval/peak, rounded half-to-even and
    clamped to [0, maxval]; 16-bit samples big-endian (image.py:289-297)."""
    if bits not in (8, 16):
        raise ValueError("bits must be 8 or 16")
    top = 2 ** bits - 1
    q = np.clip(np.rint(img.data * (top / img.peak)), 0, top)
    body = q.astype(np.dtype(">u2") if bits == 16 else np.uint8).tobytes()
    Path(path).write_bytes(b"P5\n%d %d\n%d\n" % (img.width, img.height, top) + body)


def _pgm_header(raw: bytes, path) -> tuple[list[bytes], int]:
    """Four whitespace-separated header fields (magic, width, height, maxval),
    '#' comments allowed between them; returns the fields and the offset of
    the single whitespace byte that ends the header."""
    fields, i, n = [], 0, len(raw)
    while len(fields) < 4:
        while i < n and (raw[i:i + 1].isspace() or raw[i:i + 1] == b"#"):
            if raw[i:i + 1] == b"#":
                j = raw.find(b"\n", i)
                if j < 0:
                    raise ValueError(f"truncated PGM header in {path}")
                i = j + 1
            else:
                i += 1
        if i >= n:
            raise ValueError(f"truncated PGM header in {path}")
        j = i
        while j < n and not raw[j:j + 1].isspace():
            j += 1
        fields.append(raw[i:j])
        i = j
    return fields, i


def read_pgm(path) -> Image:
    """P5 file -> Image with peak = stored maxval (image.py:300-317)."""
    raw = Path(path).read_bytes()
    (magic, w, h, mv), end = _pgm_header(raw, path)
    if magic != b"P5":
        raise ValueError(f"not a binary PGM file: {path}")
    w, h, mv = int(w), int(h), int(mv)
    sample = np.dtype(">u2") if mv > 255 else np.dtype(np.uint8)
    px = np.frombuffer(raw, dtype=sample, count=w * h, offset=end + 1)
    return Image(px.reshape(h, w).astype(np.float64), float(mv))


def write_csv(img: Image, path) -> None:
    """Comma-separated rows at 17 significant digits, plus '<path>.json' with
    peak / width / height (image.py:320-325)."""
    p = Path(path)
    np.savetxt(p, img.data, delimiter=",", fmt="%.17g")
    meta = {"peak": img.peak, "width": img.width, "height": img.height}
    Path(str(p) + ".json").write_text(json.dumps(meta))


def read_csv(path) -> Image:
    """CSV (+ optional sidecar; peak 255 without one) -> Image (image.py:328-335)."""
    p = Path(path)
    side = Path(str(p) + ".json")
    peak = float(json.loads(side.read_text())["peak"]) if side.exists() else 255.0
    return Image(np.loadtxt(p, delimiter=",", ndmin=2), peak)
