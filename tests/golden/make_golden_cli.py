"""Golden outputs of the REFERENCE command-line harness (curvemg.cli,
/root/reference/pkg/src/curvemg/cli.py) for the CLI parity tests.

    python tests/golden/make_golden_cli.py

Runs ``curvemg.cli.main`` (denoise and bench commands) in a subprocess with
the reference on sys.path and keeps its output directories under
tests/golden/cli/<case>/ (trace seconds and report wall_time vary run to run;
the tests compare everything else).
"""

from __future__ import annotations

import shutil
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent / "cli"
REF = "/root/reference/pkg/src"

CASES = {
    "denoise_triangle": ["denoise", "--phantom", "triangle", "--size", "64", "--sigma", "12", "--seed", "3",
                         "--max-outer", "8", "--threads", "1"],
    "denoise_shepp_gc_rel_u": ["denoise", "--phantom", "shepp_logan", "--size", "48", "--sigma", "0.05",
                               "--mode", "gaussian", "--stop", "u", "--epsilon", "1e-3", "--layers", "4",
                               "--max-outer", "30", "--threads", "1", "--clip"],
    "bench_sizes": ["bench", "--sizes", "64,96", "--bench-iters", "4", "--threads", "1"],
    "mri_radial": ["mri", "--phantom", "shepp_logan", "--size", "48", "--sigma", "4", "--rate", "0.3",
                   "--layers", "2", "--max-outer", "4", "--epsilon", "1e-300", "--threads", "1"],
}


def phantoms():
    """SHA-256 of the reference phantoms (image.py:199-281) at a few sizes."""
    import hashlib
    import json

    sys.path.insert(0, REF)
    from curvemg.image import phantom

    out = {}
    for kind in ("shepp_logan", "triangle", "shapes"):
        for size in (32, 64, 100, 257):
            img = phantom(kind, size)
            out[f"{kind}_{size}"] = {"peak": img.peak, "sha256": hashlib.sha256(img.data.tobytes()).hexdigest()}
    (HERE / "phantoms.json").write_text(json.dumps(out, indent=1))


def main():
    phantoms()
    for name, argv in CASES.items():
        out = HERE / name
        shutil.rmtree(out, ignore_errors=True)
        code = (f"import sys; sys.path.insert(0, {REF!r}); from curvemg.cli import main; "
                f"main({argv + ['--output-dir', str(out)]!r})")
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
        (out / "exit_code").write_text(f"{r.returncode}\n")
        print(name, "exit", r.returncode, sorted(p.name for p in out.iterdir()))


if __name__ == "__main__":
    main()
