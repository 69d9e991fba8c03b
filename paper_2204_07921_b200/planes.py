"""Tangent-plane stencil tables (host side).

Restates the plane enumeration of the reference ``tangent.plane_set``
(/root/reference/pkg/src/curvemg/tangent.py:95-133): level ``j`` keeps every
plane of level ``j-1`` and, for each new direction ``p`` on the Chebyshev ring
of radius ``2**(j-1)`` (half-ring representatives sorted by angle, directions
deduplicated by gcd), appends the planes ``(p, rot90 p, -p)`` and
``(p, -p, -rot90 p)``.  The CUDA kernels read the same tables from
``csrc/planes_table.h``, which ``tools/gen_planes.py`` writes from this module.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

MAX_LAYER = 6  # tangent.py:43


@dataclass(frozen=True)
class Plane:
    x: tuple[int, int]
    y: tuple[int, int]
    z: tuple[int, int]
    ds2: float

    @property
    def nz(self) -> int:
        dy0, dy1 = self.y[0] - self.x[0], self.y[1] - self.x[1]
        dz0, dz1 = self.z[0] - self.x[0], self.z[1] - self.x[1]
        return dz0 * dy1 - dz1 * dy0


def _rot90(p):
    return (-p[1], p[0])


@lru_cache(maxsize=None)
def planes(layer: int) -> tuple[Plane, ...]:
    """Ordered plane list of one level (count ``2**(layer+2)``)."""
    if not 1 <= layer <= MAX_LAYER:
        raise ValueError(f"layer must be in [1, {MAX_LAYER}], got {layer}")
    out = [] if layer == 1 else list(planes(layer - 1))
    have = set()
    for pl in out:
        g = math.gcd(abs(pl.x[0]), abs(pl.x[1]))
        have.add((pl.x[0] // g, pl.x[1] // g))
    r = 2 ** (layer - 1)
    ring = [(a, b) for a in range(-r, r + 1) for b in range(-r, r + 1) if max(abs(a), abs(b)) == r]
    reps = sorted((p for p in ring if p[0] < 0 or (p[0] == 0 and p[1] > 0)),
                  key=lambda p: math.atan2(-p[0], p[1]))
    for p in reps:
        g = math.gcd(abs(p[0]), abs(p[1]))
        if (p[0] // g, p[1] // g) in have:
            continue
        q = _rot90(p)
        neg = (-p[0], -p[1])
        ds2 = float(p[0] * p[0] + p[1] * p[1])
        out.append(Plane(p, q, neg, ds2))
        out.append(Plane(p, neg, (-q[0], -q[1]), ds2))
    assert len(out) == 2 ** (layer + 2)
    assert all(pl.nz < 0 for pl in out)
    return tuple(out)


def patch_side(layer: int) -> int:
    """hierarchy.py:37-38 -- side = 2**j - 1."""
    return 2 ** layer - 1


def radius(layer: int) -> int:
    """tangent.py:81-83 -- Chebyshev radius 2**(j-1)."""
    return 2 ** (layer - 1)
