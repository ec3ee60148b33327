"""Mirror of atlaspack.metrics (metrics.py:1-161).

These run after the per-frame path (quality evaluation,
"next" rows §8f-1/2).  The digest / efficiency helpers are host functions
over the layout value objects, exactly as in the reference.
`scene_stretch_arrays` evaluates the stretch metric for a whole frame in
closed form (2x2 singular values) vectorised over triangles.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .packing import AtlasLayout

DIGEST_ALGORITHM = "sha256"


class MetricsError(Exception):
    pass


class DegenerateTriangle(MetricsError):
    """The atlas-space triangle has zero area; the map is undefined."""


class NoValidTriangles(MetricsError):
    """No triangle pair survived validation."""


@dataclass(frozen=True)
class StretchReport:
    l2: float
    linf: float
    per_triangle: tuple | None = None


@dataclass(frozen=True)
class LayoutDigest:
    digest: str
    algorithm: str = DIGEST_ALGORITHM


def packing_efficiency(layout: AtlasLayout) -> float:
    """metrics.py:52-55."""
    area = sum(p.w * p.h for p in layout.placements)
    return area / float(layout.omega * layout.omega)


def _sv2(m):
    """Singular values of 2x2 matrices (..., 2, 2) -> (big, small), the
    stable closed form the GPU uses (fa_uv.cu): big = (|q| + |r|) / 2 with
    q = (a + d, c - b), r = (a - d, c + b); small = |det| / big."""
    a, b, c, d = m[..., 0, 0], m[..., 0, 1], m[..., 1, 0], m[..., 1, 1]
    big = 0.5 * (np.hypot(a + d, c - b) + np.hypot(a - d, c + b))
    det = np.abs(a * d - b * c)
    small = np.divide(det, big, out=np.zeros_like(big), where=big > 0)
    return big, np.minimum(small, big)


def triangle_stretch(screen_tri, atlas_tri) -> tuple[float, float]:
    """metrics.py:58-75: singular values (max, min) of one triangle pair's
    atlas-to-screen map, through this module's closed form (the reference
    calls LAPACK's SVD; the two agree to rounding).  DegenerateTriangle for
    a zero-area atlas triangle."""
    big, small, ok, _ = _pair_singular_values(np.asarray(screen_tri, dtype=np.float64).reshape(1, 3, 2),
                                              np.asarray(atlas_tri, dtype=np.float64).reshape(1, 3, 2))
    if not ok[0]:
        raise DegenerateTriangle("atlas triangle has zero area")
    return float(big[0]), float(small[0])


def _pair_singular_values(s, a):
    """(n,3,2) screen / atlas triangles -> singular values (big, small) of
    M = Es Ea^-1 for the pairs with a non-degenerate atlas triangle, the
    mask of those pairs, and their screen areas."""
    ea = np.stack([a[:, 1] - a[:, 0], a[:, 2] - a[:, 0]], axis=2)
    es = np.stack([s[:, 1] - s[:, 0], s[:, 2] - s[:, 0]], axis=2)
    det = ea[:, 0, 0] * ea[:, 1, 1] - ea[:, 0, 1] * ea[:, 1, 0]
    ok = det != 0.0
    ea, es, det, sk = ea[ok], es[ok], det[ok], s[ok]
    inv = np.empty_like(ea)
    inv[:, 0, 0] = ea[:, 1, 1] / det
    inv[:, 0, 1] = -ea[:, 0, 1] / det
    inv[:, 1, 0] = -ea[:, 1, 0] / det
    inv[:, 1, 1] = ea[:, 0, 0] / det
    big, small = _sv2(es @ inv)
    e1 = sk[:, 1] - sk[:, 0]
    e2 = sk[:, 2] - sk[:, 0]
    area = np.abs(e1[:, 0] * e2[:, 1] - e1[:, 1] * e2[:, 0]) / 2.0
    return big, small, ok, area


def scene_stretch(pairs: Iterable[tuple], keep_per_triangle: bool = False) -> StretchReport:
    """metrics.py:84-111."""
    pairs = list(pairs)
    if not pairs:
        raise NoValidTriangles("no valid triangle pairs")
    s = np.array([np.asarray(p[0], dtype=np.float64).reshape(3, 2) for p in pairs])
    a = np.array([np.asarray(p[1], dtype=np.float64).reshape(3, 2) for p in pairs])
    return scene_stretch_arrays(s, a, keep_per_triangle)


def scene_stretch_arrays(screen, atlas, keep_per_triangle: bool = False) -> StretchReport:
    """Vectorised metrics.py:84-111 over (n,3,2) screen and atlas triangles."""
    s = np.asarray(screen, dtype=np.float64).reshape(-1, 3, 2)
    a = np.asarray(atlas, dtype=np.float64).reshape(-1, 3, 2)
    big, small, ok, area = _pair_singular_values(s, a)
    if not np.any(ok):
        raise NoValidTriangles("no valid triangle pairs")
    weighted = float(np.sum(area * (big * big + small * small) / 2.0))
    total = float(np.sum(area))
    l2 = float(np.sqrt(weighted / total)) if total > 0 else 0.0
    per = tuple(zip(big.tolist(), small.tolist())) if keep_per_triangle else None
    return StretchReport(l2=l2, linf=float(big.max()), per_triangle=per)


def effective_shading_rate(layout: AtlasLayout, screen_fragments: int, texels_read: int | None = None) -> float:
    """metrics.py:114-127."""
    if screen_fragments <= 0:
        raise MetricsError("effective shading rate undefined: no visible fragments")
    if texels_read is None:
        texels_read = sum(p.w * p.h for p in layout.placements)
    return texels_read / float(screen_fragments)


def layout_digest(layout: AtlasLayout) -> LayoutDigest:
    """metrics.py:130-153: SHA-256 of the canonical little-endian serialisation."""
    h = hashlib.sha256()
    h.update(struct.pack("<QqqQ", layout.omega, layout.scale.numerator, layout.scale.denominator,
                         len(layout.placements)))
    for p in layout.placements_by_chart_id():
        h.update(struct.pack("<qqqqqBqq", p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h))
    return LayoutDigest(digest=h.hexdigest())


def layouts_equal(a: AtlasLayout, b: AtlasLayout) -> bool:
    """metrics.py:156-161."""
    return a.omega == b.omega and a.scale == b.scale and a.placements_by_chart_id() == b.placements_by_chart_id()
