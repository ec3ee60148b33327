"""Visibility stress cases for the pass-2 shortcuts (pixel winners, 8x8
hierarchical Z, single-compare edges): stacked layers whose NDC depths sit
just inside and just outside the visibility slack 1e-6*max(1,|d|)
(charts.py:309-311), mixed small / tiled / near-clipped triangles.  Every
flag, chart id and placement must equal the C oracle's.  Run with -m gpu."""

import math

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

fa = pytest.importorskip("paper_2502_17712_b200")
from paper_2502_17712_b200 import FrameEngine, FrameSettings  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()


SCREEN = (320, 240)


def _camera():
    return fa.CameraFrame.from_params(math.radians(60.0), SCREEN[0] / SCREEN[1], 0.1, 100.0,
                                      position=(0.0, 0.0, 0.0), look_at=(0.0, 0.0, -1.0))


def _ndc_z(vp, d):
    c = np.asarray(vp) @ np.array([0.0, 0.0, -d, 1.0])
    return c[2] / c[3]


def _depth_for(vp, z_target):
    """distance d on the view axis whose NDC depth is z_target (bisection)."""
    lo, hi = 0.1, 100.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if _ndc_z(vp, mid) < z_target:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _layer(d, n, half, rng, jitter):
    """n x n quad grid facing the camera at distance d (2 tris / cell, ccw)."""
    xs = np.linspace(-half, half, n + 1)
    gx, gy = np.meshgrid(xs, xs, indexing="xy")
    pos = np.stack([gx.ravel(), gy.ravel(), np.full(gx.size, -d)], 1)
    pos[:, :2] += rng.uniform(-jitter, jitter, size=(len(pos), 2)) * (2 * half / n)
    tris = []
    for j in range(n):
        for i in range(n):
            a = j * (n + 1) + i
            b, c, e = a + 1, a + n + 1, a + n + 2
            tris += [(a, b, e), (a, e, c)]
    return pos, np.asarray(tris, np.int64)


def _merge(parts):
    pos, tris, base = [], [], 0
    for p, t in parts:
        pos.append(p)
        tris.append(t + base)
        base += len(p)
    return np.vstack(pos), np.vstack(tris).astype(np.int32)


def _check(pos, tris, vp, omega=512):
    eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=SCREEN, omega=omega, uv_f64=True))
    out = eng.run(vp, check=False)
    r = oracle.run_frame(pos, tris, vp, SCREEN, omega)
    assert out.status == r.status
    h = out.to_host()
    assert np.array_equal(h["flags"].astype(bool), r.flags)
    assert np.array_equal(h["chart_of_triangle"].astype(np.int64), r.chart_of_triangle)
    if r.status == oracle.OK:
        assert np.array_equal(h["placements"], r.pack.placements)
        assert h["screen_fragments"] == r.screen_fragments
    # standalone passes (hierarchical Z without pixel winners)
    mesh = fa.Mesh(pos, tris)
    depth = fa.depth_prepass(mesh, _camera(), SCREEN)
    assert np.array_equal(depth, r.depth)  # +-0 compare equal
    vis = fa.mark_visible(mesh, _camera(), depth)
    assert np.array_equal(vis.flags, r.flags)
    return r


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_layers_around_the_slack(seed):
    rng = np.random.default_rng(seed)
    vp = _camera().view_proj
    z0 = _ndc_z(vp, 6.0)
    parts = []
    # relative NDC offsets: inside the slack (visible), at its edge, outside (hidden)
    for k, dz in enumerate([0.0, 0.2e-6, 0.9e-6, 1.1e-6, 3e-6, 1e-4]):
        d = _depth_for(vp, z0 + dz)
        n = [8, 13, 40, 21, 64, 5][k]  # big (tiled) and small (record) triangles
        parts.append(_layer(d, n, 3.0 + 0.1 * k, rng, 0.2))
    # a layer crossing the near plane (clipping path) and one far behind
    near = _layer(0.5, 6, 1.0, rng, 0.1)
    near[0][:, 2] += rng.uniform(-0.45, 0.2, size=len(near[0]))
    parts.append(near)
    parts.append(_layer(50.0, 30, 40.0, rng, 0.3))
    pos, tris = _merge(parts)
    r = _check(pos, tris, vp)
    assert r.status == oracle.OK
    assert r.flags.sum() > 0


def test_coplanar_duplicates():
    """Exact duplicates at equal depth: both copies pass the slack test."""
    rng = np.random.default_rng(7)
    vp = _camera().view_proj
    a = _layer(5.0, 30, 2.5, rng, 0.3)
    b = (a[0].copy(), a[1][:, ::-1].copy())  # same geometry, reversed winding (culled)
    c = (a[0].copy(), a[1].copy())           # same geometry, same winding
    pos, tris = _merge([a, b, c, _layer(9.0, 50, 6.0, rng, 0.4)])
    r = _check(pos, tris, vp)
    assert r.status == oracle.OK


def _screen_tris(vp_cam, pts_px, depths):
    """World triangles whose corners project to the given screen points
    (pixels, row 0 at NDC y = -1) at view distance `depths` (one per tri)."""
    W, H = SCREEN
    t = math.tan(math.radians(60.0) / 2)
    aspect = W / H
    pos = []
    for tri, d in zip(pts_px, depths):
        for sx, sy in tri:
            nx, ny = 2.0 * sx / W - 1.0, 2.0 * sy / H - 1.0
            pos.append((nx * d * t * aspect, ny * d * t, -d))
    pos = np.asarray(pos, np.float64)
    tris = np.arange(len(pos)).reshape(-1, 3)
    return pos, tris


@pytest.mark.parametrize("seed", [0, 1])
def test_edges_through_sample_centres(seed):
    """Small triangles whose corners sit on pixel centres +- 1e-12..5e-3 px,
    so their edges graze sample centres at every distance around the span
    margin (and edges are near-horizontal with |dy| around the 1e-3 / 1e-2
    span thresholds): the pruned row spans of the small-record path must
    drop no sample the reference covers (charts.py:237-249)."""
    rng = np.random.default_rng(100 + seed)
    offs = np.array([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 1e-6, -1e-6, 1e-4, -1e-4, 1e-3, -1e-3, 5e-3, -5e-3])
    pts, depths = [], []
    W, H = SCREEN
    for _ in range(3000):
        cx, cy = rng.integers(8, W - 56), rng.integers(8, H - 16)
        kind = rng.integers(0, 3)
        if kind == 0:    # compact triangle, corners on centres + tiny offsets
            c = np.array([[0, 0], [rng.integers(1, 6), rng.integers(0, 3)], [rng.integers(0, 3), rng.integers(1, 6)]],
                         np.float64)
        elif kind == 1:  # long, nearly horizontal edge (dy ~ 1e-3 .. 1e-2 over up to 40 px)
            L = rng.integers(10, 40)
            c = np.array([[0, 0], [L, rng.choice([1e-3, -1e-3, 1e-2, -1e-2, 2e-2, 0.0])], [rng.integers(0, L), 1]],
                         np.float64)
        else:            # thin sliver crossing a column of centres
            c = np.array([[0, 0], [rng.choice([1e-3, 1e-2, 0.5]), rng.integers(4, 9)], [1, rng.integers(1, 5)]],
                         np.float64)
        c = c + 0.5 + rng.choice(offs, size=(3, 2))
        c[:, 0] += cx
        c[:, 1] += cy
        tri = [tuple(p) for p in c]
        # counter-clockwise in screen space (front-facing with culling on)
        a2 = (c[1, 0] - c[0, 0]) * (c[2, 1] - c[0, 1]) - (c[2, 0] - c[0, 0]) * (c[1, 1] - c[0, 1])
        if a2 < 0:
            tri = [tri[0], tri[2], tri[1]]
        pts.append(tri)
        depths.append(rng.uniform(3.0, 9.0))
    pos, tris = _screen_tris(None, pts, depths)
    r = _check(pos, tris, _camera().view_proj)
    assert r.flags.sum() > 100


@pytest.mark.parametrize("seed", [0, 1])
def test_subpixel_triangles(seed):
    """Sub-pixel triangles, most covering no sample centre: the setup drops
    provably empty windows (no centre within the vertex box + 1e-4 px, or <= 4
    centres failing the edge test, slivers excepted -- fa_raster.cuh
    empty_window).  Boxes end at centres + {0, +-1e-12, +-1e-6, +-1e-4 +- 1e-8}
    and include near-degenerate slivers, so every branch of the test meets
    the reference's own edge arithmetic at its boundary."""
    rng = np.random.default_rng(300 + seed)
    offs = np.array([0.0, 1e-12, -1e-12, 1e-6, -1e-6, 1e-4, -1e-4, 1e-4 + 1e-8, -1e-4 - 1e-8, 1e-4 - 1e-8])
    pts, depths = [], []
    W, H = SCREEN
    for _ in range(4000):
        cx, cy = rng.integers(4, W - 8), rng.integers(4, H - 8)
        kind = rng.integers(0, 3)
        if kind == 0:    # tiny triangle anywhere in a pixel
            base = rng.uniform(0.0, 1.0, size=2)
            c = base + rng.uniform(-0.6, 0.6, size=(3, 2))
        elif kind == 1:  # a corner on a centre +- offsets, the others within a pixel
            c = np.array([[0.5, 0.5], [0.5, 0.5], [0.5, 0.5]]) + rng.uniform(-0.9, 0.9, size=(3, 2))
            c[0] = 0.5 + rng.choice(offs, size=2)
        else:            # near-degenerate sliver through / beside a centre
            a = np.array([0.5, 0.5]) + rng.choice(offs, size=2)
            d = rng.uniform(-1, 1, size=2)
            d /= np.linalg.norm(d)
            c = np.array([a - 0.8 * d, a + 0.9 * d, a + rng.choice([1e-7, 1e-5, 1e-3]) * np.array([-d[1], d[0]])])
        c[:, 0] += cx
        c[:, 1] += cy
        a2 = (c[1, 0] - c[0, 0]) * (c[2, 1] - c[0, 1]) - (c[2, 0] - c[0, 0]) * (c[1, 1] - c[0, 1])
        tri = [tuple(p) for p in c]
        if a2 < 0:
            tri = [tri[0], tri[2], tri[1]]
        pts.append(tri)
        depths.append(rng.uniform(3.0, 9.0))
    pos, tris = _screen_tris(None, pts, depths)
    r = _check(pos, tris, _camera().view_proj)
    assert r.flags.sum() > 50
