"""Deterministic synthetic scenes for the per-frame atlasing benchmarks.

These generators rebuild the scene shapes of SURVEY.md §8(d) (the reference
ships no scenes; its tests synthesise inputs from seeds, see
`/root/reference/pkg/tests/oracles.py:211-218`).  They are host-side input
builders used by bench.py, the parity tests and the golden-vector script —
not part of the per-frame hot path.

Shapes (triangle / vertex counts match SURVEY §8(d) exactly):

* C1: icosphere L4 (5,120 tris) + 75x100 ground plane  -> 20,120 tris,   512x512,   omega 1024
* C2: 8x6 sphere field at L5 + 100x85 plane            -> 1,000,040 tris, 1920x1080, omega 2048
* C3: 8x6 sphere field at L6 + 250x136 plane           -> 4,000,160 tris, 3840x2160, omega 4096, prescale 2
* C4: C2 scene, 120-frame camera arc
* C5: C2 scene, 64 golden-angle views

Every triangle is wound counter-clockwise seen from its front side, which is
the front-facing convention of the reference rasterizer
(`/root/reference/pkg/src/atlaspack/charts.py:205-219`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "icosphere",
    "ground_plane",
    "sphere_field",
    "SceneSpec",
    "CameraPose",
    "scene_c1",
    "scene_c2",
    "scene_c3",
    "camera_path_c4",
    "views_c5",
    "build_scene",
    "CONFIGS",
]


def icosphere(level: int, center=(0.0, 0.0, 0.0), radius: float = 1.0):
    """Subdivided icosahedron (20*4^level tris, 10*4^level+2 verts), outward CCW."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    verts = [
        (-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
        (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
        (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1),
    ]
    faces = [
        (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
        (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
        (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
        (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
    ]
    v = np.asarray(verts, dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.asarray(faces, dtype=np.int64)
    for _ in range(level):
        # one midpoint per undirected edge, numbered after the old vertices
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
        key = np.sort(e, axis=1)
        uniq, inv = np.unique(key, axis=0, return_inverse=True)
        inv = inv.reshape(-1)
        mid = v[uniq[:, 0]] + v[uniq[:, 1]]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        base = len(v)
        v = np.vstack([v, mid])
        nf = len(f)
        ab = base + inv[:nf]
        bc = base + inv[nf:2 * nf]
        ca = base + inv[2 * nf:]
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        f = np.concatenate([
            np.stack([a, ab, ca], 1),
            np.stack([ab, b, bc], 1),
            np.stack([ca, bc, c], 1),
            np.stack([ab, bc, ca], 1),
        ])
    pos = v * float(radius) + np.asarray(center, dtype=np.float64)
    return pos, f


def ground_plane(nx: int, nz: int, y: float = -1.3, span: float = 9.0, center_z: float = -6.0,
                 jitter: float = 1e-3, rng: np.random.Generator | None = None):
    """nx*nz quad grid (2 tris per cell) on y = const facing +y, xz jittered."""
    xs = np.linspace(-span, span, nx + 1)
    zs = np.linspace(center_z - span, center_z + span, nz + 1)
    gx, gz = np.meshgrid(xs, zs, indexing="xy")  # (nz+1, nx+1)
    px = gx.reshape(-1).copy()
    pz = gz.reshape(-1).copy()
    if jitter and rng is not None:
        px += rng.uniform(-jitter, jitter, size=px.shape)
        pz += rng.uniform(-jitter, jitter, size=pz.shape)
    pos = np.column_stack([px, np.full(px.shape, float(y)), pz])
    row = nx + 1
    j, i = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
    v00 = (j * row + i).reshape(-1)
    v10 = v00 + 1
    v01 = v00 + row
    v11 = v01 + 1
    # +y normal: (b-a) x (c-a) must point up; z grows along rows
    t1 = np.stack([v00, v01, v10], 1)
    t2 = np.stack([v10, v01, v11], 1)
    tris = np.empty((2 * len(v00), 3), dtype=np.int64)
    tris[0::2] = t1
    tris[1::2] = t2
    return pos, tris


def sphere_field(level: int, seed: int = 11):
    """8x6 grid of jittered icospheres."""
    rng = np.random.default_rng(seed)
    unit_pos, unit_tris = icosphere(level)
    positions, triangles = [], []
    base = 0
    for gz in range(6):
        for gx in range(8):
            cx = -5.6 + 1.6 * gx + rng.uniform(-0.2, 0.2)
            cy = -0.6 + rng.uniform(-0.3, 0.3)
            cz = -4.0 - 1.6 * gz
            r = 0.55 + rng.uniform(-0.1, 0.1)
            positions.append(unit_pos * r + np.array([cx, cy, cz]))
            triangles.append(unit_tris + base)
            base += len(unit_pos)
    return np.vstack(positions), np.vstack(triangles), rng


def _merge(*parts):
    positions, triangles, base = [], [], 0
    for pos, tris in parts:
        positions.append(pos)
        triangles.append(tris + base)
        base += len(pos)
    return np.vstack(positions), np.vstack(triangles)


@dataclass(frozen=True)
class CameraPose:
    position: tuple
    look_at: tuple = (0.0, -0.2, -6.0)
    up: tuple = (0.0, 1.0, 0.0)
    fov_y_deg: float = 60.0
    near: float = 0.1
    far: float = 1000.0


@dataclass
class SceneSpec:
    name: str
    positions: np.ndarray
    triangles: np.ndarray
    screen: tuple
    omega: int
    prescale: float = 1.0
    n_scales: int = 64
    min_dim: int = 1
    padding: int = 0
    backface_cull: bool = True
    poses: list = field(default_factory=list)

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)


DEFAULT_POSE = CameraPose(position=(0.0, 1.0, 0.0))


def scene_c1() -> SceneSpec:
    rng = np.random.default_rng(11)
    sphere = icosphere(4, center=(0.2, 0.3, -6.0), radius=1.5)
    plane = ground_plane(75, 100, rng=rng)
    pos, tris = _merge(sphere, plane)
    return SceneSpec("C1", pos, tris, (512, 512), 1024, poses=[DEFAULT_POSE])


def _field_scene(name, level, nx, nz, screen, omega, prescale):
    fpos, ftris, rng = sphere_field(level)
    plane = ground_plane(nx, nz, rng=rng)
    pos, tris = _merge((fpos, ftris), plane)
    return SceneSpec(name, pos, tris, screen, omega, prescale=prescale, poses=[DEFAULT_POSE])


def scene_c2() -> SceneSpec:
    return _field_scene("C2", 5, 100, 85, (1920, 1080), 2048, 1.0)


def scene_c3() -> SceneSpec:
    return _field_scene("C3", 6, 250, 136, (3840, 2160), 4096, 2.0)


def camera_path_c4(n_frames: int = 120) -> list:
    poses = []
    for f in range(n_frames):
        th = (math.pi / 2.0) * f / max(1, n_frames - 1)
        poses.append(CameraPose(position=(6.0 * math.sin(th), 1.0, -6.0 + 6.0 * math.cos(th))))
    return poses


def views_c5(n_views: int = 64) -> list:
    rng = np.random.default_rng(20240811)
    poses = []
    for k in range(n_views):
        th = (k * 2.399963229728653) % (2.0 * math.pi)
        dy = float(rng.uniform(-0.3, 0.3))
        poses.append(CameraPose(position=(6.0 * math.sin(th), 1.0 + dy, -6.0 + 6.0 * math.cos(th))))
    return poses


CONFIGS = {"C1": scene_c1, "C2": scene_c2, "C3": scene_c3}


def build_scene(name: str) -> SceneSpec:
    if name in CONFIGS:
        return CONFIGS[name]()
    if name == "C4":
        s = scene_c2()
        s.name, s.poses = "C4", camera_path_c4()
        return s
    if name == "C5":
        s = scene_c2()
        s.name, s.poses = "C5", views_c5()
        return s
    raise ValueError(f"unknown scene config {name!r}")
