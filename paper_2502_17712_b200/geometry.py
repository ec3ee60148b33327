"""Drop-in mirror of atlaspack.geometry (geometry.py:1-362).

Camera construction (A1 in SURVEY §8a) stays on the host exactly as the
reference computes it — it is 16 doubles per frame.  Everything the
per-frame path computes per triangle / per chart (blinn_clamped_ndc,
select_side_plane, chart_bbox, viewport_box) runs in the CUDA library
(paper_2502_17712_b200/csrc/fa_bounds.cu).  `project_vertex`,
`project_points`, `clip_near` and `conservative_blinn_box` are standalone
helpers that the per-frame pipeline never calls (SURVEY §2.1 marks them out
of scope); they are kept here as thin host functions for API completeness.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import NamedTuple, Sequence

import numpy as np

from . import _native as nat

W_EPSILON = 1e-9  # geometry.py:19
SIDE_PLANES = ("left", "right", "bottom", "top")  # geometry.py:21


class GeometryError(Exception):
    pass


class AllClipped(GeometryError):
    """No vertex of the triangle passes the near half-space test."""


class DegenerateChart(GeometryError):
    """No triangle of the chart survives clipping."""


class HPoint(NamedTuple):
    x: float
    y: float
    z: float
    w: float


@dataclass
class CameraFrame:
    """Perspective camera (geometry.py:45-92)."""

    fov_y: float
    aspect: float
    near: float
    far: float
    view: np.ndarray = field(repr=False)
    proj: np.ndarray = field(repr=False)

    def __post_init__(self):
        if not (self.near > 0 and self.far > self.near):
            raise ValueError("camera requires 0 < near < far")
        self.view = np.asarray(self.view, dtype=np.float64).reshape(4, 4)
        self.proj = np.asarray(self.proj, dtype=np.float64).reshape(4, 4)

    @classmethod
    def from_params(cls, fov_y: float, aspect: float, near: float, far: float,
                    position: Sequence[float] = (0.0, 0.0, 0.0), look_at: Sequence[float] = (0.0, 0.0, -1.0),
                    up: Sequence[float] = (0.0, 1.0, 0.0)) -> "CameraFrame":
        if not (0 < fov_y < math.pi):
            raise ValueError("fov_y must be in (0, pi)")
        if aspect <= 0:
            raise ValueError("aspect must be positive")
        view = look_at_matrix(position, look_at, up)
        proj = perspective_matrix(fov_y, aspect, near, far)
        return cls(fov_y=fov_y, aspect=aspect, near=near, far=far, view=view, proj=proj)

    @property
    def view_proj(self) -> np.ndarray:
        return self.proj @ self.view


class RawCamera:
    """A camera given directly by its 4x4 view_proj (e.g. from golden vectors)."""

    def __init__(self, view_proj):
        self._vp = np.ascontiguousarray(np.asarray(view_proj, dtype=np.float64).reshape(4, 4))

    @property
    def view_proj(self) -> np.ndarray:
        return self._vp


def perspective_matrix(fov_y: float, aspect: float, near: float, far: float) -> np.ndarray:
    """geometry.py:95-103."""
    f = 1.0 / math.tan(fov_y / 2.0)
    m = np.zeros((4, 4), dtype=np.float64)
    m[0, 0] = f / aspect
    m[1, 1] = f
    m[2, 2] = (far + near) / (near - far)
    m[2, 3] = 2.0 * far * near / (near - far)
    m[3, 2] = -1.0
    return m


def look_at_matrix(position, target, up) -> np.ndarray:
    """geometry.py:106-124."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - pos
    n = np.linalg.norm(fwd)
    if n == 0:
        raise ValueError("look_at target coincides with position")
    fwd = fwd / n
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    n = np.linalg.norm(right)
    if n == 0:
        raise ValueError("up vector is parallel to the view direction")
    right = right / n
    true_up = np.cross(right, fwd)
    m = np.eye(4, dtype=np.float64)
    m[0, :3] = right
    m[1, :3] = true_up
    m[2, :3] = -fwd
    m[:3, 3] = m[:3, :3] @ (-pos)
    return m


@dataclass(frozen=True)
class NdcBox:
    """geometry.py:127-150."""

    min_x: float
    min_y: float
    max_x: float
    max_y: float

    def __post_init__(self):
        if self.min_x > self.max_x or self.min_y > self.max_y:
            raise ValueError("NdcBox requires min <= max componentwise")

    @property
    def area(self) -> float:
        return (self.max_x - self.min_x) * (self.max_y - self.min_y)

    def contains(self, other: "NdcBox", tol: float = 0.0) -> bool:
        return (self.min_x <= other.min_x + tol and self.min_y <= other.min_y + tol
                and self.max_x >= other.max_x - tol and self.max_y >= other.max_y - tol)


@dataclass(frozen=True)
class ClipPolygon:
    """geometry.py:153-166."""

    vertices: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.vertices, dtype=np.float64)
        if v.ndim != 2 or v.shape[1] != 4 or v.shape[0] not in (3, 4):
            raise ValueError("ClipPolygon holds 3 or 4 homogeneous vertices")
        object.__setattr__(self, "vertices", v)

    def __len__(self) -> int:
        return self.vertices.shape[0]


# ---------------------------------------------------------------------------
# per-frame path functions: CUDA
# ---------------------------------------------------------------------------

def _dev(a, dtype, device):
    torch = nat._torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=dtype)).to(device)


def blinn_clamped_ndc(p) -> tuple[float, float]:
    """geometry.py:185-200 (computed by the fa_blinn_clamped_ndc kernel)."""
    out = blinn_clamped_ndc_batch(np.asarray([float(v) for v in p], dtype=np.float64).reshape(1, 4))
    return float(out[0, 0]), float(out[0, 1])


def blinn_clamped_ndc_batch(points) -> np.ndarray:
    """Batched geometry.py:185-200 over (n, 4) clip points -> (n, 2)."""
    ctx = nat.default_context()
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 4)
    if len(pts) == 0:
        return np.zeros((0, 2))
    d_in = _dev(pts, np.float64, ctx.torch_device)
    d_out = nat._torch().empty((len(pts), 2), dtype=nat._torch().float64, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_blinn_clamped_ndc(ctx.h, nat.ptr(d_in), len(pts), nat.ptr(d_out),
                                                    ctx.stream_ptr()))
    return d_out.cpu().numpy()


def select_side_plane(tri) -> str | None:
    """geometry.py:257-278 (fa_select_side_plane kernel)."""
    v = np.asarray(tri, dtype=np.float64).reshape(1, 3, 4)
    idx = select_side_plane_batch(v)[0]
    return None if idx < 0 else SIDE_PLANES[idx]


def select_side_plane_batch(tris) -> np.ndarray:
    ctx = nat.default_context()
    t = np.ascontiguousarray(tris, dtype=np.float64).reshape(-1, 3, 4)
    if len(t) == 0:
        return np.zeros(0, dtype=np.int32)
    d_in = _dev(t, np.float64, ctx.torch_device)
    d_out = nat._torch().empty(len(t), dtype=nat._torch().int32, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_select_side_plane(ctx.h, nat.ptr(d_in), len(t), nat.ptr(d_out), ctx.stream_ptr()))
    return d_out.cpu().numpy()


def chart_bbox(triangles, cam) -> NdcBox:
    """geometry.py:281-322 (fa_chart_bbox kernel); raises DegenerateChart."""
    tris = np.ascontiguousarray(triangles, dtype=np.float64).reshape(-1, 3, 3)
    if tris.shape[0] == 0:
        raise DegenerateChart("chart has no triangles")
    ctx = nat.default_context()
    d_in = _dev(tris, np.float64, ctx.torch_device)
    vp = nat.vp_host(cam.view_proj)
    box = np.zeros(4)
    nat.raise_for_status(ctx.L.fa_chart_bbox(ctx.h, vp.ctypes.data_as(ctypes.c_void_p), nat.ptr(d_in), len(tris),
                                             box.ctypes.data_as(ctypes.c_void_p), ctx.stream_ptr()))
    return NdcBox(float(box[0]), float(box[1]), float(box[2]), float(box[3]))


def viewport_box(box: NdcBox, screen_w: int, screen_h: int) -> tuple[int, int]:
    """geometry.py:352-362 (fa_viewport_box kernel)."""
    if screen_w < 1 or screen_h < 1:
        raise ValueError("screen dimensions must be >= 1")
    out = viewport_box_batch(np.array([[box.min_x, box.min_y, box.max_x, box.max_y]]), screen_w, screen_h)
    return int(out[0, 0]), int(out[0, 1])


def viewport_box_batch(boxes, screen_w: int, screen_h: int) -> np.ndarray:
    ctx = nat.default_context()
    b = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 4)
    if len(b) == 0:
        return np.zeros((0, 2), dtype=np.int64)
    d_in = _dev(b, np.float64, ctx.torch_device)
    d_out = nat._torch().empty((len(b), 2), dtype=nat._torch().int64, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_viewport_box(ctx.h, nat.ptr(d_in), len(b), int(screen_w), int(screen_h),
                                               nat.ptr(d_out), ctx.stream_ptr()))
    return d_out.cpu().numpy()


# ---------------------------------------------------------------------------
# standalone helpers outside the per-frame path (host; SURVEY §2.1 out of scope)
# ---------------------------------------------------------------------------
# The reference's scalar host helpers, kept for API completeness.  They are
# not on the per-frame path (the frame projects and clips on the GPU:
# k_frame_init, tri_setup_warp); their arithmetic is the reference's own
# (numpy matmul for the projection, so the same OpenBLAS bits).

def project_points(points: np.ndarray, cam: CameraFrame) -> np.ndarray:
    """geometry.py:178-182: (n,3) points -> (n,4) clip coordinates."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    homo = np.concatenate([pts, np.ones((len(pts), 1))], axis=1)
    return homo @ cam.view_proj.T


def project_vertex(p: Sequence[float], cam: CameraFrame) -> HPoint:
    """geometry.py:169-175: one finite 3D point -> HPoint."""
    q = np.asarray(p, dtype=np.float64)
    if q.shape != (3,) or not np.isfinite(q).all():
        raise ValueError("expected a finite 3D point")
    x, y, z, w = cam.view_proj @ np.append(q, 1.0)
    return HPoint(x, y, z, w)


def clip_near(tri) -> ClipPolygon:
    """geometry.py:223-236: clip a clip-space triangle to w > W_EPSILON
    (strict, unlike the frustum clip of charts.py:178-189, which keeps d >= 0)."""
    v = np.asarray(tri, dtype=np.float64).reshape(3, 4)
    d = v[:, 3] - W_EPSILON
    inside = d > 0
    if inside.all():
        return ClipPolygon(v)
    if not inside.any():
        raise AllClipped("triangle lies entirely behind the camera")
    poly = []
    for i in range(3):
        j = (i + 1) % 3
        if inside[i]:
            poly.append(v[i])
        if inside[i] != inside[j]:  # the edge crosses the plane
            t = d[i] / (d[i] - d[j])
            poly.append(v[i] + t * (v[j] - v[i]))
    return ClipPolygon(np.array(poly, dtype=np.float64).reshape(-1, 4))


def conservative_blinn_box(triangles, cam: CameraFrame) -> NdcBox:
    """geometry.py:325-349 (clamp-only test baseline, not used by the pipeline)."""
    tris = np.asarray(triangles, dtype=np.float64).reshape(-1, 3, 3)
    if len(tris) == 0:
        raise DegenerateChart("chart has no triangles")
    clip = np.concatenate([tris, np.ones((len(tris), 3, 1))], axis=2) @ cam.view_proj.T
    pts = clip.reshape(-1, 4)
    if np.any(pts[:, 3] <= W_EPSILON):
        return NdcBox(-1.0, -1.0, 1.0, 1.0)
    nd = blinn_clamped_ndc_batch(pts)
    return NdcBox(float(nd[:, 0].min()), float(nd[:, 1].min()), float(nd[:, 0].max()), float(nd[:, 1].max()))
