"""Drop-in mirror of atlaspack.charts (charts.py:1-406).

depth_prepass / mark_visible / connected_charts / merge_shared_vertices run
in the CUDA library (csrc/fa_raster.cu, csrc/fa_charts.cu).  Meshes keep
their numpy arrays (the reference's value semantics) plus a cached device
copy (float64 positions, int32 triangles) so repeated frames never re-upload.

`load_obj` (host file ingestion) and the edge adjacency used by the
standalone `connected_charts` are per-mesh, not per-frame (SURVEY §3.1 step
2, §8f-3); adjacency is built lazily on first use with a vectorised sort.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _native as nat
from .geometry import CameraFrame, W_EPSILON  # noqa: F401  (re-exported like the reference)

DEPTH_EPSILON = 1e-6  # charts.py:26


def _device_adjacency(tris_dev, ctx):
    """charts.py:64-77 on the GPU (fa_build_adjacency: edge hash table)."""
    torch = nat._torch()
    T = tris_dev.shape[0]
    adj = torch.empty((max(T, 1), 3), dtype=torch.int32, device=ctx.torch_device)
    if T:
        nat.raise_for_status(ctx.L.fa_build_adjacency(ctx.h, nat.ptr(adj), ctx.stream_ptr()))
    return adj[:T]


def build_adjacency(triangles: np.ndarray) -> np.ndarray:
    """charts.py:64-77: link edges used by exactly two (triangle, edge) slots (GPU)."""
    tris = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
    if len(tris) == 0:
        return np.full((0, 3), -1, dtype=np.int64)
    n = int(tris.max()) + 1
    return Mesh(np.zeros((n, 3)), tris).adjacency


class Mesh:
    """Indexed triangle soup (charts.py:29-61) with a cached device copy."""

    def __init__(self, positions, triangles, adjacency=None):
        self.positions = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        self.triangles = np.asarray(triangles, dtype=np.int64).reshape(-1, 3)
        if self.triangles.size and (self.triangles.min() < 0 or self.triangles.max() >= len(self.positions)):
            raise ValueError("triangle indices out of range")
        self._adjacency = None if adjacency is None else np.asarray(adjacency, dtype=np.int64).reshape(-1, 3)
        self._dev = {}

    @property
    def adjacency(self) -> np.ndarray:
        """Edge adjacency (charts.py:64-77), built once per mesh on the GPU."""
        if self._adjacency is None:
            ctx = nat.default_context()
            self._adjacency = self.device_adjacency(ctx.torch_device).cpu().numpy().astype(np.int64)
        return self._adjacency

    @adjacency.setter
    def adjacency(self, value):
        self._adjacency = np.asarray(value, dtype=np.int64).reshape(-1, 3)
        self._dev = {k: v for k, v in self._dev.items() if k[0] != "adj"}

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)

    @property
    def n_vertices(self) -> int:
        return len(self.positions)

    def triangle_corners(self, indices=None) -> np.ndarray:
        tris = self.triangles if indices is None else self.triangles[indices]
        return self.positions[tris]

    # -- device residency -------------------------------------------------
    def device_arrays(self, device):
        """(positions float64 (V,3), triangles int32 (T,3)) on `device`, uploaded once."""
        torch = nat._torch()
        key = ("mesh", str(device), id(self.positions), id(self.triangles))
        got = self._dev.get(key)
        if got is None:
            self._dev = {k: v for k, v in self._dev.items() if k[0] != "mesh"}
            pos = torch.as_tensor(np.ascontiguousarray(self.positions)).to(device)
            tris = torch.as_tensor(np.ascontiguousarray(self.triangles, dtype=np.int32)).to(device)
            got = (pos, tris)
            self._dev[key] = got
        return got

    def device_adjacency(self, device):
        torch = nat._torch()
        key = ("adj", str(device))
        got = self._dev.get(key)
        if got is None:
            if self._adjacency is not None:  # caller-supplied adjacency (Mesh(adjacency=...))
                got = torch.as_tensor(np.ascontiguousarray(self._adjacency, dtype=np.int32)).to(device)
            else:
                ctx = nat.default_context(torch.device(device).index)
                pos, tris = self.device_arrays(device)
                ctx.set_mesh(pos, tris)
                got = _device_adjacency(tris, ctx)
            self._dev[key] = got
        return got


def _obj_vertex_index(token: str, n_vertices: int) -> int:
    """An OBJ face token ('i', 'i/t', 'i/t/n') as a 0-based vertex index;
    negative indices count back from the vertices read so far."""
    i = int(token.split("/", 1)[0])
    return i - 1 if i > 0 else n_vertices + i


def load_obj(path) -> Mesh:
    """charts.py:80-110 restated (host file ingestion, outside the per-frame
    path): 'v x y z' and 'f ...' records, '#' comments, polygons
    fan-triangulated around their first vertex; the reference's error
    messages for short records."""
    verts: list[tuple[float, float, float]] = []
    tris: list[tuple[int, int, int]] = []
    with open(path, "r", encoding="utf-8", errors="replace") as fh:
        for lineno, raw in enumerate(fh, start=1):
            tok = raw.partition("#")[0].split()
            if not tok:
                continue
            kind, args = tok[0], tok[1:]
            if kind == "v":
                if len(args) < 3:
                    raise ValueError(f"{path}:{lineno}: vertex needs 3 coordinates")
                verts.append((float(args[0]), float(args[1]), float(args[2])))
            elif kind == "f":
                ids = [_obj_vertex_index(t, len(verts)) for t in args]
                if len(ids) < 3:
                    raise ValueError(f"{path}:{lineno}: face needs >= 3 vertices")
                tris.extend((ids[0], b, c) for b, c in zip(ids[1:-1], ids[2:]))
    return Mesh(positions=np.array(verts, dtype=np.float64).reshape(-1, 3),
                triangles=np.array(tris, dtype=np.int64).reshape(-1, 3))


class VisibilityBuffer:
    """charts.py:113-125."""

    def __init__(self, flags, sample_res):
        self.flags = np.asarray(flags, dtype=bool)
        self.sample_res = tuple(sample_res)

    @property
    def visible_indices(self) -> np.ndarray:
        return np.flatnonzero(self.flags)

    def __eq__(self, other):
        return (isinstance(other, VisibilityBuffer) and np.array_equal(self.flags, other.flags)
                and self.sample_res == other.sample_res)


def _charts_from_labels(labels: np.ndarray) -> dict:
    vis = np.flatnonzero(labels >= 0)
    if len(vis) == 0:
        return {}
    lab = labels[vis]
    order = np.argsort(lab, kind="stable")
    sl = lab[order]
    members = vis[order]
    starts = np.flatnonzero(np.concatenate([[True], sl[1:] != sl[:-1]]))
    ends = np.concatenate([starts[1:], [len(sl)]])
    return {int(sl[s]): members[s:e].astype(np.int64) for s, e in zip(starts, ends)}


class ChartSet:
    """charts.py:128-145, with lazily materialised dict views.

    Constructed either like the reference (chart_of_triangle, charts,
    vertex_to_chart) or from the GPU arrays (labels, vertex array)."""

    def __init__(self, chart_of_triangle, charts=None, vertex_to_chart=None, *, vertex_chart_array=None):
        self.chart_of_triangle = np.asarray(chart_of_triangle, dtype=np.int64)
        self._charts = charts
        self._v2c = vertex_to_chart
        self._v2c_arr = None if vertex_chart_array is None else np.asarray(vertex_chart_array, dtype=np.int64)

    @property
    def charts(self) -> dict:
        if self._charts is None:
            self._charts = _charts_from_labels(self.chart_of_triangle)
        return self._charts

    @charts.setter
    def charts(self, v):
        self._charts = v

    @property
    def vertex_to_chart(self) -> dict:
        if self._v2c is None:
            if self._v2c_arr is None:
                self._v2c = {}
            else:
                idx = np.flatnonzero(self._v2c_arr >= 0)
                self._v2c = dict(zip(idx.tolist(), self._v2c_arr[idx].tolist()))
        return self._v2c

    @vertex_to_chart.setter
    def vertex_to_chart(self, v):
        self._v2c = v

    @property
    def vertex_chart_array(self) -> np.ndarray | None:
        return self._v2c_arr

    @property
    def n_charts(self) -> int:
        if self._charts is not None:
            return len(self._charts)
        lab = self.chart_of_triangle
        return int(np.count_nonzero(lab == np.arange(len(lab))))


# ---------------------------------------------------------------------------
# per-frame path (CUDA)
# ---------------------------------------------------------------------------

def _ctx_and_mesh(mesh: Mesh):
    ctx = nat.default_context()
    pos, tris = mesh.device_arrays(ctx.torch_device)
    ctx.set_mesh(pos, tris)
    return ctx


def depth_prepass(mesh: Mesh, cam: CameraFrame, res, backface_cull: bool = True) -> np.ndarray:
    """charts.py:285-299 -> (H, W) float64, +inf where uncovered."""
    width, height = int(res[0]), int(res[1])
    if width < 1 or height < 1:
        raise ValueError("resolution must be at least 1x1")
    torch = nat.require_device()
    ctx = _ctx_and_mesh(mesh)
    vp = nat.vp_host(cam.view_proj)
    out = torch.empty((height, width), dtype=torch.float64, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_depth_prepass(ctx.h, vp.ctypes.data_as(ctypes.c_void_p), width, height,
                                                int(bool(backface_cull)), nat.ptr(out), ctx.stream_ptr()))
    return out.cpu().numpy()


def mark_visible(mesh: Mesh, cam: CameraFrame, depth: np.ndarray, backface_cull: bool = True) -> VisibilityBuffer:
    """charts.py:302-313."""
    torch = nat.require_device()
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    height, width = depth.shape
    ctx = _ctx_and_mesh(mesh)
    vp = nat.vp_host(cam.view_proj)
    d_depth = torch.as_tensor(depth).to(ctx.torch_device)
    flags = torch.empty(max(mesh.n_triangles, 1), dtype=torch.uint8, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_mark_visible(ctx.h, vp.ctypes.data_as(ctypes.c_void_p), nat.ptr(d_depth), width,
                                               height, int(bool(backface_cull)), nat.ptr(flags), ctx.stream_ptr()))
    return VisibilityBuffer(flags=flags[:mesh.n_triangles].cpu().numpy().astype(bool), sample_res=(width, height))


def connected_charts(mesh: Mesh, vis: VisibilityBuffer) -> ChartSet:
    """charts.py:343-359 (edge-adjacency union-find on the GPU)."""
    flags = np.asarray(vis.flags, dtype=bool)
    if len(flags) != mesh.n_triangles:
        raise ValueError("visibility buffer does not match the mesh")
    torch = nat.require_device()
    ctx = _ctx_and_mesh(mesh)
    adj = mesh.device_adjacency(ctx.torch_device)
    d_flags = torch.as_tensor(flags.astype(np.uint8)).to(ctx.torch_device)
    labels = torch.empty(max(mesh.n_triangles, 1), dtype=torch.int32, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_connected_charts(ctx.h, nat.ptr(adj), nat.ptr(d_flags), nat.ptr(labels),
                                                   ctx.stream_ptr()))
    return ChartSet(labels[:mesh.n_triangles].cpu().numpy().astype(np.int64), vertex_to_chart={})


def merge_shared_vertices(cs: ChartSet, mesh: Mesh) -> ChartSet:
    """charts.py:362-386 (vertex union-find on the GPU)."""
    torch = nat.require_device()
    ctx = _ctx_and_mesh(mesh)
    lab = np.asarray(cs.chart_of_triangle, dtype=np.int64)
    d_in = torch.as_tensor(lab.astype(np.int32)).to(ctx.torch_device)
    out = torch.empty(max(mesh.n_triangles, 1), dtype=torch.int32, device=ctx.torch_device)
    v2c = torch.empty(max(len(mesh.positions), 1), dtype=torch.int32, device=ctx.torch_device)
    nat.raise_for_status(ctx.L.fa_merge_shared_vertices(ctx.h, nat.ptr(d_in), nat.ptr(out), nat.ptr(v2c),
                                                        ctx.stream_ptr()))
    return ChartSet(out[:mesh.n_triangles].cpu().numpy().astype(np.int64),
                    vertex_chart_array=v2c[:len(mesh.positions)].cpu().numpy().astype(np.int64))


__all__ = ["DEPTH_EPSILON", "Mesh", "build_adjacency", "load_obj", "VisibilityBuffer", "ChartSet", "depth_prepass",
           "mark_visible", "connected_charts", "merge_shared_vertices"]
