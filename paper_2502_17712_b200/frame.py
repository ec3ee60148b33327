"""Resident per-frame atlas engine: run_scene_pipeline (cli.py:360-406) as
one CUDA-graph replay per frame.

A `FrameEngine` binds one mesh to one device context.  Each frame uploads
only the 4x4 camera matrix, replays the captured kernel graph
(project -> depth pass -> visibility pass -> visible compaction ->
union-find charts -> per-chart bounds -> box dims -> radix order ->
64-candidate pack -> selection -> UVs) and exposes the outputs as zero-copy
device tensors.  Reference-typed objects (ChartSet dicts, Placement tuples,
NdcBox dicts) are materialised lazily, outside any timed region.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native as nat
from .charts import ChartSet, Mesh
from .geometry import NdcBox
from .packing import AtlasLayout, ChartBox, placements_from_array


@dataclass
class FrameSettings:
    screen: tuple = (1920, 1080)
    omega: int = 2048
    n_scales: int = 64
    min_dim: int = 1
    padding: int = 0
    prescale: float = 1.0
    backface_cull: bool = True
    uv_f64: bool = False
    want_depth: bool = False
    use_graph: bool = True
    profile: bool = False
    packer: str = "fastatlas"   # make_packer name (cli.py:318-339); the comparison packers run ungraphed
    block_size: int = 0         # superblock block size, 0 = default_block_size(omega)

    def params(self) -> nat.FrameParams:
        p = nat.FrameParams()
        p.width, p.height = int(self.screen[0]), int(self.screen[1])
        p.omega, p.n_scales = int(self.omega), int(self.n_scales)
        p.min_dim, p.padding = int(self.min_dim), int(self.padding)
        p.prescale = float(self.prescale)
        p.backface_cull = int(bool(self.backface_cull))
        p.uv_f64 = int(bool(self.uv_f64))
        p.want_depth = int(bool(self.want_depth))
        p.use_graph = int(bool(self.use_graph))
        p.profile = int(bool(self.profile))
        p.packer = nat.PACKER_CODES.get(self.packer, -1)  # unknown: ValueError after the NothingVisible check
        p.block_size = int(self.block_size)
        return p


class FrameOutput:
    """Device views of one frame's results (valid until the engine's next frame)."""

    def __init__(self, res: nat.FrameResult, settings: FrameSettings, T: int, V: int, device, owner=None):
        self._owner = owner  # keeps the context (and its buffers) alive while the views exist
        self.status = int(res.status)
        self.n_visible = int(res.n_visible)
        self.n_charts = int(res.n_charts)
        self.scale = Fraction(int(res.scale_num), int(res.scale_den)) if res.scale_den else None
        self.screen_fragments = int(res.screen_fragments)
        self.texels_allocated = int(res.texels_allocated)
        self.stretch_l2 = float(res.stretch_l2)
        self.stretch_linf = float(res.stretch_linf)
        self.stretch_count = int(res.stretch_count)
        self.settings = settings
        C, nv = self.n_charts, self.n_visible
        W, H = settings.screen
        v = nat.device_view
        self.flags = v(res.flags, (T,), np.uint8, device)
        self.visible = v(res.visible, (nv,), np.int32, device)
        self.chart_of_triangle = v(res.chart_of_triangle, (T,), np.int32, device)
        self.vertex_to_chart = v(res.vertex_to_chart, (V,), np.int32, device)
        self.roots = v(res.roots, (C,), np.int32, device)
        self.ndc = v(res.ndc, (C, 4), np.float64, device)
        self.px = v(res.px, (C, 2), np.int32, device)
        self.target = v(res.target, (C, 2), np.int64, device)
        self.placements = v(res.placements, (C, 8), np.int64, device)
        self.uv = v(res.uv, (nv, 6), np.float64 if settings.uv_f64 else np.float32, device)
        self.depth = v(res.depth, (H, W), np.float64, device) if settings.want_depth and res.depth else None

    # tensors that a caller may want to keep past the next frame
    TENSORS = ("flags", "visible", "chart_of_triangle", "vertex_to_chart", "roots", "ndc", "px", "target",
               "placements", "uv", "depth")

    def clone(self) -> "FrameOutput":
        out = object.__new__(FrameOutput)
        out.__dict__.update(self.__dict__)
        for k in self.TENSORS:
            t = getattr(self, k)
            setattr(out, k, None if t is None else t.clone())
        return out

    def to_host(self) -> dict:
        d = {k: (None if getattr(self, k) is None else getattr(self, k).cpu().numpy()) for k in self.TENSORS}
        d.update(status=self.status, n_visible=self.n_visible, n_charts=self.n_charts, scale=self.scale,
                 screen_fragments=self.screen_fragments, texels_allocated=self.texels_allocated)
        return d

    # -- reference-typed views (materialised on demand) --------------------
    def chart_set(self) -> ChartSet:
        return ChartSet(self.chart_of_triangle.cpu().numpy().astype(np.int64),
                        vertex_chart_array=self.vertex_to_chart.cpu().numpy().astype(np.int64))

    def boxes(self) -> list:
        r = self.roots.cpu().numpy()
        t = self.target.cpu().numpy()
        return [ChartBox(target_w=int(t[i, 0]), target_h=int(t[i, 1]), chart_id=int(r[i]), min_tri=int(r[i]))
                for i in range(len(r))]

    def layout(self) -> AtlasLayout:
        return AtlasLayout(omega=int(self.settings.omega), scale=self.scale,
                           placements=placements_from_array(self.placements.cpu().numpy()))

    def stretch(self):
        """StretchReport of the frame (computed on the GPU in the UV kernel), None if no valid pair."""
        from .metrics import StretchReport
        if self.stretch_count == 0:
            return None
        return StretchReport(l2=self.stretch_l2, linf=self.stretch_linf)

    def chart_ndc(self) -> dict:
        r = self.roots.cpu().numpy()
        b = self.ndc.cpu().numpy()
        return {int(r[i]): NdcBox(*map(float, b[i])) for i in range(len(r))}

    def chart_px(self) -> dict:
        r = self.roots.cpu().numpy()
        p = self.px.cpu().numpy()
        return {int(r[i]): (int(p[i, 0]), int(p[i, 1])) for i in range(len(r))}


class FrameEngine:
    """One mesh resident on one GPU; `run(camera)` produces one atlas."""

    def __init__(self, mesh: Mesh, device: int | None = None, settings: FrameSettings | None = None,
                 private_mesh: bool = False):
        torch = nat.require_device()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.ctx = nat.Context(self.device)  # private context: outputs survive other API calls
        self.mesh = mesh
        self.pos, self.tris = mesh.device_arrays(self.ctx.torch_device)
        if private_mesh:  # own device copy (e.g. one replica per pipeline slot)
            self.pos, self.tris = self.pos.clone(), self.tris.clone()
        self.ctx.set_mesh(self.pos, self.tris)
        self.settings = settings or FrameSettings()
        self._res = nat.FrameResult()

    @property
    def n_triangles(self) -> int:
        return self.mesh.n_triangles

    def launch(self, view_proj, settings: FrameSettings | None = None, stream=None) -> None:
        """Enqueue one frame (asynchronous)."""
        s = settings or self.settings
        self._last_settings = s
        vp = nat.vp_host(view_proj)
        self._params = s.params()
        st = ctypes.c_void_p(stream.cuda_stream) if stream is not None else self.ctx.stream_ptr()
        self._stream = st
        self.ctx.set_mesh(self.pos, self.tris)
        nat.raise_for_status(self.ctx.L.fa_frame_launch(self.ctx.h, vp.ctypes.data_as(ctypes.c_void_p),
                                                        ctypes.byref(self._params), st))

    def finish(self, check: bool = True) -> FrameOutput:
        """Wait for the launched frame; raise the reference exception on failure."""
        code = self.ctx.L.fa_frame_finish(self.ctx.h, ctypes.byref(self._res), self._stream)
        if check:
            nat.raise_for_status(code)
        return FrameOutput(self._res, self._last_settings, self.mesh.n_triangles, len(self.mesh.positions),
                           self.ctx.torch_device, owner=self)

    def run(self, view_proj, settings: FrameSettings | None = None, stream=None, check: bool = True) -> FrameOutput:
        for _ in range(4):
            self.launch(view_proj, settings, stream)
            code = self.ctx.L.fa_frame_finish(self.ctx.h, ctypes.byref(self._res), self._stream)
            if code == nat.FA_INTERNAL_ERROR and "rerun" in nat.last_error():
                continue
            if check:
                nat.raise_for_status(code)
            return FrameOutput(self._res, self._last_settings, self.mesh.n_triangles, len(self.mesh.positions),
                               self.ctx.torch_device, owner=self)
        raise RuntimeError("frame work queues kept overflowing")

    def run_views(self, views, settings: FrameSettings | None = None, stream=None) -> list:
        """Sequential convenience: one cloned FrameOutput per view."""
        return [self.run(v, settings, stream).clone() for v in views]

    def launch_count(self) -> int:
        return int(self.ctx.L.fa_last_launch_count(self.ctx.h))

    COUNTERS = ("small_records", "large_records", "clipped", "generic_setups", "tiles", "visible", "charts",
                "screen_fragments", "live_clusters")

    def counters(self) -> dict:
        """Work-queue counters of the last finished frame (fa_frame_counters)."""
        buf = (ctypes.c_int64 * 9)()
        n = self.ctx.L.fa_frame_counters(self.ctx.h, buf, 9)
        return {self.COUNTERS[i]: int(buf[i]) for i in range(n)}

    def stage_times(self) -> dict:
        """{stage name: ms} of the last frame run with settings.profile=True."""
        buf = (ctypes.c_float * 16)()
        n = self.ctx.L.fa_stage_times(self.ctx.h, buf, 16, self._stream)
        return {self.ctx.L.fa_stage_name(i).decode(): float(buf[i]) for i in range(n)}


class HostFrame:
    """One pipelined view's results in pinned host memory.

    The arrays are views into a pipeline slot and are overwritten once the
    slot is reused (`depth` views later): `on_frame` consumers that keep them
    must copy.  `error` holds the reference exception (NothingVisible,
    PackFailure, ...) when the frame failed; the arrays are then None.

    Chart ids arrive sparse by default (`visible_chart`: the chart of each
    visible triangle; every other triangle's chart is -1, charts.py:136-141);
    `chart_of_triangle` rebuilds the dense (T,) int32 array on first access
    (or is the downloaded dense array when the pipeline asked for it).

    UVs arrive per visible vertex by default (`visible_vertices`,
    `vertex_uv`: float32 pairs, NaN at/behind the camera plane): a vertex's
    UV depends on the vertex and its chart only (cli.py:436-449), so `uv`
    rebuilds the (n_visible, 6) float32 rows on first access -- NaN rows
    where any corner is NaN -- bit-identical to the frame's float32 rows (or
    is the downloaded rows when the pipeline asked for "uv")."""

    __slots__ = ("index", "status", "error", "n_visible", "n_charts", "scale", "screen_fragments",
                 "texels_allocated", "_cot", "_T", "_visible", "_visible_chart", "_uv", "_uv_copied", "placements",
                 "_visible_vertices", "vertex_uv", "_tris", "_V", "_packed")

    def __init__(self, index: int, n_triangles: int = 0, triangles=None, n_vertices: int = 0):
        self.index = index
        self.status = 0
        self.error = None
        self.n_visible = self.n_charts = 0
        self.scale = None
        self.screen_fragments = self.texels_allocated = 0
        self._cot = self._visible = self._visible_chart = self._uv = self.placements = None
        self._visible_vertices = self.vertex_uv = None
        self._uv_copied = False
        self._T = n_triangles
        self._tris = triangles
        self._V = n_vertices
        # packed wire format (fa_frame_download_packed): (visible bit mask,
        # 16-bit chart index per visible triangle, chart ids, vertex bit mask,
        # vertex order); the lists below are decoded from it on first access
        self._packed = None

    @property
    def visible(self):
        if self._visible is None and self._packed is not None:
            m = self._packed[0]
            self._visible = np.flatnonzero(np.unpackbits(m.view(np.uint8), bitorder="little",
                                                         count=self._T)).astype(np.int32)
        return self._visible

    @visible.setter
    def visible(self, v):
        self._visible = v

    @property
    def visible_chart(self):
        if self._visible_chart is None and self._packed is not None:
            self._visible_chart = self._packed[2][self._packed[1]].astype(np.int32)
        return self._visible_chart

    @visible_chart.setter
    def visible_chart(self, v):
        self._visible_chart = v

    @property
    def visible_vertices(self):
        if self._visible_vertices is None and self._packed is not None:
            bits = np.unpackbits(self._packed[3].view(np.uint8), bitorder="little", count=self._V)
            self._visible_vertices = self._packed[4][np.flatnonzero(bits)]
        return self._visible_vertices

    @visible_vertices.setter
    def visible_vertices(self, v):
        self._visible_vertices = v

    @property
    def uv(self):
        if self._uv is None and self.vertex_uv is not None and self.visible is not None:
            full = np.full((self._V, 2), np.nan, dtype=np.float32)
            full[self.visible_vertices] = self.vertex_uv
            rows = full[self._tris[self.visible]].reshape(-1, 6)
            rows[np.isnan(rows).any(axis=1)] = np.nan
            self._uv = rows
        return self._uv

    @property
    def chart_of_triangle(self):
        if self._cot is None and self.visible is not None and self.visible_chart is not None:
            cot = np.full(self._T, -1, dtype=np.int32)
            cot[self.visible] = self.visible_chart
            self._cot = cot
        return self._cot

    def d2h_bytes(self) -> int:
        """Bytes copied device -> host for this view (a rebuilt dense chart
        array is host work, not a copy)."""
        if self._packed is not None:
            arrs = self._packed[:4] + (self.vertex_uv, self.placements)
        else:
            arrs = (self._visible, self._visible_chart, self._uv if self._uv_copied else None, self.placements,
                    self._visible_vertices, self.vertex_uv)
        n = sum(a.nbytes for a in arrs if a is not None)
        if self._cot is not None and self.visible_chart is None:
            n += self._cot.nbytes
        return n


class FramePipeline:
    """Independent views (streaming clients, camera paths) through `depth`
    resident FrameEngines, each replaying its frame graph on its own CUDA
    stream.  While one slot's frame computes, the others' kernels fill the
    SMs its latency-bound stages leave idle and the copy engines return the
    finished frames' chart ids, visible list, UVs and placements to pinned
    host memory.  Results are delivered in view order through
    `on_frame(HostFrame)`.  With the default compact outputs the copies use
    the packed wire format (fa_frame_download_packed: visibility and vertex
    bit masks, 16-bit chart indices; about half the bytes), decoded into the
    same HostFrame lists on first access; packed=False copies the int32
    lists."""

    def __init__(self, mesh: Mesh, device: int | None = None, settings: FrameSettings | None = None,
                 depth: int = 4, outputs: tuple = ("visible", "visible_chart", "vertex_uv", "placements"),
                 mesh_replicas: bool = False, packed: bool = True):
        torch = nat.require_device()
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.settings = settings or FrameSettings()
        self.engines = [FrameEngine(mesh, device, self.settings, private_mesh=mesh_replicas) for _ in range(depth)]
        self.device = self.engines[0].device
        self.streams = [torch.cuda.Stream(device=self.device) for _ in range(depth)]
        self._cstreams = [torch.cuda.Stream(device=self.device) for _ in range(depth)]  # D2H copies
        self.outputs = tuple(outputs)
        T = mesh.n_triangles
        uv_dt = torch.float64 if self.settings.uv_f64 else torch.float32
        self._host = []
        for _ in range(depth):
            h = {}
            if "chart_of_triangle" in outputs:
                h["chart_of_triangle"] = torch.empty(T, dtype=torch.int32).pin_memory()
            if "visible" in outputs or "visible_chart" in outputs:
                h["visible"] = torch.empty(T, dtype=torch.int32).pin_memory()
            if "visible_chart" in outputs:
                h["visible_chart"] = torch.empty(T, dtype=torch.int32).pin_memory()
            if "uv" in outputs or ("vertex_uv" in outputs and self.settings.uv_f64):
                # (float64 UVs have no compact form: the rows are downloaded)
                h["uv"] = torch.empty((T, 6), dtype=uv_dt).pin_memory()
            elif "vertex_uv" in outputs:
                h["visible_vertices"] = torch.empty(mesh.n_vertices, dtype=torch.int32).pin_memory()
                h["vertex_uv"] = torch.empty((mesh.n_vertices, 2), dtype=torch.float32).pin_memory()
                if packed and "visible" in outputs and "visible_chart" in outputs and "chart_of_triangle" not in outputs:
                    # the packed wire format (about half the bytes); the int32
                    # lists above stay for frames with more than 65535 charts
                    h["p_vis_mask"] = torch.empty(T // 32 + 1, dtype=torch.int32).pin_memory()
                    h["p_cidx"] = torch.empty(T + 1, dtype=torch.int16).pin_memory()
                    h["p_roots"] = torch.empty(T + 1, dtype=torch.int32).pin_memory()
                    h["p_vtx_mask"] = torch.empty(mesh.n_vertices // 32 + 1, dtype=torch.int32).pin_memory()
            if "placements" in outputs:
                h["placements"] = torch.empty((T + 1, 8), dtype=torch.int64).pin_memory()
            self._host.append(h)
        self._np = [{k: t.numpy() for k, t in h.items()} for h in self._host]
        for h in self._np:  # unsigned views of the packed arrays
            for k, dt in (("p_vis_mask", np.uint32), ("p_cidx", np.uint16), ("p_vtx_mask", np.uint32)):
                if k in h:
                    h[k] = h[k].view(dt)
        self._vorder = [None] * depth  # each slot context's vertex order (fa_vertex_order), fetched once
        self._tris = np.asarray(mesh.triangles)
        self._V = mesh.n_vertices

    @property
    def depth(self) -> int:
        return len(self.engines)

    def _finish(self, slot: int, index: int, view) -> HostFrame:
        """Wait for the slot's frame, then queue its D2H copies on the slot
        stream (fa_frame_download; no device tensors are built per frame)."""
        eng, st = self.engines[slot], self.streams[slot]
        L, h_ctx, res = eng.ctx.L, eng.ctx.h, eng._res
        sp = ctypes.c_void_p(st.cuda_stream)
        # the copies go on the slot's copy stream: the frame is complete here
        # (fa_frame_finish synchronised it), and the slot's next frame waits
        # on the device for them only before it rewrites the downloaded
        # buffers (the context's copy_done event), so the two overlap
        spc = ctypes.c_void_p(self._cstreams[slot].cuda_stream)
        hf = HostFrame(index, self.engines[slot].n_triangles, self._tris, self._V)
        for _ in range(4):
            code = L.fa_frame_finish(h_ctx, ctypes.byref(res), sp)
            if code == nat.FA_INTERNAL_ERROR and "rerun" in nat.last_error():
                eng.launch(view, stream=st)  # work queues grown: replay the same view
                continue
            break
        else:
            hf.status, hf.error = -2, RuntimeError("frame work queues kept overflowing")
            return hf
        if code != nat.FA_OK:
            hf.status = int(code)
            try:
                nat.raise_for_status(code)
            except Exception as exc:  # the reference exception (NothingVisible, PackFailure, ...)
                hf.error = exc
            return hf
        nv, C = int(res.n_visible), int(res.n_charts)
        hf.n_visible, hf.n_charts = nv, C
        hf.scale = Fraction(int(res.scale_num), int(res.scale_den)) if res.scale_den else None
        hf.screen_fragments, hf.texels_allocated = int(res.screen_fragments), int(res.texels_allocated)
        h = self._host[slot]
        ptr = {k: ctypes.c_void_p(t.data_ptr()) if k in h else None
               for k, t in ((k, h.get(k)) for k in ("chart_of_triangle", "visible", "visible_chart", "uv",
                                                     "placements", "visible_vertices", "vertex_uv"))}
        if "p_vis_mask" in h and C <= 65535:
            if self._vorder[slot] is None:
                vo = np.empty(self._V, dtype=np.int32)
                nat.raise_for_status(L.fa_vertex_order(h_ctx, ctypes.c_void_p(vo.ctypes.data), spc))
                self._vorder[slot] = vo
            pp = {k: ctypes.c_void_p(h[k].data_ptr()) for k in ("p_vis_mask", "p_cidx", "p_roots", "p_vtx_mask")}
            nat.raise_for_status(L.fa_frame_download_packed(h_ctx, ctypes.byref(res), pp["p_vis_mask"], pp["p_cidx"],
                                                            pp["p_roots"], pp["p_vtx_mask"], ptr["vertex_uv"],
                                                            ptr["placements"], spc))
            n = self._np[slot]
            nvv = int(res.n_visible_vertices)
            hf._packed = (n["p_vis_mask"][:(self._tris.shape[0] + 31) // 32], n["p_cidx"][:nv], n["p_roots"][:C],
                          n["p_vtx_mask"][:(self._V + 31) // 32], self._vorder[slot])
            hf.vertex_uv = n["vertex_uv"][:nvv]
            if "placements" in h:
                hf.placements = n["placements"][:C]
            return hf
        if ptr["vertex_uv"] is not None:
            nat.raise_for_status(L.fa_frame_download_compact(h_ctx, ctypes.byref(res), ptr["visible"],
                                                             ptr["visible_chart"], ptr["visible_vertices"],
                                                             ptr["vertex_uv"], ptr["placements"], spc))
            if ptr["chart_of_triangle"] is not None:
                nat.raise_for_status(L.fa_frame_download(h_ctx, ctypes.byref(res), ptr["chart_of_triangle"],
                                                         None, None, None, spc))
        elif ptr["chart_of_triangle"] is not None:
            nat.raise_for_status(L.fa_frame_download(h_ctx, ctypes.byref(res), ptr["chart_of_triangle"],
                                                     ptr["visible"], ptr["uv"], ptr["placements"], spc))
        elif any(p is not None for p in ptr.values()):
            nat.raise_for_status(L.fa_frame_download_visible(h_ctx, ctypes.byref(res), ptr["visible"],
                                                             ptr["visible_chart"], ptr["uv"], ptr["placements"],
                                                             spc))
        if "chart_of_triangle" in h:
            hf._cot = self._np[slot]["chart_of_triangle"]
        if "visible_chart" in h:
            hf.visible_chart = self._np[slot]["visible_chart"][:nv]
        if "visible" in h:
            hf.visible = self._np[slot]["visible"][:nv]
        if "uv" in h:
            hf._uv = self._np[slot]["uv"][:nv]
            hf._uv_copied = True
        if "vertex_uv" in h:
            nvv = int(res.n_visible_vertices)
            hf.visible_vertices = self._np[slot]["visible_vertices"][:nvv]
            hf.vertex_uv = self._np[slot]["vertex_uv"][:nvv]
        if "placements" in h:
            hf.placements = self._np[slot]["placements"][:C]
        return hf

    def run(self, views, on_frame=None, before_launch=None) -> int:
        """Process `views` (4x4 view-projection matrices) in order.

        on_frame(HostFrame) is called once per view, in view order, after its
        host copies completed.  before_launch(stream) (optional) runs just
        before each frame is enqueued on its slot stream.  Returns the number
        of views processed."""
        P = self.depth
        inflight = [None] * P   # (index, view) launched, not finished
        copied = [None] * P     # HostFrame whose copies are queued
        done_ev = [None] * P
        torch = nat._torch()
        n = 0

        def deliver(slot):
            if copied[slot] is not None:
                done_ev[slot].synchronize()
                if on_frame is not None:
                    on_frame(copied[slot])
                copied[slot] = None

        def retire(slot):
            if inflight[slot] is not None:
                idx, v = inflight[slot]
                copied[slot] = self._finish(slot, idx, v)
                ev = torch.cuda.Event()
                ev.record(self._cstreams[slot])
                done_ev[slot] = ev
                inflight[slot] = None

        for i, view in enumerate(views):
            slot = i % P
            deliver(slot)
            retire(slot)
            st = self.streams[slot]
            if before_launch is not None:
                before_launch(st)
            self.engines[slot].launch(view, stream=st)
            inflight[slot] = (i, view)
            n += 1
        # drain in view order
        order = sorted((inflight[s][0], s) for s in range(P) if inflight[s] is not None)
        pend = sorted((copied[s].index, s) for s in range(P) if copied[s] is not None)
        for _, s in pend:
            deliver(s)
        for _, s in order:
            retire(s)
            deliver(s)
        return n
