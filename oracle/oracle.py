"""ctypes front end of the CPU parity oracle (oracle/fa_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` leg.  The product package never
imports this module.  Each function names the reference function it restates
(file:line under /root/reference/pkg/src/atlaspack/).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfa_oracle.so")

OK, VALUE_ERROR, PACK_FAILURE, NOTHING_VISIBLE, HEIGHT_OVERFLOW = 0, 1, 2, 3, 4
MAX_BOX_DIM = 1 << 23


class OracleError(RuntimeError):
    pass


def build() -> str:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        ci = ctypes.c_int
        cd = ctypes.c_double
        L.orc_project.argtypes = [vp, i64, vp, vp]
        L.orc_depth_prepass.argtypes = [vp, i64, vp, i64, vp, ci, ci, ci, vp]
        L.orc_mark_visible.argtypes = [vp, i64, vp, i64, vp, vp, ci, ci, ci, vp]
        L.orc_build_adjacency.argtypes = [vp, i64, vp]
        L.orc_connected_charts.argtypes = [vp, vp, i64, vp]
        L.orc_merge_shared_vertices.argtypes = [vp, i64, i64, vp, vp, vp]
        L.orc_chart_bbox.argtypes = [vp, i64, vp, vp]
        L.orc_viewport_box.argtypes = [vp, ci, ci, vp]
        L.orc_chart_boxes.argtypes = [vp, i64, vp, i64, vp, vp, ci, ci, cd, vp, vp, vp, vp]
        L.orc_chart_boxes.restype = i64
        L.orc_fold.argtypes = [vp, i64, i64, vp, vp, vp]
        L.orc_push_up.argtypes = [vp, vp, vp, vp, i64, i64, vp, vp]
        L.orc_pack_arrays.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp]
        L.orc_orient_order.argtypes = [vp, vp, vp, i64, i64, vp, vp, vp, vp]
        L.orc_pack.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp]
        L.orc_uv.argtypes = [vp, i64, vp, vp, vp, i64, vp, vp, vp, vp, ci, ci, i64, vp]
        L.orc_signed_area2.argtypes = [vp, vp, ci]
        L.orc_signed_area2.restype = ctypes.c_double
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# --- projection / raster (charts.py:269-313) --------------------------------

def project(positions, vp):
    pos = _f64(positions, (-1, 3))
    out = np.empty((len(pos), 4))
    lib().orc_project(_p(pos), len(pos), _p(_f64(vp, (4, 4))), _p(out))
    return out


def signed_area2(xs, ys) -> float:
    """charts.py:251-253 through the OpenBLAS ddot restatement."""
    x, y = _f64(xs), _f64(ys)
    return lib().orc_signed_area2(_p(x), _p(y), len(x))


def depth_prepass(positions, triangles, vp, res, cull=True):
    """charts.py:285-299; returns (H, W) float64."""
    W, H = int(res[0]), int(res[1])
    pos, tris, m = _f64(positions, (-1, 3)), _i64(triangles).reshape(-1, 3), _f64(vp, (4, 4))
    depth = np.empty((max(H, 0), max(W, 0)))
    st = lib().orc_depth_prepass(_p(pos), len(pos), _p(tris), len(tris), _p(m), W, H, int(cull), _p(depth))
    if st == VALUE_ERROR:
        raise ValueError("resolution must be at least 1x1")
    if st:
        raise OracleError(f"depth_prepass status {st}")
    return depth


def mark_visible(positions, triangles, vp, depth, cull=True):
    """charts.py:302-313; returns (T,) bool."""
    pos, tris, m = _f64(positions, (-1, 3)), _i64(triangles).reshape(-1, 3), _f64(vp, (4, 4))
    depth = _f64(depth)
    H, W = depth.shape
    flags = np.zeros(len(tris), dtype=np.uint8)
    st = lib().orc_mark_visible(_p(pos), len(pos), _p(tris), len(tris), _p(m), _p(depth), W, H,
                                int(cull), _p(flags))
    if st:
        raise OracleError(f"mark_visible status {st}")
    return flags.astype(bool)


# --- charts (charts.py:64-77, 343-406) --------------------------------------

def build_adjacency(triangles):
    tris = _i64(triangles).reshape(-1, 3)
    adj = np.empty_like(tris)
    lib().orc_build_adjacency(_p(tris), len(tris), _p(adj))
    return adj


def connected_charts(adjacency, flags):
    adj = _i64(adjacency).reshape(-1, 3)
    fl = np.ascontiguousarray(flags, dtype=np.uint8)
    labels = np.empty(len(fl), dtype=np.int64)
    lib().orc_connected_charts(_p(adj), _p(fl), len(fl), _p(labels))
    return labels


def merge_shared_vertices(triangles, n_vertices, labels):
    tris = _i64(triangles).reshape(-1, 3)
    lab = _i64(labels)
    out = np.empty_like(lab)
    v2c = np.empty(int(n_vertices), dtype=np.int64)
    lib().orc_merge_shared_vertices(_p(tris), len(tris), int(n_vertices), _p(lab), _p(out), _p(v2c))
    return out, v2c


# --- bounds (geometry.py:281-362, cli.py:371-384) ---------------------------

def chart_bbox(world_tris, vp):
    """geometry.py:281-322 -> (min_x, min_y, max_x, max_y) or None (DegenerateChart)."""
    t = _f64(world_tris, (-1, 3, 3))
    box = np.empty(4)
    st = lib().orc_chart_bbox(_p(t), len(t), _p(_f64(vp, (4, 4))), _p(box))
    if st < 0:
        raise OracleError(f"chart_bbox status {st}")
    return tuple(box) if st == 1 else None


def viewport_box(box, W, H):
    b = _f64(box)
    out = np.empty(2, dtype=np.int64)
    lib().orc_viewport_box(_p(b), int(W), int(H), _p(out))
    return int(out[0]), int(out[1])


@dataclass
class ChartBoxes:
    roots: np.ndarray   # (C,) ascending chart roots that produced a box
    ndc: np.ndarray     # (C, 4) min_x, min_y, max_x, max_y
    px: np.ndarray      # (C, 2) viewport w_px, h_px
    target: np.ndarray  # (C, 2) target_w, target_h after prescale


def chart_boxes(positions, triangles, vp, labels, screen, prescale=1.0):
    pos, tris, m = _f64(positions, (-1, 3)), _i64(triangles).reshape(-1, 3), _f64(vp, (4, 4))
    lab = _i64(labels)
    n = int(np.count_nonzero(lab == np.arange(len(lab))))
    roots = np.empty(n, dtype=np.int64)
    ndc = np.empty((n, 4))
    px = np.empty((n, 2), dtype=np.int64)
    tg = np.empty((n, 2), dtype=np.int64)
    c = lib().orc_chart_boxes(_p(pos), len(pos), _p(tris), len(tris), _p(m), _p(lab),
                              int(screen[0]), int(screen[1]), float(prescale),
                              _p(roots), _p(ndc), _p(px), _p(tg))
    if c < 0:
        raise OracleError(f"chart_boxes status {c}")
    return ChartBoxes(roots[:c], ndc[:c], px[:c], tg[:c])


# --- packing (packing.py:109-362) -------------------------------------------

def fold(widths, omega):
    w = _i64(widths)
    rows, xs, m = np.empty_like(w), np.empty_like(w), np.zeros(1, dtype=np.int64)
    st = lib().orc_fold(_p(w), len(w), int(omega), _p(rows), _p(xs), _p(m))
    if st:
        raise ValueError("bad fold arguments")
    return rows, xs, int(m[0])


def push_up(rows, xs, widths, heights, omega):
    rows, xs, w, h = _i64(rows), _i64(xs), _i64(widths), _i64(heights)
    y = np.empty_like(w)
    used = np.zeros(1, dtype=np.int64)
    lib().orc_push_up(_p(rows), _p(xs), _p(w), _p(h), len(w), int(omega), _p(y), _p(used))
    return y, int(used[0])


def orient_order(tw, th, min_tri, max_h=MAX_BOX_DIM):
    tw, th, mt = _i64(tw), _i64(th), _i64(min_tri)
    n = len(tw)
    perm, ow, oh = np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int64)
    rot = np.empty(n, np.uint8)
    st = lib().orc_orient_order(_p(tw), _p(th), _p(mt), n, int(max_h), _p(perm), _p(ow), _p(oh), _p(rot))
    if st == HEIGHT_OVERFLOW:
        raise OverflowError("box height exceeds capacity")
    return perm, ow, oh, rot.astype(bool)


def pack_arrays(ow, oh, num, den, omega, min_dim=1, padding=0):
    """packing.py:245-292 -> None or dict(x, y, w, h, num, den)."""
    ow, oh = _i64(ow), _i64(oh)
    n = len(ow)
    x, y, w, h = (np.empty(n, np.int64) for _ in range(4))
    sn, sd = np.zeros(1, np.int64), np.zeros(1, np.int64)
    ok = lib().orc_pack_arrays(_p(ow), _p(oh), n, int(num), int(den), int(omega), int(min_dim),
                               int(padding), _p(x), _p(y), _p(w), _p(h), _p(sn), _p(sd))
    if not ok:
        return None
    return dict(x=x, y=y, w=w, h=h, num=int(sn[0]), den=int(sd[0]))


@dataclass
class PackResult:
    status: int
    placements: np.ndarray  # (C, 8) chart_id x y w h rotated target_w target_h, packing order
    scale: tuple            # (num, den)
    accept: np.ndarray | None = None


def pack(tw, th, chart_id, min_tri, omega, n_scales=64, min_dim=1, padding=0, want_accept=False):
    """packing.py:295-345."""
    tw, th, cid, mt = _i64(tw), _i64(th), _i64(chart_id), _i64(min_tri)
    n = len(tw)
    plc = np.zeros((n, 8), dtype=np.int64)
    sn, sd = np.zeros(1, np.int64), np.zeros(1, np.int64)
    acc = np.zeros(int(n_scales), np.uint8) if want_accept else None
    st = lib().orc_pack(_p(tw), _p(th), _p(cid), _p(mt), n, int(omega), int(n_scales), int(min_dim),
                        int(padding), _p(plc), _p(sn), _p(sd), _p(acc))
    return PackResult(st, plc, (int(sn[0]), int(sd[0])), acc)


def uv(positions, triangles, vp, vis_list, chart_of_vis, ndc, px, placements_by_chart, screen, padding=0):
    """cli.py:424-450 -> (n_vis, 6) float64, NaN rows for skipped triangles."""
    pos, tris, m = _f64(positions, (-1, 3)), _i64(triangles).reshape(-1, 3), _f64(vp, (4, 4))
    vl, cv = _i64(vis_list), _i64(chart_of_vis)
    out = np.empty((len(vl), 6))
    lib().orc_uv(_p(pos), len(pos), _p(tris), _p(m), _p(vl), len(vl), _p(cv), _p(_f64(ndc)),
                 _p(_i64(px)), _p(_i64(placements_by_chart)), int(screen[0]), int(screen[1]),
                 int(padding), _p(out))
    return out


# --- whole frame (cli.py:360-406) -------------------------------------------

@dataclass
class FrameResult:
    status: int
    depth: np.ndarray
    flags: np.ndarray
    chart_of_triangle: np.ndarray
    vertex_to_chart: np.ndarray
    boxes: ChartBoxes | None = None
    pack: PackResult | None = None
    uv: np.ndarray | None = None
    screen_fragments: int = 0
    texels_allocated: int = 0


def run_frame(positions, triangles, vp, screen, omega, n_scales=64, min_dim=1, padding=0,
              prescale=1.0, cull=True, adjacency=None) -> FrameResult:
    """The reference run_scene_pipeline (cli.py:360-406) restated on arrays."""
    pos, tris = _f64(positions, (-1, 3)), _i64(triangles).reshape(-1, 3)
    depth = depth_prepass(pos, tris, vp, screen, cull)
    flags = mark_visible(pos, tris, vp, depth, cull)
    if not flags.any():
        return FrameResult(NOTHING_VISIBLE, depth, flags, np.full(len(tris), -1, np.int64),
                           np.full(len(pos), -1, np.int64))
    adj = build_adjacency(tris) if adjacency is None else adjacency
    pre = connected_charts(adj, flags)
    labels, v2c = merge_shared_vertices(tris, len(pos), pre)
    boxes = chart_boxes(pos, tris, vp, labels, screen, prescale)
    C = len(boxes.roots)
    pk = pack(boxes.target[:, 0], boxes.target[:, 1], boxes.roots, boxes.roots, omega,
              n_scales, min_dim, padding)
    res = FrameResult(pk.status, depth, flags, labels, v2c, boxes, pk,
                      screen_fragments=int(np.isfinite(depth).sum()))
    if pk.status != OK:
        return res
    # placements by chart index (boxes are in ascending root order)
    order = np.argsort(pk.placements[:, 0], kind="stable")
    by_chart = pk.placements[order]
    root_to_c = {int(r): i for i, r in enumerate(boxes.roots)}
    vis_list = np.flatnonzero(flags)
    cv = np.array([root_to_c.get(int(labels[t]), -1) for t in vis_list], dtype=np.int64)
    res.uv = uv(pos, tris, vp, vis_list, cv, boxes.ndc, boxes.px, by_chart, screen, padding)
    res.texels_allocated = int(sum(max(0, p[3] - 2 * padding) * max(0, p[4] - 2 * padding)
                                   for p in pk.placements))
    _ = C
    return res
