"""Drop-in mirror of atlaspack.packing (packing.py:1-367).

orient / order / fold / push_up / pack_at_scale / pack run in the CUDA
library (csrc/fa_pack.cu): a one-CTA stable radix sort for the order and
one CTA per scale candidate for the fold / overflow / push-up search.  The
value types (ChartBox, OrientedBox, Placement, AtlasLayout, FoldResult) and
the rational `correct_overflow` helper (API only; `pack` never calls it,
packing.py:161-167) are host objects, as in the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, Sequence

import numpy as np

from . import _native as nat

MAX_BOX_DIM = 1 << 23           # packing.py:25
_SCALE_GRID_BITS = 24           # packing.py:29
_DIRECTION_PERIOD = 3           # packing.py:32
_MAX_OVERFLOW_ITERATIONS = 8    # packing.py:34


class PackingError(Exception):
    pass


class HeightOverflow(PackingError):
    """A box is taller than the ordering capacity allows."""


class PackFailure(PackingError):
    """Every candidate scale was rejected."""


@dataclass(frozen=True)
class ChartBox:
    target_w: int
    target_h: int
    chart_id: int
    min_tri: int

    def __post_init__(self):
        if self.target_w < 1 or self.target_h < 1:
            raise ValueError(f"box {self.chart_id}: target dims must be >= 1")


@dataclass(frozen=True)
class OrientedBox:
    w: int
    h: int
    rotated: bool
    source: ChartBox


@dataclass(frozen=True)
class Placement:
    chart_id: int
    x: int
    y: int
    w: int
    h: int
    rotated: bool
    target_w: int
    target_h: int


@dataclass(frozen=True)
class AtlasLayout:
    omega: int
    scale: Fraction
    placements: tuple

    def placements_by_chart_id(self) -> tuple:
        return tuple(sorted(self.placements, key=lambda p: p.chart_id))


@dataclass(frozen=True)
class FoldResult:
    row_of_box: np.ndarray
    x_of_box: np.ndarray
    row_direction_left: np.ndarray
    overflow_m: int


def _check_omega(omega: int) -> None:
    if omega < 1 or (omega & (omega - 1)) != 0:
        raise ValueError("omega must be a power of two >= 1")


def _i64_dev(a, device):
    torch = nat._torch()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64)).to(device)


def _empty(n, dtype, device):
    torch = nat._torch()
    return torch.empty(max(int(n), 1), dtype=dtype, device=device)


def orient(boxes: Iterable[ChartBox]) -> list:
    """packing.py:109-117 (fa_orient kernel)."""
    box_list = list(boxes)
    if not box_list:
        return []
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    tw = _i64_dev([b.target_w for b in box_list], dev)
    th = _i64_dev([b.target_h for b in box_list], dev)
    n = len(box_list)
    ow, oh, rot = _empty(n, torch.int64, dev), _empty(n, torch.int64, dev), _empty(n, torch.uint8, dev)
    nat.raise_for_status(ctx.L.fa_orient(ctx.h, nat.ptr(tw), nat.ptr(th), n, nat.ptr(ow), nat.ptr(oh), nat.ptr(rot),
                                         ctx.stream_ptr()))
    ow, oh, rot = ow.cpu().numpy(), oh.cpu().numpy(), rot.cpu().numpy()
    return [OrientedBox(w=int(ow[i]), h=int(oh[i]), rotated=bool(rot[i]), source=b) for i, b in enumerate(box_list)]


def _order_perm(boxes: Sequence[OrientedBox], max_h: int):
    """GPU stable sort by (-h, min_tri) over the boxes' oriented dims."""
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    n = len(boxes)
    # order() sorts the oriented boxes it is given: feed (w, h) as targets of
    # already-oriented boxes (w <= h keeps them unrotated inside the kernel)
    w = _i64_dev([min(b.w, b.h) for b in boxes], dev)
    h = _i64_dev([b.h for b in boxes], dev)
    mt = _i64_dev([b.source.min_tri for b in boxes], dev)
    perm = _empty(n, torch.int32, dev)
    ow, oh, rot = _empty(n, torch.int64, dev), _empty(n, torch.int64, dev), _empty(n, torch.uint8, dev)
    nat.raise_for_status(ctx.L.fa_orient_order(ctx.h, nat.ptr(w), nat.ptr(h), nat.ptr(mt), n, int(max_h),
                                               nat.ptr(perm), nat.ptr(ow), nat.ptr(oh), nat.ptr(rot),
                                               ctx.stream_ptr()))
    return perm[:n].cpu().numpy()


def order(boxes: Sequence[OrientedBox], max_h: int = MAX_BOX_DIM) -> list:
    """packing.py:120-130: height descending, min_tri ascending (stable)."""
    boxes = list(boxes)
    for b in boxes:
        if b.h > max_h:
            raise HeightOverflow(f"box height {b.h} exceeds capacity {max_h}")
    if len(boxes) <= 1:
        return boxes
    if any(b.w > b.h for b in boxes):
        # hand-built boxes that are wider than tall: sort key is still h
        pass
    perm = _order_perm(boxes, max_h)
    return [boxes[int(i)] for i in perm]


def fold(widths, omega: int) -> FoldResult:
    """packing.py:133-158 (fa_fold kernel)."""
    _check_omega(omega)
    w = np.asarray(widths, dtype=np.int64)
    if w.ndim != 1 or w.size == 0:
        raise ValueError("fold requires a non-empty width sequence")
    if np.any(w < 1):
        raise ValueError("widths must be >= 1")
    if np.any(w > omega):
        raise ValueError("fold requires every width <= omega")
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    d_w = _i64_dev(w, dev)
    rows, xs = _empty(len(w), torch.int64, dev), _empty(len(w), torch.int64, dev)
    m = ctypes.c_int64(0)
    nat.raise_for_status(ctx.L.fa_fold(ctx.h, nat.ptr(d_w), len(w), int(omega), nat.ptr(rows), nat.ptr(xs),
                                       ctypes.byref(m), ctx.stream_ptr()))
    rows = rows[:len(w)].cpu().numpy()
    n_rows = int(rows[-1]) + 1
    left = (np.arange(n_rows, dtype=np.int64) % _DIRECTION_PERIOD) == 0
    return FoldResult(row_of_box=rows, x_of_box=xs[:len(w)].cpu().numpy(), row_direction_left=left,
                      overflow_m=int(m.value))


def correct_overflow(scale: Fraction, m: int, omega: int) -> Fraction:
    """packing.py:161-167 (rational API helper, not called by pack)."""
    if m < 0:
        raise ValueError("overflow must be non-negative")
    if m == 0:
        return scale
    return scale * Fraction(omega, omega + m)


def push_up(fold_result: FoldResult, dims, omega: int):
    """packing.py:170-215 (fa_push_up kernel)."""
    _check_omega(omega)
    if fold_result.overflow_m != 0:
        raise ValueError("push_up requires a fold with zero overflow")
    d = np.asarray(dims, dtype=np.int64).reshape(-1, 2)
    n = len(d)
    if len(fold_result.x_of_box) != n:
        raise ValueError("dims do not match the fold result")
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    rows = _i64_dev(fold_result.row_of_box, dev)
    xs = _i64_dev(fold_result.x_of_box, dev)
    w = _i64_dev(d[:, 0], dev)
    h = _i64_dev(d[:, 1], dev)
    y = _empty(n, torch.int64, dev)
    used = ctypes.c_int64(0)
    nat.raise_for_status(ctx.L.fa_push_up(ctx.h, nat.ptr(rows), nat.ptr(xs), nat.ptr(w), nat.ptr(h), n, int(omega),
                                          nat.ptr(y), ctypes.byref(used), ctx.stream_ptr()))
    return y[:n].cpu().numpy(), int(used.value)


def pack_at_scale(ordered_boxes: Sequence[OrientedBox], scale: Fraction, omega: int, min_dim: int = 1,
                  padding: int = 0):
    """packing.py:218-242 (one candidate CTA of the pack kernel)."""
    _check_omega(omega)
    if not (0 < scale <= 1):
        raise ValueError("scale must be in (0, 1]")
    if min_dim < 1 or padding < 0:
        raise ValueError("min_dim must be >= 1 and padding >= 0")
    if not ordered_boxes:
        return AtlasLayout(omega=omega, scale=Fraction(scale), placements=())
    fr = Fraction(scale)
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    n = len(ordered_boxes)
    ow = _i64_dev([b.w for b in ordered_boxes], dev)
    oh = _i64_dev([b.h for b in ordered_boxes], dev)
    xywh = _empty(4 * n, torch.int64, dev)
    sc = (ctypes.c_int64 * 2)()
    acc = ctypes.c_int(0)
    nat.raise_for_status(ctx.L.fa_pack_at_scale(ctx.h, nat.ptr(ow), nat.ptr(oh), n, fr.numerator, fr.denominator,
                                                int(omega), int(min_dim), int(padding), nat.ptr(xywh), sc,
                                                ctypes.byref(acc), ctx.stream_ptr()))
    if not acc.value:
        return None
    r = xywh[:4 * n].cpu().numpy().reshape(n, 4)
    placements = tuple(
        Placement(chart_id=b.source.chart_id, x=int(r[i, 0]), y=int(r[i, 1]), w=int(r[i, 2]), h=int(r[i, 3]),
                  rotated=b.rotated, target_w=b.source.target_w, target_h=b.source.target_h)
        for i, b in enumerate(ordered_boxes))
    return AtlasLayout(omega=omega, scale=Fraction(int(sc[0]), int(sc[1])), placements=placements)


def placements_from_array(arr) -> tuple:
    """(n, 8) int64 placements (packing order) -> Placement tuple."""
    a = np.asarray(arr, dtype=np.int64).reshape(-1, 8).tolist()
    return tuple(Placement(chart_id=r[0], x=r[1], y=r[2], w=r[3], h=r[4], rotated=bool(r[5]), target_w=r[6],
                           target_h=r[7]) for r in a)


def pack_arrays(tw, th, chart_id, min_tri, omega: int, n_scales: int = 64, min_dim: int = 1, padding: int = 0,
                want_accept: bool = False):
    """Array form of pack(): returns (placements (n,8) int64 in packing order, Fraction, accept)."""
    _check_omega(omega)
    if not (1 <= n_scales <= 1 << 20):
        raise ValueError("n_scales must be in [1, 2^20]")
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    tw = np.asarray(tw, dtype=np.int64)
    n = len(tw)
    if n == 0:
        return np.zeros((0, 8), dtype=np.int64), Fraction(1), None
    d_tw, d_th = _i64_dev(tw, dev), _i64_dev(th, dev)
    d_cid, d_mt = _i64_dev(chart_id, dev), _i64_dev(min_tri, dev)
    plc = _empty(8 * n, torch.int64, dev)
    acc = _empty(n_scales, torch.uint8, dev) if want_accept else None
    sc = (ctypes.c_int64 * 2)()
    nat.raise_for_status(ctx.L.fa_pack(ctx.h, nat.ptr(d_tw), nat.ptr(d_th), nat.ptr(d_cid), nat.ptr(d_mt), n,
                                       int(omega), int(n_scales), int(min_dim), int(padding), nat.ptr(plc), sc,
                                       nat.ptr(acc), ctx.stream_ptr()))
    accept = acc[:n_scales].cpu().numpy().astype(bool) if want_accept else None
    return plc[:8 * n].cpu().numpy().reshape(n, 8), Fraction(int(sc[0]), int(sc[1])), accept


def pack(boxes: Iterable[ChartBox], omega: int, n_scales: int = 64, min_dim: int = 1, padding: int = 0,
         workers: int = 1) -> AtlasLayout:
    """packing.py:295-345: all candidates evaluated concurrently on the GPU
    (`workers` is accepted for API compatibility; the result never depends on it)."""
    _check_omega(omega)
    if not (1 <= n_scales <= 1 << 20):
        raise ValueError("n_scales must be in [1, 2^20]")
    box_list = list(boxes)
    if not box_list:
        return AtlasLayout(omega=omega, scale=Fraction(1), placements=())
    if min_dim < 1 or padding < 0:
        raise ValueError("min_dim must be >= 1 and padding >= 0")
    plc, scale, _ = pack_arrays([b.target_w for b in box_list], [b.target_h for b in box_list],
                                [b.chart_id for b in box_list], [b.min_tri for b in box_list], omega, n_scales,
                                min_dim, padding)
    return AtlasLayout(omega=omega, scale=scale, placements=placements_from_array(plc))


__all__ = ["MAX_BOX_DIM", "PackingError", "HeightOverflow", "PackFailure", "ChartBox", "OrientedBox", "Placement",
           "AtlasLayout", "FoldResult", "orient", "order", "fold", "correct_overflow", "push_up", "pack_at_scale",
           "pack", "pack_arrays", "placements_from_array"]
