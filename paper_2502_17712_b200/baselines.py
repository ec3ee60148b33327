"""Mirror of the comparison packers of atlaspack.baselines (baselines.py:1-261).

sequential_scale_search and superblock_pack run in the CUDA library
(csrc/fa_baselines.cu): candidates / halving levels in parallel CTAs, the
inherently serial row walk and first-fit loop inside each.  sequential_fold
and sequential_pack (single-scale helpers) use the same kernel with one
candidate.  The tiny-instance exhaustive_optimal test oracle
(baselines.py:267-344) is not part of this package (SURVEY §8f-4 scope).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

import numpy as np

from . import _native as nat
from .packing import AtlasLayout, ChartBox, FoldResult, OrientedBox, PackFailure, Placement, _check_omega, \
    placements_from_array

SUPERBLOCK_FLOOR = 16  # baselines.py:31


@dataclass(frozen=True)
class SuperblockConfig:
    block_size: int
    halving_enabled: bool = True

    def __post_init__(self):
        if self.block_size < 1 or (self.block_size & (self.block_size - 1)) != 0:
            raise ValueError("block_size must be a power of two")


@dataclass(frozen=True)
class SuperblockLayout(AtlasLayout):
    block_size: int = 0


def _dev_boxes(boxes, ctx):
    torch = nat._torch()
    dev = ctx.torch_device
    f = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int64)).to(dev)  # noqa: E731
    return (f([b.target_w for b in boxes]), f([b.target_h for b in boxes]), f([b.chart_id for b in boxes]),
            f([b.min_tri for b in boxes]))


def sequential_scale_search(boxes: Sequence[ChartBox], omega: int, n_scales: int = 64, min_dim: int = 1,
                            padding: int = 0) -> AtlasLayout:
    """baselines.py:110-141 (all candidates concurrently on the GPU)."""
    _check_omega(omega)
    box_list = list(boxes)
    if not box_list:
        return AtlasLayout(omega=omega, scale=Fraction(1), placements=())
    torch = nat.require_device()
    ctx = nat.default_context()
    tw, th, cid, mt = _dev_boxes(box_list, ctx)
    n = len(box_list)
    plc = torch.empty(8 * n, dtype=torch.int64, device=ctx.torch_device)
    sc = (ctypes.c_int64 * 2)()
    nat.raise_for_status(ctx.L.fa_sequential_scale_search(ctx.h, nat.ptr(tw), nat.ptr(th), nat.ptr(cid), nat.ptr(mt),
                                                          n, int(omega), int(n_scales), int(min_dim), int(padding),
                                                          nat.ptr(plc), sc, ctx.stream_ptr()))
    return AtlasLayout(omega=omega, scale=Fraction(int(sc[0]), int(sc[1])),
                       placements=placements_from_array(plc.cpu().numpy()))


def _sequential(widths, heights, omega):
    """fa_sequential_pack: (rows, xs, ys, used) of the row walk + push-up, caller's order."""
    torch = nat.require_device()
    ctx = nat.default_context()
    dev = ctx.torch_device
    n = len(widths)
    w = torch.as_tensor(np.asarray(widths, dtype=np.int64)).to(dev)
    h = torch.as_tensor(np.asarray(heights, dtype=np.int64)).to(dev)
    rows, xs, ys = (torch.empty(n, dtype=torch.int64, device=dev) for _ in range(3))
    used = ctypes.c_int64(0)
    nat.raise_for_status(ctx.L.fa_sequential_pack(ctx.h, nat.ptr(w), nat.ptr(h), n, int(omega), nat.ptr(rows),
                                                  nat.ptr(xs), nat.ptr(ys), ctypes.byref(used), ctx.stream_ptr()))
    return rows.cpu().numpy(), xs.cpu().numpy(), ys.cpu().numpy(), int(used.value)


def sequential_fold(widths: Sequence[int], omega: int) -> FoldResult:
    """baselines.py:53-76: walk the boxes; a box that would cross the atlas
    edge starts the next row (overflow 0 by construction)."""
    _check_omega(omega)
    w = [int(v) for v in widths]
    for v in w:
        if v < 1 or v > omega:
            raise ValueError("widths must be in [1, omega]")
    if not w:
        return FoldResult(row_of_box=np.zeros(0, np.int64), x_of_box=np.zeros(0, np.int64),
                          row_direction_left=np.ones(1, bool), overflow_m=0)
    rows, xs, _, _ = _sequential(w, [1] * len(w), omega)
    left = (np.arange(int(rows[-1]) + 1, dtype=np.int64) % 3) == 0
    return FoldResult(row_of_box=rows, x_of_box=xs, row_direction_left=left, overflow_m=0)


def sequential_pack(ordered_boxes: Sequence[OrientedBox], omega: int) -> AtlasLayout | None:
    """baselines.py:79-107: place ordered boxes at their stated dims, push up; None on overflow."""
    if not ordered_boxes:
        return AtlasLayout(omega=omega, scale=Fraction(1), placements=())
    _check_omega(omega)
    for b in ordered_boxes:
        if b.w < 1 or b.w > omega:
            raise ValueError("widths must be in [1, omega]")
    rows, xs, ys, used = _sequential([b.w for b in ordered_boxes], [b.h for b in ordered_boxes], omega)
    if used > omega:
        return None
    placements = tuple(Placement(chart_id=b.source.chart_id, x=int(xs[i]), y=int(ys[i]), w=b.w, h=b.h,
                                 rotated=b.rotated, target_w=b.source.target_w, target_h=b.source.target_h)
                       for i, b in enumerate(ordered_boxes))
    return AtlasLayout(omega=omega, scale=Fraction(1), placements=placements)


def superblock_pack(boxes: Sequence[ChartBox], omega: int, cfg: SuperblockConfig) -> SuperblockLayout | None:
    """baselines.py:187-218 (halving levels in parallel CTAs); None when the floor fails."""
    _check_omega(omega)
    if cfg.block_size > omega:
        raise ValueError("block_size must not exceed omega")
    if omega % cfg.block_size != 0:
        raise ValueError("omega must be divisible by block_size")
    box_list = list(boxes)
    if not box_list:
        return SuperblockLayout(omega=omega, scale=Fraction(1), placements=(), block_size=cfg.block_size)
    torch = nat.require_device()
    ctx = nat.default_context()
    tw, th, cid, mt = _dev_boxes(box_list, ctx)
    n = len(box_list)
    plc = torch.empty(8 * n, dtype=torch.int64, device=ctx.torch_device)
    sc = (ctypes.c_int64 * 2)()
    blk = ctypes.c_int64(0)
    code = ctx.L.fa_superblock_pack(ctx.h, nat.ptr(tw), nat.ptr(th), nat.ptr(cid), nat.ptr(mt), n, int(omega),
                                    int(cfg.block_size), int(bool(cfg.halving_enabled)), nat.ptr(plc), sc,
                                    ctypes.byref(blk), ctx.stream_ptr())
    if code == nat.FA_PACK_FAILURE:
        return None
    nat.raise_for_status(code)
    return SuperblockLayout(omega=omega, scale=Fraction(int(sc[0]), int(sc[1])),
                            placements=placements_from_array(plc.cpu().numpy()), block_size=int(blk.value))


__all__ = ["SUPERBLOCK_FLOOR", "SuperblockConfig", "SuperblockLayout", "sequential_fold", "sequential_pack",
           "sequential_scale_search", "superblock_pack", "PackFailure"]
