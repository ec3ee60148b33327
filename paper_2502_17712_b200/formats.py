"""Wire formats of the streaming-client output.

Text formats of the reference CLI — box lists (cli.py:86-123), layouts with a
SHA-256 canonical digest (cli.py:145-203, metrics.py:130-153) and chart
assignments (cli.py:457-463) — over the value types this package returns.
Host I/O: these touch no per-frame arithmetic.  Outputs are written
atomically (temp file + rename, cli.py:501-512).
"""

from __future__ import annotations

import os
import tempfile
from fractions import Fraction
from pathlib import Path

import numpy as np

from .metrics import DIGEST_ALGORITHM, layout_digest
from .packing import AtlasLayout, ChartBox, Placement

FORMAT_VERSION = "0.1.0"


class InputError(Exception):
    """Malformed input file; the message names the offending record."""


def write_atomic(path, text: str) -> None:
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    fd, tmp = tempfile.mkstemp(dir=path.parent, prefix=path.name, suffix=".tmp")
    try:
        with os.fdopen(fd, "w", encoding="utf-8") as fh:
            fh.write(text)
        os.replace(tmp, path)
    except BaseException:
        if os.path.exists(tmp):
            os.unlink(tmp)
        raise


def _records(path):
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            body = raw.split("#", 1)[0].strip()
            if body:
                yield lineno, body.split()


def parse_box_file(path) -> list:
    """(chart_id, min_tri, w, h) per record; ids unique, dims >= 1."""
    boxes, ids, tris = [], set(), set()
    for lineno, f in _records(path):
        if len(f) != 4:
            raise InputError(f"{path}:{lineno}: expected 4 fields, got {len(f)}")
        try:
            cid, mt, w, h = (int(x) for x in f)
        except ValueError:
            raise InputError(f"{path}:{lineno}: fields must be unsigned integers") from None
        if min(cid, mt) < 0:
            raise InputError(f"{path}:{lineno}: ids must be non-negative")
        if w < 1 or h < 1:
            raise InputError(f"{path}:{lineno}: box dimensions must be >= 1 (chart {cid}: {w}x{h})")
        if cid in ids:
            raise InputError(f"{path}:{lineno}: duplicate chart_id {cid}")
        if mt in tris:
            raise InputError(f"{path}:{lineno}: duplicate min_tri {mt}")
        ids.add(cid)
        tris.add(mt)
        boxes.append(ChartBox(target_w=w, target_h=h, chart_id=cid, min_tri=mt))
    return boxes


def write_box_file(boxes, path) -> None:
    rows = ["# chart_id min_tri w h"] + [f"{b.chart_id} {b.min_tri} {b.target_w} {b.target_h}" for b in boxes]
    write_atomic(path, "\n".join(rows) + "\n")


def write_layout_file(layout: AtlasLayout, path) -> None:
    """Header keys, then placements sorted by chart id (canonical order)."""
    rows = [
        "# atlaspack layout v1",
        f"version {FORMAT_VERSION}",
        f"omega {layout.omega}",
        f"scale {layout.scale.numerator}/{layout.scale.denominator}",
        f"digest_algorithm {DIGEST_ALGORITHM}",
        f"digest {layout_digest(layout).digest}",
        f"count {len(layout.placements)}",
        "# chart_id x y w h rotated target_w target_h",
    ]
    rows += [f"{p.chart_id} {p.x} {p.y} {p.w} {p.h} {int(p.rotated)} {p.target_w} {p.target_h}"
             for p in layout.placements_by_chart_id()]
    write_atomic(path, "\n".join(rows) + "\n")


def parse_layout_file(path) -> AtlasLayout:
    """Inverse of write_layout_file; verifies count and digest when present."""
    header, placements = {}, []
    for lineno, f in _records(path):
        if len(f) == 2 and not f[0].isdigit():
            header[f[0]] = f[1]
            continue
        if len(f) != 8:
            raise InputError(f"{path}:{lineno}: expected 8 placement fields")
        try:
            cid, x, y, w, h, rot, tw, th = (int(v) for v in f)
        except ValueError:
            raise InputError(f"{path}:{lineno}: placement fields must be integers") from None
        placements.append(Placement(chart_id=cid, x=x, y=y, w=w, h=h, rotated=bool(rot), target_w=tw, target_h=th))
    for key in ("omega", "scale", "count"):
        if key not in header:
            raise InputError(f"{path}: missing header key '{key}'")
    if len(placements) != int(header["count"]):
        raise InputError(f"{path}: count says {header['count']} placements, found {len(placements)}")
    num, _, den = header["scale"].partition("/")
    layout = AtlasLayout(omega=int(header["omega"]), scale=Fraction(int(num), int(den or "1")),
                         placements=tuple(placements))
    if "digest" in header and layout_digest(layout).digest != header["digest"]:
        raise InputError(f"{path}: digest mismatch, file corrupted or edited")
    return layout


def write_charts_file(chart_set, path) -> None:
    """'t <triangle> <chart>' for visible triangles, then 'v <vertex> <chart>' by vertex."""
    rows = ["# chart assignments v1", "# t <triangle> <chart>  /  v <vertex> <chart>"]
    lab = np.asarray(chart_set.chart_of_triangle)
    vis = np.flatnonzero(lab >= 0)
    rows += [f"t {t} {c}" for t, c in zip(vis.tolist(), lab[vis].tolist())]
    arr = getattr(chart_set, "vertex_chart_array", None)
    if arr is not None:
        idx = np.flatnonzero(arr >= 0)
        rows += [f"v {v} {c}" for v, c in zip(idx.tolist(), arr[idx].tolist())]
    else:
        rows += [f"v {v} {chart_set.vertex_to_chart[v]}" for v in sorted(chart_set.vertex_to_chart)]
    write_atomic(path, "\n".join(rows) + "\n")
