"""Wire formats: layout files round-trip with their SHA-256
digest, reproduce the reference's golden digests, and reject tampering.
CPU only (the layouts come from the reference golden vectors)."""

from fractions import Fraction

import numpy as np
import pytest

from goldens import pack_cases
from paper_2502_17712_b200 import formats
from paper_2502_17712_b200.charts import ChartSet
from paper_2502_17712_b200.packing import AtlasLayout, ChartBox, Placement


def _layout(case):
    pl = tuple(Placement(chart_id=p[0], x=p[1], y=p[2], w=p[3], h=p[4], rotated=bool(p[5]), target_w=p[6],
                         target_h=p[7]) for p in case["placements"])
    return AtlasLayout(omega=case["omega"], scale=Fraction(*case["scale"]), placements=pl)


def test_golden_digests_and_roundtrip(tmp_path):
    from paper_2502_17712_b200.metrics import layout_digest, layouts_equal
    n = 0
    for c in pack_cases()["pack"]:
        if c["status"] != "ok":
            continue
        lay = _layout(c)
        assert layout_digest(lay).digest == c["digest"]
        p = tmp_path / f"l{n}.layout.txt"
        formats.write_layout_file(lay, p)
        back = formats.parse_layout_file(p)
        assert layouts_equal(back, lay) and back.scale == lay.scale
        n += 1
    assert n > 50


def test_tampering_detected(tmp_path):
    c = next(c for c in pack_cases()["pack"] if c["status"] == "ok" and len(c["placements"]) > 3)
    p = tmp_path / "t.layout.txt"
    formats.write_layout_file(_layout(c), p)
    lines = p.read_text().splitlines()
    i = next(k for k, l in enumerate(lines) if l and l[0].isdigit())
    f = lines[i].split()
    f[1] = str(int(f[1]) + 1)
    lines[i] = " ".join(f)
    p.write_text("\n".join(lines) + "\n")
    with pytest.raises(formats.InputError, match="digest"):
        formats.parse_layout_file(p)


def test_count_and_fields(tmp_path):
    p = tmp_path / "bad.layout.txt"
    p.write_text("omega 64\nscale 1/1\ncount 2\n0 0 0 8 8 0 8 8\n")
    with pytest.raises(formats.InputError, match="count"):
        formats.parse_layout_file(p)


def test_box_files(tmp_path):
    boxes = [ChartBox(3, 4, 0, 10), ChartBox(7, 2, 1, 3)]
    p = tmp_path / "b.txt"
    formats.write_box_file(boxes, p)
    assert formats.parse_box_file(p) == boxes
    p.write_text("# h\n1 1 4 4\n2 2 0 5\n")
    with pytest.raises(formats.InputError, match="b.txt:3"):
        formats.parse_box_file(p)
    p.write_text("1 1 4 4\n1 2 5 5\n")
    with pytest.raises(formats.InputError, match="duplicate chart_id"):
        formats.parse_box_file(p)


def test_charts_file(tmp_path):
    cs = ChartSet(np.array([-1, 1, 1, 3]), vertex_chart_array=np.array([1, 1, -1, 3, 3]))
    p = tmp_path / "c.txt"
    formats.write_charts_file(cs, p)
    body = [l for l in p.read_text().splitlines() if not l.startswith("#")]
    assert body == ["t 1 1", "t 2 1", "t 3 3", "v 0 1", "v 1 1", "v 3 3", "v 4 3"]
