"""Full-size frames pinned DIRECTLY to the reference: SHA-256 digests of the
reference's own run_scene_pipeline (cli.py:360-406) at C2, C3 (prescale 2),
a C4 camera-path frame, a C5 streaming view, and C2 with the comparison
packers, written by tests/golden/make_golden.py --digest / --c2 in the build
container (each reference frame takes minutes there; C3 about half an hour).

Compared per frame: depth (sign of zero folded), visibility flags,
chart_of_triangle, vertex_to_chart, chart NDC boxes, targets, placements
(packing order), scale, layout digest, screen_fragments, texels_allocated,
the float64 UV rows in the reference's emission order (cli.py:424-450)
together with the triangle id of each row, and the stretch report.

CPU (not gpu): the C oracle against the digests (the stages up to the boxes
for the comparison packers, which the oracle does not restate).
GPU (-m gpu): the CUDA frame through FrameEngine against the same digests.
"""

import glob
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from goldens import GOLDEN, canon

FILES = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "*_reference.json")))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    ref = json.load(open(os.path.join(GOLDEN, name)))
    ref.setdefault("scene", "C2")  # the round-1 C2 file predates these keys
    ref.setdefault("pose", 0)
    ref.setdefault("packer", "fastatlas")
    from paper_2502_17712_b200 import scenes
    spec = scenes.build_scene(ref["scene"])
    ref.setdefault("prescale", spec.prescale)
    return ref, spec


def reference_uv_order(vis, chart_of_vis, uv):
    """Rows of the per-visible-triangle UVs (ascending triangle id, NaN rows =
    no UV) in the reference's emission order: charts by ascending root,
    members ascending, triangles reaching behind the camera skipped."""
    order = np.lexsort((vis, chart_of_vis))
    keep = ~np.isnan(uv[order]).any(axis=1)
    rows = order[keep]
    return vis[rows].astype(np.int64), uv[rows]


def check_common(ref, depth, flags, chart, v2c):
    assert sha(canon(depth)) == ref["depth_sha"]
    assert sha(flags.astype(np.uint8)) == ref["flags_sha"]
    assert int(flags.sum()) == ref["n_visible"]
    assert sha(chart.astype(np.int64)) == ref["chart_sha"]
    assert sha(v2c.astype(np.int64)) == ref["v2c_sha"]


@pytest.mark.slow
@pytest.mark.parametrize("name", FILES)
def test_oracle_vs_reference_digest(name):
    ref, s = load(name)
    vp = np.array(ref["vp"])
    r = oracle.run_frame(s.positions, s.triangles, vp, s.screen, s.omega, prescale=ref["prescale"])
    check_common(ref, r.depth, r.flags, r.chart_of_triangle, r.vertex_to_chart)
    assert len(r.boxes.roots) == ref["n_charts"]
    assert r.boxes.target.tolist() == ref["target"]
    assert sha(r.boxes.ndc) == ref["ndc_sha"]
    if ref["packer"] != "fastatlas":
        return
    assert r.status == oracle.OK
    assert r.pack.placements.tolist() == ref["placements"]
    assert list(r.pack.scale) == ref["scale"]
    assert r.screen_fragments == ref["screen_fragments"]
    assert r.texels_allocated == ref["texels_allocated"]
    vis = np.flatnonzero(r.flags)
    tris, uv = reference_uv_order(vis, r.chart_of_triangle[vis], r.uv)
    assert sha(tris) == ref["uv_tris_sha"]
    assert sha(uv) == ref["uv_sha"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", FILES)
def test_gpu_frame_vs_reference_digest(name):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_17712_b200 as fa
    from paper_2502_17712_b200 import FrameEngine, FrameSettings
    ref, s = load(name)
    settings = FrameSettings(screen=tuple(s.screen), omega=s.omega, prescale=ref["prescale"], uv_f64=True,
                             want_depth=True, packer=ref["packer"])
    out = FrameEngine(fa.Mesh(s.positions, s.triangles), settings=settings).run(np.array(ref["vp"]))
    h = out.to_host()
    check_common(ref, h["depth"], h["flags"], h["chart_of_triangle"], h["vertex_to_chart"])
    assert out.n_charts == ref["n_charts"]
    assert h["target"].tolist() == ref["target"]
    assert sha(h["ndc"]) == ref["ndc_sha"]
    assert h["placements"].tolist() == ref["placements"]
    assert [out.scale.numerator, out.scale.denominator] == ref["scale"]
    assert fa.layout_digest(out.layout()).digest == ref["digest"]
    assert out.screen_fragments == ref["screen_fragments"]
    assert out.texels_allocated == ref["texels_allocated"]
    vis = h["visible"]
    tris, uv = reference_uv_order(vis, h["chart_of_triangle"][vis], h["uv"])
    assert sha(tris) == ref["uv_tris_sha"]
    assert sha(uv) == ref["uv_sha"]
    st = out.stretch()
    assert st.l2 == pytest.approx(ref["stretch"][0], rel=1e-9)
    assert st.linf == pytest.approx(ref["stretch"][1], rel=1e-9)
