"""GPU parity: the CUDA path against the reference's golden vectors and the
C oracle (CPU restatement pinned to those vectors).  Run with -m gpu.

Bar: depth (up to the sign of zero), flags, chart ids, vertex
map, boxes, placements, packing order and scale are bit-exact; float64 UVs
are bit-exact; float32 UVs are within 1e-5 relative (|d| <= 1e-5 * max(1,|x|)).
"""

import math

import numpy as np
import pytest

import oracle
from goldens import canon, group, meta, npz, pack_cases, same_bits

pytestmark = pytest.mark.gpu

fa = pytest.importorskip("paper_2502_17712_b200")
from paper_2502_17712_b200 import FrameEngine, FrameSettings, RawCamera  # noqa: E402
from paper_2502_17712_b200 import packing as fpk  # noqa: E402
from paper_2502_17712_b200 import scenes  # noqa: E402

UV_F32_RTOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    oracle.build()


# ---------------------------------------------------------------- raster ----
class TestRaster:
    @pytest.mark.parametrize("case", [m["name"] for m in meta()["raster"]])
    def test_depth_flags_vs_reference(self, case):
        m = next(x for x in meta()["raster"] if x["name"] == case)
        g = group(npz("raster.npz"), case)
        mesh = fa.Mesh(g["pos"], g["tris"])
        cam = RawCamera(g["vp"])
        depth = fa.depth_prepass(mesh, cam, m["res"], backface_cull=m["cull"])
        assert same_bits(canon(depth), g["depth"])
        vis = fa.mark_visible(mesh, cam, depth, backface_cull=m["cull"])
        assert np.array_equal(vis.flags, g["flags"])

    def test_empty_mesh(self):
        mesh = fa.Mesh(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
        cam = fa.CameraFrame.from_params(math.radians(90), 1.0, 0.1, 100.0)
        depth = fa.depth_prepass(mesh, cam, (16, 8))
        assert depth.shape == (8, 16) and np.all(np.isinf(depth))

    def test_bad_resolution(self):
        mesh = fa.Mesh(np.zeros((3, 3)), np.array([[0, 1, 2]]))
        cam = fa.CameraFrame.from_params(math.radians(90), 1.0, 0.1, 100.0)
        with pytest.raises(ValueError):
            fa.depth_prepass(mesh, cam, (0, 4))

    def test_large_triangles_match_oracle(self):
        """Screen-filling triangles exercise the tiled (large) raster path."""
        rng = np.random.default_rng(3)
        tri = rng.normal(scale=3.0, size=(60, 3, 3))
        tri[:, :, 2] -= 4.0
        pos = tri.reshape(-1, 3)
        tris = np.arange(len(pos)).reshape(-1, 3)
        cam = fa.CameraFrame.from_params(math.radians(70), 1.5, 0.1, 50.0)
        for res, cull in [((300, 200), True), ((257, 131), False)]:
            mesh = fa.Mesh(pos, tris)
            d = fa.depth_prepass(mesh, cam, res, backface_cull=cull)
            rd = oracle.depth_prepass(pos, tris, cam.view_proj, res, cull)
            assert same_bits(canon(d), canon(rd))
            f = fa.mark_visible(mesh, cam, d, backface_cull=cull).flags
            assert np.array_equal(f, oracle.mark_visible(pos, tris, cam.view_proj, rd, cull))


# ---------------------------------------------------------------- charts ----
class TestCharts:
    @pytest.mark.parametrize("case", meta()["charts"])
    def test_vs_reference(self, case):
        g = group(npz("charts.npz"), case)
        mesh = fa.Mesh(g["pos"], g["tris"], adjacency=g["adj"])
        vis = fa.VisibilityBuffer(g["flags"], (8, 8))
        pre = fa.connected_charts(mesh, vis)
        assert np.array_equal(pre.chart_of_triangle, g["pre"])
        merged = fa.merge_shared_vertices(pre, mesh)
        assert np.array_equal(merged.chart_of_triangle, g["merged"])
        assert np.array_equal(merged.vertex_chart_array, g["v2c"])
        assert list(merged.charts.keys()) == g["roots"].tolist()

    def test_gpu_adjacency_matches_reference(self):
        """build_adjacency (charts.py:64-77) incl. non-manifold edges, on the GPU."""
        for case in meta()["charts"]:
            g = group(npz("charts.npz"), case)
            assert np.array_equal(fa.Mesh(g["pos"], g["tris"]).adjacency, g["adj"])
        assert fa.Mesh(np.zeros((5, 3)), [(0, 1, 2), (0, 1, 3), (0, 1, 4)]).adjacency.tolist() == [[-1] * 3] * 3

    def test_gpu_adjacency_full_size(self):
        spec = scenes.build_scene("C2")
        adj = fa.Mesh(spec.positions, spec.triangles).adjacency
        assert np.array_equal(adj, oracle.build_adjacency(spec.triangles))

    def test_connected_charts_with_gpu_adjacency(self):
        for case in meta()["charts"][:12]:
            g = group(npz("charts.npz"), case)
            mesh = fa.Mesh(g["pos"], g["tris"])  # adjacency built on the GPU
            pre = fa.connected_charts(mesh, fa.VisibilityBuffer(g["flags"], (8, 8)))
            assert np.array_equal(pre.chart_of_triangle, g["pre"])


# ---------------------------------------------------------------- bounds ----
class TestBounds:
    def test_chart_bbox_vs_reference(self):
        g = npz("bounds.npz")
        for i in range(len(g["tris"])):  # all 3000 reference cases
            tri = g["tris"][i]
            tri = tri[~np.isnan(tri[:, 0, 0])]
            cam = RawCamera(g["vps"][g["cam"][i]])
            if g["degenerate"][i]:
                with pytest.raises(fa.DegenerateChart):
                    fa.chart_bbox(tri, cam)
            else:
                b = fa.chart_bbox(tri, cam)
                assert np.array_equal([b.min_x, b.min_y, b.max_x, b.max_y], g["boxes"][i]), i

    def test_viewport_box(self):
        from paper_2502_17712_b200.geometry import viewport_box_batch
        g = npz("bounds.npz")
        for W, H in {(int(r[4]), int(r[5])) for r in g["vb_in"][:20]}:
            sel = (g["vb_in"][:, 4] == W) & (g["vb_in"][:, 5] == H)
            assert np.array_equal(viewport_box_batch(g["vb_in"][sel, :4], W, H), g["vb_out"][sel])
        assert fa.viewport_box(fa.NdcBox(-1, -1, 1, 1), 1920, 1080) == (1920, 1080)
        assert fa.viewport_box(fa.NdcBox(0.25, -0.5, 0.25, -0.5), 640, 480) == (1, 1)

    def test_blinn_and_side_plane_kats(self):
        """tests/test_geometry.py:66-146 restated."""
        assert fa.blinn_clamped_ndc((0.5, -0.5, 0.0, 1.0)) == (0.5, -0.5)
        assert fa.blinn_clamped_ndc((5.0, 0.0, 0.0, 2.0)) == (1.0, 0.0)
        assert fa.blinn_clamped_ndc((3.0, -7.0, 0.0, -2.0)) == (1.0, -1.0)
        assert fa.blinn_clamped_ndc((2.0, -0.1, 0.0, 0.0)) == (1.0, -1.0)
        assert fa.blinn_clamped_ndc((0.0, 0.0, 0.0, 0.0)) == (1.0, 1.0)
        assert fa.select_side_plane(np.array([[0.1, 0.1, 0, 1], [0.5, 0.1, 0, 1], [0.1, 0.5, 0, 1]], float)) is None
        assert fa.select_side_plane(np.array([[0.5, 0.0, 0, 1], [1.5, 0.1, 0, 1], [0.6, 0.3, 0, 1]], float)) == "right"
        assert fa.select_side_plane(np.array([[0.2, 0.5, 0, 1], [2.0, 0.9, 0, 1], [0.4, -2.0, 0, 1]], float)) == "right"
        assert fa.select_side_plane(np.array([[1.5, 0.0, 0, 1], [2.5, 0.1, 0, 1], [1.6, 0.3, 0, 1]], float)) is None


# ---------------------------------------------------------------- packing ---
STATUS_EXC = {"PackFailure": fa.PackFailure, "ValueError": ValueError, "HeightOverflow": fa.HeightOverflow}


class TestPack:
    @pytest.fixture(autouse=True, params=["smem_tail", "global_tail"])
    def _tail(self, request, monkeypatch):
        """Both push-up tails of k_pack: boxes in shared memory (default) and
        the global-memory rows (FASTATLAS_PACK_SMEM_TAIL=0, the path of frames
        with more than 4096 charts)."""
        monkeypatch.setenv("FASTATLAS_PACK_SMEM_TAIL", "1" if request.param == "smem_tail" else "0")

    @pytest.mark.parametrize("idx", range(len(pack_cases()["pack"])))
    def test_pack_vs_reference(self, idx):
        c = pack_cases()["pack"][idx]
        boxes = [fa.ChartBox(int(b[0]), int(b[1]), int(b[2]), int(b[3])) for b in c["boxes"]]
        if c["status"] != "ok":
            with pytest.raises(STATUS_EXC[c["status"]]):
                fa.pack(boxes, c["omega"], n_scales=c["n_scales"], min_dim=c["min_dim"], padding=c["padding"])
            return
        lay = fa.pack(boxes, c["omega"], n_scales=c["n_scales"], min_dim=c["min_dim"], padding=c["padding"])
        assert [lay.scale.numerator, lay.scale.denominator] == c["scale"]
        got = [[p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h] for p in lay.placements]
        assert got == c["placements"]
        assert fa.layout_digest(lay).digest == c["digest"]
        if c.get("accept") is not None and boxes:
            b = np.array(c["boxes"], dtype=np.int64)
            _, _, acc = fpk.pack_arrays(b[:, 0], b[:, 1], b[:, 2], b[:, 3], c["omega"], c["n_scales"],
                                        c["min_dim"], c["padding"], want_accept=True)
            assert acc.tolist() == c["accept"]

    def test_fold_push_up_vs_reference(self):
        for rec in pack_cases()["prim"]:
            if rec["kind"] != "fold":
                continue
            f = fa.fold(rec["widths"], rec["omega"])
            assert f.row_of_box.tolist() == rec["rows"] and f.x_of_box.tolist() == rec["x"]
            assert f.overflow_m == rec["m"]
            if "y" in rec:
                y, used = fa.push_up(f, np.stack([rec["widths"], rec["heights"]], 1), rec["omega"])
                assert y.tolist() == rec["y"] and used == rec["used"]

    def test_pack_at_scale_vs_reference(self):
        from fractions import Fraction
        for rec in pack_cases()["prim"]:
            if rec["kind"] != "pack_at_scale":
                continue
            ordered = [fa.OrientedBox(w=o[0], h=o[1], rotated=bool(o[2]),
                                      source=fa.ChartBox(o[3], o[4], o[5], o[6])) for o in rec["ordered"]]
            lay = fa.pack_at_scale(ordered, Fraction(rec["num"], rec["den"]), rec["omega"], rec["min_dim"],
                                   rec["padding"])
            if rec["result"] is None:
                assert lay is None
                continue
            assert [lay.scale.numerator, lay.scale.denominator] == rec["result"]["scale"]
            got = [[p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h] for p in lay.placements]
            assert got == rec["result"]["placements"]

    def test_orient_order_kats(self):
        """tests/test_packing.py:29-69 restated."""
        (o,) = fa.orient([fa.ChartBox(7, 2, 0, 0)])
        assert (o.w, o.h, o.rotated) == (2, 7, True)
        (o,) = fa.orient([fa.ChartBox(4, 4, 0, 0)])
        assert (o.w, o.h, o.rotated) == (4, 4, False)
        box = lambda w, h, i: fa.ChartBox(w, h, i, i)  # noqa: E731
        boxes = [fa.OrientedBox(1, 7, False, box(1, 7, 40)), fa.OrientedBox(1, 5, False, box(1, 5, 10)),
                 fa.OrientedBox(1, 7, False, box(1, 7, 3))]
        assert [(b.h, b.source.min_tri) for b in fa.order(boxes)] == [(7, 3), (7, 40), (5, 10)]
        with pytest.raises(fa.HeightOverflow):
            fa.order([fa.OrientedBox(1, 100, False, box(1, 100, 0))], max_h=50)

    def test_permutation_invariance(self):
        from paper_2502_17712_b200.cli import generate_boxes
        boxes = generate_boxes(40, 128, np.random.default_rng(5))
        ref = fa.layout_digest(fa.pack(boxes, 128))
        rng = np.random.default_rng(1)
        for _ in range(3):
            sh = list(boxes)
            rng.shuffle(sh)
            assert fa.layout_digest(fa.pack(sh, 128)) == ref


# ---------------------------------------------------------------- frames ----
def _frame_case(name):
    m = next(x for x in meta()["frames"] if x["name"] == name)
    g = group(npz("frames.npz"), name)
    if name.startswith("C"):
        s = scenes.build_scene(name)
        pos, tris = s.positions, s.triangles
    else:
        pos, tris = g["pos"], g["tris"]
    return m, g, pos, tris


class TestFrames:
    @pytest.mark.parametrize("case", [m["name"] for m in meta()["frames"]])
    @pytest.mark.parametrize("use_graph", [False, True])
    def test_frame_vs_reference(self, case, use_graph):
        m, g, pos, tris = _frame_case(case)
        settings = FrameSettings(screen=tuple(m["screen"]), omega=m["omega"], min_dim=m["min_dim"],
                                 padding=m["padding"], prescale=m["prescale"], uv_f64=True, want_depth=True,
                                 use_graph=use_graph)
        eng = FrameEngine(fa.Mesh(pos, tris), settings=settings)
        out = eng.run(g["vp"], check=False)
        h = out.to_host()
        assert same_bits(canon(h["depth"]), g["depth"])
        assert np.array_equal(h["flags"].astype(bool), g["flags"])
        if m["status"] == "NothingVisible":
            assert out.status == 3
            return
        assert np.array_equal(h["chart_of_triangle"].astype(np.int64), g["chart_of_triangle"])
        assert np.array_equal(h["vertex_to_chart"].astype(np.int64), g["vertex_to_chart"])
        assert np.array_equal(h["roots"].astype(np.int64), g["box_roots"])
        assert np.array_equal(h["target"], g["target"])
        if m["status"] == "PackFailure":
            assert out.status == 2
            return
        assert out.status == 0
        assert same_bits(h["ndc"], g["ndc"])
        assert np.array_equal(h["px"].astype(np.int64), g["px"])
        assert np.array_equal(h["placements"], g["placements"])
        assert [out.scale.numerator, out.scale.denominator] == g["scale"].tolist()
        assert out.screen_fragments == m["screen_fragments"]
        assert out.texels_allocated == m["texels_allocated"]
        assert fa.layout_digest(out.layout()).digest == m["digest"]
        # stretch (metrics.py:84-111): GPU closed form vs the reference's LAPACK SVD
        if m.get("stretch") is None:
            assert out.stretch() is None
        else:
            st = out.stretch()
            assert st.l2 == pytest.approx(m["stretch"][0], rel=1e-9)
            assert st.linf == pytest.approx(m["stretch"][1], rel=1e-9)
        vis = h["visible"]
        assert np.array_equal(vis, np.flatnonzero(g["flags"]))
        pos_of = {int(t): k for k, t in enumerate(vis)}
        rows = np.array([pos_of[int(t)] for t in g["uv_tris"]], dtype=np.int64)
        assert same_bits(h["uv"][rows], g["uv"])
        mask = np.ones(len(vis), bool)
        mask[rows] = False
        assert np.all(np.isnan(h["uv"][mask]))

    def test_uv_f32_within_tolerance(self):
        m, g, pos, tris = _frame_case("C1")
        eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=tuple(m["screen"]), omega=m["omega"]))
        h = eng.run(g["vp"]).to_host()
        pos_of = {int(t): k for k, t in enumerate(h["visible"])}
        rows = np.array([pos_of[int(t)] for t in g["uv_tris"]])
        got = h["uv"][rows].astype(np.float64)
        assert np.all(np.abs(got - g["uv"]) <= UV_F32_RTOL * np.maximum(1.0, np.abs(g["uv"])))

    def test_engine_reuse_is_deterministic(self):
        m, g, pos, tris = _frame_case("mini_v0")
        eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=tuple(m["screen"]), omega=m["omega"],
                                                                     uv_f64=True))
        a = eng.run(g["vp"]).clone()
        _, g2, _, _ = _frame_case("mini_v1")
        eng.run(g2["vp"])
        b = eng.run(g["vp"])
        for k in ("chart_of_triangle", "placements", "uv"):
            assert np.array_equal(getattr(a, k).cpu().numpy().view(np.uint8),
                                  getattr(b, k).cpu().numpy().view(np.uint8)), k

    def test_run_scene_pipeline_api(self, tmp_path):
        """tests/test_cli.py:164-199 scene KATs, through run_scene_pipeline."""
        obj = tmp_path / "quad.obj"
        obj.write_text("v -2 -2 -2\nv 2 -2 -2\nv 2 2 -2\nv -2 2 -2\nf 1 2 3 4\n")
        cfg = fa.SceneConfig(mesh_path=obj, fov_y_deg=90, near=0.1, far=100, screen=(128, 128), omega=256)
        res = fa.run_scene_pipeline(cfg)
        assert res.chart_set.n_charts == 1 and len(res.layout.placements) == 1
        p = res.layout.placements[0]
        assert 120 <= p.w <= 130 and 120 <= p.h <= 130
        assert res.stretch.l2 == pytest.approx(1.0, abs=0.02)
        assert res.chart_set.chart_of_triangle[0] == 0 and res.chart_set.vertex_to_chart[0] == 0
        cfg.omega = 64
        assert fa.run_scene_pipeline(cfg).stretch.l2 == pytest.approx(2.0, abs=0.1)
        cfg.look_at = (0, 0, 1)
        with pytest.raises(fa.NothingVisible):
            fa.run_scene_pipeline(cfg)


# ------------------------------------------- frames with comparison packers ---
def _packer_case(key):
    m = next(x for x in meta()["frames_packers"] if f"{x['packer']}/{x['name']}" == key)
    g = group(npz("frames_packers.npz"), key)
    if m["name"].startswith("C"):
        s = scenes.build_scene(m["name"])
        pos, tris = s.positions, s.triangles
    else:  # every mini frame renders the same mini scene
        mini = group(npz("frames.npz"), "mini_v0")
        pos, tris = mini["pos"], mini["tris"]
    return m, g, pos, tris


class TestFramePackers:
    """run_scene_pipeline(cfg, packer=...) with the comparison packers of
    make_packer (cli.py:318-339,386-387) vs the reference frame."""

    @pytest.mark.parametrize("key", [f"{m['packer']}/{m['name']}" for m in meta()["frames_packers"]])
    def test_frame_vs_reference(self, key):
        m, g, pos, tris = _packer_case(key)
        settings = FrameSettings(screen=tuple(m["screen"]), omega=m["omega"], min_dim=m["min_dim"],
                                 padding=m["padding"], prescale=m["prescale"], uv_f64=True, packer=m["packer"])
        eng = FrameEngine(fa.Mesh(pos, tris), settings=settings)
        if m["status"] == "ValueError":
            with pytest.raises(ValueError):
                eng.run(g["vp"])
            return
        out = eng.run(g["vp"], check=False)
        if m["status"] == "PackFailure":
            assert out.status == 2
            return
        assert out.status == 0
        h = out.to_host()
        assert np.array_equal(h["roots"].astype(np.int64), g["box_roots"])
        assert np.array_equal(h["target"], g["target"])
        assert np.array_equal(h["placements"], g["placements"])
        assert [out.scale.numerator, out.scale.denominator] == g["scale"].tolist()
        assert out.texels_allocated == m["texels_allocated"]
        assert out.screen_fragments == m["screen_fragments"]
        assert fa.layout_digest(out.layout()).digest == m["digest"]
        if m.get("stretch") is None:
            assert out.stretch() is None
        else:
            st = out.stretch()
            assert st.l2 == pytest.approx(m["stretch"][0], rel=1e-9)
            assert st.linf == pytest.approx(m["stretch"][1], rel=1e-9)
        pos_of = {int(t): k for k, t in enumerate(h["visible"])}
        rows = np.array([pos_of[int(t)] for t in g["uv_tris"]], dtype=np.int64)
        assert same_bits(h["uv"][rows], g["uv"])
        mask = np.ones(len(h["visible"]), bool)
        mask[rows] = False
        assert np.all(np.isnan(h["uv"][mask]))

    def test_engine_switches_packers(self):
        """One engine alternating the graphed FastAtlas frame and an ungraphed
        comparison frame: each result equals a fresh engine's."""
        m, g, pos, tris = _packer_case("sequential/mini_v0")
        base = dict(screen=tuple(m["screen"]), omega=m["omega"], uv_f64=True)
        eng = FrameEngine(fa.Mesh(pos, tris))
        a = eng.run(g["vp"], FrameSettings(**base)).clone()
        b = eng.run(g["vp"], FrameSettings(packer="sequential", **base)).clone()
        c = eng.run(g["vp"], FrameSettings(**base))
        assert np.array_equal(b.placements.cpu().numpy(), g["placements"])
        for k in ("placements", "uv"):
            assert np.array_equal(getattr(a, k).cpu().numpy().view(np.uint8), getattr(c, k).cpu().numpy().view(np.uint8))

    def test_run_scene_pipeline_packer_argument(self, tmp_path):
        """The packer argument reaches the frame; an unknown name is InputError
        only after the NothingVisible check (cli.py:366-368 before :386)."""
        obj = tmp_path / "quad.obj"
        obj.write_text("v -2 -2 -2\nv 2 -2 -2\nv 2 2 -2\nv -2 2 -2\nf 1 2 3 4\n")
        cfg = fa.SceneConfig(mesh_path=obj, fov_y_deg=90, near=0.1, far=100, screen=(128, 128), omega=256)
        ref = {p: fa.run_scene_pipeline(cfg, packer=p).layout for p in ("fastatlas", "sequential", "superblock")}
        assert ref["sequential"].scale == 1 and len(ref["superblock"].placements) == 1
        from paper_2502_17712_b200.cli import InputError
        with pytest.raises(InputError):
            fa.run_scene_pipeline(cfg, packer="nope")
        cfg.look_at = (0, 0, 1)
        with pytest.raises(fa.NothingVisible):
            fa.run_scene_pipeline(cfg, packer="nope")


# ------------------------------------------------- full-size configurations ---
def _scene_vp(spec, pose):
    cam = fa.CameraFrame.from_params(math.radians(pose.fov_y_deg), spec.screen[0] / spec.screen[1], pose.near,
                                     pose.far, position=pose.position, look_at=pose.look_at, up=pose.up)
    return cam.view_proj


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_size_vs_oracle(cfg):
    spec = scenes.build_scene(cfg)
    vp = _scene_vp(spec, spec.poses[0])
    eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                      settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale,
                                             uv_f64=True))
    h = eng.run(vp).to_host()
    r = oracle.run_frame(spec.positions, spec.triangles, vp, spec.screen, spec.omega, prescale=spec.prescale)
    assert np.array_equal(h["flags"].astype(bool), r.flags)
    assert np.array_equal(h["chart_of_triangle"].astype(np.int64), r.chart_of_triangle)
    assert np.array_equal(h["vertex_to_chart"].astype(np.int64), r.vertex_to_chart)
    assert np.array_equal(h["placements"], r.pack.placements)
    assert (h["scale"].numerator, h["scale"].denominator) == r.pack.scale
    assert same_bits(h["uv"], r.uv)
    assert h["screen_fragments"] == r.screen_fragments
    # size-independent properties: placements inside the atlas and disjoint
    p = h["placements"]
    om = spec.omega
    assert np.all(p[:, 1] >= 0) and np.all(p[:, 2] >= 0)
    assert np.all(p[:, 1] + p[:, 3] <= om) and np.all(p[:, 2] + p[:, 4] <= om)
    grid = np.zeros((om, om), np.int32)
    for q in p:
        grid[q[2]:q[2] + q[4], q[1]:q[1] + q[3]] += 1
    assert grid.max() <= 1


def test_stretch_sums_are_reproducible():
    """k_uv adds its per-block stretch partials in a fixed order (last block),
    so repeated frames report bit-identical L2 / Linf stretch."""
    spec = scenes.build_scene("C2")
    eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                      settings=FrameSettings(screen=spec.screen, omega=spec.omega))
    vp = _scene_vp(spec, spec.poses[0])
    seen = set()
    for _ in range(5):
        st = eng.run(vp).stretch()
        seen.add((np.float64(st.l2).tobytes(), np.float64(st.linf).tobytes()))
    assert len(seen) == 1


def _check_vs_oracle(h, r, status_ok=True):
    assert np.array_equal(h["flags"].astype(bool), r.flags)
    assert np.array_equal(h["chart_of_triangle"].astype(np.int64), r.chart_of_triangle)
    assert np.array_equal(h["vertex_to_chart"].astype(np.int64), r.vertex_to_chart)
    if status_ok:
        assert np.array_equal(h["placements"], r.pack.placements)
        assert (h["scale"].numerator, h["scale"].denominator) == r.pack.scale
        assert same_bits(h["uv"], r.uv)
        assert h["screen_fragments"] == r.screen_fragments
        assert h["texels_allocated"] == r.texels_allocated


@pytest.mark.parametrize("cfg,idx", [("C4", 0), ("C4", 59), ("C4", 119), ("C5", 0), ("C5", 1), ("C5", 2),
                                     ("C5", 37)])
def test_camera_path_and_views_vs_oracle(cfg, idx):
    """C4 (120-frame path) and C5 (64 streaming views) poses on the 1M-triangle scene."""
    spec = scenes.build_scene(cfg)
    vp = _scene_vp(spec, spec.poses[idx])
    eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                      settings=FrameSettings(screen=spec.screen, omega=spec.omega, uv_f64=True))
    h = eng.run(vp).to_host()
    r = oracle.run_frame(spec.positions, spec.triangles, vp, spec.screen, spec.omega)
    assert r.status == oracle.OK
    _check_vs_oracle(h, r)


def test_no_cull_frame_vs_oracle():
    """backface_cull=False (charts.py:216-219 flips clockwise polygons)."""
    fpos, ftris, rng = scenes.sphere_field(1)
    pos, tris = scenes._merge((fpos, ftris), scenes.ground_plane(20, 16, rng=rng))
    spec = scenes.build_scene("C1")
    vp = _scene_vp(spec, scenes.views_c5(8)[3])
    eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=(300, 200), omega=256, uv_f64=True,
                                                                 backface_cull=False, padding=1, min_dim=2))
    out = eng.run(vp, check=False)
    r = oracle.run_frame(pos, tris, vp, (300, 200), 256, min_dim=2, padding=1, cull=False)
    assert out.status == r.status
    _check_vs_oracle(out.to_host(), r, status_ok=r.status == oracle.OK)


def test_height_overflow_frame():
    """A prescale pushing a chart box past 2^23 raises HeightOverflow like order() (packing.py:127-129)."""
    m, g, pos, tris = _frame_case("mini_v0")
    eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=tuple(m["screen"]), omega=m["omega"],
                                                                 prescale=1e6))
    with pytest.raises(fa.HeightOverflow):
        eng.run(g["vp"])


@pytest.mark.parametrize("frac", [0.18, 0.5])
def test_union_find_under_contention(frac):
    """Random visibility on the 4M-triangle mesh: many small components and
    heavy hook contention; repeated runs must equal the oracle every time."""
    spec = scenes.build_scene("C3")
    T = len(spec.triangles)
    lab0 = np.where(np.random.default_rng(0).random(T) < frac, np.arange(T), -1)
    ref, ref_v2c = oracle.merge_shared_vertices(spec.triangles, len(spec.positions), lab0)
    mesh = fa.Mesh(spec.positions, spec.triangles)
    for _ in range(3):
        cs = fa.merge_shared_vertices(fa.ChartSet(lab0), mesh)
        assert np.array_equal(cs.chart_of_triangle, ref)
        assert np.array_equal(cs.vertex_chart_array, ref_v2c)


# ---------------------------------------------- comparison packers (§8f-4) ---
def _bl_cases():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "baselines.json")) as fh:
        return json.load(fh)


def _plc(lay):
    return [[p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h] for p in lay.placements]


class TestBaselines:
    def test_sequential_scale_search_vs_reference(self):
        from paper_2502_17712_b200.baselines import sequential_scale_search
        for c in _bl_cases()["sequential"]:
            boxes = [fa.ChartBox(*b) for b in c["boxes"]]
            if c["status"] != "ok":
                with pytest.raises(fa.PackFailure):
                    sequential_scale_search(boxes, c["omega"], c["n_scales"], c["min_dim"], c["padding"])
                continue
            lay = sequential_scale_search(boxes, c["omega"], c["n_scales"], c["min_dim"], c["padding"])
            assert [lay.scale.numerator, lay.scale.denominator] == c["scale"]
            assert _plc(lay) == c["placements"]

    def test_superblock_vs_reference(self):
        from paper_2502_17712_b200.baselines import SuperblockConfig, superblock_pack
        for c in _bl_cases()["superblock"]:
            boxes = [fa.ChartBox(*b) for b in c["boxes"]]
            lay = superblock_pack(boxes, c["omega"], SuperblockConfig(c["block_size"], c["halving"]))
            if c["status"] != "ok":
                assert lay is None
                continue
            assert lay.block_size == c["block_used"]
            assert [lay.scale.numerator, lay.scale.denominator] == c["scale"]
            assert _plc(lay) == c["placements"]

    def test_sequential_fold_and_pack_vs_reference(self):
        from paper_2502_17712_b200.baselines import sequential_fold, sequential_pack
        for c in _bl_cases()["prim"]:
            f = sequential_fold(c["widths"], c["omega"])
            assert f.row_of_box.tolist() == c["rows"] and f.x_of_box.tolist() == c["x"]
            ordered = [fa.OrientedBox(w=o[0], h=o[1], rotated=False, source=fa.ChartBox(o[0], o[1], o[2], o[2]))
                       for o in c["ordered"]]
            lay = sequential_pack(ordered, c["omega"])
            if c["pack"] is None:
                assert lay is None
            else:
                assert [[p.chart_id, p.x, p.y, p.w, p.h] for p in lay.placements] == c["pack"]

    def test_make_packer_registry(self):
        from paper_2502_17712_b200.cli import make_packer
        c = next(c for c in _bl_cases()["sequential"] if c["status"] == "ok")
        boxes = [fa.ChartBox(*b) for b in c["boxes"]]
        for name in ("fastatlas", "sequential"):
            lay = make_packer(name, 64, 1, 0)(boxes, c["omega"])
            assert len(lay.placements) == len(boxes)
        sb = next(s for s in _bl_cases()["superblock"] if s["status"] == "ok")
        lay = make_packer("superblock", 64, 1, 0, block_size=sb["block_size"])(
            [fa.ChartBox(*b) for b in sb["boxes"]], sb["omega"])
        assert _plc(lay) == sb["placements"]
        bad = next(s for s in _bl_cases()["superblock"] if s["status"] != "ok" and s["halving"])
        with pytest.raises(fa.PackFailure):
            make_packer("superblock", 64, 1, 0, block_size=bad["block_size"])(
                [fa.ChartBox(*b) for b in bad["boxes"]], bad["omega"])


@pytest.mark.parametrize("order", ["1", "0"])
def test_shuffled_vertices_and_unused_vertices(order, monkeypatch):
    """fa_set_mesh renumbers vertices in order of first use (FASTATLAS_VERTEX_ORDER=1,
    the default) or keeps the caller's numbering (=0); with shuffled vertex ids
    and vertices no triangle uses, every output -- the per-vertex map in the
    caller's numbering included (unused vertices -1) -- equals the oracle's."""
    monkeypatch.setenv("FASTATLAS_VERTEX_ORDER", order)
    spec = scenes.build_scene("C1")
    rng = np.random.default_rng(5)
    V = len(spec.positions)
    extra = rng.normal(size=(300, 3))                      # never referenced
    pos = np.vstack([spec.positions, extra])
    perm = rng.permutation(len(pos))                       # new id of each old vertex
    pos_s = np.empty_like(pos)
    pos_s[perm] = pos
    tris_s = perm[spec.triangles.astype(np.int64)].astype(np.int32)
    vp = _scene_vp(spec, spec.poses[0])
    eng = FrameEngine(fa.Mesh(pos_s, tris_s), settings=FrameSettings(screen=spec.screen, omega=spec.omega,
                                                                      uv_f64=True))
    h = eng.run(vp).to_host()
    r = oracle.run_frame(pos_s, tris_s, vp, spec.screen, spec.omega)
    _check_vs_oracle(h, r)
    assert np.all(h["vertex_to_chart"][perm[V:]] == -1)


# ------------------------------------------------------------ mesh binding ---
def test_in_place_mesh_update_is_rebound():
    """A deforming mesh: updating the engine's device positions in place
    rebinds the mesh (torch version counter), and the frame equals a fresh
    engine's frame of the moved mesh."""
    m, g, pos, tris = _frame_case("mini_v0")
    st = FrameSettings(screen=tuple(m["screen"]), omega=m["omega"], uv_f64=True)
    eng = FrameEngine(fa.Mesh(pos, tris), settings=st)
    eng.run(g["vp"])
    moved = pos + np.array([0.05, -0.02, 0.03])
    eng.pos.copy_(eng.pos.new_tensor(moved))
    a = eng.run(g["vp"]).clone()
    b = FrameEngine(fa.Mesh(moved, tris), settings=st).run(g["vp"])
    for k in ("flags", "chart_of_triangle", "placements", "uv"):
        assert np.array_equal(getattr(a, k).cpu().numpy().view(np.uint8), getattr(b, k).cpu().numpy().view(np.uint8)), k


def test_invalid_mesh_leaves_no_mesh_bound():
    """fa_set_mesh validates indices on the device before binding; a failed
    bind leaves an empty mesh (frames see nothing), never the invalid one."""
    import ctypes
    import torch
    from paper_2502_17712_b200 import _native as nat
    ctx = nat.Context(0)
    pos = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    for bad in ([[0, 1, 4]], [[0, -1, 2]]):
        tri = torch.tensor(bad, dtype=torch.int32, device="cuda")
        code = ctx.L.fa_set_mesh(ctx.h, ctypes.c_void_p(pos.data_ptr()), 4, ctypes.c_void_p(tri.data_ptr()), 1)
        assert code == nat.FA_VALUE_ERROR and b"out of range" in ctx.L.fa_last_error()
        p = FrameSettings(screen=(8, 8), omega=16).params()
        res = nat.FrameResult()
        vp = np.eye(4)
        code = ctx.L.fa_frame(ctx.h, vp.ctypes.data_as(ctypes.c_void_p), ctypes.byref(p), ctypes.byref(res),
                              ctx.stream_ptr())
        assert code == nat.FA_NOTHING_VISIBLE


@pytest.mark.parametrize("seed", range(16))
def test_random_frames_vs_oracle(seed):
    """Seeded random frames: sphere fields (icosphere level 1-2, jittered by
    the seed) over a ground plane, a random camera (sometimes inside the field
    or grazing the plane, so the near plane and the frustum sides clip), a
    random screen and atlas, cull on/off, min_dim/padding; the whole CUDA
    frame against the C oracle (status, depth, flags, charts, placements, f64
    UVs)."""
    rng = np.random.default_rng(1000 + seed)
    fpos, ftris, frng = scenes.sphere_field(int(rng.integers(1, 3)), seed=seed)
    pos, tris = scenes._merge((fpos, ftris), scenes.ground_plane(int(rng.integers(4, 24)), int(rng.integers(4, 24)),
                                                                 rng=frng))
    W, H = int(rng.integers(48, 700)), int(rng.integers(48, 500))
    omega = int(2 ** rng.integers(7, 12))
    eye = np.array([rng.uniform(-7, 7), rng.uniform(-1.2, 4.0), rng.uniform(-12, 6)])
    target = np.array([rng.uniform(-5, 5), rng.uniform(-1.3, 0.5), rng.uniform(-12, -3)])
    if np.linalg.norm(target - eye) < 1e-3:
        target = eye + np.array([0.0, 0.0, -1.0])
    near = float(rng.choice([0.01, 0.1, 0.5, 1.5]))
    cam = fa.CameraFrame.from_params(math.radians(rng.uniform(25, 110)), W / H, near, near + rng.uniform(5, 60),
                                     position=eye, look_at=target, up=(0.0, 1.0, 0.0))
    cull = bool(rng.integers(0, 4) > 0)
    min_dim, padding = int(rng.integers(1, 4)), int(rng.integers(0, 3))
    eng = FrameEngine(fa.Mesh(pos, tris), settings=FrameSettings(screen=(W, H), omega=omega, uv_f64=True,
                                                                 backface_cull=cull, padding=padding, min_dim=min_dim))
    out = eng.run(cam.view_proj, check=False)
    r = oracle.run_frame(pos, tris, cam.view_proj, (W, H), omega, min_dim=min_dim, padding=padding, cull=cull)
    assert out.status == r.status
    if r.status == oracle.NOTHING_VISIBLE:
        return
    _check_vs_oracle(out.to_host(), r, status_ok=r.status == oracle.OK)
