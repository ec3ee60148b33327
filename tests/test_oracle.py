"""Pin the C oracle (oracle/fa_oracle.c) against the reference's golden vectors.

CPU only.  Every golden vector was produced by the unmodified reference
(tests/golden/make_golden.py); the oracle must reproduce it bit for bit.
"""

import json
import os

import numpy as np
import pytest

import oracle
from goldens import GOLDEN, canon, group, meta, npz, pack_cases, same_bits


@pytest.fixture(scope="module", autouse=True)
def _built():
    oracle.build()


class TestRaster:
    @pytest.mark.parametrize("case", [m["name"] for m in meta()["raster"]])
    def test_depth_and_flags_bit_exact(self, case):
        m = next(x for x in meta()["raster"] if x["name"] == case)
        g = group(npz("raster.npz"), case)
        depth = oracle.depth_prepass(g["pos"], g["tris"], g["vp"], m["res"], m["cull"])
        assert same_bits(canon(depth), g["depth"])
        flags = oracle.mark_visible(g["pos"], g["tris"], g["vp"], depth, m["cull"])
        assert np.array_equal(flags, g["flags"])

    def test_kat_flags(self):
        """tests/test_charts.py:122-159 expectations restated."""
        d = npz("raster.npz")
        assert group(d, "occluded")["flags"].tolist() == [True, True, False]
        assert not group(d, "subpixel")["flags"][0]
        assert group(d, "offscreen_corner")["flags"][0]
        assert not group(d, "backface_cull")["flags"][0]
        assert group(d, "backface_nocull")["flags"][0]

    def test_empty_mesh_all_inf(self):
        depth = oracle.depth_prepass(np.zeros((0, 3)), np.zeros((0, 3), np.int64), np.eye(4), (16, 8))
        assert depth.shape == (8, 16) and np.all(np.isinf(depth))

    def test_bad_resolution(self):
        with pytest.raises(ValueError):
            oracle.depth_prepass(np.zeros((0, 3)), np.zeros((0, 3), np.int64), np.eye(4), (0, 8))


class TestCharts:
    @pytest.mark.parametrize("case", meta()["charts"])
    def test_components(self, case):
        g = group(npz("charts.npz"), case)
        adj = oracle.build_adjacency(g["tris"])
        assert np.array_equal(adj, g["adj"])
        pre = oracle.connected_charts(adj, g["flags"])
        assert np.array_equal(pre, g["pre"])
        merged, v2c = oracle.merge_shared_vertices(g["tris"], len(g["pos"]), pre)
        assert np.array_equal(merged, g["merged"])
        assert np.array_equal(v2c, g["v2c"])
        roots = np.flatnonzero(merged == np.arange(len(merged)))
        assert np.array_equal(roots, g["roots"])


class TestBounds:
    def test_chart_bbox_bit_exact(self):
        g = npz("bounds.npz")
        for i in range(len(g["tris"])):
            tri = g["tris"][i]
            tri = tri[~np.isnan(tri[:, 0, 0])]
            box = oracle.chart_bbox(tri, g["vps"][g["cam"][i]])
            if g["degenerate"][i]:
                assert box is None
            else:
                assert box is not None
                assert np.array_equal(np.array(box), g["boxes"][i]), i

    def test_viewport_box(self):
        g = npz("bounds.npz")
        for row, want in zip(g["vb_in"], g["vb_out"]):
            assert oracle.viewport_box(row[:4], int(row[4]), int(row[5])) == tuple(want)

    def test_viewport_kats(self):
        """tests/test_geometry.py:214-222."""
        assert oracle.viewport_box([-1, -1, 1, 1], 1920, 1080) == (1920, 1080)
        assert oracle.viewport_box([0, 0, 1, 1], 256, 256) == (128, 128)
        assert oracle.viewport_box([0.25, -0.5, 0.25, -0.5], 640, 480) == (1, 1)


STATUS = {"ok": oracle.OK, "PackFailure": oracle.PACK_FAILURE, "ValueError": oracle.VALUE_ERROR,
          "HeightOverflow": oracle.HEIGHT_OVERFLOW}


class TestPack:
    @pytest.mark.parametrize("idx", range(len(pack_cases()["pack"])))
    def test_pack_cases(self, idx):
        c = pack_cases()["pack"][idx]
        b = np.array(c["boxes"], dtype=np.int64).reshape(-1, 4)
        r = oracle.pack(b[:, 0], b[:, 1], b[:, 2], b[:, 3], c["omega"], c["n_scales"], c["min_dim"],
                        c["padding"], want_accept=c.get("accept") is not None)
        assert r.status == STATUS[c["status"]], c["tag"]
        if c["status"] != "ok":
            return
        assert list(r.scale) == c["scale"]
        assert r.placements.tolist() == c["placements"]
        if c.get("accept") is not None and len(b):
            assert r.accept.astype(bool).tolist() == c["accept"]

    def test_fold_and_push_up(self):
        for rec in pack_cases()["prim"]:
            if rec["kind"] != "fold":
                continue
            rows, xs, m = oracle.fold(rec["widths"], rec["omega"])
            assert rows.tolist() == rec["rows"] and xs.tolist() == rec["x"] and m == rec["m"]
            if "y" in rec:
                y, used = oracle.push_up(rows, xs, rec["widths"], rec["heights"], rec["omega"])
                assert y.tolist() == rec["y"] and used == rec["used"]

    def test_pack_at_scale(self):
        for rec in pack_cases()["prim"]:
            if rec["kind"] != "pack_at_scale":
                continue
            o = np.array(rec["ordered"], dtype=np.int64).reshape(-1, 7)
            r = oracle.pack_arrays(o[:, 0], o[:, 1], rec["num"], rec["den"], rec["omega"],
                                   rec["min_dim"], rec["padding"])
            if rec["result"] is None:
                assert r is None
                continue
            assert r is not None
            assert [r["num"], r["den"]] == rec["result"]["scale"]
            got = [[int(o[i, 5]), int(r["x"][i]), int(r["y"][i]), int(r["w"][i]), int(r["h"][i]),
                    int(o[i, 2]), int(o[i, 3]), int(o[i, 4])] for i in range(len(o))]
            assert got == rec["result"]["placements"]

    def test_kats(self):
        """tests/test_packing.py:337-411 fold / push-up KATs."""
        rows, xs, m = oracle.fold([4, 4, 4, 4], 8)
        assert rows.tolist() == [0, 0, 1, 1] and xs.tolist() == [0, 4, 4, 0] and m == 0
        assert oracle.fold([5, 5], 8)[2] == 2
        rows, xs, _ = oracle.fold([4, 4, 4, 4], 8)
        y, used = oracle.push_up(rows, xs, [4] * 4, [10, 3, 3, 2], 8)
        assert y.tolist() == [0, 0, 3, 10] and used == 12


class TestFrames:
    @pytest.mark.parametrize("case", [m["name"] for m in meta()["frames"]])
    def test_frame_bit_exact(self, case):
        m = next(x for x in meta()["frames"] if x["name"] == case)
        g = group(npz("frames.npz"), case)
        if case.startswith("C"):
            from paper_2502_17712_b200 import scenes
            s = scenes.build_scene(case)
            pos, tris = s.positions, s.triangles
        else:
            pos, tris = g["pos"], g["tris"]
        r = oracle.run_frame(pos, tris, g["vp"], m["screen"], m["omega"], 64, m["min_dim"], m["padding"],
                             m["prescale"])
        assert same_bits(canon(r.depth), g["depth"])
        assert np.array_equal(r.flags, g["flags"])
        if m["status"] == "NothingVisible":
            assert r.status == oracle.NOTHING_VISIBLE
            return
        assert np.array_equal(r.chart_of_triangle, g["chart_of_triangle"])
        assert np.array_equal(r.vertex_to_chart, g["vertex_to_chart"])
        assert np.array_equal(r.boxes.roots, g["box_roots"])
        assert np.array_equal(r.boxes.target, g["target"])
        if m["status"] == "PackFailure":
            assert r.status == oracle.PACK_FAILURE
            return
        assert same_bits(r.boxes.ndc, g["ndc"])
        assert np.array_equal(r.boxes.px, g["px"])
        assert r.status == oracle.OK
        assert np.array_equal(r.pack.placements, g["placements"])
        assert list(r.pack.scale) == g["scale"].tolist()
        assert r.screen_fragments == m["screen_fragments"]
        assert r.texels_allocated == m["texels_allocated"]
        # UVs: reference emits rows in (chart, member) order; map through tri ids
        vis_list = np.flatnonzero(r.flags)
        pos_of = {int(t): k for k, t in enumerate(vis_list)}
        rows = np.array([pos_of[int(t)] for t in g["uv_tris"]], dtype=np.int64)
        assert same_bits(r.uv[rows], g["uv"])
        mask = np.ones(len(vis_list), bool)
        mask[rows] = False
        assert np.all(np.isnan(r.uv[mask]))


