"""Generate golden vectors by running the REFERENCE atlaspack package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py [--c2]

It imports the unmodified reference from /root/reference/pkg/src, feeds it
seeded inputs (scene generators in paper_2502_17712_b200/scenes.py plus the
random-input recipes of /root/reference/pkg/tests), and writes small
fixtures next to this script.  The fixtures pin the C oracle
(tests/test_oracle.py, CPU) and, through it, the CUDA product
(tests/test_gpu_*.py on a B200).  Camera matrices are stored in the
fixtures so the GPU box never recomputes them with its own BLAS.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import tempfile
import time
from fractions import Fraction

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import atlaspack as ap  # noqa: E402  (the reference)
from atlaspack import cli as apcli  # noqa: E402
from atlaspack.cli import generate_boxes  # noqa: E402

from paper_2502_17712_b200 import scenes  # noqa: E402


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def canon_depth(d):
    """Depth bits with -0.0 folded to +0.0 (np.minimum's zero sign is order dependent)."""
    d = np.array(d, dtype=np.float64, copy=True)
    d[d == 0] = 0.0
    return d


def cam(fov_deg, aspect, near, far, pos=(0, 0, 0), look=(0, 0, -1), up=(0, 1, 0)):
    return ap.CameraFrame.from_params(math.radians(fov_deg), aspect, near, far, position=pos,
                                      look_at=look, up=up)


# ---------------------------------------------------------------- raster ----

def raster_cases():
    rng = np.random.default_rng(20240811)
    cases = []

    def flat(tris, coords, z):
        coords = np.asarray(coords, dtype=np.float64)
        return np.column_stack([coords, np.full(len(coords), z)]), np.asarray(tris, dtype=np.int64)

    def quad(z, half=2.0):
        s = half * abs(z)
        return flat([(0, 1, 2), (0, 2, 3)], [(-s, -s), (s, -s), (s, s), (-s, s)], z)

    c90 = cam(90, 1.0, 0.1, 100.0)
    # KAT scenes restated from tests/test_charts.py:98-159
    p, t = quad(-1.0)
    cases.append(("screen_quad", p, t, c90, (32, 32), True))
    pn, tn = quad(-1.0)
    pf, tf = quad(-5.0)
    cases.append(("overlap", np.vstack([pn, pf]), np.vstack([tn, tf + 4]), c90, (16, 16), True))
    pb, tb = flat([(0, 1, 2)], [(-0.5, -0.5), (0.5, -0.5), (0.0, 0.5)], -5.0)
    cases.append(("occluded", np.vstack([pn, pb]), np.vstack([tn, tb + 4]), c90, (32, 32), True))
    p, t = flat([(0, 1, 2)], [(0.02, 0.02), (0.05, 0.02), (0.03, 0.05)], -1.0)
    cases.append(("subpixel", p, t, c90, (8, 8), True))
    p, t = flat([(0, 1, 2)], [(-3.0, -0.9), (-0.8, -0.9), (-0.8, -0.8)], -1.0)
    cases.append(("offscreen_corner", p, t, c90, (8, 8), True))
    p, t = flat([(0, 1, 2)], [(-1.0, -1.0), (0.0, 1.0), (1.0, -1.0)], -2.0)
    cases.append(("backface_cull", p, t, c90, (16, 16), True))
    cases.append(("backface_nocull", p, t, c90, (16, 16), False))
    # random soups around the camera: every clip plane, near crossings, w<0
    for k in range(6):
        n = 150
        tri = rng.normal(scale=2.0, size=(n, 3, 3))
        tri[:, :, 2] -= rng.uniform(0.0, 3.0)
        p = tri.reshape(-1, 3)
        t = np.arange(3 * n, dtype=np.int64).reshape(-1, 3)
        W, H = [(40, 30), (64, 48), (33, 17), (48, 48), (25, 40), (64, 64)][k]
        cc = cam(50 + 10 * k, W / H, 0.1, 50.0, pos=(0.1 * k, 0.2, 0.5), look=(0, 0, -3))
        cases.append((f"soup{k}", p, t, cc, (W, H), bool(k % 2 == 0)))
    # shared-vertex grids (exercise the top-left rule on shared edges)
    for k in range(3):
        pos, tris = scenes.ground_plane(12 + k, 9 + k, y=-1.0, span=2.0, center_z=-3.0,
                                        jitter=0.05 * k, rng=np.random.default_rng(k))
        cc = cam(70, 1.25, 0.1, 100.0, pos=(0.0, 0.8, 0.0), look=(0.0, -1.0, -3.0))
        cases.append((f"grid{k}", pos, tris, cc, (40, 32), True))
    # a sphere with exact pixel-centre-aligned geometry avoided by jitter
    pos, tris = scenes.icosphere(2, center=(0.1, -0.2, -3.0), radius=1.0)
    cases.append(("sphere", pos, tris, cam(60, 1.5, 0.1, 100.0), (60, 40), True))
    return cases


def gen_raster(out):
    arrays, meta = {}, []
    for name, pos, tris, camf, res, cull in raster_cases():
        mesh = ap.Mesh(positions=pos, triangles=tris)
        depth = ap.depth_prepass(mesh, camf, res, backface_cull=cull)
        vis = ap.mark_visible(mesh, camf, depth, backface_cull=cull)
        arrays[f"{name}/pos"] = mesh.positions
        arrays[f"{name}/tris"] = mesh.triangles
        arrays[f"{name}/vp"] = camf.view_proj
        arrays[f"{name}/depth"] = canon_depth(depth)
        arrays[f"{name}/flags"] = vis.flags
        meta.append(dict(name=name, res=list(res), cull=cull))
    np.savez_compressed(os.path.join(out, "raster.npz"), **arrays)
    return meta


# ---------------------------------------------------------------- charts ----

def delaunay_mesh(rng, n_points, z=-5.0):
    from scipy.spatial import Delaunay
    pts = rng.random((max(n_points, 4), 2)) * 4.0 - 2.0
    tri = Delaunay(pts)
    positions = np.column_stack([pts, np.full(len(pts), z)])
    return positions, np.asarray(tri.simplices, dtype=np.int64)


def gen_charts(out):
    rng = np.random.default_rng(20240811)
    arrays, meta = {}, []
    specs = [(int(rng.integers(5, 120)), 0.6) for _ in range(30)]
    specs += [(200, 0.3), (300, 0.9), (50, 1.0), (20, 0.0)]
    for i, (npts, frac) in enumerate(specs):
        pos, tris = delaunay_mesh(rng, npts)
        if i % 5 == 4 and len(tris) > 3:
            # non-manifold fan: three triangles on one edge
            extra = np.array([[tris[0, 0], tris[0, 1], tris[1, 2]]], dtype=np.int64)
            tris = np.vstack([tris, extra])
        mesh = ap.Mesh(positions=pos, triangles=tris)
        flags = rng.random(mesh.n_triangles) < frac
        vis = ap.VisibilityBuffer(flags=flags, sample_res=(8, 8))
        pre = ap.connected_charts(mesh, vis)
        merged = ap.merge_shared_vertices(pre, mesh)
        v2c = np.full(len(pos), -1, dtype=np.int64)
        for v, c in merged.vertex_to_chart.items():
            v2c[v] = c
        k = f"m{i}"
        arrays[f"{k}/pos"] = pos
        arrays[f"{k}/tris"] = mesh.triangles
        arrays[f"{k}/adj"] = mesh.adjacency
        arrays[f"{k}/flags"] = flags
        arrays[f"{k}/pre"] = pre.chart_of_triangle
        arrays[f"{k}/merged"] = merged.chart_of_triangle
        arrays[f"{k}/v2c"] = v2c
        arrays[f"{k}/roots"] = np.array(list(merged.charts.keys()), dtype=np.int64)
        meta.append(k)
    np.savez_compressed(os.path.join(out, "charts.npz"), **arrays)
    return meta


# ---------------------------------------------------------------- bounds ----

def gen_bounds(out):
    rng = np.random.default_rng(7)
    c90 = cam(90, 1.0, 0.1, 100.0)
    cams = [c90, cam(65, 1.5, 0.05, 500.0, pos=(3, -2, 8), look=(0, 1, 0))]
    arrays = {}
    tris_all, cam_idx, boxes, degen = [], [], [], []
    for ci, cc in enumerate(cams):
        for _ in range(1500):
            n = int(rng.integers(1, 4))
            tri = rng.normal(scale=2.0 if ci == 0 else 6.0, size=(n, 3, 3))
            try:
                b = ap.chart_bbox(tri, cc)
                boxes.append([b.min_x, b.min_y, b.max_x, b.max_y])
                degen.append(False)
            except ap.DegenerateChart:
                boxes.append([np.nan] * 4)
                degen.append(True)
            pad = np.full((3, 3, 3), np.nan)
            pad[:n] = tri
            tris_all.append(pad)
            cam_idx.append(ci)
    arrays["tris"] = np.array(tris_all)
    arrays["cam"] = np.array(cam_idx)
    arrays["vps"] = np.array([c.view_proj for c in cams])
    arrays["boxes"] = np.array(boxes)
    arrays["degenerate"] = np.array(degen)
    # viewport KATs + random boxes (geometry.py:352-362)
    vb_in, vb_out = [], []
    for _ in range(500):
        a, b = np.sort(rng.uniform(-1, 1, 2)), np.sort(rng.uniform(-1, 1, 2))
        W, H = int(rng.integers(1, 4000)), int(rng.integers(1, 4000))
        box = ap.NdcBox(a[0], b[0], a[1], b[1])
        vb_in.append([a[0], b[0], a[1], b[1], W, H])
        vb_out.append(ap.viewport_box(box, W, H))
    arrays["vb_in"] = np.array(vb_in)
    arrays["vb_out"] = np.array(vb_out, dtype=np.int64)
    np.savez_compressed(os.path.join(out, "bounds.npz"), **arrays)


# ---------------------------------------------------------------- packing ---

def layout_rec(layout):
    return dict(
        scale=[layout.scale.numerator, layout.scale.denominator],
        placements=[[p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h]
                    for p in layout.placements],
        digest=ap.layout_digest(layout).digest,
    )


def gen_pack(out):
    rng = np.random.default_rng(123)
    cases = []

    def run(boxes, omega, n_scales=64, min_dim=1, padding=0, tag=""):
        rec = dict(tag=tag, omega=omega, n_scales=n_scales, min_dim=min_dim, padding=padding,
                   boxes=[[b.target_w, b.target_h, b.chart_id, b.min_tri] for b in boxes])
        try:
            lay = ap.pack(boxes, omega, n_scales=n_scales, min_dim=min_dim, padding=padding)
            rec.update(status="ok", **layout_rec(lay))
            ordered = ap.order(ap.orient(boxes))
            rec["accept"] = [
                ap.pack_at_scale(ordered, Fraction(i, n_scales), omega, min_dim, padding) is not None
                for i in range(1, n_scales + 1)] if n_scales <= 64 and len(boxes) <= 400 else None
        except ap.PackFailure:
            rec["status"] = "PackFailure"
        except ap.HeightOverflow:
            rec["status"] = "HeightOverflow"
        except ValueError:
            rec["status"] = "ValueError"
        cases.append(rec)

    box = lambda w, h, i: ap.ChartBox(target_w=w, target_h=h, chart_id=i, min_tri=i)  # noqa: E731
    # KATs from tests/test_packing.py
    run([box(10, 12, i) for i in range(8)], 256, tag="fit_full_scale")
    run([], 128, tag="empty")
    run([box(256, 256, i) for i in range(16)], 256, tag="sixteen_full")
    run([box(6400, 6400, 0)], 64, tag="floor_fail")
    run([ap.ChartBox(4, 4, 0, 7), ap.ChartBox(5, 5, 1, 7)], 64, tag="dup_min_tri")
    run([box(1000, 1000, 0)], 64, tag="iterated_overflow")
    run([box(32, 32, i) for i in range(4)], 64, tag="four_half")
    run([box(9000000, 3, 0)], 1 << 20, tag="height_overflow")
    for seed in range(40):
        run(generate_boxes(int(3 + seed % 20), 128, np.random.default_rng(seed)), 128, tag=f"rand128_{seed}")
    for seed in range(30):
        om = int(2 ** rng.integers(4, 12))
        cnt = int(rng.integers(1, 300))
        md = int(rng.integers(1, 4))
        pad = int(rng.integers(0, 3))
        ns = int(rng.choice([1, 7, 16, 64, 100]))
        run(generate_boxes(cnt, om, np.random.default_rng(1000 + seed)), om, ns, md, pad, tag=f"rand_{seed}")
    for cnt, om in [(1000, 2048), (2000, 4096), (3000, 2048), (10000, 2048), (10000, 8192)]:
        run(generate_boxes(cnt, om, np.random.default_rng(cnt + om)), om, tag=f"big_{cnt}_{om}")
    # chart-like boxes: many small boxes, a few large (pipeline-shaped)
    for seed in range(6):
        r = np.random.default_rng(50 + seed)
        n = int(r.integers(100, 1500))
        w = np.clip((r.pareto(1.5, n) * 4 + 1).astype(int), 1, 900)
        h = np.clip((r.pareto(1.5, n) * 4 + 1).astype(int), 1, 900)
        mt = np.sort(r.choice(n * 50, n, replace=False))
        run([ap.ChartBox(int(w[i]), int(h[i]), int(mt[i]), int(mt[i])) for i in range(n)], 2048,
            tag=f"chartlike_{seed}")

    # fold / push_up / pack_at_scale primitives
    prim = []
    for _ in range(300):
        omega = int(2 ** rng.integers(2, 10))
        n = int(rng.integers(1, 60))
        widths = np.clip((omega * rng.random(n) ** 3).astype(int), 1, omega)
        f = ap.fold(widths, omega)
        rec = dict(kind="fold", omega=omega, widths=widths.tolist(), rows=f.row_of_box.tolist(),
                   x=f.x_of_box.tolist(), m=f.overflow_m)
        if f.overflow_m == 0:
            hts = rng.integers(1, omega + 1, size=n)
            y, used = ap.push_up(f, np.stack([widths, hts], 1), omega)
            rec.update(heights=hts.tolist(), y=y.tolist(), used=used)
        prim.append(rec)
    for seed in range(60):
        r = np.random.default_rng(seed)
        om = int(2 ** r.integers(4, 10))
        boxes = generate_boxes(int(r.integers(1, 40)), om, r)
        ordered = ap.order(ap.orient(boxes))
        num, den = int(r.integers(1, 64)), 64
        md, pad = int(r.integers(1, 3)), int(r.integers(0, 3))
        lay = ap.pack_at_scale(ordered, Fraction(num, den), om, md, pad)
        prim.append(dict(kind="pack_at_scale", omega=om, num=num, den=den, min_dim=md, padding=pad,
                         ordered=[[b.w, b.h, int(b.rotated), b.source.target_w, b.source.target_h,
                                   b.source.chart_id, b.source.min_tri] for b in ordered],
                         result=None if lay is None else layout_rec(lay)))
    with open(os.path.join(out, "pack.json"), "w") as fh:
        json.dump(dict(pack=cases, prim=prim), fh)


# ---------------------------------------------------------------- frames ----

def write_obj(path, pos, tris):
    with open(path, "w") as fh:
        for p in pos:
            fh.write(f"v {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}\n")
        for t in tris:
            fh.write(f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}\n")


def run_reference_frame(pos, tris, pose, screen, omega, prescale=1.0, n_scales=64, min_dim=1,
                        padding=0, cull=True, packer="fastatlas"):
    """Run the reference run_scene_pipeline (cli.py:360-406) and capture its
    intermediate arrays and the UV pairs it hands to scene_stretch."""
    captured = {}
    orig_dp, orig_mv, orig_ss = apcli.depth_prepass, apcli.mark_visible, apcli.scene_stretch
    orig_msv, orig_mp = apcli.merge_shared_vertices, apcli.make_packer

    def msv(*a, **k):
        captured["cs"] = orig_msv(*a, **k)
        return captured["cs"]

    def mp(*a, **k):
        fn = orig_mp(*a, **k)

        def run(boxes, omega):
            captured["boxes"] = list(boxes)
            return fn(boxes, omega)
        return run

    def dp(*a, **k):
        captured["depth"] = orig_dp(*a, **k)
        return captured["depth"]

    def mv(*a, **k):
        captured["vis"] = orig_mv(*a, **k)
        return captured["vis"]

    def ss(pairs, *a, **k):
        pairs = list(pairs)
        captured["pairs"] = pairs
        return orig_ss(pairs, *a, **k)

    apcli.depth_prepass, apcli.mark_visible, apcli.scene_stretch = dp, mv, ss
    apcli.merge_shared_vertices, apcli.make_packer = msv, mp
    try:
        with tempfile.TemporaryDirectory() as td:
            write_obj(os.path.join(td, "m.obj"), pos, tris)
            cfg = apcli.SceneConfig(mesh_path=os.path.join(td, "m.obj"), fov_y_deg=pose.fov_y_deg,
                                    near=pose.near, far=pose.far, position=tuple(pose.position),
                                    look_at=tuple(pose.look_at), up=tuple(pose.up), screen=tuple(screen),
                                    omega=omega, n_scales=n_scales, min_dim=min_dim, padding=padding,
                                    backface_cull=cull, prescale=prescale)
            t0 = time.perf_counter()
            try:
                res = apcli.run_scene_pipeline(cfg, packer=packer)
                status = "ok"
            except ap.PackFailure:
                res, status = None, "PackFailure"
            except apcli.NothingVisible:
                res, status = None, "NothingVisible"
            except ValueError:  # e.g. superblock's block_size > omega (baselines.py:211-214)
                res, status = None, "ValueError"
            wall = time.perf_counter() - t0
            vp = cfg.camera().view_proj
    finally:
        apcli.depth_prepass, apcli.mark_visible, apcli.scene_stretch = orig_dp, orig_mv, orig_ss
        apcli.merge_shared_vertices, apcli.make_packer = orig_msv, orig_mp
    out = dict(status=status, vp=vp, depth=canon_depth(captured["depth"]), flags=captured["vis"].flags,
               wall_s=wall)
    if "cs" in captured:
        cs = captured["cs"]
        v2c = np.full(len(pos), -1, dtype=np.int64)
        for v, c in cs.vertex_to_chart.items():
            v2c[v] = c
        out.update(chart_of_triangle=cs.chart_of_triangle, vertex_to_chart=v2c,
                   roots=np.array(list(cs.charts.keys()), dtype=np.int64))
    if "boxes" in captured:
        bx = captured["boxes"]
        out.update(box_roots=np.array([b.chart_id for b in bx], dtype=np.int64),
                   target=np.array([[b.target_w, b.target_h] for b in bx], dtype=np.int64))
    if res is None:
        return out
    # UV rows in the reference's own emission order (cli.py:424-450)
    placements = {p.chart_id: p for p in res.layout.placements}
    clip = np.concatenate([pos[tris], np.ones((len(tris), 3, 1))], axis=2) @ vp.T
    uv_tris = []
    for root, members in cs.charts.items():
        if placements.get(root) is None or root not in res.chart_ndc:
            continue
        for t in members:
            if np.any(clip[t][:, 3] <= ap.geometry.W_EPSILON):
                continue
            uv_tris.append(t)
    pairs = captured.get("pairs", [])
    assert len(pairs) == len(uv_tris)
    uv = np.array([p[1] for p in pairs]).reshape(-1, 6) if pairs else np.zeros((0, 6))
    out.update(
        box_roots=np.array([b.chart_id for b in res.boxes], dtype=np.int64),
        ndc=np.array([[res.chart_ndc[b.chart_id].min_x, res.chart_ndc[b.chart_id].min_y,
                       res.chart_ndc[b.chart_id].max_x, res.chart_ndc[b.chart_id].max_y] for b in res.boxes]),
        px=np.array([res.chart_px[b.chart_id] for b in res.boxes], dtype=np.int64),
        target=np.array([[b.target_w, b.target_h] for b in res.boxes], dtype=np.int64),
        placements=np.array([[p.chart_id, p.x, p.y, p.w, p.h, int(p.rotated), p.target_w, p.target_h]
                             for p in res.layout.placements], dtype=np.int64),
        scale=np.array([res.layout.scale.numerator, res.layout.scale.denominator], dtype=np.int64),
        digest=ap.layout_digest(res.layout).digest,
        uv_tris=np.array(uv_tris, dtype=np.int64), uv=uv,
        screen_fragments=res.screen_fragments, texels_allocated=res.texels_allocated,
        n_visible=res.n_visible,
        stretch=[res.stretch.l2, res.stretch.linf] if res.stretch else None,
    )
    return out


def mini_scene(level=1, nx=20, nz=16):
    fpos, ftris, rng = scenes.sphere_field(level)
    plane = scenes.ground_plane(nx, nz, rng=rng)
    return scenes._merge((fpos, ftris), plane)


def gen_frames(out, with_c1=True):
    arrays, meta = {}, []
    frames = []
    pos, tris = mini_scene()
    poses = scenes.views_c5(8)
    for k in range(4):
        frames.append((f"mini_v{k}", pos, tris, poses[k], (320, 180), 256, 1.0, 1, 0))
    path = scenes.camera_path_c4(120)
    for f in (0, 59, 119):
        frames.append((f"mini_p{f}", pos, tris, path[f], (240, 160), 128, 1.0, 1, 0))
    frames.append(("mini_pad", pos, tris, poses[4], (200, 150), 256, 1.5, 2, 1))
    frames.append(("mini_fail", pos, tris, poses[5], (320, 180), 8, 1.0, 1, 0))
    frames.append(("mini_away", pos, tris, scenes.CameraPose(position=(0, 1, 0), look_at=(0, 1, 5)),
                   (64, 64), 64, 1.0, 1, 0))
    if with_c1:
        s = scenes.scene_c1()
        frames.append(("C1", s.positions, s.triangles, s.poses[0], s.screen, s.omega, 1.0, 1, 0))
    for name, p, t, pose, screen, omega, prescale, md, pad in frames:
        r = run_reference_frame(p, t, pose, screen, omega, prescale=prescale, min_dim=md, padding=pad)
        print(f"  frame {name}: {r['status']} {r['wall_s']:.2f}s", flush=True)
        m = dict(name=name, screen=list(screen), omega=omega, prescale=prescale, min_dim=md, padding=pad,
                 status=r["status"], wall_s=r["wall_s"])
        if not name.startswith("C"):
            arrays[f"{name}/pos"] = p
            arrays[f"{name}/tris"] = t
        for key in ("vp", "depth", "flags", "chart_of_triangle", "vertex_to_chart", "roots", "box_roots",
                    "ndc", "px", "target", "placements", "scale", "uv_tris", "uv"):
            if key in r:
                arrays[f"{name}/{key}"] = r[key]
        for key in ("digest", "screen_fragments", "texels_allocated", "n_visible", "stretch"):
            if key in r:
                m[key] = r[key]
        meta.append(m)
    np.savez_compressed(os.path.join(out, "frames.npz"), **arrays)
    return meta


def gen_frames_packers(out):
    """run_scene_pipeline(cfg, packer=p) for the comparison packers
    (cli.py:318-339,386-387): layouts, UV rows and stretch of mini frames and
    C1, including a superblock PackFailure (omega 16) and a ValueError
    (omega 8 < the default 16-texel block)."""
    arrays, meta = {}, []
    pos, tris = mini_scene()
    poses = scenes.views_c5(8)
    path = scenes.camera_path_c4(120)
    frames = [(f"mini_v{k}", pos, tris, poses[k], (320, 180), 256, 1.0, 1, 0) for k in range(2)]
    frames += [("mini_p59", pos, tris, path[59], (240, 160), 128, 1.0, 1, 0),
               ("mini_pad", pos, tris, poses[4], (200, 150), 256, 1.5, 2, 1),
               ("mini_tiny", pos, tris, poses[5], (320, 180), 16, 1.0, 1, 0),
               ("mini_fail", pos, tris, poses[5], (320, 180), 8, 1.0, 1, 0)]
    s = scenes.scene_c1()
    frames.append(("C1", s.positions, s.triangles, s.poses[0], s.screen, s.omega, 1.0, 1, 0))
    for packer in ("sequential", "superblock"):
        for name, p, t, pose, screen, omega, prescale, md, pad in frames:
            r = run_reference_frame(p, t, pose, screen, omega, prescale=prescale, min_dim=md, padding=pad,
                                    packer=packer)
            key = f"{packer}/{name}"
            print(f"  frame {key}: {r['status']} {r['wall_s']:.2f}s", flush=True)
            m = dict(name=name, packer=packer, screen=list(screen), omega=omega, prescale=prescale, min_dim=md,
                     padding=pad, status=r["status"])
            arrays[f"{key}/vp"] = r["vp"]
            for k in ("placements", "scale", "uv_tris", "uv", "box_roots", "target"):
                if k in r:
                    arrays[f"{key}/{k}"] = r[k]
            for k in ("digest", "screen_fragments", "texels_allocated", "n_visible", "stretch"):
                if k in r:
                    m[k] = r[k]
            meta.append(m)
    np.savez_compressed(os.path.join(out, "frames_packers.npz"), **arrays)
    return meta


def gen_c2(out):
    gen_digest(out, "c2_reference.json", scenes.scene_c2(), 0)


def gen_digest(out, fname, s, pose_idx, packer="fastatlas"):
    """One full-size reference frame reduced to SHA-256 digests of its arrays
    (depth, flags, chart ids, vertex map, NDC boxes, UV rows) plus the layout."""
    r = run_reference_frame(s.positions, s.triangles, s.poses[pose_idx], s.screen, s.omega,
                            prescale=s.prescale, packer=packer)
    rec = dict(scene=s.name, pose=pose_idx, packer=packer, prescale=s.prescale,
               screen=list(s.screen), omega=s.omega, status=r["status"], wall_s=r["wall_s"], vp=r["vp"].tolist(),
               depth_sha=sha(r["depth"]), flags_sha=sha(r["flags"].astype(np.uint8)),
               n_visible=int(r["flags"].sum()),
               chart_sha=sha(r["chart_of_triangle"].astype(np.int64)),
               v2c_sha=sha(r["vertex_to_chart"].astype(np.int64)),
               n_charts=len(r["roots"]), digest=r["digest"],
               scale=r["scale"].tolist(), placements=r["placements"].tolist(),
               target=r["target"].tolist(), ndc_sha=sha(r["ndc"]),
               uv_sha=sha(r["uv"]), uv_tris_sha=sha(r["uv_tris"]),
               screen_fragments=r["screen_fragments"], texels_allocated=r["texels_allocated"],
               stretch=r["stretch"])
    with open(os.path.join(out, fname), "w") as fh:
        json.dump(rec, fh)
    print(f"  {fname}: {r['status']} {r['wall_s']:.1f}s charts={rec['n_charts']} vis={rec['n_visible']}")


def gen_baselines(out):
    """Comparison packers (baselines.py:53-261) on seeded box sets."""
    from atlaspack import baselines as bl
    rng = np.random.default_rng(77)
    seq, sb, prim = [], [], []

    def boxrecs(boxes):
        return [[b.target_w, b.target_h, b.chart_id, b.min_tri] for b in boxes]

    for k in range(36):
        om = int(2 ** rng.integers(5, 12))
        cnt = int(rng.integers(1, 400))
        boxes = generate_boxes(cnt, om, np.random.default_rng(500 + k))
        ns = int(rng.choice([8, 16, 64]))
        md, pad = int(rng.integers(1, 3)), int(rng.integers(0, 2))
        rec = dict(omega=om, n_scales=ns, min_dim=md, padding=pad, boxes=boxrecs(boxes))
        try:
            lay = bl.sequential_scale_search(boxes, om, n_scales=ns, min_dim=md, padding=pad)
            rec.update(status="ok", **layout_rec(lay))
        except ap.PackFailure:
            rec["status"] = "PackFailure"
        seq.append(rec)
        blk = max(16, min(om, om // 8))
        for halving, bsz in ((True, blk), (False, blk), (True, om)):
            r2 = dict(omega=om, block_size=bsz, halving=halving, boxes=boxrecs(boxes))
            lay = bl.superblock_pack(boxes, om, bl.SuperblockConfig(block_size=bsz, halving_enabled=halving))
            if lay is None:
                r2["status"] = "None"
            else:
                r2.update(status="ok", block_used=lay.block_size, **layout_rec(lay))
            sb.append(r2)
    for _ in range(100):
        om = int(2 ** rng.integers(2, 10))
        n = int(rng.integers(1, 60))
        widths = np.clip((om * rng.random(n) ** 3).astype(int), 1, om)
        f = bl.sequential_fold(widths.tolist(), om)
        heights = rng.integers(1, om + 1, size=n)
        ordered = ap.order([ap.OrientedBox(w=int(w), h=int(h), rotated=False,
                                           source=ap.ChartBox(int(w), int(h), i, i))
                            for i, (w, h) in enumerate(zip(widths, heights))])
        lay = bl.sequential_pack(ordered, om)
        prim.append(dict(omega=om, widths=widths.tolist(), rows=f.row_of_box.tolist(), x=f.x_of_box.tolist(),
                         ordered=[[b.w, b.h, b.source.chart_id] for b in ordered],
                         pack=None if lay is None else [[p.chart_id, p.x, p.y, p.w, p.h] for p in lay.placements]))
    with open(os.path.join(out, "baselines.json"), "w") as fh:
        json.dump(dict(sequential=seq, superblock=sb, prim=prim), fh)


def main():
    ap_ = argparse.ArgumentParser()
    ap_.add_argument("--c2", action="store_true", help="also run the ~6 min C2 reference frame")
    ap_.add_argument("--only", default=None)
    ap_.add_argument("--digest", default=None,
                     help="SCENE:POSE[:PACKER] full-size reference digest, e.g. C3:0, C4:59, C5:37")
    args = ap_.parse_args()
    out = HERE
    meta = {}
    only = set(args.only.split(",")) if args.only else (set() if (args.c2 or args.digest) else None)
    if only is None or "raster" in only:
        meta["raster"] = gen_raster(out)
    if only is None or "charts" in only:
        meta["charts"] = gen_charts(out)
    if only is None or "bounds" in only:
        gen_bounds(out)
    if only is None or "pack" in only:
        gen_pack(out)
    if only is None or "baselines" in only:
        gen_baselines(out)
    if only is None or "frames" in only:
        meta["frames"] = gen_frames(out)
    if only is None or "frames_packers" in only:
        meta["frames_packers"] = gen_frames_packers(out)
    if meta:
        mp = os.path.join(out, "meta.json")
        old = json.load(open(mp)) if os.path.exists(mp) else {}
        old.update(meta)
        with open(mp, "w") as fh:
            json.dump(old, fh, indent=1)
    if args.c2:
        gen_c2(out)
    if args.digest:
        parts = args.digest.split(":")
        name, pose = parts[0], int(parts[1])
        packer = parts[2] if len(parts) > 2 else "fastatlas"
        suffix = "" if packer == "fastatlas" else f"_{packer}"
        gen_digest(out, f"{name.lower()}_p{pose}{suffix}_reference.json", scenes.build_scene(name), pose,
                   packer=packer)


if __name__ == "__main__":
    main()
