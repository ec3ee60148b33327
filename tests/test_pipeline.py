"""FramePipeline (independent views on concurrent slot streams, host copies
overlapped): every delivered frame equals the sequential engine's frame for
the same view, bit for bit, and frames arrive in view order.  Run with -m gpu."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fa = pytest.importorskip("paper_2502_17712_b200")
from paper_2502_17712_b200 import FrameEngine, FramePipeline, FrameSettings, scenes  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _vps(spec, poses):
    out = []
    for p in poses:
        cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                         position=p.position, look_at=p.look_at, up=p.up)
        out.append(cam.view_proj)
    return out


@pytest.mark.parametrize("depth,outputs,packed", [(1, None, True), (3, None, True), (3, None, False),
                                                  (2, ("chart_of_triangle", "visible", "uv", "placements"), True)])
def test_pipeline_matches_sequential(depth, outputs, packed):
    """Sparse chart ids (default: visible_chart, dense array rebuilt on the
    host) and the dense download give the sequential engine's outputs."""
    spec = scenes.build_scene("C5")
    mesh = fa.Mesh(spec.positions, spec.triangles)
    settings = FrameSettings(screen=spec.screen, omega=spec.omega)
    vps = _vps(spec, spec.poses[:7])
    seq = FrameEngine(mesh, settings=settings)
    want = []
    for vp in vps:
        o = seq.run(vp)
        want.append({"chart": o.chart_of_triangle.cpu().numpy(), "vis": o.visible.cpu().numpy(),
                     "uv": o.uv.cpu().numpy(), "plc": o.placements.cpu().numpy(), "scale": o.scale,
                     "frag": o.screen_fragments})
    got = []

    def on_frame(hf):
        assert hf.error is None, hf.error
        got.append((hf.index, {"chart": hf.chart_of_triangle.copy(), "vis": hf.visible.copy(), "uv": hf.uv.copy(),
                               "plc": hf.placements.copy(), "scale": hf.scale, "frag": hf.screen_fragments,
                               "vchart": None if hf.visible_chart is None else hf.visible_chart.copy(),
                               "vv": None if hf.visible_vertices is None else np.sort(hf.visible_vertices)}))

    kw = {"packed": packed} if outputs is None else {"outputs": outputs}
    pipe = FramePipeline(mesh, settings=settings, depth=depth, **kw)
    assert pipe.run(vps, on_frame) == len(vps)
    assert [i for i, _ in got] == list(range(len(vps)))
    for (_, g), w in zip(got, want):
        assert np.array_equal(g["chart"], w["chart"])
        assert np.array_equal(g["vis"], w["vis"])
        assert np.array_equal(g["uv"].view(np.uint32), w["uv"].view(np.uint32))
        assert np.array_equal(g["plc"], w["plc"])
        assert g["scale"] == w["scale"] and g["frag"] == w["frag"]
        if g["vchart"] is not None:
            assert np.array_equal(g["vchart"], w["chart"][w["vis"]])
        if g["vv"] is not None:  # every vertex of a visible triangle, once
            assert np.array_equal(g["vv"], np.unique(spec.triangles[w["vis"]]))


def test_pipeline_reports_failures_in_order():
    """A view that sees nothing is delivered with its NothingVisible error;
    the views around it are unaffected."""
    spec = scenes.build_scene("C1")
    mesh = fa.Mesh(spec.positions, spec.triangles)
    settings = FrameSettings(screen=spec.screen, omega=spec.omega)
    good = _vps(spec, spec.poses[:1])[0]
    away = np.array(good, dtype=np.float64).copy()
    away[3, :] = [0.0, 0.0, 0.0, -1.0]  # every vertex behind the camera (w < 0)
    got = []

    def on_frame(h):  # slot arrays are reused: keep copies
        got.append((h.index, h.error, None if h.chart_of_triangle is None else h.chart_of_triangle.copy()))

    FramePipeline(mesh, settings=settings, depth=2).run([good, away, good], on_frame)
    assert [g[0] for g in got] == [0, 1, 2]
    assert got[0][1] is None and got[2][1] is None
    assert isinstance(got[1][1], fa.NothingVisible)
    assert got[1][2] is None
    assert np.array_equal(got[0][2], got[2][2])


def test_compact_uv_rows_match_engine_rows():
    """The compact download (f32 UV per visible vertex) rebuilds the engine's
    f32 rows bit for bit, NaN rows of triangles with a corner at/behind the
    camera plane (cli.py:433-435) included: a grid through the camera plane."""
    rng = np.random.default_rng(3)
    # a background grid plus long triangles reaching from in front of the
    # camera to behind it (third corner at z = +1: w < 0)
    nx = 20
    gx, gz = np.meshgrid(np.linspace(-4.0, 4.0, nx + 1), np.linspace(-9.0, -5.0, 5))
    grid = np.stack([gx.ravel(), gz.ravel() * 0.0 - 1.0 + 0.05 * gz.ravel(), gz.ravel()], 1)
    tris = []
    for j in range(4):
        for i in range(nx):
            a = j * (nx + 1) + i
            tris += [(a, a + nx + 2, a + 1), (a, a + nx + 1, a + nx + 2)]
    pos = [grid]
    base = len(grid)
    for k in range(6):
        x0 = -1.5 + 0.6 * k + rng.uniform(-0.05, 0.05)
        pos.append(np.array([[x0, -0.4, -3.0], [x0 + 0.5, -0.4, -3.0], [x0 + 0.25, -0.6, 1.0]]))
        tris.append((base, base + 1, base + 2))
        base += 3
    pos = np.vstack(pos)
    tris = np.asarray(tris, np.int32)
    mesh = fa.Mesh(pos, tris)
    cam = fa.CameraFrame.from_params(math.radians(70.0), 1.5, 0.1, 50.0, position=(0.0, 0.0, 0.0),
                                     look_at=(0.0, -0.2, -1.0))
    settings = FrameSettings(screen=(240, 160), omega=512, backface_cull=False)
    o = FrameEngine(mesh, settings=settings).run(cam.view_proj)
    want = o.uv.cpu().numpy()
    assert np.isnan(want).any(), "the scene must have rows with a corner behind the camera"
    got = []
    FramePipeline(mesh, settings=settings, depth=2).run([cam.view_proj] * 3,
                                                        lambda hf: got.append(hf.uv.copy()))
    assert len(got) == 3
    for g in got:
        assert g.dtype == np.float32 and g.shape == want.shape
        assert np.array_equal(g.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("no_wait", [False, True])
def test_copies_overlap_next_frame_safely(no_wait):
    """The slot's downloads run on a copy stream beside its next frame; the
    frame waits (device side, the context's copy_done event) before it
    rewrites the downloaded buffers.  With the copies delayed 2 ms, results
    stay exact -- and without the wait (debug knob) they would not, which
    shows the test exercises the race."""
    import subprocess
    import sys
    env = dict(__import__("os").environ, FASTATLAS_DEBUG_COPY_DELAY="2000")
    if no_wait:
        env["FASTATLAS_DEBUG_NO_COPY_WAIT"] = "1"
    code = (
        "import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import numpy as np, test_pipeline as tp;"
        "tp.test_pipeline_matches_sequential(2, None, True)"
    )
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    if no_wait:
        assert r.returncode != 0, "the unprotected overlap was expected to corrupt a delayed download"
    else:
        assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.parametrize("use_graph", [True, False])
def test_queue_overflow_reruns(use_graph, monkeypatch):
    """Frames whose large-triangle and tile queues overflow (contexts created
    with FASTATLAS_QUEUE_INIT=32) grow the queues and rerun; the results equal
    a default context's, through the engine and through the pipeline (whose
    slots rerun inside FramePipeline._finish)."""
    spec = scenes.build_scene("C5")
    mesh = fa.Mesh(spec.positions, spec.triangles)
    settings = FrameSettings(screen=spec.screen, omega=spec.omega, use_graph=use_graph)
    vps = _vps(spec, spec.poses[:4])
    ref = FrameEngine(mesh, settings=settings)
    want = [{"chart": o.chart_of_triangle.cpu().numpy(), "uv": o.uv.cpu().numpy(), "plc": o.placements.cpu().numpy(),
             "scale": o.scale, "counters": ref.counters()} for o in (ref.run(vp) for vp in vps)]
    assert all(w["counters"]["tiles"] > 32 and w["counters"]["large_records"] > 32 for w in want)
    monkeypatch.setenv("FASTATLAS_QUEUE_INIT", "32")
    eng = FrameEngine(mesh, settings=settings)
    # the first launch really overflows (and asks for a rerun)
    import ctypes
    from paper_2502_17712_b200 import _native as nat
    eng.launch(vps[0])
    code = eng.ctx.L.fa_frame_finish(eng.ctx.h, ctypes.byref(eng._res), eng._stream)
    assert code == nat.FA_INTERNAL_ERROR and "rerun" in nat.last_error()
    for vp, w in zip(vps, want):
        o = eng.run(vp)
        assert np.array_equal(o.chart_of_triangle.cpu().numpy(), w["chart"])
        assert np.array_equal(o.uv.cpu().numpy().view(np.uint32), w["uv"].view(np.uint32))
        assert np.array_equal(o.placements.cpu().numpy(), w["plc"]) and o.scale == w["scale"]
    got = []
    pipe = FramePipeline(mesh, settings=settings, depth=2,
                         outputs=("chart_of_triangle", "visible", "uv", "placements"))
    assert pipe.run(vps, lambda hf: got.append((hf.error, hf.chart_of_triangle.copy(), hf.uv.copy(),
                                                hf.placements.copy(), hf.scale))) == len(vps)
    for (err, chart, uv, plc, scale), w in zip(got, want):
        assert err is None, err
        assert np.array_equal(chart, w["chart"])
        assert np.array_equal(uv.view(np.uint32), w["uv"].view(np.uint32))
        assert np.array_equal(plc, w["plc"]) and scale == w["scale"]
