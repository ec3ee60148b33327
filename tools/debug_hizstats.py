"""Hierarchical-Z rejection counters (needs FASTATLAS_LIB=tools/libfa_hizstats.so,
built with -DFA_HIZ_STATS, and FA_VIS_COOP=0 so the per-record kernel runs)."""
import ctypes
import math
import sys

sys.path.insert(0, ".")
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, _native, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = scenes.build_scene(cfg)
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale,
                                         use_graph=False))
L = _native.load_library()
L.fa_debug_hiz_stats.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 6)()
for k in range(3):
    p = spec.poses[0] if k == 0 else scenes.views_c5(8)[k]
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    L.fa_debug_hiz_stats(buf)
    out = eng.run(cam.view_proj)
    L.fa_debug_hiz_stats(buf)
    print(cfg, k, "vis", out.n_visible, "small: hiz rejected", buf[0], "sampled", buf[1], "| tiles: tested", buf[2],
          "hiz rejected", buf[3], "skipped visible", buf[4])
