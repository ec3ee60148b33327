"""Union-find work counters (needs FASTATLAS_LIB=tools/libfa_ufstats.so, built with -DFA_UF_STATS)."""
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
                                         use_graph=False, profile=True))
L = _native.load_library()
L.fa_debug_uf_stats.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 5)()
for k in range(3):
    p = scenes.views_c5(8)[k]
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    L.fa_debug_uf_stats(buf)
    out = eng.run(cam.view_proj)
    L.fa_debug_uf_stats(buf)
    print(cfg, k, "vis", out.n_visible, "charts", out.n_charts, "unions", buf[0], "cas", buf[1], "casfail", buf[2],
          "hops", buf[3], "maxhops", buf[4], "uf_ms", round(eng.stage_times()["union-find"], 4))
