"""Small records by window size and whether any sample was covered (needs
FASTATLAS_LIB=tools/lib_coopstats.so built with -DFA_COOP_STATS)."""
import ctypes
import math
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, _native, scenes

spec = scenes.build_scene(sys.argv[1] if len(sys.argv) > 1 else "C2")
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles), settings=FrameSettings(screen=spec.screen, omega=spec.omega))
L = _native.load_library()
L.fa_debug_coop_stats.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(10, np.uint64)
for p in scenes.views_c5(4):
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    L.fa_debug_coop_stats(buf.ctypes.data, 1)
    eng.run(cam.view_proj)
    L.fa_debug_coop_stats(buf.ctypes.data, 1)
    b = buf.reshape(5, 2)
    print("window <=4 / <=9 / <=16 / <=48 / >48:  none-covered", b[:, 0].tolist(), " covered", b[:, 1].tolist())
