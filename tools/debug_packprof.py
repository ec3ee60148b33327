"""Per-candidate pack phase timings (needs FASTATLAS_LIB=tools/libfa_packprof.so, built with -DFA_PACK_PROF).
Columns: cycles at fold done / heights done / row starts done / rows done, overflow iterations, rows."""
import ctypes
import math
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, _native, scenes

spec = scenes.build_scene("C2")
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, use_graph=False))
L = _native.load_library()
L.fa_debug_pack_prof.argtypes = [ctypes.c_void_p]
buf = np.zeros((256, 12), np.int64)
p = spec.poses[0]
cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                 position=p.position, look_at=p.look_at, up=p.up)
for _ in range(3):
    out = eng.run(cam.view_proj)
L.fa_debug_pack_prof(buf.ctypes.data)
print("charts", out.n_charts, "scale", out.scale)
for i in range(64):
    r = buf[i]
    print(i, "fold %.1f us  heights %.1f  rowstart %.1f  rows %.1f  iters %d  n_rows %d | round 2: widths %d cyc, "
          "+scan %d cyc +max2 %d +snap %d | loaded %d cyc, round 1 done %d cyc" % (r[0] / 1920, r[1] / 1920, r[2] / 1920,
                                    r[3] / 1920, r[4], r[5], r[6], r[7], r[8], r[9], r[10], r[11]))
