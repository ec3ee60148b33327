"""Work-queue counters of a few frames (records, tiles, clipped triangles, ...).

usage (GPU box): python tools/frame_counters.py [C2|C3|C1] [n_views]"""
import math
import sys

sys.path.insert(0, ".")
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = scenes.build_scene(cfg)
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale))
for k, p in enumerate(scenes.views_c5(n)):
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    eng.run(cam.view_proj)
    print(cfg, "view", k, eng.counters())
