"""Small driver for ncu: a few C2 frames through the non-graph path."""
import math
import sys

sys.path.insert(0, ".")
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
spec = scenes.build_scene(cfg)
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale,
                                         use_graph=False))
views = scenes.views_c5(8)
for k in range(n):
    p = views[k]
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    out = eng.run(cam.view_proj, check=False)
torch.cuda.synchronize()
print("frames", n, "visible", out.n_visible, "charts", out.n_charts, "launches/frame", eng.launch_count())
