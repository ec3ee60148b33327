"""Host-side ceiling of FramePipeline: views/s on the tiny C1 scene (GPU work
per view is small, so the rate is bounded by the Python/driver loop).
GPU box: python tools/host_rate.py"""
import math
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FramePipeline, FrameSettings, scenes

spec = scenes.build_scene("C1")
p = spec.poses[0]
cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                 position=p.position, look_at=p.look_at, up=p.up)
N = 200
pin = torch.empty((N, 16), dtype=torch.float64).pin_memory()
pin.copy_(torch.as_tensor(np.tile(np.asarray(cam.view_proj).reshape(1, 16), (N, 1))))
cams = [pin[i].numpy().reshape(4, 4) for i in range(N)]
mesh = fa.Mesh(spec.positions, spec.triangles)
st = FrameSettings(screen=spec.screen, omega=spec.omega)
for outs in [(), ("visible", "visible_chart", "uv", "placements")]:
    pipe = FramePipeline(mesh, settings=st, depth=6, outputs=outs)
    pipe.run(cams[:20])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pipe.run(cams)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"outputs={len(outs)}: {N / dt:.0f} views/s host-bound ceiling ({1e6 * dt / N:.1f} us/view)")
