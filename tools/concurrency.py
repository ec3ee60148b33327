"""Throughput of P FrameEngines on P CUDA streams (independent views) vs one."""
import math
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, scenes

spec = scenes.build_scene("C2")
mesh = fa.Mesh(spec.positions, spec.triangles)
views = scenes.views_c5(16)
vps = []
for p in views:
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    vps.append(cam.view_proj)
settings = FrameSettings(screen=spec.screen, omega=spec.omega)
K = 32
for P in (1, 2, 3, 4):
    engines = [FrameEngine(mesh, settings=settings) for _ in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    for e, s in zip(engines, streams):
        for i in range(3):
            e.run(vps[i], stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rnd in range(K // P):
        for j, (e, s) in enumerate(zip(engines, streams)):
            e.launch(vps[(rnd * P + j) % len(vps)], stream=s)
        for e in engines:
            e.finish()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    n = (K // P) * P
    print(f"P={P}: {1e3 * dt / n:.4f} ms/frame wall, {n / dt:.1f} atlases/s")
