"""Pipelined throughput vs slot count and downloaded outputs (GPU box):
python tools/e2e_exp.py"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameSettings, scenes
import bench
spec = scenes.scene_c2()
mesh = fa.Mesh(spec.positions, spec.triangles)
settings = FrameSettings(screen=spec.screen, omega=spec.omega, n_scales=64, prescale=1.0)
views = bench._views()
N = 48
vps = [bench._vp(views[i % len(views)], spec.screen) for i in range(N)]
pin = torch.empty((N, 16), dtype=torch.float64).pin_memory()
pin.copy_(torch.as_tensor(np.stack([v.reshape(-1) for v in vps])))
cams = [pin[i].numpy().reshape(4, 4) for i in range(N)]
full = ("chart_of_triangle", "visible", "uv", "placements")
for depth, outs in [(6, full), (8, full), (10, full), (8, ()), (10, ()), (12, ())]:
    p = fa.FramePipeline(mesh, settings=settings, depth=depth, outputs=outs, mesh_replicas=True)
    p.run(cams[:2 * depth]); torch.cuda.synchronize()
    r = []
    for rep in range(2):
        t0 = time.perf_counter(); p.run(cams); torch.cuda.synchronize(); r.append(N / (time.perf_counter() - t0))
    print(depth, len(outs), "views/s %.0f %.0f" % tuple(r))
    del p
    torch.cuda.empty_cache()
