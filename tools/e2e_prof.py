import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameSettings, scenes
import bench
spec = scenes.scene_c2()
mesh = fa.Mesh(spec.positions, spec.triangles)
settings = FrameSettings(screen=spec.screen, omega=spec.omega, n_scales=64, prescale=1.0)
views = bench._views()
N = 64
vps = [bench._vp(views[i % len(views)], spec.screen) for i in range(N)]
pin = torch.empty((N, 16), dtype=torch.float64).pin_memory()
pin.copy_(torch.as_tensor(np.stack([v.reshape(-1) for v in vps])))
cams = [pin[i].numpy().reshape(4, 4) for i in range(N)]
for outs in [(), ("visible", "visible_chart", "vertex_uv", "placements")]:
    p = fa.FramePipeline(mesh, settings=settings, depth=6, outputs=outs, mesh_replicas=True)
    p.run(cams); torch.cuda.synchronize()
    t0 = time.perf_counter(); p.run(cams); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(len(outs), "wall views/s %.0f" % (N / dt))
    pr = cProfile.Profile(); pr.enable(); p.run(cams); torch.cuda.synchronize(); pr.disable()
    st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(12)
    del p
