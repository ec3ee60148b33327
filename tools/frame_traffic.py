"""Whole-frame DRAM traffic in the real cache state, for ncu's range replay:

    ncu --replay-mode range --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum \
        python tools/frame_traffic.py [C2] [graph|nograph]
    FASTATLAS_PROFILE_STAGE=k ncu ... python tools/frame_traffic.py C2 nograph   (stage k only)

A few warm frames run first; cudaProfilerStart/Stop then bracket exactly one
frame (the next C5 view), so the counters cover one frame's kernels with the
L2 state the previous frame left behind -- unlike the per-kernel captures,
which flush the caches before every kernel.  (The metrics ncu prints for the
range are the frame's; a run under ncu is never a timing.)"""
import math
import os
import sys

sys.path.insert(0, ".")
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
graph = (sys.argv[2] if len(sys.argv) > 2 else "graph") == "graph"
spec = scenes.build_scene(cfg)
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale,
                                         use_graph=graph))
vps = []
for p in scenes.views_c5(8):
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    vps.append(cam.view_proj)
for k in range(4):
    eng.run(vps[k], check=False)
torch.cuda.synchronize()
stage = os.environ.get("FASTATLAS_PROFILE_STAGE")  # the library brackets one stage of frame 4 itself
if stage is None:
    torch.cuda.cudart().cudaProfilerStart()
out = eng.run(vps[4], check=False)
torch.cuda.synchronize()
if stage is None:
    torch.cuda.cudart().cudaProfilerStop()
print("visible", out.n_visible, "charts", out.n_charts)
