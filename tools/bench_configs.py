"""Per-config timings on one GPU for BASELINE.json's other configs (bench.py
measures configs[1], C2).  GPU box: python tools/bench_configs.py [out.json]

  C1  20K tris, 512^2 -> 1K^2                single-view latency
  C2  1M tris, 1080p -> 2K^2                 latency + pipelined views/s (reference point)
  C3  4M tris, 4K -> 4K^2, prescale 2        latency + pipelined views/s
  C4  120-frame camera path over C2          frames/s, camera path in order (pipelined)
  C5  64 golden-angle views of C2            views/s (pipelined)

Latency: one FrameEngine, CUDA events around each graph replay, a 256 MiB L2
flush before each event pair (outside it).  Pipelined: FramePipeline (6
slots, per-slot mesh replicas, device outputs), one event pair around all
views.  Every frame's status is checked (a failing frame raises)."""
import json
import math
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FramePipeline, FrameSettings, scenes


def vps_for(spec, poses):
    out = []
    for p in poses:
        cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                         position=p.position, look_at=p.look_at, up=p.up)
        out.append(cam.view_proj)
    return out


def latency(spec, vps, flush, reps=None):
    settings = FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale)
    eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles), settings=settings)
    for v in vps[:3]:
        eng.run(v)
    stream = torch.cuda.current_stream()
    ts, vis, charts = [], [], []
    for v in (vps if reps is None else vps[:reps]):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.launch(v)
        b.record(stream)
        out = eng.finish()
        ts.append(a.elapsed_time(b))
        vis.append(out.n_visible)
        charts.append(out.n_charts)
    del eng
    return {"ms_per_frame_mean": float(np.mean(ts)), "ms_per_frame_p50": float(np.median(ts)),
            "ms_per_frame_max": float(np.max(ts)), "frames": len(ts), "mean_visible": int(np.mean(vis)),
            "mean_charts": int(np.mean(charts))}


def pipelined(spec, vps, depth=6):
    settings = FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale)
    pipe = FramePipeline(fa.Mesh(spec.positions, spec.triangles), settings=settings, depth=depth, outputs=(),
                         mesh_replicas=True)
    errors = []

    def check(hf):
        if hf.error is not None:
            errors.append(hf.error)

    pipe.run(vps[:2 * depth], check)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for st in pipe.streams:
        st.wait_stream(stream)
    pipe.run(vps, check)
    for st in pipe.streams:
        stream.wait_stream(st)
    b.record(stream)
    torch.cuda.synchronize()
    if errors:
        raise errors[0]
    ms = a.elapsed_time(b)
    del pipe
    torch.cuda.empty_cache()
    return {"views": len(vps), "ms_total": ms, "views_per_s": len(vps) / (ms * 1e-3), "ms_per_view": ms / len(vps)}


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {"gpu": torch.cuda.get_device_name(0)}
    c1 = scenes.build_scene("C1")
    res["C1"] = {"latency": latency(c1, vps_for(c1, c1.poses) * 20, flush)}
    c2 = scenes.scene_c2()
    v5 = vps_for(c2, scenes.views_c5(64))
    res["C2"] = {"latency": latency(c2, v5, flush, reps=20), "pipelined": pipelined(c2, v5[:32])}
    res["C5"] = {"pipelined": pipelined(c2, v5)}
    v4 = vps_for(c2, scenes.camera_path_c4(120))
    res["C4"] = {"latency": latency(c2, v4, flush), "pipelined": pipelined(c2, v4)}
    del c2
    c3 = scenes.scene_c3()
    v3 = vps_for(c3, scenes.views_c5(16))
    res["C3"] = {"latency": latency(c3, v3, flush, reps=10), "pipelined": pipelined(c3, v3, depth=4)}
    txt = json.dumps(res, indent=1)
    print(txt)
    if len(sys.argv) > 1:
        open(sys.argv[1], "w").write(txt + "\n")


if __name__ == "__main__":
    main()
