"""Device-side timeline of one graphed frame (kernel start/end from
%globaltimer, a build with -DFA_TRACE):

    bash tools/build_variant.sh trace -DFA_TRACE
    FASTATLAS_LIB=tools/lib_trace.so python tools/trace_frame.py [C2] [frames]

Per kernel: first block start and last block-0 thread exit relative to the
frame's first kernel, in microseconds (averaged over the frames), so the
critical path and the overlap of the concurrent branches are visible.  The
timestamps perturb the kernels slightly (two atomics per block)."""
import ctypes
import math
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import FrameEngine, FrameSettings, _native, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = scenes.build_scene(cfg)
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles),
                  settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale))
L = _native.load_library()
L.fa_debug_trace_reset.restype = ctypes.c_int
L.fa_debug_trace_read.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int]
views = scenes.views_c5(max(n, 8))
vps = []
for p in views:
    cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0] / spec.screen[1], p.near, p.far,
                                     position=p.position, look_at=p.look_at, up=p.up)
    vps.append(cam.view_proj)
for v in vps[:3]:
    eng.run(v)
acc = defaultdict(list)
total = []
for k in range(n):
    torch.cuda.synchronize()
    assert L.fa_debug_trace_reset() == 0
    eng.run(vps[k % len(vps)])
    torch.cuda.synchronize()
    names = ctypes.create_string_buffer(64 * 128)
    st = (ctypes.c_uint64 * 128)()
    en = (ctypes.c_uint64 * 128)()
    hi = (ctypes.c_uint64 * 128)()
    m = L.fa_debug_trace_read(names, st, en, hi, 128)
    recs = [(names.raw[64 * i:64 * i + 64].split(b"\0")[0].decode(), st[i], en[i], hi[i]) for i in range(m)]
    t0 = min(r[1] for r in recs)
    total.append((max(r[2] for r in recs) - t0) / 1e3)
    for name, s0, e0, h in recs:
        acc[name].append(((s0 - t0) / 1e3, (e0 - t0) / 1e3, h))
TU = {1: "fa_api.cu", 2: "fa_raster.cu", 3: "fa_charts.cu", 4: "fa_bounds.cu", 5: "fa_pack.cu", 6: "fa_uv.cu",
      7: "fa_baselines.cu", 8: "fa_mesh.cu"}
_src = {}


def kernel_name(key: str) -> str:
    """FA_TU_ID * 100000 + line of the kernel's FA_PDL_PROLOGUE -> the kernel's name."""
    k = int(key)
    tu, line = TU.get(k // 100000), k % 100000
    if tu is None:
        return key
    if tu not in _src:
        _src[tu] = open("paper_2502_17712_b200/csrc/" + tu).read().splitlines()
    lines = _src[tu]
    for i in range(min(line, len(lines)) - 1, -1, -1):
        if "__global__" in lines[i]:
            import re
            m = re.search(r"\b(k_\w+)\s*\(", " ".join(lines[i:i + 3]))
            return f"{m.group(1) if m else '?'} ({tu}:{line})"
    return key


acc = {kernel_name(k): v for k, v in acc.items()}
print(f"{cfg}: {n} graphed frames, kernel span mean {np.mean(total):.1f} us (first start -> last end)")
print(f"{'kernel':36s} {'start':>8s} {'end':>8s} {'dur':>7s}  launches")
rows = sorted(((np.mean([a[0] for a in v]), np.mean([a[1] for a in v]), int(np.mean([a[2] for a in v])), k)
               for k, v in acc.items()))
for s0, e0, h, name in rows:
    print(f"{name[:36]:36s} {s0:8.1f} {e0:8.1f} {e0 - s0:7.1f}  {h}")
