"""Time fa_set_mesh (index check, Morton triangle order, first-use vertex
renumbering, cluster culling data -- all on the GPU) for a config's mesh.

usage (GPU box): python tools/set_mesh_time.py [C3] [reps]"""
import sys

sys.path.insert(0, ".")
import torch

import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import _native as nat, scenes

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = scenes.build_scene(cfg)
mesh = fa.Mesh(spec.positions, spec.triangles)
ctx = nat.Context(0)
pos, tris = mesh.device_arrays(ctx.torch_device)
ctx.set_mesh(pos, tris)
times = []
for _ in range(reps):
    pos.add_(0.0)  # bump the version counter: Context.set_mesh rebinds
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.set_mesh(pos, tris)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
print(f"{cfg}: {len(spec.triangles)} triangles, {len(spec.positions)} vertices; fa_set_mesh "
      f"min {min(times):.3f} ms, median {sorted(times)[len(times) // 2]:.3f} ms")
