import sys, math, numpy as np
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import scenes, FrameEngine, FrameSettings
spec = scenes.build_scene(sys.argv[1] if len(sys.argv) > 1 else 'C2'); p = spec.poses[0]
cam = fa.CameraFrame.from_params(math.radians(p.fov_y_deg), spec.screen[0]/spec.screen[1], p.near, p.far, position=p.position, look_at=p.look_at, up=p.up)
vp = cam.view_proj
eng = FrameEngine(fa.Mesh(spec.positions, spec.triangles), settings=FrameSettings(screen=spec.screen, omega=spec.omega, prescale=spec.prescale, uv_f64=True))
h = eng.run(vp).to_host()
r = oracle.run_frame(spec.positions, spec.triangles, vp, spec.screen, spec.omega, prescale=spec.prescale)
g = h['chart_of_triangle'].astype(np.int64); o = r.chart_of_triangle
bad = np.flatnonzero(g != o)
print('n_vis', h['n_visible'], (o>=0).sum(), 'mismatch', len(bad), 'charts gpu', h['n_charts'], 'oracle', len(r.boxes.roots))
print('first bad', bad[:10], g[bad[:10]], o[bad[:10]])
vis = np.flatnonzero(g >= 0)
print('label<=t', np.all(g[vis] <= vis), 'idempotent', np.all(g[g[vis]] == g[vis]))
# vertex consistency: all visible tris sharing a vertex have equal label
tris = spec.triangles
lv = np.full(len(spec.positions), -1)
incons = 0
for k in range(3):
    v = tris[vis, k]
    lv[v] = g[vis]
for k in range(3):
    incons += np.sum(lv[tris[vis, k]] != g[vis])
print('vertex-inconsistent', incons)
# rerun determinism
h2 = eng.run(vp).to_host()
print('rerun equal', np.array_equal(h2['chart_of_triangle'], h['chart_of_triangle']))
# where do they differ: same partition?
from collections import defaultdict
if len(bad):
    pairs = set(zip(g[bad].tolist(), o[bad].tolist()))
    print('distinct (gpu,oracle) label pairs', len(pairs), list(pairs)[:10])
    # oracle: is it vertex-consistent?
    lv2 = np.full(len(spec.positions), -1); vis2 = np.flatnonzero(o >= 0)
    for k in range(3): lv2[tris[vis2, k]] = o[vis2]
    print('oracle vertex-inconsistent', sum(np.sum(lv2[tris[vis2, k]] != o[vis2]) for k in range(3)))
    print('oracle label<=t', np.all(o[vis2] <= vis2), 'idem', np.all(o[o[vis2]] == o[vis2]))
    print('gpu label min member?', all(g[t] == np.flatnonzero(g == g[t]).min() for t in bad[:5]))
    print('oracle label min member?', all(o[t] == np.flatnonzero(o == o[t]).min() for t in bad[:5]))
