import sys, math, numpy as np
sys.path[:0] = ['.', 'oracle']
import oracle
import paper_2502_17712_b200 as fa
from paper_2502_17712_b200 import scenes
name = sys.argv[1] if len(sys.argv) > 1 else 'C3'
spec = scenes.build_scene(name)
rng = np.random.default_rng(0)
T = len(spec.triangles)
for frac in (0.18, 0.5):
    flags = rng.random(T) < frac
    lab0 = np.where(flags, np.arange(T), -1)
    ref, _ = oracle.merge_shared_vertices(spec.triangles, len(spec.positions), lab0)
    mesh = fa.Mesh(spec.positions, spec.triangles)
    for rep in range(4):
        cs = fa.merge_shared_vertices(fa.ChartSet(lab0), mesh)
        g = cs.chart_of_triangle
        print(name, frac, rep, 'mismatch', int(np.sum(g != ref)))
