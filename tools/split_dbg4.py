import os, sys, math, json
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
n = 12
S = sw.Spectrahedron.from_instance(inst)
def w(tag, x0=None, ch=256, st=5):
    try:
        out = S.walk_sample(ch, st, 2 * math.sqrt(n), 120, 0, x0=x0, tag=tag)
        return out["stats"]["failures"], out["final_x"]
    except Exception as e:
        return str(e), None
f, X = w(3 << 28, np.zeros((256, n)), st=20); print("pilot", f)
f, _ = w(1 << 28, (1 - 2.0 ** -40) * X); print("est0 direct", f)
xs = np.random.default_rng(0).uniform(-0.05, 0.05, (256, n)); vs = np.random.default_rng(1).standard_normal((256, n))
S.boundary_oracle(xs, vs)
f, _ = w(1 << 28, (1 - 2.0 ** -40) * X); print("est0 after boundary_oracle", f)
f, _ = w(1 << 28, None); print("origin after boundary_oracle", f)
