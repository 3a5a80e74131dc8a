import math, sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw
import specgen, oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
inst = specgen.ball(n)
S = sw.Spectrahedron.from_instance(inst)
print(S.k2_config())
lmi = oracle.Lmi(inst)
# per-call interior
us = specgen.unit_vectors(16, n, 3); vs = specgen.unit_vectors(16, n, 4)
xs = np.array([0.5 * u for u in us])
res = S.boundary_oracle(xs, vs, want_kernel=True)
for k in range(16):
    r = oracle.chord(lmi, xs[k], vs[k])
    print("int", k, res["t_plus"][k], r["t_plus"], res["t_minus"][k], r["t_minus"], res["binding"][k])
# boundary starts from the oracle hits
hits, uu, ss = [], [], []
for k in range(16):
    r = oracle.chord(lmi, xs[k], vs[k]); w = oracle.normal(lmi, r["block"], r["y"])
    hits.append(xs[k] + r["t_plus"] * vs[k]); uu.append(r["y"] / np.linalg.norm(r["y"])); ss.append(oracle.reflect(vs[k], w))
hits, uu, ss = map(np.array, (hits, uu, ss))
res = S.boundary_oracle(hits, ss, u=uu)
for k in range(16):
    r = oracle.chord(lmi, hits[k], ss[k], F0=lmi.eval_block(0, hits[k]), bound=0, u=uu[k])
    print("bnd", k, res["t_plus"][k], r["t_plus"], res["binding"][k])
g = S.walk_trace(list(range(4)), steps=2, L=2 * math.sqrt(n), rho=10 * n, seed=0, max_refl=6)
for c in range(4):
    o = oracle.trace(lmi, oracle.BILLIARD, 0, c, 2, 2 * math.sqrt(n), 10 * n, 6, stop=True)
    print("traj", c, len(g[c]["t"]), len(o["t"]), g[c]["t"][:6], o["t"][:6])
