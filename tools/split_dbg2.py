import os, sys, json, math
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
tr = {}
orc = {}
for mode in ("split", "fused"):
    if mode == "fused": os.environ["SPECWALK_K2_FUSED"] = "1"
    S = sw.Spectrahedron.from_instance(inst)
    tr[mode] = S.walk_trace(np.arange(64), 20, 2 * math.sqrt(12), 120, 0, 300)
    xs = np.random.default_rng(0).uniform(-0.05, 0.05, (512, 12)); vs = np.random.default_rng(1).standard_normal((512, 12))
    orc[mode] = S.boundary_oracle(xs, vs, want_kernel=True)
    S.close()
for k in orc["split"]:
    a, b = np.asarray(orc["split"][k]), np.asarray(orc["fused"][k])
    print("oracle", k, "max diff", np.nanmax(np.abs(a - b)) if a.size else 0)
first = []
for c in range(64):
    A, B = tr["split"][c], tr["fused"][c]
    nn = min(len(A["t"]), len(B["t"]))
    d = [i for i in range(nn) if not (np.array_equal(A["hit_x"][i], B["hit_x"][i]) and A["t"][i] == B["t"][i])]
    first.append(d[0] if d else None)
    if d and len(first) < 70 and d[0] is not None:
        i = d[0]
        print("chain", c, "first diff at refl", i, "of", nn, "t", A["t"][i], B["t"][i], "bind", A["binding"][i], B["binding"][i],
              "dx", np.abs(A["hit_x"][i] - B["hit_x"][i]).max())
print("chains identical:", sum(1 for f in first if f is None), "/ 64")
