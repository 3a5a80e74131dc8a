"""Volume estimator spread: GPU over many seeds vs oracle over some seeds (same instance)."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import specgen
inst = specgen.rand_cube(12, 12, 2)
which = sys.argv[1]
seeds = range(int(sys.argv[2]), int(sys.argv[3]))
if which == "gpu":
    import paper_2010_03817_b200 as sw
    S = sw.Spectrahedron.from_instance(inst)
    v = [S.volume(0.1, s, 256, walk_len=5, burn=20) for s in seeds]
    print(json.dumps(dict(which=which, vols=[r["volume"] for r in v], phases=[r["phases"] for r in v],
                          chains=[r["chains"] for r in v])))
else:
    import oracle
    v = [oracle.volume(inst, 0.1, s, 256, W=5, burn=20) for s in seeds]
    print(json.dumps(dict(which=which, vols=[r["volume"] for r in v], phases=[r["phases"] for r in v],
                          chains=[r["chains"] for r in v])))
