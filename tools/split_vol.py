import os, sys, json
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
for mode in ("split", "fused"):
    if mode == "fused": os.environ["SPECWALK_K2_FUSED"] = "1"
    S = sw.Spectrahedron.from_instance(inst)
    for s in range(10):
        try:
            r = S.volume(0.1, s, 256, walk_len=5, burn=20)
            print(mode, s, r["volume"], r["phases"], r["calls"], flush=True)
        except Exception as e:
            print(mode, s, "ERR", e, flush=True)
    S.close()
