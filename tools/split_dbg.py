import os, sys, json, math
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
for mode in ("split", "fused"):
    if mode == "fused": os.environ["SPECWALK_K2_FUSED"] = "1"
    S = sw.Spectrahedron.from_instance(inst)
    for (x0, tag, ch) in [(None, 0, 256), (np.zeros((256, 12)), 0, 256), (None, 3 << 28, 256), (None, 0, 64), (None, 0, 1024)]:
        try:
            out = S.walk_sample(ch, 20, 2 * math.sqrt(12), 120, 0, x0=x0, tag=tag)
            print(mode, "x0" if x0 is not None else "-", tag, ch, json.dumps(out["stats"]), flush=True)
        except Exception as e:
            print(mode, "x0" if x0 is not None else "-", tag, ch, "ERR", e, flush=True)
    S.close()
