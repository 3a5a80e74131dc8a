"""Compare the K2 split path with the fused kernel on the same walk (SPECWALK_K2_FUSED toggles at create)."""
import os, sys, math, json
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
res = {}
for mode in ("split", "fused"):
    if mode == "fused": os.environ["SPECWALK_K2_FUSED"] = "1"
    else: os.environ.pop("SPECWALK_K2_FUSED", None)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_ball(np.zeros(12), float(sys.argv[1]) if len(sys.argv) > 1 else 0.3)
    try:
        out = S.walk_sample(256, 5, 2 * math.sqrt(12), 120, seed=3)
        res[mode] = (out["final_x"], out["stats"])
        print(mode, json.dumps(out["stats"]))
    except Exception as e:
        print(mode, "ERR", e)
    S.close()
if len(res) == 2:
    d = np.abs(res["split"][0] - res["fused"][0]).max()
    print("max |x_split - x_fused| =", d)
