import os, sys, json, math
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw, specgen
inst = specgen.rand_cube(12, 12, 2)
n = 12
for mode in ("split", "fused"):
    if mode == "fused": os.environ["SPECWALK_K2_FUSED"] = "1"
    S = sw.Spectrahedron.from_instance(inst)
    tag = lambda purpose, phase, ball, att=0: (purpose << 28) | (att << 20) | (phase << 1) | (1 if ball else 0)
    try:
        out = S.walk_sample(256, 20, 2 * math.sqrt(n), 120, 0, x0=np.zeros((256, n)), tag=tag(3, 0, False))
        X = out["final_x"]; print(mode, "pilot", json.dumps(out["stats"]))
        d = np.sort(np.linalg.norm(X, axis=1)); r = d[int(math.ceil(0.325 * 256)) - 1]
        inside = X[np.linalg.norm(X, axis=1) < r]
        X0 = (1 - 2.0 ** -40) * inside[np.arange(256) % len(inside)]
        S.set_ball(np.zeros(n), r)
        out = S.walk_sample(256, 5, 2 * math.sqrt(n), 120, 0, x0=X0, tag=tag(3, 1, False))
        print(mode, "phase1", r, json.dumps(out["stats"]))
        S.set_ball(np.zeros(n), 0.0)
        X0 = (1 - 2.0 ** -40) * X
        out = S.walk_sample(256, 5, 2 * math.sqrt(n), 120, 0, x0=X0, tag=tag(1, 0, False))
        print(mode, "est0", json.dumps(out["stats"]))
    except Exception as e:
        print(mode, "ERR", e)
    S.close()
