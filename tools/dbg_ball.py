import math, sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw
import specgen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
S = sw.Spectrahedron.from_instance(specgen.ball(n))
for steps in (2, 6):
    try:
        o = S.walk_sample(512, steps, 2 * math.sqrt(n), 10 * n, 0)
        print("walk", steps, o["stats"], np.linalg.norm(o["final_x"], axis=1).max())
    except Exception as e:
        print("walk", steps, "ERR", e)
os.environ["SPECWALK_DEBUG_VOLUME"] = "1"
try:
    r = S.volume(0.3, 0, 512, walk_len=4, burn=6)
    print(r)
except Exception as e:
    print("volume ERR", e)
x = np.zeros((4, n)); v = specgen.unit_vectors(4, n, 1)
print(S.boundary_oracle(x, v)["t_plus"])
