import sys, math
sys.path.insert(0,'.')
import numpy as np, torch
import paper_2010_03817_b200 as sw, specgen, oracle
inst = specgen.config_instance(4)
S = sw.Spectrahedron.from_instance(inst)
L = 2*math.sqrt(200); R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
S.walk_begin(65536, 100, L, 2000, 4)
S.walk_rounds(R)
X = torch.empty((65536, 200), dtype=torch.float64, device="cuda")
st = S.walk_end(final_x=X)
print(st)
X = X.cpu().numpy()
lmi = oracle.Lmi(inst)
for c in (0, 65535):
    xo, calls = oracle.replay(lmi, oracle.BILLIARD, 4, c, 100, L, 2000, R)
    print(c, np.linalg.norm(X[c]-xo), np.linalg.norm(xo), np.linalg.norm(X[c]))
