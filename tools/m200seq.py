import sys, math, gc
sys.path.insert(0,'.')
import numpy as np, torch
import paper_2010_03817_b200 as sw, specgen, oracle
def dev_state(S, chains, rounds, steps, L, rho, seed):
    S.walk_begin(chains, steps, L, rho, seed)
    S.walk_rounds(rounds)
    X = torch.empty((chains, S.n), dtype=torch.float64, device="cuda")
    st = S.walk_end(final_x=X)
    return X.cpu().numpy(), st
S1 = sw.Spectrahedron.from_instance(specgen.config_instance(3))
X1, st1 = dev_state(S1, 65536, 12, 100, 20.0, 1000, 4)
print("m100", st1["calls"], X1[0][:3], flush=True)
if len(sys.argv) > 1: S1.close(); del S1; gc.collect()
inst = specgen.config_instance(4)
S2 = sw.Spectrahedron.from_instance(inst)
L = 2 * math.sqrt(200)
X2, st2 = dev_state(S2, 65536, 2, 100, L, 2000, 4)
print("m200", st2, flush=True)
lmi = oracle.Lmi(inst)
for c in (0, 65535):
    xo, calls = oracle.replay(lmi, oracle.BILLIARD, 4, c, 100, L, 2000, 2)
    print(c, "diff", np.linalg.norm(X2[c] - xo), "|x|", np.linalg.norm(X2[c]), "nonzero", np.count_nonzero(X2[c]), "mem", torch.cuda.mem_get_info())
