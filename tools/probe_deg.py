import sys, math, json
sys.path.insert(0,'.')
import numpy as np
import paper_2010_03817_b200 as sw, specgen
for (n,m,seed) in [(12,12,2),(10,10,0),(40,40,2),(100,100,3)]:
    inst = specgen.rand_cube(n,m,seed) if (n,m)!=(100,100) else specgen.config_instance(3)
    S = sw.Spectrahedron.from_instance(inst)
    ch = 4096 if n < 100 else 2048
    out = S.walk_sample(ch, 20 if n<100 else 2, 2*math.sqrt(n), 10*n, seed=7)
    print(json.dumps(dict(n=n, **{k:v for k,v in out["stats"].items()})))
