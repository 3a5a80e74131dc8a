"""Quick timing probe of walk_sample on BASELINE-shaped instances (not the bench)."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen

cfgs = sys.argv[1:] or ["10:10:4096:5", "40:40:2048:2", "100:100:1024:1"]
for c in cfgs:
    n, m, chains, steps = map(int, c.split(":"))
    inst = specgen.rand_cube(n, m, 3)
    S = sw.Spectrahedron.from_instance(inst)
    S.walk_sample(min(chains, 256), 1, 2 * np.sqrt(n), 10 * n, seed=1, final=False)
    t0 = time.time()
    out = S.walk_sample(chains, steps, 2 * np.sqrt(n), 10 * n, seed=4, final=False)
    wall = time.time() - t0
    st = out["stats"]
    print(json.dumps(dict(n=n, m=m, chains=chains, steps=steps, calls=st["calls"], ms=st["device_ms"],
                          calls_per_s=st["calls"] / (st["device_ms"] * 1e-3), wall=wall,
                          refl_per_step=st["reflections"] / max(st["steps"], 1), rounds=st["rounds"],
                          rejects=st["rejects"], degenerates=st["degenerates"])), flush=True)
