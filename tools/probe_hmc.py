"""Timing probe of the HMC-r walk (K5) on the configs[3] instance."""
import json, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen
for c in sys.argv[1:] or ["100:100:1024:2"]:
    n, m, chains, steps = map(int, c.split(":"))
    inst = specgen.rand_cube(n, m, 3)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(specgen.objective(n, 3))
    S.walk_sample(min(chains, 148), 1, 1.0, 10 * n, seed=1, kind=sw.HMC, T=1.0, final=False)
    out = S.walk_sample(chains, steps, 1.0, 10 * n, seed=3, kind=sw.HMC, T=1.0, final=False)
    st = out["stats"]
    print(json.dumps(dict(n=n, m=m, chains=chains, steps=steps, calls=st["calls"], ms=st["device_ms"],
                          calls_per_s=st["calls"] / (st["device_ms"] * 1e-3),
                          refl_per_step=st["reflections"] / max(st["steps"], 1), rounds=st["rounds"])), flush=True)
