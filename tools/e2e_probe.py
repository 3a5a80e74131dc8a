"""End-to-end calls/s through walk_sample with host buffers on the M100 instance for several
(chains, steps) shapes (H2D x0, D2H end points + moments inside the timed region).
  python tools/e2e_probe.py chains:steps ..."""
import json, math, sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2010_03817_b200 as sw
import specgen

S = sw.Spectrahedron.from_instance(specgen.config_instance(3))
stream = torch.cuda.ExternalStream(S.stream())
S.walk_sample(4096, 1, 20.0, 1000, 4)  # warm-up
for arg in sys.argv[1:]:
    c, k = map(int, arg.split(":"))
    x0 = np.zeros((c, 100))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(stream)
    out = S.walk_sample(c, k, 20.0, 1000, 4, x0=x0)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    st = out["stats"]
    print(json.dumps(dict(chains=c, steps=k, calls=st["calls"], rounds=st["rounds"], ms=ms,
                          calls_per_s=st["calls"] / (ms * 1e-3), mean_calls_per_chain=st["calls"] / c)), flush=True)
