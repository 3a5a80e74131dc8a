"""Volume estimator at configs[2] (n = m = 40): burn-in / walk-length sensitivity over seeds."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2010_03817_b200 as sw
import specgen
S = sw.Spectrahedron.from_instance(specgen.config_instance(2))
S.volume(0.1, 99, 512, walk_len=2, burn=4)
for burn, wl in [(40, 10), (20, 10)]:
    vs, ts, ph = [], [], []
    for sd in range(int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[1]) if len(sys.argv) > 1 else 8):
        t = time.time()
        r = S.volume(0.1, sd, 4096, walk_len=wl, burn=burn)
        ts.append(time.time() - t); vs.append(r["volume"]); ph.append(r["phases"])
    vs = np.array(vs)
    print(json.dumps(dict(burn=burn, walk_len=wl, mean=vs.mean(), sd=vs.std(ddof=1), se=vs.std(ddof=1) / np.sqrt(len(vs)),
                          time_mean=float(np.mean(ts)), phases=ph)), flush=True)
