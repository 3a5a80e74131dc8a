"""Context timings on the paper's own instance family S-n-m (A0 = Z Z^T + I,
A_i = blockdiag(Q~, -Q~)), shaped like its Tables 2 and 3 -- not the benchmark, and not
comparable point by point (the paper's random draws and seeds are not available, and its
volume schedule differs; R12-R14):

* Table 2 (tab:volumes): volume at e = 0.1 of S-40-40 / S-60-60 (10 seeds in the
  paper; here `--seeds` instances), wall time, phases, oracle calls.
* Table 3 (tab:bill_times): time to sample 200 points with the billiard walk at
  walk length W on S-100-100 and S-200-200 (here 200 independent chains x W steps from the
  start point 0, L = diameter-scale 2 sqrt(n), rho = 10 n).
  python tools/paper_context.py [--seeds K]"""
import argparse
import json
import math
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_03817_b200 as sw  # noqa: E402
import specgen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", type=int, default=3)
ap.add_argument("--volume-n", default="40,60")
ap.add_argument("--walk-n", default="100,200")
args = ap.parse_args()
out = {"table2_volume": [], "table3_billiard_200_points": []}
for n in map(int, args.volume_n.split(",")):
    for s in range(args.seeds):
        S = sw.Spectrahedron.from_instance(specgen.paper_random(n, n, s))
        S.volume(0.1, 99, 512, walk_len=2, burn=4)  # warm-up
        t0 = time.time()
        r = S.volume(0.1, s, 4096)
        out["table2_volume"].append(dict(instance=f"S-{n}-{n} (paper generator, seed {s})", eps=0.1,
                                         seconds=time.time() - t0, volume=r["volume"], std_rel=r["std_rel"],
                                         phases=r["phases"], oracle_calls=r["calls"],
                                         paper=dict(S40=6.7, S60=28.5).get(f"S{n}")))
        print(json.dumps(out["table2_volume"][-1]), flush=True)
for n in map(int, args.walk_n.split(",")):
    S = sw.Spectrahedron.from_instance(specgen.paper_random(n, n, 0))
    S.walk_sample(200, 1, 2 * math.sqrt(n), 10 * n, 1)  # warm-up
    for W in (1, 10, 50):
        torch.cuda.synchronize()
        t0 = time.time()
        o = S.walk_sample(200, W, 2 * math.sqrt(n), 10 * n, 7)
        dt = time.time() - t0
        out["table3_billiard_200_points"].append(dict(instance=f"S-{n}-{n} (paper generator, seed 0)", walk_length=W,
                                                      seconds=dt, oracle_calls=o["stats"]["calls"],
                                                      paper_seconds={100: {1: 1.4, 10: 7.7, 50: 28.2},
                                                                     200: {1: 16.2, 10: 148, 50: 722}}[n][W]))
        print(json.dumps(out["table3_billiard_200_points"][-1]), flush=True)
print(json.dumps(out))
