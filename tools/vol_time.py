"""configs[2] volume wall time (eps 0.1, 4096 chains/phase) for given seeds: python tools/vol_time.py 0 1 2"""
import json, sys, time
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen
S = sw.Spectrahedron.from_instance(specgen.config_instance(2))
S.volume(0.1, 99, 512, walk_len=2, burn=4)  # warm-up
for a in sys.argv[1:]:
    t0 = time.time()
    r = S.volume(0.1, int(a), 4096)
    print(json.dumps(dict(seed=int(a), seconds=time.time() - t0, volume=r["volume"], phases=r["phases"], calls=r["calls"])), flush=True)
