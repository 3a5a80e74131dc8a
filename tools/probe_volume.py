"""Volume time at n = m = 40 (BASELINE.json metric, second half; configs[2] instance)."""
import json, sys, time
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen
seeds = [int(s) for s in (sys.argv[1:] or ["0"])]
inst = specgen.config_instance(2)
S = sw.Spectrahedron.from_instance(inst)
S.volume(0.1, 99, 512, walk_len=2, burn=5)  # warm-up (module load, first launches)
for s in seeds:
    t0 = time.time()
    r = S.volume(0.1, s, 4096)
    print(json.dumps(dict(seed=s, wall_s=time.time() - t0, **{k: r[k] for k in ("volume", "std_rel", "phases", "chains", "calls", "device_ms", "radii", "ratios", "q")})), flush=True)
