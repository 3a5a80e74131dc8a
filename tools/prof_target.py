"""Profiling driver: a few scheduler rounds of one bench workload (for ncu --set full).
  python tools/prof_target.py m100|m200|hmc [warm_rounds] [rounds]
m100: configs[3] instance, billiard (bench.py's timed workload); m200: configs[4]; hmc:
configs[3] HMC-r (T = 1, L = 1.09).  65536 chains, seed 4 (HMC: 3)."""
import math
import sys

sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw  # noqa: E402
import specgen  # noqa: E402

what = sys.argv[1]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if what == "m200":
    S = sw.Spectrahedron.from_instance(specgen.config_instance(4))
    S.walk_begin(65536, 100, 2 * math.sqrt(200), 2000, 4)
elif what == "hmc":
    S = sw.Spectrahedron.from_instance(specgen.config_instance(3))
    S.set_objective(specgen.objective(100, 3))
    S.walk_begin(65536, 200, 1.09, 1000, 3, kind=sw.HMC, T=1.0)
else:
    S = sw.Spectrahedron.from_instance(specgen.config_instance(3))
    S.walk_begin(65536, 100, 20.0, 1000, 4)
S.walk_rounds(warm)
S.walk_rounds(rounds)
print(what, S.walk_end())
