"""Per-phase cycle breakdown of K2 (SPECWALK_PROF=1) on a BASELINE-shaped instance.
  SPECWALK_PROF=1 python tools/prof_probe.py n:m:chains:rounds ...
Prints calls/s (device events) and the library's [specwalk prof] lines (stderr)."""
import json, math, sys
sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen

for c in sys.argv[1:] or ["100:100:8192:40"]:
    n, m, chains, rounds = map(int, c.split(":"))
    inst = specgen.config_instance(3) if (n, m) == (100, 100) else specgen.rand_cube(n, m, 3)
    S = sw.Spectrahedron.from_instance(inst)
    S.walk_begin(chains, 100, 2 * math.sqrt(n), 10 * n, 4)
    S.walk_rounds(3)
    st0 = S.walk_stats_now()
    S.kernel_timing(True)
    S.lanczos_iterations(reset=True)
    S.walk_rounds(rounds)
    st1 = S.walk_stats_now()
    lz = S.lanczos_iterations(reset=True)
    kt = S.kernel_times()
    S.walk_end()
    calls = st1["calls"] - st0["calls"]
    k2 = kt["ms"]["K2_chord"]
    print(json.dumps(dict(n=n, m=m, chains=chains, rounds=rounds, calls=calls,
                          k2_calls_per_s=calls / (k2 * 1e-3), kernel_ms=kt["ms"], k2_phases_ms=kt["k2_phases_ms"],
                          lanczos=lz)), flush=True)
