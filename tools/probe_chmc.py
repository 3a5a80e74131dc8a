"""Collocation HMC-r throughput probe: calls/s, Weyl iterations, Picard iterations per segment."""
import math
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2010_03817_b200 as sw
import specgen


def run(name, inst, pot, sigma, q, h, L, chains, rounds=3, warm=3):
    S = sw.Spectrahedron.from_instance(inst)
    S.set_potential(pot, np.zeros(inst.n), sigma)
    S.walk_begin(chains, 1000, L, 100 * inst.n, 7, kind=sw.CHMC, q=q, h=h)
    S.walk_rounds(warm)
    st0 = S.walk_stats_now()
    S.lanczos_iterations(reset=True)
    S.chmc_counters(reset=True)
    S.kernel_timing(True)
    st = torch.cuda.ExternalStream(S.stream())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    S.walk_rounds(rounds)
    e1.record(st)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    st1 = S.walk_stats_now()
    lz = S.lanczos_iterations(reset=True)
    cc = S.chmc_counters(reset=True)
    kt = S.kernel_times()
    S.walk_end()
    calls = st1["calls"] - st0["calls"]
    print(f"{name}: {calls / ms * 1e3:.4g} calls/s  ms/round {ms / rounds:.2f}  weyl/call {lz['solves'] / calls:.2f}"
          f"  J {lz['mean_j']:.1f}  picard/seg {cc['picard'] / max(cc['segments'], 1):.2f}"
          f"  congr/call {cc['congruences'] / calls:.1f} refl {st1['reflections'] - st0['reflections']}"
          f"  kms {kt['ms']}", flush=True)


if __name__ == "__main__":
    G = sw.POT_GAUSS
    run("cube_dense_10 q3", specgen.cube_dense(10), G, 0.6, 3, 0.25, 2.0, 65536)
    run("rand_10_10 q3", specgen.rand_cube(10, 10, 0), G, 1.0, 3, 0.25, 2 * math.sqrt(10), 65536)
    run("rand_40_40 q3", specgen.config_instance(2), G, 1.0, 3, 0.25, 2 * math.sqrt(40), 65536)
    run("rand_100_100 q3", specgen.config_instance(3), G, 1.0, 3, 0.25, 2 * math.sqrt(100), 16384, rounds=2)
