"""Write the oracle-side reference values the GPU statistical parity tests compare
against, where the oracle is too slow to run inside a GPU test session.

Calls ONLY the CPU oracle (oracle/) on seeded inputs from specgen/ -- nothing from
the CUDA path.  Each output JSON records the workload, the per-seed / per-chain
oracle values and the wall time.  Usage:

    python tests/golden/make_oracle_goldens.py volume_cfg2      # ~40 min on 8 cores
    python tests/golden/make_oracle_goldens.py expectation_cfg3 # ~10 min on 8 cores

Workloads (reduced equally on both sides, VERDICT r1 "Close parity"; DESIGN.md
"Statistical parity at the BASELINE configs"):

* volume_cfg2: BASELINE.json configs[2] instance (rand-cube n = m = 40, instance
  seed 2), ball-phase MMC (eq:mmc_vol P:1291-1300) at eps = 0.3 with 512 chains per
  phase, walk length 10, burn-in 20 (R25), seeds 0..9.  (configs[2]'s own eps = 0.1 with
  4096 chains/phase is ~9e6 oracle calls per seed: hours on the host.)
* expectation_cfg3: BASELINE.json configs[3] (rand-cube n = m = 100, instance seed 3,
  c = objective(100, 3)), HMC-r (Alg. 6) for exp(-c^T x / T), T = 1, L = 1.09
  (SURVEY 8(c).2 #8), rho = 1000, walk seed 3, global chain ids 0..127, 12 steps from 0:
  per-chain f values for f = c^T x and f = |x|^2.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import specgen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

VOLUME_CFG2 = dict(instance=2, eps=0.3, chains_per_phase=512, walk_len=10, burn=20, seeds=list(range(10)))
EXPECT_CFG3 = dict(instance=3, T=1.0, L=1.09, rho=1000, seed=3, chains=128, steps=12)


def volume_cfg2():
    cfg = VOLUME_CFG2
    inst = specgen.config_instance(cfg["instance"])
    out = dict(workload=cfg, seeds={}, script=os.path.relpath(__file__, ROOT))
    for s in cfg["seeds"]:
        t0 = time.time()
        r = oracle.volume(inst, cfg["eps"], s, cfg["chains_per_phase"], W=cfg["walk_len"], burn=cfg["burn"])
        r = {k: (float(v) if isinstance(v, (float, np.floating)) else v) for k, v in r.items()}
        r["radii"] = [float(x) for x in r["radii"]]
        r["ratios"] = [float(x) for x in r["ratios"]]
        r["seconds"] = time.time() - t0
        out["seeds"][str(s)] = r
        print(f"seed {s}: volume {r['volume']:.6g} phases {r['phases']} chains {r['chains']} "
              f"calls {r['calls']} {r['seconds']:.0f} s", flush=True)
        json.dump(out, open(os.path.join(HERE, "oracle_volume_cfg2.json"), "w"), indent=1)


def expectation_cfg3():
    cfg = EXPECT_CFG3
    inst = specgen.config_instance(cfg["instance"])
    c = specgen.objective(inst.n, cfg["instance"])
    lmi = oracle.Lmi(inst)
    t0 = time.time()
    X, st = oracle.walk(lmi, oracle.HMC, cfg["seed"], 0, cfg["chains"], cfg["steps"], cfg["L"], cfg["rho"],
                        T=cfg["T"], c=c)
    out = dict(workload=cfg, script=os.path.relpath(__file__, ROOT), seconds=time.time() - t0, stats=st,
               f_linear_c=[float(v) for v in X @ c], f_sqnorm=[float(v) for v in (X * X).sum(1)])
    json.dump(out, open(os.path.join(HERE, "oracle_expectation_cfg3.json"), "w"), indent=1)
    print(f"expectation_cfg3: {out['seconds']:.0f} s, stats {st}", flush=True)


if __name__ == "__main__":
    for what in sys.argv[1:]:
        globals()[what]()
