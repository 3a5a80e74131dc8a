"""Parity at BASELINE.json's configs (GPU through the C-ABI vs the CPU oracle on the
same seeded inputs; tolerances from BASELINE.json north_star):

* per trajectory: chains 0..63 through their first 20 reflections at configs[0],
  the configs[3] instance under the M100 billiard workload, configs[4], plus a
  mixed dense/cube-face body and n = m = 40 -- hit points, t, normals and
  post-reflection directions to 1e-8, binding ids exact.  Every chain must pass
  up to its chaos horizon (SURVEY P16 / DESIGN.md R27): the oracle is re-run from a
  start perturbed by 1e-13 and the comparison of a chain stops at the first
  reflection whose oracle-vs-perturbed-oracle amplification exceeds 1e4 (beyond
  it a per-call difference of 1e-12 -- 1000x below the 1e-9 per-call bound -- can
  legitimately exceed 1e-8).  The fraction of records compared is reported and
  must stay >= 0.9.  (R27: the horizon is TOL / the per-call budget the per-call tests assert.)
* per call: 256 interior and 256 boundary-start lines at m = 100 and m = 200 for
  the billiard chord (Alg. 2, Schur deflation R6) and the HMC-r chord (Alg. 6,
  eq:boltz_ode): t+ (and t-) to 1e-9 relative, normals cos >= 1 - 1e-10, binding exact.

Set SPECWALK_PARITY_REPORT=<dir> to write one JSON summary per test there."""
import json
import math
import os
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import specgen
from _traj import PER_CALL_ASSERT, PER_CALL_BUDGET_HMC, traj_parity

pytestmark = pytest.mark.gpu

TOL_TRAJ = 1e-8
TOL_T = 1e-9
TOL_COS = 1e-10
R = 20
POOL = ThreadPoolExecutor(os.cpu_count() or 4)  # the oracle's C calls release the GIL


def _report(name: str, data: dict):
    d = os.environ.get("SPECWALK_PARITY_REPORT")
    line = json.dumps(data, default=float)
    print(f"[parity] {name}: {line}")
    if d:
        os.makedirs(d, exist_ok=True)
        with open(os.path.join(d, f"{name}.json"), "w") as f:
            f.write(line + "\n")


# ---------------------------------------------------------------- trajectories
TRAJ = {
    # name: (instance, L, rho, walk seed, steps)
    "cfg0": (lambda: specgen.config_instance(0), 2 * math.sqrt(10), 100, 0, 50),
    "mixed": (lambda: specgen.rand_cube(10, 10, 1, scale=0.3), 2 * math.sqrt(10), 100, 0, 50),
    "m40": (lambda: specgen.rand_cube(40, 40, 2), 2 * math.sqrt(40), 400, 0, 50),
    "m100": (lambda: specgen.config_instance(3), 20.0, 1000, 4, 3),
    "cfg4": (lambda: specgen.config_instance(4), 2 * math.sqrt(200), 2000, 4, 3),
}


@pytest.mark.parametrize("cfg", list(TRAJ))
def test_trajectory_parity_64_chains_20_reflections(cfg):
    import paper_2010_03817_b200 as sw
    make, L, rho, seed, steps = TRAJ[cfg]
    inst = make()
    n = inst.n
    lmi = oracle.Lmi(inst)
    chains = list(range(64))
    S = sw.Spectrahedron.from_instance(inst)
    g = S.walk_trace(chains, steps=steps, L=L, rho=rho, seed=seed, max_refl=R)
    rep, fails = traj_parity(g, lmi, oracle.BILLIARD, seed, chains, steps, L, rho, R, n, POOL)
    _report(f"trajectory_{cfg}", rep)
    assert not fails, fails[:8]
    assert rep["fraction_compared"] >= 0.9, rep["fraction_compared"]


# ---------------------------------------------------------------- per call, 256 lines
PER_CALL = {"m100": lambda: specgen.config_instance(3), "m200": lambda: specgen.config_instance(4)}
N_LINES = 256


def _interior(inst, lmi, count, seed, hmc):
    n = inst.n
    us = specgen.unit_vectors(count, n, seed)
    lams = specgen.uniforms(count, seed, 0.0, 0.95)
    tps = list(POOL.map(lambda u: oracle.chord(lmi, np.zeros(n), u)["t_plus"], us))
    xs = np.array([lams[k] * min(tps[k], 1e6) * us[k] for k in range(count)])
    if hmc:  # HMC velocity v ~ N(0, I) (Alg. 6)
        vs = np.random.default_rng(seed + 7).standard_normal((count, n))
    else:
        vs = specgen.unit_vectors(count, n, seed + 1)
    return xs, vs


def _cmp_lines(res, refs, lmi, what, dw=None):
    bad, worst_t, worst_c = [], 0.0, 0.0
    for k, r in enumerate(refs):
        code = lmi.binding_code(r["block"])
        if res["binding"][k] != code:
            bad.append((k, "binding", int(res["binding"][k]), code))
            continue
        et = abs(res["t_plus"][k] - r["t_plus"]) / abs(r["t_plus"])
        if "t_minus" in r and np.isfinite(r["t_minus"]) and r["t_minus"] != 0.0:
            et = max(et, abs(res["t_minus"][k] - r["t_minus"]) / abs(r["t_minus"]))
        w = r["w"]
        if w is None:  # degenerate hit (rank <= m-2, measure zero): nothing to compare
            continue
        cos = float(res["normal"][k] @ w) / (np.linalg.norm(res["normal"][k]) * np.linalg.norm(w))
        if dw is not None:
            dw.append(float(np.linalg.norm(res["normal"][k] - w)))
        worst_t, worst_c = max(worst_t, et), max(worst_c, 1 - cos)
        if not (et <= TOL_T and 1 - cos <= TOL_COS):
            bad.append((k, what, et, 1 - cos))
    return bad, worst_t, worst_c


@pytest.mark.parametrize("name", list(PER_CALL))
@pytest.mark.parametrize("kind", ["billiard", "hmc"])
def test_per_call_parity_256_interior_and_boundary(kind, name):
    import paper_2010_03817_b200 as sw
    inst = PER_CALL[name]()
    n = inst.n
    hmc = kind == "hmc"
    T = 1.0
    c = specgen.objective(n, 3)
    lmi = oracle.Lmi(inst)
    seed = zlib.crc32(f"{kind}-{name}".encode()) % 1000
    xs, vs = _interior(inst, lmi, N_LINES, seed, hmc)

    def ref_int(k):
        if hmc:
            r = oracle.hmc_chord(lmi, xs[k], vs[k], c, T)
        else:
            r = oracle.chord(lmi, xs[k], vs[k])
        r["w"] = oracle.normal(lmi, r["block"], r["y"])  # cube blocks give +-e_i (O2)
        return r

    refs = list(POOL.map(ref_int, range(N_LINES)))
    S = sw.Spectrahedron.from_instance(inst)
    if hmc:
        S.set_objective(c)
        res = S.hmc_oracle(xs, vs, T)
    else:
        res = S.boundary_oracle(xs, vs)
    dw_i, dw_b = [], []
    bad_i, wt_i, wc_i = _cmp_lines(res, refs, lmi, "interior", dw_i)

    # boundary starts: the oracle's dense hits, unit kernel u = y/|y|, reflected velocity
    dense = [k for k in range(N_LINES) if refs[k]["block"] == 0]
    hits, us, ss = [], [], []
    for k in dense:
        t = refs[k]["t_plus"]
        if hmc:
            hit = xs[k] + t * vs[k] - c * t * t / (2 * T)
            vel = vs[k] - c * t / T
        else:
            hit = xs[k] + t * vs[k]
            vel = vs[k]
        hits.append(hit)
        us.append(refs[k]["y"] / np.linalg.norm(refs[k]["y"]))
        ss.append(oracle.reflect(vel, refs[k]["w"]))
    hits, us, ss = np.array(hits), np.array(us), np.array(ss)

    def ref_bnd(k):
        F = lmi.eval_block(0, hits[k])
        if hmc:
            r = oracle.hmc_chord(lmi, hits[k], ss[k], c, T, F0=F, bound=0, u=us[k])
        else:
            r = oracle.chord(lmi, hits[k], ss[k], F0=F, bound=0, u=us[k])
        r["w"] = oracle.normal(lmi, r["block"], r["y"])  # cube blocks give +-e_i (O2)
        return r

    brefs = list(POOL.map(ref_bnd, range(len(dense))))
    if hmc:
        bres = S.hmc_oracle(hits, ss, T, u=us)
    else:
        bres = S.boundary_oracle(hits, ss, u=us)
        assert np.all(bres["t_minus"] == 0.0)
    # lines whose boundary start the oracle rejects as outward are skipped on both sides
    keep = [k for k in range(len(dense)) if not brefs[k].get("outward", False)]
    bsub = {k: v[keep] for k, v in bres.items()}
    bad_b, wt_b, wc_b = _cmp_lines(bsub, [brefs[k] for k in keep], lmi, "boundary", dw_b)
    _report(f"per_call_{kind}_{name}", dict(interior=N_LINES, boundary=len(keep), interior_fail=len(bad_i),
                                            boundary_fail=len(bad_b), worst_rel_t_interior=wt_i,
                                            worst_1mcos_interior=wc_i, worst_rel_t_boundary=wt_b,
                                            worst_1mcos_boundary=wc_b,
                                            normal_diff_max=max(dw_i + dw_b), normal_diff_median=float(np.median(dw_i + dw_b))))
    assert len(keep) >= 200, len(keep)
    assert not bad_i, bad_i[:8]
    assert not bad_b, bad_b[:8]
    # the per-call budget the trajectory horizon assumes (tests/_traj.py, R27)
    budget = PER_CALL_BUDGET_HMC if hmc else PER_CALL_ASSERT
    assert max(dw_i + dw_b) <= budget, (max(dw_i + dw_b), budget)
