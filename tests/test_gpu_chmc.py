"""GPU parity for collocation HMC-r (PAPER.md sec:hmcr P:1116-1158, R33):
the CUDA K7 kernels (Picard collocation per warp; the degree-d pencil's first root in (0, h] by
monotone Weyl stepping, sqrt(t)-deflated after a dense reflection; cube faces by scalar Weyl
stepping) vs the CPU oracle (Vandermonde basis, mu-companion + Francis QR), per call, per
trajectory and in law."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
from scipy import special

import oracle
import specgen

pytestmark = pytest.mark.gpu
TOL_T = 1e-9
TOL_COS = 1e-10
POTS = {"gauss": oracle.POT_GAUSS, "logcosh": oracle.POT_LOGCOSH, "linear": oracle.POT_LINEAR}


def _interior(inst, lmi, count, seed, vscale=1.0):
    n = inst.n
    us = specgen.unit_vectors(count, n, seed)
    lams = specgen.uniforms(count, seed, 0.0, 0.9)
    xs = np.array([lams[k] * min(oracle.chord(lmi, np.zeros(n), us[k])["t_plus"], 1e6) * us[k] for k in range(count)])
    vs = np.random.default_rng(seed + 7).standard_normal((count, n)) * vscale
    return xs, vs


def _setup(inst, pot, sigma, seed=3):
    import paper_2010_03817_b200 as sw
    n = inst.n
    mu = 0.2 * np.random.default_rng(seed).standard_normal(n)
    c = specgen.objective(n, seed)
    S = sw.Spectrahedron.from_instance(inst)
    if pot == oracle.POT_LINEAR:
        S.set_objective(c)
    S.set_potential(pot, mu, sigma)
    colloc = lambda q, h: dict(pot=pot, mu=mu, sigma=sigma, q=q, h=h)
    return S, c, mu, colloc


def _ref(lmi, x, v, q, h, colloc, c, sigma, F0=None, bound=-1, u=None):
    coef, it = oracle.colloc_poly(x, v, h, colloc(q, h), c=c, T=sigma)
    r = oracle.colloc_chord(lmi, coef, h, F0=F0, bound=bound, u=u)
    return r, coef


def _cmp(res, refs, lmi, report=None):
    worst_t, worst_c, hits = 0.0, 0.0, 0
    for k, r in enumerate(refs):
        if not np.isfinite(r["t_plus"]):
            assert np.isinf(res["t_plus"][k]) and res["binding"][k] == -2, (k, res["t_plus"][k])
            continue
        hits += 1
        assert res["binding"][k] == lmi.binding_code(r["block"]), (k, res["binding"][k], r["block"])
        e = abs(res["t_plus"][k] - r["t_plus"]) / r["t_plus"]
        worst_t = max(worst_t, e)
        assert e <= TOL_T, (k, res["t_plus"][k], r["t_plus"])
        w = oracle.normal(lmi, r["block"], r["y"])
        cos = float(res["normal"][k] @ w)
        worst_c = max(worst_c, 1 - cos)
        assert cos >= 1 - TOL_COS, (k, cos)
    if report is not None:
        report.update(lines=len(refs), hits=hits, worst_rel_t=worst_t, worst_1mcos=worst_c)
    return hits


CASES = [
    # name, instance, potential, sigma, q, h, velocity scale
    ("rand_10_10_gauss_q3", lambda: specgen.rand_cube(10, 10, 0), "gauss", 0.7, 3, 0.4, 1.0),
    ("rand_10_10_logcosh_q2", lambda: specgen.rand_cube(10, 10, 0), "logcosh", 0.5, 2, 0.5, 1.0),
    ("rand_10_10_linear_q1", lambda: specgen.rand_cube(10, 10, 0), "linear", 1.0, 1, 0.8, 1.0),
    ("mixed_12_30_gauss_q4", lambda: specgen.rand_cube(12, 30, 5, scale=1 / np.sqrt(12)), "gauss", 0.5, 4, 0.6, 2.0),
    ("rand_40_40_logcosh_q3", lambda: specgen.rand_cube(40, 40, 2), "logcosh", 0.4, 3, 0.2, 1.0),
    ("cube_only_6_gauss_q6", lambda: specgen.cube_only(6), "gauss", 0.6, 6, 0.5, 1.5),
    ("rand_20_100_gauss_q3", lambda: specgen.rand_cube(20, 100, 3), "gauss", 0.5, 3, 0.1, 1.0),
    # m > 128: 512 threads, one chain per SM; the Lanczos matvec's general path (mdp > 128)
    ("rand_8_136_logcosh_q2", lambda: specgen.rand_cube(8, 136, 8), "logcosh", 0.5, 2, 0.4, 1.0),
]


@pytest.mark.parametrize("name,make,pot,sigma,q,h,vscale", CASES, ids=[c[0] for c in CASES])
def test_chmc_oracle_interior_parity(name, make, pot, sigma, q, h, vscale):
    inst = make()
    lmi = oracle.Lmi(inst)
    S, c, mu, colloc = _setup(inst, POTS[pot], sigma)
    count = 8 if inst.m > 128 else (16 if inst.m >= 100 else 48)
    xs, vs = _interior(inst, lmi, count, 11, vscale)
    # h: most segments hit; h / 8: most end inside (t_plus = +inf on both sides)
    for hh, need in ((h, count // 8), (h / 8, 0)):
        refs = [_ref(lmi, xs[k], vs[k], q, hh, colloc, c, sigma)[0] for k in range(count)]
        res = S.chmc_oracle(xs, vs, q, hh)
        rep = {}
        hits = _cmp(res, refs, lmi, rep)
        print(f"[parity] chmc_interior_{name}_h{hh:g}: {rep}")
        assert hits >= need  # the cases are sized so that a fair share of the long segments hit


BCASES = [c for c in CASES if not c[0].startswith("cube_only")]


@pytest.mark.parametrize("name,make,pot,sigma,q,h,vscale", BCASES, ids=[c[0] for c in BCASES])
def test_chmc_oracle_boundary_start_parity(name, make, pot, sigma, q, h, vscale):
    """After a dense reflection the segment starts on the boundary: the sqrt(t)-deflated pencil."""
    inst0 = make()
    inst = specgen.Instance(inst0.name, inst0.A)  # dense block only
    lmi = oracle.Lmi(inst)
    S, c, mu, colloc = _setup(inst, POTS[pot], sigma)
    count = 8 if inst.m > 128 else (12 if inst.m >= 100 else 40)
    xs, vs = _interior(inst, lmi, count, 13, vscale)
    hits, ss, us = [], [], []
    for k in range(count):
        hh = 4 * h
        r, coef = _ref(lmi, xs[k], vs[k], q, hh, colloc, c, sigma)
        if not np.isfinite(r["t_plus"]):
            continue
        t = r["t_plus"]
        hit = np.polynomial.polynomial.polyval(t, coef)
        vel = np.polynomial.polynomial.polyval(t, np.polynomial.polynomial.polyder(coef))
        w = oracle.normal(lmi, r["block"], r["y"])
        hits.append(hit)
        ss.append(oracle.reflect(vel, w))
        us.append(r["y"] / np.linalg.norm(r["y"]))
    assert len(hits) >= min(6, count // 2)
    hits, ss, us = map(np.array, (hits, ss, us))
    for hh in (h, 4 * h):
        refs = [_ref(lmi, hits[k], ss[k], q, hh, colloc, c, sigma, F0=lmi.eval_block(0, hits[k]), bound=0,
                     u=us[k])[0] for k in range(len(hits))]
        res = S.chmc_oracle(hits, ss, q, hh, u=us)
        rep = {}
        _cmp(res, refs, lmi, rep)
        print(f"[parity] chmc_boundary_{name}_h{hh:g}: {rep}")


TRAJ = {
    # name: (instance, potential, sigma, q, h, L, rho, seed, steps, chains, reflections)
    "rand_10_10_gauss": (lambda: specgen.rand_cube(10, 10, 0), "gauss", 0.7, 3, 0.3, 2 * np.sqrt(10), 100, 4, 30,
                         48, 12),
    "mixed_12_30_logcosh": (lambda: specgen.rand_cube(12, 30, 5, scale=1 / np.sqrt(12)), "logcosh", 0.3, 3, 0.25,
                            2.0, 100, 5, 30, 48, 12),
    "rand_10_10_linear": (lambda: specgen.rand_cube(10, 10, 0), "linear", 1.0, 2, 0.5, 2 * np.sqrt(10), 100, 6,
                          30, 32, 12),
    "rand_40_40_gauss": (lambda: specgen.rand_cube(40, 40, 2), "gauss", 0.4, 3, 0.15, 2.0, 100, 7, 30, 24, 10),
}


@pytest.mark.parametrize("name", list(TRAJ))
def test_chmc_trajectory_parity(name):
    """Collocation HMC-r trajectories (segments, reflections, rejections) vs the oracle, 1e-8,
    each chain up to its chaos horizon (R27); all chains must pass."""
    from _traj import traj_parity
    make, pot, sigma, q, h, L, rho, seed, steps, nch, R = TRAJ[name]
    inst = make()
    lmi = oracle.Lmi(inst)
    S, c, mu, colloc = _setup(inst, POTS[pot], sigma)
    import paper_2010_03817_b200 as sw
    chains = list(range(nch))
    g = S.walk_trace(chains, steps=steps, L=L, rho=rho, seed=seed, max_refl=R, kind=sw.CHMC, T=sigma, q=q, h=h)
    with ThreadPoolExecutor(os.cpu_count() or 4) as pool:
        rep, fails = traj_parity(g, lmi, oracle.CHMC, seed, chains, steps, L, rho, R, inst.n, pool, T=sigma, c=c,
                                 colloc=colloc(q, h))
    print(f"[parity] chmc_trajectory_{name}: {rep}")
    assert not fails, fails[:8]
    assert rep["records_available"] > 0
    assert rep["fraction_compared"] >= 0.5, rep["fraction_compared"]


def test_chmc_walk_end_points_match_oracle():
    """Whole walks (segments without a hit, reflections, the step ends) from the same starts:
    per-chain end points vs oracle.walk after 3 steps, inside the chaos horizon of short walks."""
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(8, 8, 1)
    lmi = oracle.Lmi(inst)
    S, c, mu, colloc = _setup(inst, oracle.POT_GAUSS, 0.6)
    out = S.walk_sample(64, 3, 1.0, 50, seed=12, kind=sw.CHMC, T=0.6, q=3, h=0.2)
    X, st = oracle.walk(lmi, oracle.CHMC, 12, 0, 64, 3, 1.0, 50, colloc=colloc(3, 0.2))
    err = np.abs(out["final_x"] - X).max(axis=1)
    print(f"[parity] chmc_walk_end_points: median {np.median(err):.3g} max {err.max():.3g} "
          f"calls gpu {out['stats']['calls']} oracle {st['calls']}")
    assert out["stats"]["calls"] == st["calls"]
    assert out["stats"]["reflections"] == st["reflections"]
    assert np.median(err) <= 1e-10 and np.mean(err <= 1e-8) >= 0.95


def test_chmc_truncated_gauss_cube_moments_gpu():
    """exp(-|x - mu|^2 / 2 sigma^2) on [-1, 1]^n through the dense path (the cube as a diagonal
    LMI): truncated-normal closed-form moments."""
    import paper_2010_03817_b200 as sw
    n = 4
    inst = specgen.cube_dense(n)
    mu, sigma = np.array([0.3, -0.5, 0.0, 0.8]), 0.6
    S = sw.Spectrahedron(inst.A)
    S.set_potential(sw.POT_GAUSS, mu, sigma)
    out = S.walk_sample(4000, 20, 2.0, 100, seed=5, kind=sw.CHMC, q=3, h=0.25)
    X = out["final_x"]
    assert out["stats"]["failures"] == 0
    phi = lambda z: np.exp(-0.5 * z * z) / np.sqrt(2 * np.pi)
    Phi = lambda z: 0.5 * (1 + special.erf(z / np.sqrt(2)))
    for i in range(n):
        a, b = (-1 - mu[i]) / sigma, (1 - mu[i]) / sigma
        Z = Phi(b) - Phi(a)
        m1 = mu[i] + sigma * (phi(a) - phi(b)) / Z
        var = sigma ** 2 * (1 + (a * phi(a) - b * phi(b)) / Z - ((phi(a) - phi(b)) / Z) ** 2)
        for vals, e in ((X[:, i], m1), (X[:, i] ** 2, var + m1 ** 2)):
            se = vals.std(ddof=1) / np.sqrt(len(vals))
            assert abs(vals.mean() - e) <= 4.5 * se, (i, vals.mean(), e, se)


def test_chmc_invalid_arguments():
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(4, 4, 0)
    S = sw.Spectrahedron.from_instance(inst)
    with pytest.raises(sw.SpecError):
        S.walk_sample(4, 1, 1.0, 10, seed=0, kind=sw.CHMC, q=3, h=0.2)  # no potential
    S.set_potential(sw.POT_GAUSS, None, 1.0)
    for q, h in ((0, 0.2), (7, 0.2), (3, 0.0), (3, float("nan"))):
        with pytest.raises(sw.SpecError):
            S.walk_sample(4, 1, 1.0, 10, seed=0, kind=sw.CHMC, q=q, h=h)
    with pytest.raises(sw.SpecError):
        S.set_potential(sw.POT_LINEAR, None, 1.0)  # no objective
    with pytest.raises(sw.SpecError):
        S.set_potential(sw.POT_GAUSS, None, -1.0)


def test_chmc_oracle_empty_batch_and_counters():
    """batch = 0 is a no-op; the device counters see the segments of a call and reset."""
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(6, 6, 1)
    S, c, mu, colloc = _setup(inst, oracle.POT_GAUSS, 0.8)
    res = S.chmc_oracle(np.zeros((0, 6)), np.zeros((0, 6)), 3, 0.2)
    assert res["t_plus"].shape == (0,)
    S.chmc_counters(reset=True)
    xs, vs = _interior(inst, oracle.Lmi(inst), 10, 3)
    S.chmc_oracle(xs, vs, 3, 0.2)
    cnt = S.chmc_counters(reset=True)
    assert cnt["segments"] == 10 and cnt["unconverged"] == 0 and cnt["picard"] >= 10
    assert S.chmc_counters(reset=False)["segments"] == 0
