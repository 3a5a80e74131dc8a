"""GPU parity for reflective HMC (Alg. 6, eq:boltz_ode): the CUDA K5 kernel
(monotone Weyl stepping on the quadratic / sqrt-deflated quartic pencil) vs the
CPU oracle (mu-companion + Francis QR), per call, per trajectory and in law."""
import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu
TOL_T = 1e-9
TOL_COS = 1e-10


def _interior(inst, lmi, count, seed, vscale=1.0):
    n = inst.n
    us = specgen.unit_vectors(count, n, seed)
    lams = specgen.uniforms(count, seed, 0.0, 0.9)
    xs = np.array([lams[k] * min(oracle.chord(lmi, np.zeros(n), us[k])["t_plus"], 1e6) * us[k] for k in range(count)])
    vs = np.random.default_rng(seed + 7).standard_normal((count, n)) * vscale
    return xs, vs


def _cmp(res, refs, lmi):
    for k, r in enumerate(refs):
        assert res["binding"][k] == lmi.binding_code(r["block"]), (k, res["binding"][k], r["block"])
        assert abs(res["t_plus"][k] - r["t_plus"]) <= TOL_T * r["t_plus"], (k, res["t_plus"][k], r["t_plus"])
        w = oracle.normal(lmi, r["block"], r["y"])
        cos = float(res["normal"][k] @ w)
        assert cos >= 1 - TOL_COS, (k, cos)


CASES = [
    ("rand_10_10", lambda: specgen.rand_cube(10, 10, 0), 1.0, 1.0),
    ("rand_40_40", lambda: specgen.rand_cube(40, 40, 2), 1.0, 1.0),
    ("rand_100_100", lambda: specgen.rand_cube(100, 100, 3), 1.0, 1.0),
    ("mixed_12_30", lambda: specgen.rand_cube(12, 30, 5, scale=1 / np.sqrt(12)), 0.5, 0.3),
    ("cube_only_6", lambda: specgen.cube_only(6), 1.0, 0.2),
    # K5 split variants: <256, KC 8> (m <= 64), <512, 13> (m <= 104), <512, 16> (m <= 112);
    # larger m runs the fused global-scratch hmc_kernel
    ("rand_16_110", lambda: specgen.rand_cube(16, 110, 7), 1.0, 1.0),
    ("rand_10_136", lambda: specgen.rand_cube(10, 136, 8), 1.0, 1.0),
]


@pytest.mark.parametrize("name,make,vscale,T", CASES, ids=[c[0] for c in CASES])
def test_hmc_oracle_interior_parity(name, make, vscale, T):
    import paper_2010_03817_b200 as sw
    inst = make()
    lmi = oracle.Lmi(inst)
    c = specgen.objective(inst.n, 3)
    count = 8 if inst.m >= 100 else 24
    xs, vs = _interior(inst, lmi, count, 11, vscale)
    refs = [oracle.hmc_chord(lmi, xs[k], vs[k], c, T) for k in range(count)]
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    res = S.hmc_oracle(xs, vs, T)
    _cmp(res, refs, lmi)


BCASES = CASES[:4] + CASES[5:]


@pytest.mark.parametrize("name,make,vscale,T", BCASES, ids=[c[0] for c in BCASES])
def test_hmc_oracle_boundary_start_parity(name, make, vscale, T):
    """After a dense reflection the segment starts on the boundary: sqrt(t) deflation (SURVEY a-10)."""
    import paper_2010_03817_b200 as sw
    inst0 = make()
    inst = specgen.Instance(inst0.name, inst0.A)  # dense block only
    lmi = oracle.Lmi(inst)
    n = inst.n
    c = specgen.objective(n, 3)
    count = 6 if inst.m >= 100 else 16
    xs, vs = _interior(inst, lmi, count, 13, vscale)
    hits, ss, us = [], [], []
    for k in range(count):
        r = oracle.hmc_chord(lmi, xs[k], vs[k], c, T)
        t = r["t_plus"]
        hit = xs[k] + t * vs[k] - c * t * t / (2 * T)
        u = vs[k] - c * t / T
        w = oracle.normal(lmi, r["block"], r["y"])
        hits.append(hit)
        ss.append(oracle.reflect(u, w))
        us.append(r["y"] / np.linalg.norm(r["y"]))
    hits, ss, us = map(np.array, (hits, ss, us))
    refs = [oracle.hmc_chord(lmi, hits[k], ss[k], c, T, F0=lmi.eval_block(0, hits[k]), bound=0, u=us[k])
            for k in range(count)]
    S = sw.Spectrahedron(inst.A)
    S.set_objective(c)
    res = S.hmc_oracle(hits, ss, T, u=us)
    _cmp(res, refs, lmi)


HMC_TRAJ = {
    # name: (instance, c, T, L, rho, walk seed, steps, chains, reflections)
    "mixed_10": (lambda: specgen.rand_cube(10, 10, 1, scale=0.5), lambda: specgen.objective(10, 1), 0.5, 2.0, 100, 2,
                 40, 64, 15),
    "m40_split": (lambda: specgen.rand_cube(12, 40, 4, scale=1 / np.sqrt(12)), lambda: specgen.objective(12, 4), 0.5,
                  2.0, 100, 6, 10, 32, 10),
    # configs[3]'s own workload (T = 1, tau = 1.09: SURVEY 8(c).2 #8)
    "configs3": (lambda: specgen.config_instance(3), lambda: specgen.objective(100, 3), 1.0, 1.09, 1000, 3, 5, 64, 20),
}


@pytest.mark.parametrize("name", list(HMC_TRAJ))
def test_hmc_trajectory_parity(name):
    """HMC-r trajectories (Alg. 6) through the first reflections of every chain vs the oracle
    (companion + QR roots), 1e-8, each chain up to its chaos horizon (R27); all chains must pass."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    import paper_2010_03817_b200 as sw
    from _traj import traj_parity
    make, mc, T, L, rho, seed, steps, nch, R = HMC_TRAJ[name]
    inst = make()
    c = mc()
    lmi = oracle.Lmi(inst)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    chains = list(range(nch))
    g = S.walk_trace(chains, steps=steps, L=L, rho=rho, seed=seed, max_refl=R, kind=sw.HMC, T=T)
    with ThreadPoolExecutor(os.cpu_count() or 4) as pool:
        rep, fails = traj_parity(g, lmi, oracle.HMC, seed, chains, steps, L, rho, R, inst.n, pool, T=T, c=c)
    print(f"[parity] hmc_trajectory_{name}: {rep}")
    assert not fails, fails[:8]
    assert rep["records_available"] > 0
    # HMC-r amplifies perturbations fast (|v| ~ sqrt(n)): the coverage is reported; R27
    assert rep["fraction_compared"] >= 0.5, rep["fraction_compared"]


def test_hmc_boltzmann_cube_moments_gpu():
    """pi ~ exp(-c.x/T) on [-1,1]^n: independent truncated exponentials (P1)."""
    import paper_2010_03817_b200 as sw
    n = 4
    inst = specgen.cube_dense(n)  # the cube as a dense diagonal LMI: exercises K5's dense path
    c = np.array([1.0, -0.6, 2.5, 0.3])
    T = 1.0
    S = sw.Spectrahedron(inst.A)
    S.set_objective(c)
    out = S.walk_sample(3000, 20, 2.0, 100, seed=5, kind=sw.HMC, T=T)
    X = out["final_x"]
    grid = np.linspace(-1, 1, 200001)
    for i in range(n):
        dens = np.exp(-c[i] * grid / T)
        Z = np.trapezoid(dens, grid)
        e1 = np.trapezoid(grid * dens, grid) / Z
        se = X[:, i].std(ddof=1) / np.sqrt(len(X))
        assert abs(X[:, i].mean() - e1) <= 4.5 * se, (i, X[:, i].mean(), e1, se)
    assert out["stats"]["failures"] == 0
