"""Pins for the oracle's collocation HMC-r (-m "not gpu", PAPER.md sec:hmcr
P:1116-1158, R33): the collocation polynomial against its defining conditions, the
harmonic-oscillator closed form (order q+2) and a library ODE solver; the degree-d PEP root
(Lemma 3 for a degree-d curve, companion P:320-354) against brute-force scanning, numpy.roots
on diagonal pencils and the Jacobi chord at d = 1; the walk against the Boltzmann HMC-r oracle
(f linear: the collocation is exact) and against closed-form / quadrature moments of
separable log-concave laws truncated to the cube."""
from math import comb

import numpy as np
import pytest
from scipy import integrate, special

import oracle
import specgen


def _gauss(mu, sigma, q, h):
    return dict(pot=oracle.POT_GAUSS, mu=mu, sigma=sigma, q=q, h=h)


def _logcosh(mu, sigma, q, h):
    return dict(pot=oracle.POT_LOGCOSH, mu=mu, sigma=sigma, q=q, h=h)


def _grad(pot, mu, sigma, x):
    if pot == oracle.POT_GAUSS:
        return (x - mu) / sigma ** 2
    return np.tanh((x - mu) / sigma) / sigma


def _peval(coef, t, der=0):
    P = np.polynomial.polynomial
    return np.array([P.polyval(t, P.polyder(coef[:, i], der) if der else coef[:, i]) for i in range(coef.shape[1])])


# ---------------------------------------------------------------- collocation basis and polynomial
@pytest.mark.parametrize("q", [1, 2, 3, 4, 6])
def test_nodes_chebyshev_and_lagrange(q):
    nodes, lc = oracle.colloc_basis(q)
    ref = (1.0 + np.polynomial.chebyshev.chebpts1(q)) / 2.0  # numpy's Chebyshev points of the first kind
    assert np.allclose(nodes, ref, rtol=0, atol=1e-15)
    for j in range(q):
        vals = np.polynomial.polynomial.polyval(nodes, lc[j])
        assert np.allclose(vals, np.eye(q)[j], rtol=0, atol=1e-12)


def test_colloc_linear_force_is_exact_quadratic():
    """f = c^T x / T: p'' = -c/T is constant, so the polynomial is p + v t - c t^2 / (2T)
    (the HMC-r trajectory of eq:boltz_ode P:1440-1446) for every q."""
    rng = np.random.default_rng(3)
    n = 5
    x0, v0, c = rng.normal(size=n), rng.normal(size=n), rng.normal(size=n)
    T = 0.7
    for q in (1, 2, 3, 5):
        coef, it = oracle.colloc_poly(x0, v0, 0.4, dict(pot=oracle.POT_LINEAR, q=q, h=0.4), c=c, T=T)
        assert 1 <= it <= 2
        assert np.array_equal(coef[0], x0) and np.array_equal(coef[1], v0)
        assert np.allclose(coef[2], -c / (2 * T), rtol=1e-13, atol=1e-15)
        assert np.abs(coef[3:]).max(initial=0.0) <= 1e-12


@pytest.mark.parametrize("pot", [oracle.POT_GAUSS, oracle.POT_LOGCOSH])
def test_colloc_conditions(pot):
    """The defining conditions: p(0) = x0, p'(0) = v0 and
    p''(s_j h) = -grad f(p(s_j h)) at every node."""
    rng = np.random.default_rng(5)
    n = 6
    mu = 0.3 * rng.normal(size=n)
    for q in (1, 2, 3, 4):
        for h in (0.05, 0.3):
            x0, v0 = 0.5 * rng.normal(size=n), rng.normal(size=n)
            cfg = dict(pot=pot, mu=mu, sigma=0.6, q=q, h=h)
            coef, it = oracle.colloc_poly(x0, v0, h, cfg)
            assert it > 0
            assert coef.shape == (q + 2, n)
            assert np.allclose(_peval(coef, 0.0), x0, atol=1e-15)
            assert np.allclose(_peval(coef, 0.0, 1), v0, atol=1e-15)
            nodes, _ = oracle.colloc_basis(q)
            for s in nodes:
                xs = _peval(coef, s * h)
                assert np.allclose(_peval(coef, s * h, 2), -_grad(pot, mu, 0.6, xs), rtol=1e-11, atol=1e-11)


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_colloc_gauss_order_vs_harmonic_closed_form(q):
    """f = |x - mu|^2 / (2 sigma^2): p(t) = mu + (x0 - mu) cos(wt) + v0 sin(wt) / w, w = 1/sigma.
    The error of the degree-(q+1) collocation polynomial on [0, h] is O(h^(q+2))."""
    rng = np.random.default_rng(7)
    n = 4
    mu, sigma = 0.2 * rng.normal(size=n), 0.7
    x0, v0 = 0.3 * rng.normal(size=n), rng.normal(size=n)
    w = 1.0 / sigma

    def err(h):
        coef, _ = oracle.colloc_poly(x0, v0, h, _gauss(mu, sigma, q, h))
        ts = np.linspace(0, h, 21)
        return max(np.abs(_peval(coef, t) - (mu + (x0 - mu) * np.cos(w * t) + v0 / w * np.sin(w * t))).max()
                   for t in ts)

    e1, e2, e3 = err(0.4), err(0.2), err(0.1)
    order = q + 2
    assert e1 / e2 >= 0.6 * 2 ** order and e2 / e3 >= 0.6 * 2 ** order, (e1, e2, e3)
    amp = np.abs(x0 - mu).max() + np.abs(v0).max() / w
    assert e3 <= amp * (w * 0.1) ** order, (e3, amp)


def test_colloc_logcosh_vs_library_ode_solver():
    """f = sum log cosh((x - mu)/sigma): against scipy's DOP853 at rtol 1e-13."""
    rng = np.random.default_rng(9)
    n = 3
    mu, sigma = 0.1 * rng.normal(size=n), 0.5
    x0, v0 = 0.4 * rng.normal(size=n), rng.normal(size=n)
    h = 0.2

    def rhs(t, y):
        return np.concatenate([y[n:], -_grad(oracle.POT_LOGCOSH, mu, sigma, y[:n])])

    ts = np.linspace(0, h, 11)
    sol = integrate.solve_ivp(rhs, (0, h), np.concatenate([x0, v0]), method="DOP853", rtol=1e-13, atol=1e-15,
                              t_eval=ts)
    errs = []
    for q in (2, 3, 4, 5):
        coef, it = oracle.colloc_poly(x0, v0, h, _logcosh(mu, sigma, q, h))
        errs.append(max(np.abs(_peval(coef, t) - sol.y[:n, k]).max() for k, t in enumerate(ts)))
    assert errs[-1] <= 1e-8 and all(errs[i + 1] < errs[i] for i in range(3)), errs


# ---------------------------------------------------------------- degree-d PEP root
def _brute_first_root(Bs, tmax, dt=2e-4):
    f = lambda t: np.linalg.eigvalsh(sum(B * t ** k for k, B in enumerate(Bs)))[0]
    t = dt
    while t <= tmax and f(t) > 0:
        t += dt
    if t > tmax:
        return np.inf if f(tmax) > 0 else None
    lo, hi = t - dt, t
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mid in (lo, hi):
            break
        if f(mid) > 0:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _rsym(rng, m, s):
    A = rng.normal(size=(m, m)) * s
    return (A + A.T) / 2


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5])
def test_pep_interior_vs_brute_force(d):
    rng = np.random.default_rng(20 + d)
    for m in (1, 3, 5):
        for _ in range(3):
            Z = rng.normal(size=(m, m))
            Bs = [Z @ Z.T + m * np.eye(m)] + [_rsym(rng, m, 3.0) for _ in range(d)]
            tp, y = oracle.pep_root(Bs, 3.0)
            tb = _brute_first_root(Bs, 3.0)
            if tb is None:
                continue
            if np.isinf(tb):
                assert np.isinf(tp)
                continue
            assert abs(tp - tb) <= 1e-9 * tb, (d, m, tp, tb)
            G = sum(B * tp ** k for k, B in enumerate(Bs))
            scale = sum(np.linalg.norm(B) * tp ** k for k, B in enumerate(Bs))
            assert np.linalg.norm(G @ y) <= 1e-12 * scale


def test_pep_beyond_tmax_is_inf():
    rng = np.random.default_rng(31)
    m = 4
    Z = rng.normal(size=(m, m))
    Bs = [Z @ Z.T + np.eye(m), _rsym(rng, m, 2.0), _rsym(rng, m, 2.0)]
    t_all, _ = oracle.pep_root(Bs, np.inf)
    assert np.isfinite(t_all)
    assert np.isinf(oracle.pep_root(Bs, 0.999 * t_all)[0])
    assert oracle.pep_root(Bs, 1.001 * t_all)[0] == t_all


def test_pep_diagonal_vs_numpy_roots():
    """Diagonal coefficients: det = prod_i p_i(t), so t+ = min_i first positive root of p_i."""
    rng = np.random.default_rng(33)
    for d in (2, 3, 4, 5):
        m = 4
        D = [np.abs(rng.normal(size=m)) + 0.5] + [rng.normal(size=m) * 2 for _ in range(d)]
        Bs = [np.diag(c) for c in D]
        best = np.inf
        for i in range(m):
            r = np.roots([D[k][i] for k in range(d, -1, -1)])
            r = r[(np.abs(r.imag) <= 1e-9) & (r.real > 0)].real
            if len(r):
                best = min(best, r.min())
        tp, _ = oracle.pep_root(Bs, np.inf)
        assert abs(tp - best) <= 1e-10 * best, (d, tp, best)


def test_pep_degree1_matches_jacobi_chord():
    """d = 1 is the linear pencil of Alg. 2; the chord oracle solves it by Jacobi instead."""
    inst = specgen.rand_cube(6, 7, 2, cube=False)
    lmi = oracle.Lmi(inst)
    rng = np.random.default_rng(35)
    for _ in range(5):
        x = 0.05 * rng.normal(size=6)
        v = rng.normal(size=6)
        r = oracle.chord(lmi, x, v)
        tp, _ = oracle.pep_root([lmi.eval_block(0, x), lmi.dir_block(0, v)], np.inf)
        assert abs(tp - r["t_plus"]) <= 1e-11 * r["t_plus"]


@pytest.mark.parametrize("d", [2, 3, 4])
def test_pep_boundary_start_vs_brute_force(d):
    """Start on the boundary: shift an interior pencil to its first root t1 (Taylor
    coefficients C_j = sum_k binom(k, j) t1^(k-j) B_k); the next root after t1 from the
    boundary-start branch must be the brute-force one."""
    rng = np.random.default_rng(40 + d)
    done = 0
    for _ in range(12):
        m = 5
        Z = rng.normal(size=(m, m))
        Bs = [Z @ Z.T + np.eye(m)] + [_rsym(rng, m, 2.0) for _ in range(d)]
        t1, y1 = oracle.pep_root(Bs, 10.0)
        if not np.isfinite(t1):
            continue
        Cs = [sum(comb(k, j) * t1 ** (k - j) * Bs[k] for k in range(j, d + 1)) for j in range(d + 1)]
        u = y1 / np.linalg.norm(y1)
        if u @ Cs[1] @ u <= 0:  # crossing outward at t1: walk the reversed curve back inside
            Cs = [C * (-1) ** j for j, C in enumerate(Cs)]
        tb = _brute_first_root(Cs, 6.0)
        if tb is None:
            continue
        t2, y2 = oracle.pep_root(Cs, 6.0, u=u)
        if np.isinf(tb):
            assert np.isinf(t2)
        else:
            assert abs(t2 - tb) <= 1e-8 * tb, (t2, tb)
        done += 1
    assert done >= 6


# ---------------------------------------------------------------- walks
def test_chmc_linear_force_equals_hmc_trace():
    """f = c^T x / T and h >= tau: one collocation segment per chord, exactly the HMC-r
    trajectory; the two oracles' reflections agree up to rounding (different PEP degree)."""
    inst = specgen.config_instance(0)
    lmi = oracle.Lmi(inst)
    n = inst.n
    c = specgen.objective(n, 1)
    T, L = 1.0, 2 * np.sqrt(n)
    for chain in range(6):
        a = oracle.trace(lmi, oracle.HMC, 3, chain, 30, L, 100, 8, T=T, c=c)
        b = oracle.trace(lmi, oracle.CHMC, 3, chain, 30, L, 100, 8, T=T, c=c,
                         colloc=dict(pot=oracle.POT_LINEAR, q=3, h=10 * L))
        k = min(len(a["t"]), len(b["t"]), 5)
        assert k >= 3
        assert np.array_equal(a["binding"][:k], b["binding"][:k])
        assert np.allclose(a["t"][:k], b["t"][:k], rtol=1e-8, atol=0)
        assert np.allclose(a["hit_x"][:k], b["hit_x"][:k], rtol=0, atol=1e-8)
        assert np.allclose(a["v_after"][:k], b["v_after"][:k], rtol=0, atol=1e-7)


def _check_moment(vals, expect, nsig=4.5):
    se = vals.std(ddof=1) / np.sqrt(len(vals))
    assert abs(vals.mean() - expect) <= nsig * se + 1e-12, (vals.mean(), expect, se)


def test_chmc_truncated_gauss_cube_moments():
    """exp(-|x - mu|^2 / 2 sigma^2) on [-1, 1]^n: independent truncated normals, whose first two
    moments are closed forms in phi and Phi."""
    n = 3
    inst = specgen.cube_only(n)
    lmi = oracle.Lmi(inst)
    mu, sigma = np.array([0.3, -0.5, 0.0]), 0.6
    X, st = oracle.walk(lmi, oracle.CHMC, 8, 0, 800, 20, 2.0, 100, colloc=_gauss(mu, sigma, 3, 0.25))
    assert st["failures"] == 0 and st["reflections"] > 0
    phi = lambda z: np.exp(-0.5 * z * z) / np.sqrt(2 * np.pi)
    Phi = lambda z: 0.5 * (1 + special.erf(z / np.sqrt(2)))
    for i in range(n):
        a, b = (-1 - mu[i]) / sigma, (1 - mu[i]) / sigma
        Z = Phi(b) - Phi(a)
        m1 = mu[i] + sigma * (phi(a) - phi(b)) / Z
        var = sigma ** 2 * (1 + (a * phi(a) - b * phi(b)) / Z - ((phi(a) - phi(b)) / Z) ** 2)
        _check_moment(X[:, i], m1)
        _check_moment(X[:, i] ** 2, var + m1 ** 2)


def test_chmc_logcosh_cube_moments():
    """exp(-sum log cosh((x_i - mu_i)/sigma)) on [-1, 1]^n: separable; 1-d moments by quadrature."""
    n = 3
    inst = specgen.cube_only(n)
    lmi = oracle.Lmi(inst)
    mu, sigma = np.array([0.4, -0.2, 0.0]), 0.3
    X, st = oracle.walk(lmi, oracle.CHMC, 9, 0, 800, 20, 2.0, 100, colloc=_logcosh(mu, sigma, 3, 0.2))
    assert st["failures"] == 0 and st["reflections"] > 0
    for i in range(n):
        dens = lambda x: 1.0 / np.cosh((x - mu[i]) / sigma)
        Z = integrate.quad(dens, -1, 1, epsabs=1e-14)[0]
        m1 = integrate.quad(lambda x: x * dens(x), -1, 1, epsabs=1e-14)[0] / Z
        m2 = integrate.quad(lambda x: x * x * dens(x), -1, 1, epsabs=1e-14)[0] / Z
        _check_moment(X[:, i], m1)
        _check_moment(X[:, i] ** 2, m2)


def test_chmc_replay_matches_trace_and_walk():
    """orc_replay's call budget for CHMC: the budget of a whole s-step walk ends where the walk
    ends (bit for bit)."""
    inst = specgen.rand_cube(6, 6, 3)
    lmi = oracle.Lmi(inst)
    cfg = _gauss(np.zeros(6), 0.8, 3, 0.3)
    X, st = oracle.walk(lmi, oracle.CHMC, 2, 4, 5, 3, 2.0, 60, colloc=cfg, nthreads=1)
    x, calls = oracle.replay(lmi, oracle.CHMC, 2, 4, 3, 2.0, 60, st["calls"], colloc=cfg)
    assert calls == st["calls"]
    assert np.array_equal(x, X[0])
