"""Pins for the oracle's walks and QEP (-m "not gpu"): closed-form moments of
uniform / Boltzmann distributions on bodies with known laws (P1-P3), HMC
energy conservation (P11), QEP root vs brute-force scanning (P12), and
sharding determinism (P15)."""
import numpy as np
import pytest

import oracle
import specgen


def _lmi_full(inst, x):
    return inst.A[0] + np.tensordot(x, inst.A[1:], axes=1)


def _brute_first_root(B0, B1, B2, t0=0.0, dt=1e-3, tmax=50.0):
    """Scan lambda_min(B0 + t B1 + t^2 B2) (LAPACK) for the first sign change after t0, then bisect."""
    f = lambda t: np.linalg.eigvalsh(B0 + t * B1 + t * t * B2)[0]
    t = t0 + dt
    while t < tmax and f(t) > 0:
        t += dt
    if t >= tmax:
        return np.inf
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


# ---------------------------------------------------------------- P12 QEP
def test_qep_interior_vs_brute_force():
    rng = np.random.default_rng(11)
    for m in (1, 3, 6, 10):
        for _ in range(4):
            Z = rng.standard_normal((m, m))
            B0 = Z @ Z.T + np.eye(m)
            B1 = rng.standard_normal((m, m)); B1 = B1 + B1.T
            B2 = rng.standard_normal((m, m)); B2 = -(B2 @ B2.T) / 4 + 0.3 * (B2 + B2.T)
            tp, y = oracle.qep_root(B0, B1, B2)
            tb = _brute_first_root(B0, B1, B2)
            if np.isinf(tb):
                assert np.isinf(tp) or tp > 49
                continue
            assert abs(tp - tb) <= 1e-11 * max(1, tb), (m, tp, tb)
            G = B0 + tp * B1 + tp * tp * B2
            yn = y / np.linalg.norm(y)
            scale = max(np.abs(B0).max(), tp * np.abs(B1).max(), tp * tp * np.abs(B2).max())
            assert np.linalg.norm(G @ yn) <= 1e-12 * scale


def test_qep_boundary_start_vs_brute_force():
    rng = np.random.default_rng(12)
    for m in (1, 4, 8):
        for _ in range(4):
            Z = rng.standard_normal((m, m))
            B0 = Z @ Z.T + np.eye(m)
            B1 = rng.standard_normal((m, m)); B1 = B1 + B1.T
            B2 = -np.eye(m) * 0.5
            t1, y = oracle.qep_root(B0, B1, B2)
            assert np.isfinite(t1)
            # move to the hit; the new pencil in s = t - t1 starts on the boundary
            C0 = B0 + t1 * B1 + t1 * t1 * B2
            C1 = -(B1 + 2 * t1 * B2)  # reverse direction -> inward start
            u = y / np.linalg.norm(y)
            if u @ C1 @ u <= 0:
                continue
            t2, _ = oracle.qep_root(C0, C1, B2, u=u)
            tb = _brute_first_root(C0, C1, B2, t0=1e-7, dt=1e-3)
            assert abs(t2 - tb) <= 1e-9 * max(1, tb), (m, t2, tb)


# ---------------------------------------------------------------- P11 HMC energy
def test_hmc_energy_conserved_across_reflections():
    inst = specgen.rand_cube(5, 6, 13)
    L = oracle.Lmi(inst)
    c = specgen.objective(5, 13)
    T = 0.7
    for chain in range(4):
        tr = oracle.trace(L, oracle.HMC, seed=3, chain=chain, steps=1, L=6.0, rho=200, max_refl=50, T=T, c=c)
        g, _ = oracle.step_draws(3, 0, chain, 0, 5)
        E0 = 0.5 * g @ g  # x0 = 0
        for k in range(len(tr["t"])):
            E = c @ tr["hit_x"][k] / T + 0.5 * tr["v_after"][k] @ tr["v_after"][k]
            assert abs(E - E0) <= 1e-12 * max(1.0, abs(E0))


# ---------------------------------------------------------------- billiard trace invariants
def test_billiard_trace_invariants():
    inst = specgen.rand_cube(8, 8, 14)
    L = oracle.Lmi(inst)
    tr = oracle.trace(L, oracle.BILLIARD, seed=0, chain=3, steps=20, L=2 * np.sqrt(8), rho=80, max_refl=20)
    assert len(tr["t"]) == 20
    for k in range(20):
        assert abs(np.linalg.norm(tr["v_after"][k]) - 1) < 1e-14
        x = tr["hit_x"][k]
        if tr["binding"][k] == 0:
            F = _lmi_full(inst, x)
            assert abs(np.linalg.eigvalsh(F)[0]) <= 1e-12 * np.abs(F).max()
        else:
            i = (tr["binding"][k] - 1) // 2
            assert abs(abs(x[i]) - 1) < 1e-14
        # specular law: w . v_after = -(w . v_before) and v_after tangential part matches
        assert tr["w"][k] @ tr["v_after"][k] < 0


# ---------------------------------------------------------------- P15 sharding determinism
def test_walk_sharding_bit_identical():
    inst = specgen.rand_cube(6, 6, 15)
    L = oracle.Lmi(inst)
    a, sa = oracle.walk(L, oracle.BILLIARD, 5, 0, 12, 10, 2 * np.sqrt(6), 60, nthreads=3)
    b1, _ = oracle.walk(L, oracle.BILLIARD, 5, 0, 5, 10, 2 * np.sqrt(6), 60, nthreads=1)
    b2, _ = oracle.walk(L, oracle.BILLIARD, 5, 5, 12, 10, 2 * np.sqrt(6), 60, nthreads=2)
    assert np.array_equal(a, np.vstack([b1, b2]))
    assert sa["steps"] == 120 and sa["calls"] >= 120


# ---------------------------------------------------------------- P1-P3 uniform moments
def _check_moment(vals, expect, nsig=4.5):
    se = vals.std(ddof=1) / np.sqrt(len(vals))
    assert abs(vals.mean() - expect) <= nsig * se + 1e-12, (vals.mean(), expect, se)


@pytest.mark.parametrize("body", ["cube", "cube_dense", "ball", "elliptope3"])
def test_billiard_uniform_moments(body):
    if body == "cube":
        inst, ex2 = specgen.cube_only(3), 1 / 3
    elif body == "cube_dense":
        inst, ex2 = specgen.cube_dense(3), 1 / 3
    elif body == "ball":
        inst, ex2 = specgen.ball(4), 1 / 6  # E[x_i^2] = 1/(n+2)
    else:
        inst, ex2 = specgen.elliptope(3), 1 / 4  # E[x^2] = 1/(k+1)
    L = oracle.Lmi(inst)
    n = inst.n
    X, st = oracle.walk(L, oracle.BILLIARD, 21, 0, 600, 25, 2 * np.sqrt(n), 10 * n)
    # coordinates are exchangeable: average per chain to get iid samples
    _check_moment((X ** 2).mean(axis=1), ex2)
    _check_moment(X.mean(axis=1), 0.0)
    assert st["failures"] == 0


def test_hmc_boltzmann_cube_moments():
    """pi(x) ~ exp(-c.x/T) on [-1,1]^n: independent truncated exponentials (P1, V7)."""
    n = 3
    inst = specgen.cube_only(n)
    L = oracle.Lmi(inst)
    c = np.array([1.0, -0.6, 2.5])
    T = 1.0
    X, st = oracle.walk(L, oracle.HMC, 4, 0, 800, 20, 2.0, 100, T=T, c=c)
    grid = np.linspace(-1, 1, 200001)
    for i in range(n):
        dens = np.exp(-c[i] * grid / T)
        Z = np.trapezoid(dens, grid)
        e1 = np.trapezoid(grid * dens, grid) / Z
        e2 = np.trapezoid(grid ** 2 * dens, grid) / Z
        _check_moment(X[:, i], e1)
        _check_moment(X[:, i] ** 2, e2)
    assert st["failures"] == 0


# ---------------------------------------------------------------- orc_replay / orc_trace budget semantics
def test_replay_one_call_cube_closed_form():
    """Replay budget = 1 call on the cube [-1,1]^n (P1): from x0 = 0 the billiard's first
    segment (Alg. 5) ends at min(l, t+) v, with l = -L ln eta and
    t+ = min_i (sgn v_i - 0)/v_i = 1/max|v_i| (closed form), v = g/|g| from the step draws."""
    n = 6
    lmi = oracle.Lmi(specgen.cube_only(n))
    for chain in range(20):
        for L in (0.3, 3.0):
            g, eta = oracle.step_draws(5, 0, chain, 0, n)
            v = g / np.linalg.norm(g)
            ell = -L * np.log(eta)
            tp = 1.0 / np.max(np.abs(v))
            x, calls = oracle.replay(lmi, oracle.BILLIARD, 5, chain, 10, L, 100, 1)
            assert calls == 1
            expect = min(ell, tp) * v
            assert np.allclose(x, expect, rtol=0, atol=1e-14), (chain, L, x, expect)


def test_replay_matches_walk_and_trace():
    """Replay with the budget of s whole steps ends exactly where an s-step walk ends; a budget
    inside a step ends at the last recorded hit point of the trace (bit for bit: same chains)."""
    inst = specgen.rand_cube(8, 8, 3)
    lmi = oracle.Lmi(inst)
    L, rho = 2 * np.sqrt(8), 80
    for chain in (0, 5, 11):
        for s in (1, 3):
            X, st = oracle.walk(lmi, oracle.BILLIARD, 7, chain, chain + 1, s, L, rho, nthreads=1)
            x, calls = oracle.replay(lmi, oracle.BILLIARD, 7, chain, 50, L, rho, st["calls"])
            assert calls == st["calls"]
            assert np.array_equal(x, X[0]), (chain, s)
        tr = oracle.trace(lmi, oracle.BILLIARD, 7, chain, 50, L, rho, 6, stop=True)
        full = oracle.trace(lmi, oracle.BILLIARD, 7, chain, 50, L, rho, 6)
        for k in ("hit_x", "t", "w", "v_after", "binding"):
            assert np.array_equal(tr[k], full[k])
        # the first step of these chains reflects at least 6 times before it ends
        g, eta = oracle.step_draws(7, 0, chain, 0, 8)
        assert len(tr["t"]) == 6 and -L * np.log(eta) > tr["t"].sum()
        x, calls = oracle.replay(lmi, oracle.BILLIARD, 7, chain, 50, L, rho, 6)
        assert calls == 6
        assert np.array_equal(x, tr["hit_x"][5])


# ---------------------------------------------------------------- Hit-and-Run / coordinate Hit-and-Run
@pytest.mark.parametrize("kind", [oracle.HNR, oracle.CHNR])
def test_hnr_one_step_cube_closed_form(kind):
    """One W-HnR / W-CHnR step (Alg. 4) on the cube [-1,1]^n from x0:
    the chord through x0 along v has t+ = min_i (sgn v_i - x0_i)/v_i and
    t- = max_i (-sgn v_i - x0_i)/v_i (closed form), the next point x0 + (t- + eta (t+ - t-)) v."""
    n = 5
    lmi = oracle.Lmi(specgen.cube_only(n))
    x0 = np.array([0.3, -0.2, 0.0, 0.7, -0.9])
    for chain in range(25):
        if kind == oracle.HNR:
            g, eta = oracle.step_draws(2, 0, chain, 0, n)
            v = g / np.linalg.norm(g)
        else:
            eta, u2 = oracle.step_uniforms(2, 0, chain, 0, n)
            v = np.zeros(n)
            v[min(int(u2 * n), n - 1)] = 1.0
        nz = v != 0
        tp = np.min((np.sign(v[nz]) - x0[nz]) / v[nz])
        tm = np.max((-np.sign(v[nz]) - x0[nz]) / v[nz])
        X, st = oracle.walk(lmi, kind, 2, chain, chain + 1, 1, 1.0, 10, x0=x0, nthreads=1)
        assert st["calls"] == 1 and st["reflections"] == 0
        assert np.allclose(X[0], x0 + (tm + eta * (tp - tm)) * v, rtol=0, atol=1e-14)


@pytest.mark.parametrize("kind", [oracle.HNR, oracle.CHNR])
@pytest.mark.parametrize("body", ["cube_dense", "ball", "elliptope3"])
def test_hnr_uniform_moments(kind, body):
    """W-HnR / W-CHnR target the uniform law: E[x_i] = 0 and E[x_i^2] = 1/3 (cube), 1/(n+2)
    (ball), 1/(k+1) (elliptope) over chain end points."""
    if body == "cube_dense":
        inst, ex2 = specgen.cube_dense(3), 1 / 3
    elif body == "ball":
        inst, ex2 = specgen.ball(4), 1 / 6
    else:
        inst, ex2 = specgen.elliptope(3), 1 / 4
    lmi = oracle.Lmi(inst)
    X, st = oracle.walk(lmi, kind, 21, 0, 3000, 40, 1.0, 10)
    assert st["calls"] == 3000 * 40 and st["steps"] == 3000 * 40
    x2 = (X ** 2).mean(1)
    se = x2.std(ddof=1) / np.sqrt(len(x2))
    assert abs(x2.mean() - ex2) <= 4 * se, (x2.mean(), ex2, se)
    mx = X.mean(1)
    assert abs(mx.mean()) <= 4 * mx.std(ddof=1) / np.sqrt(len(mx))


@pytest.mark.parametrize("kind", [oracle.HNR, oracle.CHNR])
def test_hnr_boltzmann_cube_moments(kind):
    """W-HnR / W-CHnR with pi_l the restriction of exp(-c.x/T) (sec:optimization P:1408-1424)
    on [-1,1]^n: independent truncated exponentials (P1, V7), moments by quadrature."""
    n = 3
    lmi = oracle.Lmi(specgen.cube_only(n))
    c = np.array([1.0, -0.6, 2.5])
    T = 0.7
    X, st = oracle.walk(lmi, kind, 8, 0, 3000, 30, 1.0, 10, T=T, c=c)
    assert st["calls"] == 3000 * 30
    grid = np.linspace(-1, 1, 200001)
    for i in range(n):
        dens = np.exp(-c[i] * grid / T)
        Z = np.trapezoid(dens, grid)
        _check_moment(X[:, i], np.trapezoid(grid * dens, grid) / Z)
        _check_moment(X[:, i] ** 2, np.trapezoid(grid ** 2 * dens, grid) / Z)
