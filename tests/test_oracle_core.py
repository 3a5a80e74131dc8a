"""Pins for the CPU oracle's geometric operations (-m "not gpu").

Each test pins an oracle function to something other than itself: a value
the paper prints, a closed form, a library routine (LAPACK via numpy), brute
force, or an invariant (DESIGN.md "Oracle pins" P1-P16)."""
import os

import numpy as np
import pytest

import oracle
import specgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _lam_min(F):
    return np.linalg.eigvalsh(F)[0]


def _lmi_full(inst, x):
    return inst.A[0] + np.tensordot(x, inst.A[1:], axes=1)


def _bisect_tplus(inst, x, v, t_lo=0.0, t_hi=None, cube=True, it=200):
    """P5: t+ from the concavity of t -> lambda_min(F(x+tv)) by bisection on
    LAPACK eigenvalues of the literal matrix (no pencil, no Cholesky)."""
    def feasible(t):
        p = x + t * v
        ok = _lam_min(_lmi_full(inst, p)) >= 0.0
        if cube and inst.lo is not None:
            ok = ok and np.all(p <= inst.hi) and np.all(p >= inst.lo)
        return ok
    if t_hi is None:
        t_hi = 1.0
        while feasible(t_hi):
            t_hi *= 2.0
    lo, hi = t_lo, t_hi
    for _ in range(it):
        mid = 0.5 * (lo + hi)
        if mid == lo or mid == hi:
            break
        if feasible(mid):
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _read_golden(name):
    d = {}
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            k, *vals = line.split()
            d[k] = np.array([float(v) for v in vals])
    return d


# ---------------------------------------------------------------- P14 RNG
def test_philox_known_answers():
    with open(os.path.join(GOLD, "philox_kat.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        vals = [int(x, 16) for x in r]
        out = oracle.philox(vals[0:4], vals[4:6])
        assert out.tolist() == vals[6:10]


def test_u01_open_interval_and_normals():
    assert oracle.u01(0, 0) > 0.0 and oracle.u01(0, 0) == 0.5 * 2.0 ** -52
    assert oracle.u01(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    assert oracle.u01(0xFFFFFFFF, 0xFFFFFFFF) < 1.0
    # Box-Muller normals: sample moments over many draws (N(0,1))
    zs = np.concatenate([oracle.step_draws(7, 0, c, 0, 64)[0] for c in range(400)])
    assert abs(zs.mean()) < 4 / np.sqrt(len(zs))
    assert abs(zs.var() - 1.0) < 6 * np.sqrt(2.0 / len(zs))
    etas = np.array([oracle.step_draws(7, 0, c, 3, 4)[1] for c in range(2000)])
    assert np.all((etas > 0) & (etas < 1)) and abs(etas.mean() - 0.5) < 4 * np.sqrt(1 / 12 / 2000)


# ---------------------------------------------------------------- dense LA
def test_cholesky_and_jacobi_vs_lapack():
    rng = np.random.default_rng(0)
    for m in (1, 2, 5, 17, 40):
        B = rng.standard_normal((m, m))
        A = B @ B.T + m * np.eye(m)
        L = oracle.cholesky(A)
        assert np.allclose(L @ L.T, A, rtol=0, atol=1e-12 * np.abs(A).max())
        assert np.allclose(np.triu(L, 1), 0)
        S = rng.standard_normal((m, m))
        S = S + S.T
        ev, V = oracle.jacobi(S)
        ref = np.linalg.eigvalsh(S)
        assert np.allclose(np.sort(ev), ref, rtol=0, atol=1e-13 * np.abs(ref).max())
        assert np.allclose(V.T @ V, np.eye(m), atol=1e-13)
        assert np.allclose(S @ V, V * ev, atol=1e-12 * np.abs(ref).max())
    assert oracle.cholesky(np.array([[1.0, 2.0], [2.0, 1.0]])) is None


# ---------------------------------------------------------------- P7 worked example
def test_paper_worked_example():
    g = _read_golden("paper_example.txt")
    inst = specgen.paper_example()
    L = oracle.Lmi(inst)
    r = oracle.chord(L, g["p0"], g["u"])
    tol = 0.15  # reading R2: the paper's matrices are rounded to one decimal
    assert abs(r["t_minus"] - g["t_minus"][0]) < tol
    assert abs(r["t_plus"] - g["t_plus"][0]) < tol
    p1 = g["p0"] + r["t_plus"] * g["u"]
    assert np.allclose(p1, g["p1"], atol=tol)
    w = oracle.normal(L, r["block"], r["y"])
    wp = g["w"] / np.linalg.norm(g["w"])
    assert min(np.linalg.norm(w - wp), np.linalg.norm(w + wp)) < tol
    s = oracle.reflect(g["u"], w)
    assert np.allclose(s, g["u_reflected"], atol=tol + 0.1)
    # the hit is on the boundary (P4) and the endpoints agree with bisection (P5)
    F = _lmi_full(inst, p1)
    assert abs(_lam_min(F)) <= 1e-13 * np.abs(F).max()
    assert abs(r["t_plus"] - _bisect_tplus(inst, g["p0"], g["u"])) < 1e-13
    assert abs(r["t_minus"] + _bisect_tplus(inst, g["p0"], -g["u"])) < 1e-13


# ---------------------------------------------------------------- P1 cube
@pytest.mark.parametrize("dense", [False, True])
def test_cube_closed_form_chords(dense):
    n = 6
    inst = specgen.cube_dense(n) if dense else specgen.cube_only(n)
    L = oracle.Lmi(inst)
    rng = np.random.default_rng(1)
    for _ in range(30):
        x = rng.uniform(-0.9, 0.9, n)
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        r = oracle.chord(L, x, v)
        tp = np.min(np.where(v > 0, (1 - x) / v, (-1 - x) / v))
        tm = np.max(np.where(v > 0, (-1 - x) / v, (1 - x) / v))
        assert abs(r["t_plus"] - tp) <= 1e-14 * max(1, tp)
        assert abs(r["t_minus"] - tm) <= 1e-14 * max(1, abs(tm))
        i = int(np.argmin(np.where(v > 0, (1 - x) / v, (-1 - x) / v)))
        w = oracle.normal(L, r["block"], r["y"])
        e = np.zeros(n)
        e[i] = np.sign(v[i])  # outward normal of the face that is hit
        assert np.allclose(w, e, atol=1e-12)
        if not dense:
            assert r["binding"] == (1 + 2 * i if v[i] > 0 else 2 + 2 * i)


# ---------------------------------------------------------------- P3 ball
def test_ball_closed_form_chords_and_normals():
    n = 7
    inst = specgen.ball(n)
    L = oracle.Lmi(inst)
    rng = np.random.default_rng(2)
    for _ in range(30):
        x = rng.standard_normal(n)
        x *= rng.uniform(0, 0.95) / np.linalg.norm(x)
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        r = oracle.chord(L, x, v)
        xv = x @ v
        tp = -xv + np.sqrt(xv ** 2 + 1 - x @ x)
        tm = -xv - np.sqrt(xv ** 2 + 1 - x @ x)
        assert abs(r["t_plus"] - tp) <= 1e-13
        assert abs(r["t_minus"] - tm) <= 1e-13
        w = oracle.normal(L, r["block"], r["y"])
        hit = x + tp * v
        assert np.allclose(w, hit / np.linalg.norm(hit), atol=1e-12)


# ---------------------------------------------------------------- P4 / P5 random instances
@pytest.mark.parametrize("n,m", [(10, 10), (40, 40), (12, 30)])
def test_random_instance_chord_vs_bisection(n, m):
    inst = specgen.rand_cube(n, m, 5)
    L = oracle.Lmi(inst)
    rng = np.random.default_rng(3)
    for _ in range(6):
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        x = 0.3 * rng.uniform() * v
        r = oracle.chord(L, x, v)
        tb = _bisect_tplus(inst, x, v)
        assert abs(r["t_plus"] - tb) <= 1e-12 * max(1.0, tb)
        tmb = -_bisect_tplus(inst, x, -v)
        assert abs(r["t_minus"] - tmb) <= 1e-12 * max(1.0, abs(tmb))
        if r["block"] == 0:
            F = _lmi_full(inst, x + r["t_plus"] * v)
            assert abs(_lam_min(F)) <= 1e-13 * np.abs(F).max()
            # y is the kernel vector of F(x + t+ v)
            y = r["y"] / np.linalg.norm(r["y"])
            assert np.linalg.norm(F @ y) <= 1e-12 * np.abs(F).max()


# ---------------------------------------------------------------- P6 boundary start (deflation)
@pytest.mark.parametrize("n,m", [(10, 10), (20, 16)])
def test_boundary_start_deflation_vs_bisection(n, m):
    inst = specgen.rand_cube(n, m, 6, cube=False)
    L = oracle.Lmi(inst, cube=False)
    rng = np.random.default_rng(4)
    for _ in range(6):
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        x = np.zeros(n)
        r = oracle.chord(L, x, v)
        hit = x + r["t_plus"] * v
        w = oracle.normal(L, r["block"], r["y"])
        s = oracle.reflect(v, w)
        u = r["y"] / np.linalg.norm(r["y"])
        F = _lmi_full(inst, hit)
        rb = oracle.chord(L, hit, s, F0=F, bound=0, u=u)
        assert rb["t_minus"] == 0.0
        # bisection from just inside along s (lambda_min(F(hit + t s)) concave, = 0 at t=0)
        tb = _bisect_tplus(inst, hit, s, t_lo=1e-9 * rb["t_plus"], cube=False)
        assert abs(rb["t_plus"] - tb) <= 1e-11 * max(1.0, tb)
        F2 = _lmi_full(inst, hit + rb["t_plus"] * s)
        assert abs(_lam_min(F2)) <= 1e-12 * np.abs(F2).max()


# ---------------------------------------------------------------- P9 finite differences
@pytest.mark.parametrize("which", ["rand", "ball", "example"])
def test_normal_vs_finite_differences(which):
    if which == "rand":
        inst = specgen.rand_cube(5, 6, 8, cube=False)
    elif which == "ball":
        inst = specgen.ball(4)
    else:
        inst = specgen.paper_example()
    L = oracle.Lmi(inst, cube=False)
    rng = np.random.default_rng(5)
    n = inst.n
    x0 = np.array([-1.0, 1.0]) if which == "example" else np.zeros(n)
    for _ in range(5):
        v = rng.standard_normal(n)
        v /= np.linalg.norm(v)
        r = oracle.chord(L, x0, v)
        hit = x0 + r["t_plus"] * v
        w = oracle.normal(L, r["block"], r["y"])
        h = 1e-5
        g = np.array([(np.linalg.det(_lmi_full(inst, hit + h * e)) - np.linalg.det(_lmi_full(inst, hit - h * e)))
                      / (2 * h) for e in np.eye(n)])
        g = -g / np.linalg.norm(g)  # outward = -grad det (det > 0 inside)
        ang = np.arccos(np.clip(abs(w @ g), -1, 1))
        assert ang <= 1e-4
        assert w @ g > 0  # orientation: outward


# ---------------------------------------------------------------- P10 reflection invariants
def test_reflection_invariants():
    rng = np.random.default_rng(6)
    for n in (2, 5, 50):
        u = rng.standard_normal(n)
        w = rng.standard_normal(n)
        w /= np.linalg.norm(w)
        s = oracle.reflect(u, w)
        assert abs(np.linalg.norm(s) - np.linalg.norm(u)) <= 1e-14 * np.linalg.norm(u)
        assert abs(s @ w + u @ w) <= 1e-14 * np.linalg.norm(u)
        assert np.allclose(oracle.reflect(u, -w), s, atol=1e-15 * np.linalg.norm(u))
        # tangential part unchanged
        assert np.allclose(s - (s @ w) * w, u - (u @ w) * w, atol=1e-14 * np.linalg.norm(u))


# ---------------------------------------------------------------- P13 literal vs split blocks
def test_literal_vs_split_blocks():
    inst = specgen.rand_cube(6, 8, 9, scale=0.5)  # dense, cube and ball all bind
    Ls = oracle.Lmi(inst, ball_c=np.zeros(6), ball_r=1.4)
    Ll = oracle.Lmi(inst, ball_c=np.zeros(6), ball_r=1.4, literal=True)
    assert Ll.nblocks == 1 and Ll.block_size(0) == 8 + 12 + 7
    rng = np.random.default_rng(7)
    kinds = set()
    for _ in range(40):
        v = rng.standard_normal(6)
        v /= np.linalg.norm(v)
        x = rng.uniform(-0.3, 0.3, 6)
        rs, rl = oracle.chord(Ls, x, v), oracle.chord(Ll, x, v)
        kinds.add(rs["binding"] if rs["binding"] <= 0 else 1)
        assert abs(rs["t_plus"] - rl["t_plus"]) <= 1e-13 * max(1, rs["t_plus"])
        assert abs(rs["t_minus"] - rl["t_minus"]) <= 1e-13 * max(1, abs(rs["t_minus"]))
        ws = oracle.normal(Ls, rs["block"], rs["y"])
        wl = oracle.normal(Ll, rl["block"], rl["y"])
        assert np.allclose(ws, wl, atol=1e-9)
    assert kinds >= {0, 1, -1}  # dense, cube and ball all bound at least once


# ---------------------------------------------------------------- membership (Alg. 1)
def test_membership():
    inst = specgen.ball(3)
    L = oracle.Lmi(inst)
    assert oracle.membership(L, [0.0, 0.0, 0.0])
    assert oracle.membership(L, [0.5, 0.5, 0.5])
    assert not oracle.membership(L, [0.6, 0.6, 0.6])
    assert not oracle.membership(L, [1.0, 0.0, 0.0])  # boundary: measure zero, counted outside
    cube = oracle.Lmi(specgen.cube_only(3))
    assert oracle.membership(cube, [0.99, -0.99, 0.0]) and not oracle.membership(cube, [1.01, 0, 0])
