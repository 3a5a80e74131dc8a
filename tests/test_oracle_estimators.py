"""Pins for the oracle's estimators (-m "not gpu"): the ball-phase MMC volume
against closed-form volumes (cube, ball, elliptope, an elongated box that needs
several phases) and against an independent polar quadrature of the paper's 2-D
example (P8; the paper prints 10.23 for its unrounded matrices), and
E[f] against closed forms."""
import math

import numpy as np
import pytest

import oracle
import specgen


def _box(sides):
    n = len(sides)
    A = np.zeros((n + 1, 1, 1))
    A[0, 0, 0] = 1.0
    half = np.array(sides) / 2
    return specgen.Instance("box", A, -half, half)


def _check(inst, truth, seeds=(0, 1, 2), N=400, nsig=3.0):
    ests, sigs, phases = [], [], []
    for s in seeds:
        r = oracle.volume(inst, 0.1, s, N, W=8, burn=30)
        ests.append(r["volume"])
        sigs.append(r["std_rel"])
        phases.append(r["phases"])
    m = np.mean(ests)
    se = np.mean(sigs) * truth / math.sqrt(len(seeds))
    assert abs(m - truth) <= nsig * se + 1e-12, (m, truth, se, ests)
    return phases


def test_volume_cube_ball_elliptope():
    _check(specgen.cube_only(5), 32.0)
    _check(specgen.ball(4), oracle.ball_volume(4))
    _check(specgen.elliptope(3), math.pi ** 2 / 2)  # BASELINE.json pin


def test_volume_elongated_box_multiphase():
    sides = [6.0, 2.0, 0.6, 0.4]
    phases = _check(_box(sides), float(np.prod(sides)))
    assert max(phases) >= 2  # the schedule needs several ball phases here


def _polar_area_example():
    """Independent area of the App.-B spectrahedron (-Q~, R1): 0.5 * int r(phi)^2 dphi
    around the interior point p0 = (-1, 1), r by bisection on LAPACK lambda_min."""
    inst = specgen.paper_example()
    p0 = np.array([-1.0, 1.0])
    A = inst.A

    def inside(p):
        return np.linalg.eigvalsh(A[0] + p[0] * A[1] + p[1] * A[2])[0] >= 0

    K = 720
    phis = (np.arange(K) + 0.5) * 2 * math.pi / K
    rs = []
    for ph in phis:
        d = np.array([math.cos(ph), math.sin(ph)])
        lo, hi = 0.0, 1.0
        while inside(p0 + hi * d):
            hi *= 2
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if inside(p0 + mid * d):
                lo = mid
            else:
                hi = mid
        rs.append(lo)
    rs = np.array(rs)
    return 0.5 * np.sum(rs ** 2) * 2 * math.pi / K  # midpoint rule, smooth periodic integrand


def test_volume_paper_example_area():
    area = _polar_area_example()
    assert abs(area - 10.4531336720527) < 1e-4  # SURVEY V2 (independent quadrature)
    # the walk starts at c0 = 0, which is interior for the App.-B body
    _check(specgen.paper_example(), area)


def test_expectation_closed_forms():
    # uniform on the cube: E|x|^2 = n/3; E[c.x] = 0
    inst = specgen.cube_only(3)
    c = np.array([0.6, -0.8, 0.0])
    r = oracle.expectation(inst, "sqnorm", 1, 800, 20, 2 * math.sqrt(3), 30)
    assert abs(r["est"] - 1.0) <= 4 * r["stderr"]
    r = oracle.expectation(inst, "linear_c", 1, 800, 20, 2 * math.sqrt(3), 30, c=c)
    assert abs(r["est"]) <= 4 * r["stderr"]
    # half-space union on the square [-1,1]^2 with c = e1: P(x1 <= -0.5 or x1 >= 0.5) = 0.5
    inst2 = specgen.cube_only(2)
    r = oracle.expectation(inst2, "halfspace_union", 2, 1000, 20, 2 * math.sqrt(2), 20, c=np.array([1.0, 0.0]),
                           b1=-0.5, b2=0.5)
    assert abs(r["est"] - 0.5) <= 4 * r["stderr"]
    # Boltzmann on the cube (HMC): E[c.x] = sum_i c_i (1/a_i - coth a_i), a_i = c_i/T
    cc = np.array([1.0, 0.5, -1.5])
    r = oracle.expectation(inst, "linear_c", 3, 800, 20, 2.0, 100, T=1.0, c=cc)
    truth = float(np.sum(cc * (1 / cc - 1 / np.tanh(cc))))
    assert abs(r["est"] - truth) <= 4 * r["stderr"], (r, truth)


@pytest.mark.parametrize("kind", [oracle.HMC, oracle.HNR])
@pytest.mark.parametrize("body", ["cube", "ball"])
def test_sdp_anneal_lp_closed_forms(kind, body):
    """SDP by simulated annealing (eq:sdp P:1406, sec:optimization P:1408-1434) on LPs with
    closed-form optima (SURVEY 8(f)#2 pins): min c^T x over [-1,1]^n is -|c|_1 (at -sign c),
    over the unit ball -|c|_2 (at -c/|c|).  The paper's stop rule: relative error <= 0.05."""
    n = 5
    c = np.array([0.9, -0.4, 0.2, 1.3, -0.7])
    inst, fstar = (specgen.cube_dense(n), -np.abs(c).sum()) if body == "cube" else (specgen.ball(n), -np.linalg.norm(c))
    r = oracle.sdp_anneal(inst, c, kind, 16, 80, walk_len=1 if kind == oracle.HMC else 4 * n, seed=3)
    assert r["best"] >= fstar - 1e-9  # never below the optimum (every point is in S)
    assert r["best"] - fstar <= 0.05 * abs(fstar), (r["best"], fstar)
    assert abs(r["best_x"] @ c - r["best"]) <= 1e-12
    assert all(a >= b for a, b in zip(r["history"], r["history"][1:]))  # monotone best
