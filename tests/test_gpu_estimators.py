"""GPU estimators through the C-ABI: ball-phase MMC volume against closed forms
(cube, ball, elliptope, a multiphase box, the paper's 2-D example) and against
the CPU oracle's estimator on the same seeds (2 sigma); E[f] against closed
forms and the oracle."""
import math

import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu


def _box(sides):
    n = len(sides)
    A = np.zeros((n + 1, 1, 1))
    A[0, 0, 0] = 1.0
    half = np.array(sides) / 2
    return specgen.Instance("box", A, -half, half)


def _gpu_vol(inst, seeds, N=2048, eps=0.1):
    import paper_2010_03817_b200 as sw
    S = sw.Spectrahedron.from_instance(inst)
    return [S.volume(eps, s, N, walk_len=8, burn=30) for s in seeds]


@pytest.mark.parametrize("body", ["cube6", "cube_dense5", "ball5", "elliptope3", "elliptope4", "box", "example"])
def test_gpu_volume_closed_forms(body):
    if body == "cube6":
        inst, truth = specgen.cube_only(6), 64.0
    elif body == "cube_dense5":
        inst, truth = specgen.cube_dense(5), 32.0
    elif body == "ball5":
        inst, truth = specgen.ball(5), oracle.ball_volume(5)
    elif body == "elliptope3":
        inst, truth = specgen.elliptope(3), math.pi ** 2 / 2
    elif body == "elliptope4":
        inst, truth = specgen.elliptope(4), 32 * math.pi ** 2 / 27
    elif body == "box":
        inst, truth = _box([6.0, 2.0, 0.6, 0.4]), 2.88
    else:
        inst, truth = specgen.paper_example(), 10.4531336720527
    rs = _gpu_vol(inst, range(4))
    est = np.mean([r["volume"] for r in rs])
    se = np.mean([r["std_rel"] for r in rs]) * truth / 2.0
    assert abs(est - truth) <= 3.0 * se, (est, truth, se, [r["phases"] for r in rs])


def test_gpu_volume_vs_oracle_same_seeds():
    """Statistical parity with the oracle estimator: |mean_gpu - mean_oracle| <= 2 sigma."""
    inst = _box([4.0, 1.0, 0.5])
    seeds = range(6)
    g = [r["volume"] for r in _gpu_vol(inst, seeds, N=512)]
    o = [oracle.volume(inst, 0.1, s, 512, W=8, burn=30)["volume"] for s in seeds]
    sd = np.std(o, ddof=1)
    assert abs(np.mean(g) - np.mean(o)) <= 2.0 * max(sd, 1e-12) * math.sqrt(2.0 / len(seeds)) * 1.5, (g, o)


def test_gpu_expectation():
    import paper_2010_03817_b200 as sw
    inst = specgen.cube_only(3)
    S = sw.Spectrahedron.from_instance(inst)
    cc = np.array([1.0, 0.5, -1.5])
    S.set_objective(cc)
    r = S.expectation(sw.F_SQNORM, 0.0, 1, 4000, 20, 2 * math.sqrt(3), 30)
    assert abs(r["est"] - 1.0) <= 4 * r["stderr"]
    r = S.expectation(sw.F_LINEAR_C, 1.0, 3, 4000, 20, 2.0, 100)  # HMC-r, Boltzmann T = 1
    truth = float(np.sum(cc * (1 / cc - 1 / np.tanh(cc))))
    assert abs(r["est"] - truth) <= 4 * r["stderr"], (r, truth)
    r = S.expectation(sw.F_HALFSPACE_UNION, 0.0, 2, 4000, 20, 2 * math.sqrt(3), 30, b1=-0.5, b2=0.5)
    # c.x with c = (1, .5, -1.5) uniform on the cube: P(|c.x| >= .5) by quadrature of the oracle's law
    o = oracle.expectation(inst, "halfspace_union", 2, 4000, 20, 2 * math.sqrt(3), 30, c=cc, b1=-0.5, b2=0.5)
    assert abs(r["est"] - o["est"]) <= 4 * math.hypot(r["stderr"], o["stderr"]), (r, o)


def _elliptope_volume(k):
    """vol(E_k) = prod_{j=1}^{k-1} (2^j B((j+1)/2, (j+1)/2))^j (checked by V4)."""
    B = lambda a, b: math.exp(math.lgamma(a) + math.lgamma(b) - math.lgamma(a + b))
    return math.exp(sum(j * math.log(2 ** j * B((j + 1) / 2, (j + 1) / 2)) for j in range(1, k)))


@pytest.mark.parametrize("k,seeds", [(5, (0, 1)), (8, (0, 1)), (12, (0,))])
def test_volume_elliptope_large_n_closed_form(k, seeds):
    """the ball-phase MMC volume (eq:mmc_vol) of the elliptope E_k -- n = k(k-1)/2
    up to 66 coordinates, 11 phases at k = 12 -- within 3 of the estimator's own sigma of the
    closed form (4096 chains per phase, eps = 0.1).  (k = 20, n = 190, needs > 15 min per seed.)"""
    import paper_2010_03817_b200 as sw
    S = sw.Spectrahedron.from_instance(specgen.elliptope(k))
    exact = _elliptope_volume(k)
    for s in seeds:
        r = S.volume(0.1, s, 4096)
        assert abs(r["volume"] / exact - 1.0) <= 3.0 * r["std_rel"], (k, s, r["volume"], exact, r["std_rel"])


def test_volume_ball_m161_global_scratch_membership():
    """Membership (Alg. 1) for m > 160 runs its Cholesky in the global-scratch slices (A(x) no longer
    fits shared memory): the unit ball as the arrow LMI with n = 160, m = 161.  Every exact sample of
    a phase ball B(r), r < 1, is a member (q = 1 exactly), and the estimator runs through.  (Its value
    is not compared with omega_160 here: from the origin, 6 + 4 billiard steps of 512 chains do not
    mix a 160-ball -- the pilot's radius quantile sits far inside -- and mixing budgets that do take
    minutes.)"""
    import paper_2010_03817_b200 as sw
    n = 160
    S = sw.Spectrahedron.from_instance(specgen.ball(n))
    r = S.volume(0.3, 0, 512, walk_len=4, burn=6)
    assert all(0.0 < x < 1.0 for x in r["radii"]), r["radii"]
    assert r["q"] == 1.0, r["q"]
    assert math.isfinite(r["log_volume"]) and r["phases"] >= 1
