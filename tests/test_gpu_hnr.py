"""GPU parity for Hit-and-Run (Alg. 4) and coordinate-directions
Hit-and-Run (W-CHnR) through walk_sample (kinds SPEC_WALK_HNR /
SPEC_WALK_CHNR): end points of seeded chains vs the oracle pointwise (one chord per
step and no reflection, so there is no chaotic amplification to bound), one
boundary-oracle call per step, and the uniform law on bodies with closed-form
moments.  One instance per K2 launch variant."""
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu
POOL = ThreadPoolExecutor(os.cpu_count() or 4)

CASES = [
    ("cfg0_10_10", lambda: specgen.config_instance(0), 64, 30),
    ("m40", lambda: specgen.rand_cube(40, 40, 2), 64, 20),
    ("m60", lambda: specgen.rand_cube(16, 60, 13), 64, 20),
    ("m100", lambda: specgen.config_instance(3), 64, 12),
    ("m200", lambda: specgen.config_instance(4), 32, 6),
    ("mixed_12_30", lambda: specgen.rand_cube(12, 30, 5, scale=1 / math.sqrt(12)), 64, 30),
]


@pytest.mark.parametrize("kind_name", ["HNR", "CHNR"])
@pytest.mark.parametrize("name,make,chains,steps", CASES, ids=[c[0] for c in CASES])
def test_hnr_end_points_vs_oracle(kind_name, name, make, chains, steps):
    import paper_2010_03817_b200 as sw
    kind = getattr(sw, kind_name)
    okind = getattr(oracle, kind_name)
    inst = make()
    lmi = oracle.Lmi(inst)
    S = sw.Spectrahedron.from_instance(inst)
    out = S.walk_sample(chains, steps, 1.0, 10, seed=17, kind=kind)
    st = out["stats"]
    assert st["calls"] == chains * steps and st["steps"] == chains * steps
    assert st["reflections"] == 0 and st["rejects"] == 0 and st["failures"] == 0
    per = [POOL.submit(oracle.walk, lmi, okind, 17, c, c + 1, steps, 1.0, 10, None, 1.0, None, 0, 1)
           for c in range(chains)]
    Xo = np.vstack([f.result()[0] for f in per])
    X = out["final_x"]
    err = np.linalg.norm(X - Xo, axis=1) / np.maximum(np.linalg.norm(Xo, axis=1), 0.1)
    print(f"[parity] hnr {kind_name} {name}: worst rel {err.max():.3g} median {np.median(err):.3g}")
    assert err.max() <= 1e-8, (err.max(), int(err.argmax()))
    # sums agree with the end points
    assert np.allclose(out["sum_x"], X.sum(0), rtol=0, atol=1e-9 * chains)


@pytest.mark.parametrize("kind_name", ["HNR", "CHNR"])
@pytest.mark.parametrize("body", ["cube_dense", "ball", "elliptope4"])
def test_hnr_uniform_moments(kind_name, body):
    """E[x_i^2] = 1/3 (cube), 1/(n+2) (ball), 1/(k+1) (elliptope), E[x] = 0."""
    import paper_2010_03817_b200 as sw
    if body == "cube_dense":
        inst, ex2 = specgen.cube_dense(4), 1 / 3
    elif body == "ball":
        inst, ex2 = specgen.ball(5), 1 / 7
    else:
        inst, ex2 = specgen.elliptope(4), 1 / 5
    S = sw.Spectrahedron.from_instance(inst)
    out = S.walk_sample(8192, 60, 1.0, 10, seed=3, kind=getattr(sw, kind_name))
    X = out["final_x"]
    x2 = (X ** 2).mean(1)
    se = x2.std(ddof=1) / math.sqrt(len(x2))
    assert abs(x2.mean() - ex2) <= 4.5 * se, (x2.mean(), ex2, se)
    mx = X.mean(1)
    assert abs(mx.mean()) <= 4.5 * mx.std(ddof=1) / math.sqrt(len(mx))


@pytest.mark.parametrize("kind_name", ["HNR", "CHNR"])
def test_hnr_boltzmann_cube_moments(kind_name):
    """Hit-and-Run for exp(-c.x/T) (sec:optimization P:1408-1424) on [-1,1]^3: independent
    truncated exponentials (P1, V7), moments by quadrature."""
    import paper_2010_03817_b200 as sw
    S = sw.Spectrahedron.from_instance(specgen.cube_only(3))
    c = np.array([1.0, -0.6, 2.5])
    T = 0.7
    S.set_objective(c)
    out = S.walk_sample(16384, 30, 1.0, 10, seed=8, kind=getattr(sw, kind_name), T=T)
    X = out["final_x"]
    grid = np.linspace(-1, 1, 200001)
    for i in range(3):
        dens = np.exp(-c[i] * grid / T)
        Z = np.trapezoid(dens, grid)
        for vals, e in ((X[:, i], np.trapezoid(grid * dens, grid) / Z),
                        (X[:, i] ** 2, np.trapezoid(grid ** 2 * dens, grid) / Z)):
            se = vals.std(ddof=1) / math.sqrt(len(vals))
            assert abs(vals.mean() - e) <= 4.5 * se, (i, vals.mean(), e, se)


def test_hnr_boltzmann_end_points_vs_oracle():
    """Boltzmann Hit-and-Run end points vs the oracle pointwise (configs[3]-shaped body at m = 40)."""
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(40, 40, 2)
    c = specgen.objective(40, 3)
    lmi = oracle.Lmi(inst)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    for kind_name in ("HNR", "CHNR"):
        out = S.walk_sample(64, 20, 1.0, 10, seed=5, kind=getattr(sw, kind_name), T=0.05)
        Xo, _ = oracle.walk(lmi, getattr(oracle, kind_name), 5, 0, 64, 20, 1.0, 10, T=0.05, c=c)
        err = np.linalg.norm(out["final_x"] - Xo, axis=1) / np.maximum(np.linalg.norm(Xo, axis=1), 0.1)
        assert err.max() <= 1e-8, (kind_name, err.max())
