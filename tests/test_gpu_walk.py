"""GPU parity for the billiard walk (Alg. 5): per-chain trajectories through
the first 20 reflections vs the oracle (relative 1e-8), closed-form moments of
uniform laws, determinism and chain-id sharding (P15)."""
import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu
TOL_TRAJ = 1e-8


# (per-trajectory parity with the chaos horizon: tests/test_gpu_parity_configs.py)


def test_walk_end_points_match_oracle_short_walks():
    """Few steps -> few reflections: end points agree pointwise."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(0)
    lmi = oracle.Lmi(inst)
    S = sw.Spectrahedron.from_instance(inst)
    L = 0.3
    X_o, st_o = oracle.walk(lmi, oracle.BILLIARD, 11, 0, 64, 3, L, 100)
    out = S.walk_sample(64, 3, L, 100, 11)
    d = np.linalg.norm(out["final_x"] - X_o, axis=1)
    assert np.mean(d <= 1e-9) >= 0.95
    assert out["stats"]["steps"] == 64 * 3


def test_walk_determinism_and_sharding():
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(12, 12, 4)
    S = sw.Spectrahedron.from_instance(inst)
    a = S.walk_sample(40, 8, 2 * np.sqrt(12), 120, seed=9)
    b = S.walk_sample(40, 8, 2 * np.sqrt(12), 120, seed=9)
    assert np.array_equal(a["final_x"], b["final_x"])
    assert np.array_equal(a["sum_xx"], b["sum_xx"])
    c1 = S.walk_sample(17, 8, 2 * np.sqrt(12), 120, seed=9, chain_begin=0)
    c2 = S.walk_sample(23, 8, 2 * np.sqrt(12), 120, seed=9, chain_begin=17)
    assert np.array_equal(np.vstack([c1["final_x"], c2["final_x"]]), a["final_x"])
    assert np.allclose(a["sum_x"], a["final_x"].sum(0), rtol=0, atol=1e-12)


def _mom(vals, expect, nsig=4.5):
    se = vals.std(ddof=1) / np.sqrt(len(vals))
    assert abs(vals.mean() - expect) <= nsig * se + 1e-12, (vals.mean(), expect, se)


@pytest.mark.parametrize("body", ["cube_dense", "ball", "elliptope4"])
def test_gpu_uniform_moments(body):
    import paper_2010_03817_b200 as sw
    if body == "cube_dense":
        inst, ex2 = specgen.cube_dense(4), 1 / 3
    elif body == "ball":
        inst, ex2 = specgen.ball(5), 1 / 7
    else:
        inst, ex2 = specgen.elliptope(4), 1 / 5
    S = sw.Spectrahedron.from_instance(inst)
    n = inst.n
    out = S.walk_sample(4000, 30, 2 * np.sqrt(n), 10 * n, seed=3)
    X = out["final_x"]
    _mom((X ** 2).mean(1), ex2)
    _mom(X.mean(1), 0.0)
    assert out["stats"]["failures"] == 0
