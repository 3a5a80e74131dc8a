"""GPU SDP by simulated annealing (eq:sdp P:1406, sec:optimization P:1408-1434) through
the C-ABI sdp_anneal: LPs with closed-form optima (min c^T x over the cube = -|c|_1, over
the unit ball = -|c|_2; SURVEY 8(f)#2 pins) reached to the paper's relative error 0.05 by
HMC-r with walk length 1 and by Hit-and-Run, and agreement with the oracle's annealing
(same seeds, tags and chains) on a configs-shaped spectrahedron."""
import math

import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu
C5 = np.array([0.9, -0.4, 0.2, 1.3, -0.7])


@pytest.mark.parametrize("kind_name", ["HMC", "HNR", "CHNR"])
@pytest.mark.parametrize("body", ["cube", "cube_dense", "ball"])
def test_sdp_anneal_lp_closed_forms(kind_name, body):
    import paper_2010_03817_b200 as sw
    n = 5
    if body == "cube":
        inst, fstar = specgen.cube_only(n), -np.abs(C5).sum()
    elif body == "cube_dense":
        inst, fstar = specgen.cube_dense(n), -np.abs(C5).sum()
    else:
        inst, fstar = specgen.ball(n), -np.linalg.norm(C5)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(C5)
    kind = getattr(sw, kind_name)
    r = S.sdp_anneal(kind, 256, 80, seed=3, walk_len=1 if kind == sw.HMC else 4 * n)
    assert r["best"] >= fstar - 1e-9
    assert r["best"] - fstar <= 0.05 * abs(fstar), (r["best"], fstar)
    assert abs(r["best_x"] @ C5 - r["best"]) <= 1e-12
    h = r["history"]
    assert np.all(h[1:] <= h[:-1])
    # with the optimum given, the run stops at the paper's tolerance
    r2 = S.sdp_anneal(kind, 256, 80, seed=3, walk_len=1 if kind == sw.HMC else 4 * n, f_target=fstar, eps=0.05)
    assert r2["iters"] <= r["iters"] and r2["best"] - fstar <= 0.05 * abs(fstar)


def test_sdp_anneal_vs_oracle_rand_cube():
    """Same annealing on both sides (rand-cube n = m = 12, 64 chains, HMC-r walk length 1, T_0 and
    tau given): both reach best values within 1% of each other after 40 temperatures (the
    chains' trajectories part chaotically -- R = max |x| of the starts differs by a few % --
    the law does not)."""
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(12, 12, 6)
    c = specgen.objective(12, 6)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    g = S.sdp_anneal(sw.HMC, 64, 40, seed=11, T0=1.0, L=1.0)
    o = oracle.sdp_anneal(inst, c, oracle.HMC, 64, 40, seed=11, T0=1.0, L=1.0)
    assert g["T0"] == o["T0"] == 1.0
    assert abs(g["best"] - o["best"]) <= 0.01 * abs(o["best"]), (g["best"], o["best"])
    assert g["iters"] == o["iters"] == 40
