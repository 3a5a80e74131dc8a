"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (65536 chains through the round scheduler): sampled chains are compared
with the oracle replaying exactly the same number of boundary-oracle calls
(one call per chain per round), plus full-population laws with closed forms
and oracle-vs-GPU statistics at configs the oracle can finish."""
import math

import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu
SAMPLED = [0, 1, 777, 32768, 65535]


def _device_state(S, chains, rounds, steps, L, rho, seed, kind=0, T=1.0):
    import torch
    S.walk_begin(chains, steps, L, rho, seed, kind=kind, T=T)
    S.walk_rounds(rounds)
    X = torch.empty((chains, S.n), dtype=torch.float64, device="cuda")
    st = S.walk_end(final_x=X)
    return X.cpu().numpy(), st


def test_m100_bench_configuration_sampled_chains():
    """bench.py's workload: configs[3] instance, 65536 billiard chains, L=2sqrt(n), rho=10n, seed 4."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(3)
    S = sw.Spectrahedron.from_instance(inst)
    R = 12
    X, st = _device_state(S, 65536, R, 100, 20.0, 1000, 4)
    assert st["calls"] == 65536 * R
    lmi = oracle.Lmi(inst)
    for c in SAMPLED:
        xo, calls = oracle.replay(lmi, oracle.BILLIARD, 4, c, 100, 20.0, 1000, R)
        assert calls == R
        assert np.linalg.norm(X[c] - xo) <= 1e-8 * max(np.linalg.norm(xo), 0.1), c


def test_m200_configs4_sampled_chains():
    """configs[4]: n = m = 200 (global-scratch K2 variant), 65536 chains, seed 4."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(4)
    S = sw.Spectrahedron.from_instance(inst)
    R = 2
    L = 2 * math.sqrt(200)
    X, st = _device_state(S, 65536, R, 100, L, 2000, 4)
    lmi = oracle.Lmi(inst)
    for c in (0, 65535):
        xo, calls = oracle.replay(lmi, oracle.BILLIARD, 4, c, 100, L, 2000, R)
        assert np.linalg.norm(X[c] - xo) <= 1e-8 * max(np.linalg.norm(xo), 0.1), c


def test_hmc_configs3_sampled_chains():
    """configs[3] HMC-r workload (65536 chains, T = 1, c ~ N(0, I) normalised), sampled."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(3)
    c = specgen.objective(100, 3)
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    R, L = 2, 1.09  # L = diam_est
    X, st = _device_state(S, 65536, R, 200, L, 1000, 3, kind=sw.HMC, T=1.0)
    lmi = oracle.Lmi(inst)
    for ch in (0, 40000):
        xo, calls = oracle.replay(lmi, oracle.HMC, 3, ch, 200, L, 1000, R, T=1.0, c=c)
        assert np.linalg.norm(X[ch] - xo) <= 1e-8 * max(np.linalg.norm(xo), 0.1), ch


def test_elliptope_configs1_moments():
    """configs[1]: elliptope k=20 (n=190, m=20), 16384 chains from 0, L=2sqrt(n):
    uniform law has E[x]=0, E[x^2]=1/(k+1)=1/21."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(1)
    S = sw.Spectrahedron.from_instance(inst)
    out = S.walk_sample(16384, 100, 2 * math.sqrt(190), 1900, seed=1)  # BASELINE.json configs[1]: 100 steps
    X = out["final_x"]
    per_chain_x2 = (X ** 2).mean(1)
    se = per_chain_x2.std(ddof=1) / math.sqrt(len(X))
    assert abs(per_chain_x2.mean() - 1 / 21) <= 4 * se, (per_chain_x2.mean(), 1 / 21, se)
    mx = X.mean(1)
    assert abs(mx.mean()) <= 4 * mx.std(ddof=1) / math.sqrt(len(X))
    # sum_x / sum_xx outputs agree with the end points
    assert np.allclose(out["sum_x"], X.sum(0), rtol=0, atol=1e-9)


def test_configs0_full_walk_statistics_vs_oracle():
    """configs[0]: 64 chains x 1000 steps, L=2sqrt(n), rho=10n, seed 0 -- GPU and oracle
    end-point laws agree (chaos makes long walks differ pointwise)."""
    import paper_2010_03817_b200 as sw
    inst = specgen.config_instance(0)
    S = sw.Spectrahedron.from_instance(inst)
    L = 2 * math.sqrt(10)
    g = S.walk_sample(64, 1000, L, 100, seed=0)
    o, st = oracle.walk(oracle.Lmi(inst), oracle.BILLIARD, 0, 0, 64, 1000, L, 100)
    a, b = (g["final_x"] ** 2).mean(1), (o ** 2).mean(1)
    se = math.sqrt(a.var(ddof=1) / 64 + b.var(ddof=1) / 64)
    assert abs(a.mean() - b.mean()) <= 4 * se
    assert g["stats"]["steps"] == 64 * 1000
    # reflection rate matches the oracle's within sampling noise
    rg = g["stats"]["reflections"] / g["stats"]["steps"]
    ro = st["reflections"] / st["steps"]
    assert abs(rg - ro) <= 0.1 * ro


def _sigma_oracle(o_vals, o_std_rel):
    """The oracle's Monte-Carlo standard deviation of one estimate (R28): the larger
    of the sample sd over its 10 seeds and the estimator's own binomial sigma (O8 step 6,
    mean over seeds) -- a 10-seed sample sd is itself uncertain by about +-24%."""
    o = np.asarray(o_vals)
    return max(o.std(ddof=1), float(np.mean(np.asarray(o_std_rel) * o)))


def test_volume_vs_oracle_rand_cube_10_seeds():
    """configs[2]-style body at reduced size (rand-cube n=m=12): GPU and oracle volume
    estimators over the same 10 seeds: |mean_gpu - mean_oracle| <= 2 sigma_oracle
    (north_star) and every GPU seed within 3 sigma_oracle of the oracle mean."""
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(12, 12, 2)
    S = sw.Spectrahedron.from_instance(inst)
    seeds = range(10)
    g = [S.volume(0.1, s, 256, walk_len=5, burn=20) for s in seeds]
    o = [oracle.volume(inst, 0.1, s, 256, W=5, burn=20) for s in seeds]
    gv = np.array([r["volume"] for r in g])
    ov = np.array([r["volume"] for r in o])
    sd = _sigma_oracle(ov, [r["std_rel"] for r in o])
    assert abs(gv.mean() - ov.mean()) <= 2 * sd, (gv.mean(), ov.mean(), sd)
    assert np.all(np.abs(gv - ov.mean()) <= 3 * sd), (gv, ov.mean(), sd)


def _golden(name):
    import json
    import os
    return json.load(open(os.path.join(os.path.dirname(__file__), "golden", name)))


def test_volume_configs2_instance_vs_oracle_10_seeds():
    """The configs[2] instance itself (rand-cube n = m = 40), seeds 0..9, at the reduced
    workload of tests/golden/make_oracle_goldens.py (eps = 0.3, 512 chains per phase, the
    same on both sides): mean within 2 sigma_oracle, every seed within 3 sigma_oracle."""
    import paper_2010_03817_b200 as sw
    gold = _golden("oracle_volume_cfg2.json")
    w = gold["workload"]
    inst = specgen.config_instance(w["instance"])
    S = sw.Spectrahedron.from_instance(inst)
    seeds = w["seeds"]
    g = [S.volume(w["eps"], s, w["chains_per_phase"], walk_len=w["walk_len"], burn=w["burn"]) for s in seeds]
    o = [gold["seeds"][str(s)] for s in seeds]
    gv = np.array([r["volume"] for r in g])
    ov = np.array([r["volume"] for r in o])
    sd = _sigma_oracle(ov, [r["std_rel"] for r in o])
    print(f"[parity] volume_cfg2: gpu mean {gv.mean():.6g} sd {gv.std(ddof=1):.3g} phases "
          f"{[r['phases'] for r in g]}; oracle mean {ov.mean():.6g} sigma {sd:.3g} phases {[r['phases'] for r in o]}")
    assert abs(gv.mean() - ov.mean()) <= 2 * sd, (gv.mean(), ov.mean(), sd)
    assert np.all(np.abs(gv - ov.mean()) <= 3 * sd), (gv, ov.mean(), sd)


def test_expectation_configs3_vs_oracle():
    """configs[3]: E[c^T x] and E[|x|^2] under exp(-c^T x / T), T = 1, by HMC-r from 0 at the
    reduced workload of tests/golden/make_oracle_goldens.py (global chain ids 0..127 on the
    oracle, 12 steps).  The GPU runs 8192 chains with the same ids first (the oracle's 128
    included): its 128-chain mean and its 8192-chain estimate lie within 2 standard errors of
    the oracle's estimate (north_star: 2x the oracle's Monte-Carlo sd)."""
    import paper_2010_03817_b200 as sw
    gold = _golden("oracle_expectation_cfg3.json")
    w = gold["workload"]
    inst = specgen.config_instance(w["instance"])
    c = specgen.objective(inst.n, w["instance"])
    S = sw.Spectrahedron.from_instance(inst)
    S.set_objective(c)
    out = S.walk_sample(8192, w["steps"], w["L"], w["rho"], seed=w["seed"], kind=sw.HMC, T=w["T"])
    X = out["final_x"]
    assert out["stats"]["failures"] == 0
    for key, fg in (("f_linear_c", X @ c), ("f_sqnorm", (X * X).sum(1))):
        fo = np.asarray(gold[key])
        k = len(fo)
        se_o = fo.std(ddof=1) / math.sqrt(k)
        print(f"[parity] expectation_cfg3 {key}: oracle {fo.mean():.6g} +- {se_o:.3g} (N={k}); "
              f"gpu same ids {fg[:k].mean():.6g}; gpu N=8192 {fg.mean():.6g} +- {fg.std(ddof=1) / math.sqrt(len(fg)):.3g}")
        assert abs(fg[:k].mean() - fo.mean()) <= 2 * se_o, key
        assert abs(fg.mean() - fo.mean()) <= 2 * se_o, key
    # the C-ABI estimator reproduces the same walk's mean (same seed and global ids)
    e = S.expectation(sw.F_LINEAR_C, w["T"], w["seed"], 8192, w["steps"], w["L"], w["rho"])
    assert abs(e["est"] - (X @ c).mean()) <= 1e-12 * max(1.0, abs(e["est"]))
