"""GPU parity: the CUDA boundary oracle (through the C-ABI) vs the CPU oracle
on identical seeded inputs.  Tolerances from BASELINE.json north_star:
t+/t- relative 1e-9, normals cos >= 1 - 1e-10, binding exact."""
import zlib

import numpy as np
import pytest

import oracle
import specgen

pytestmark = pytest.mark.gpu

TOL_T = 1e-9
TOL_COS = 1e-10


def _interior_batch(inst, lmi, count, seed, lam_max=0.95):
    """x = lam * t+(0, u) * u with u a random unit and lam ~ U(0, lam_max); v a random unit."""
    n = inst.n
    us = specgen.unit_vectors(count, n, seed)
    vs = specgen.unit_vectors(count, n, seed + 1)
    lams = specgen.uniforms(count, seed, 0.0, lam_max)
    xs = np.zeros((count, n))
    for k in range(count):
        r = oracle.chord(lmi, np.zeros(n), us[k])
        xs[k] = lams[k] * min(r["t_plus"], 1e6) * us[k]
    return xs, vs


def _compare(res, refs, n):
    for k, r in enumerate(refs):
        tp, tm = res["t_plus"][k], res["t_minus"][k]
        assert res["binding"][k] == r["binding"], (k, res["binding"][k], r["binding"])
        assert abs(tp - r["t_plus"]) <= TOL_T * abs(r["t_plus"]), (k, tp, r["t_plus"])
        if np.isfinite(r["t_minus"]):
            assert abs(tm - r["t_minus"]) <= TOL_T * max(abs(r["t_minus"]), 1e-300), (k, tm, r["t_minus"])
        w = res["normal"][k]
        wo = r["w"]
        cos = float(w @ wo) / (np.linalg.norm(w) * np.linalg.norm(wo))
        assert cos >= 1 - TOL_COS, (k, cos)


def _oracle_refs(lmi, xs, vs, bound=-1, us=None):
    refs = []
    for k in range(len(xs)):
        kw = {}
        if us is not None:
            F = lmi.eval_block(0, xs[k])
            kw = dict(F0=F, bound=0, u=us[k])
        r = oracle.chord(lmi, xs[k], vs[k], **kw)
        r["w"] = oracle.normal(lmi, r["block"], r["y"])
        refs.append(r)
    return refs


CASES = [
    ("rand_10_10", lambda: specgen.rand_cube(10, 10, 0)),
    ("rand_40_40", lambda: specgen.rand_cube(40, 40, 2)),
    ("rand_100_100", lambda: specgen.rand_cube(100, 100, 3)),
    ("rand_200_200", lambda: specgen.rand_cube(200, 200, 4)),
    ("elliptope_20", lambda: specgen.elliptope(20)),
    ("mixed_binding_12_30", lambda: specgen.rand_cube(12, 30, 5, scale=1 / np.sqrt(12))),
    ("cube_dense_5", lambda: specgen.cube_dense(5)),
    ("ball_7", lambda: specgen.ball(7)),
    # a rank-2 pencil A(v) on the split path (m = 101: factor | lanczos2 | tail): the Lanczos
    # space becomes invariant after 2-3 steps (the residual is rounding, lanczos2's DGKS pass)
    ("ball_100", lambda: specgen.ball(100)),
    ("paper_example", specgen.paper_example),
    ("rand_3_1", lambda: specgen.rand_cube(3, 1, 9)),
]
# one instance per K2 launch variant (csrc/specwalk.cu): 128-thread fused (m <= 32), 192-thread
# fused (m <= 48), 256-thread fused (m <= 64), split with 13 column pairs (m <= 104, here with
# mp = 72 < 104: padded columns), split with 16 pairs (104 < m <= 128), global scratch (m > 128)
VARIANTS = [
    ("v4_rand_8_30", lambda: specgen.rand_cube(8, 30, 11)),
    ("v5_rand_12_44", lambda: specgen.rand_cube(12, 44, 12)),
    ("v0_rand_16_60", lambda: specgen.rand_cube(16, 60, 13)),
    ("v1_rand_20_72", lambda: specgen.rand_cube(20, 72, 14)),
    # factor_t_kernel's tile-count edges: m = 65 (a deflated start has md = 64: no padding),
    # m = 97 (md = 96, 12 tiles), m = 104 (mp = 104, 13 tiles, md = 103)
    ("v1_rand_10_65", lambda: specgen.rand_cube(10, 65, 18)),
    ("v1_rand_12_97", lambda: specgen.rand_cube(12, 97, 19)),
    ("v1_rand_14_104", lambda: specgen.rand_cube(14, 104, 20)),
    ("v3_rand_16_110", lambda: specgen.rand_cube(16, 110, 17)),  # fused <512, smem, KC 16> (104 < mp <= 112)
    ("v2_rand_24_120", lambda: specgen.rand_cube(24, 120, 15)),  # mp = 120: matrices no longer fit shared memory
    ("v2_rand_10_136", lambda: specgen.rand_cube(10, 136, 16)),
    # factor_g_kernel's tile-count edges: m = 113 (mp = 120; a deflated start has md = 112: 14 tiles,
    # no padding), m = 201 (mp = 208, 26 tiles; md = 200: 25 tiles), m = 208 (26 tiles, md = 207)
    ("v2_rand_8_113", lambda: specgen.rand_cube(8, 113, 21)),
    ("v2_rand_6_201", lambda: specgen.rand_cube(6, 201, 22)),
    ("v2_rand_6_208", lambda: specgen.rand_cube(6, 208, 23)),
]


@pytest.mark.parametrize("name,make", CASES + VARIANTS, ids=[c[0] for c in CASES + VARIANTS])
def test_boundary_oracle_interior_parity(name, make):
    import paper_2010_03817_b200 as sw
    inst = make()
    lmi = oracle.Lmi(inst)
    count = 6 if inst.m >= 200 else (24 if inst.m >= 100 else 64)
    xs, vs = _interior_batch(inst, lmi, count, seed=zlib.crc32(name.encode()) % 1000)
    refs = _oracle_refs(lmi, xs, vs)
    S = sw.Spectrahedron.from_instance(inst)
    res = S.boundary_oracle(xs, vs)
    _compare(res, refs, inst.n)
    # the hit is on the boundary: lambda_min(F(x + t+ v)) ~ 0 for dense hits (P4)
    for k in range(count):
        if res["binding"][k] == 0:
            p = xs[k] + res["t_plus"][k] * vs[k]
            F = inst.A[0] + np.tensordot(p, inst.A[1:], axes=1)
            scale = np.abs(inst.A[0]).max() + np.abs(p) @ np.abs(inst.A[1:]).max(axis=(1, 2))
            assert abs(np.linalg.eigvalsh(F)[0]) <= 1e-12 * scale


BCASES = CASES[:6] + [c for c in CASES if c[0] == "ball_100"] + VARIANTS


@pytest.mark.parametrize("name,make", BCASES, ids=[c[0] for c in BCASES])
def test_boundary_oracle_boundary_start_parity(name, make):
    """Segments that start on the dense boundary (after a reflection): Schur deflation (R6)."""
    import paper_2010_03817_b200 as sw
    inst = make()
    lmi = oracle.Lmi(inst, cube=False)
    inst_nc = specgen.Instance(inst.name, inst.A)  # dense block only so every hit is dense
    n = inst.n
    count = 4 if inst.m >= 200 else (16 if inst.m >= 100 else 48)
    xs0, vs0 = _interior_batch(inst_nc, lmi, count, seed=7)
    hits, us, ss = [], [], []
    for k in range(count):
        r = oracle.chord(lmi, xs0[k], vs0[k])
        hit = xs0[k] + r["t_plus"] * vs0[k]
        w = oracle.normal(lmi, r["block"], r["y"])
        hits.append(hit)
        us.append(r["y"] / np.linalg.norm(r["y"]))
        ss.append(oracle.reflect(vs0[k], w))
    hits, us, ss = np.array(hits), np.array(us), np.array(ss)
    refs = _oracle_refs(lmi, hits, ss, us=us)
    S = sw.Spectrahedron(inst.A)
    res = S.boundary_oracle(hits, ss, u=us)
    _compare(res, refs, n)
    assert np.all(res["t_minus"] == 0.0)


def test_boundary_oracle_errors_and_edge_cases():
    import paper_2010_03817_b200 as sw
    inst = specgen.rand_cube(6, 6, 1)
    S = sw.Spectrahedron.from_instance(inst)
    out = S.boundary_oracle(np.zeros((0, 6)), np.zeros((0, 6)))
    assert out["t_plus"].shape == (0,)
    dense = oracle.Lmi(inst, cube=False)
    u = np.ones(6) / np.sqrt(6)
    x_out = 1.5 * oracle.chord(dense, np.zeros(6), u)["t_plus"] * u  # beyond the dense boundary
    with pytest.raises(sw.SpecError) as ei:
        sw.Spectrahedron(inst.A).boundary_oracle(x_out[None], u[None])
    assert ei.value.code == 2  # EPRECOND: x not interior
    with pytest.raises(sw.SpecError):
        sw.Spectrahedron(np.stack([np.eye(3), np.triu(np.ones((3, 3)))]))  # asymmetric -> EINVAL
    # ragged batch sizes that span several chord CTAs and GEMM tiles with a tail
    lmi = oracle.Lmi(inst)
    xs, vs = _interior_batch(inst, lmi, 333, seed=3)
    res = S.boundary_oracle(xs, vs)
    refs = _oracle_refs(lmi, xs[::37], vs[::37])
    _compare({k: (v[::37] if hasattr(v, "__len__") else v) for k, v in res.items()}, refs, 6)
