"""Debug: GPU boundary_oracle vs CPU oracle, per-case diagnostics."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle, specgen
import paper_2010_03817_b200 as sw

for spec in sys.argv[1:] or ["10:10", "40:40", "100:100"]:
    n, m = map(int, spec.split(":"))
    inst = specgen.rand_cube(n, m, 0)
    lmi = oracle.Lmi(inst)
    S = sw.Spectrahedron.from_instance(inst)
    us = specgen.unit_vectors(8, n, 1); vs = specgen.unit_vectors(8, n, 2)
    xs = np.array([0.4 * oracle.chord(lmi, np.zeros(n), u)["t_plus"] * u for u in us])
    res = S.boundary_oracle(xs, vs, want_kernel=True)
    for k in range(8):
        r = oracle.chord(lmi, xs[k], vs[k]); w = oracle.normal(lmi, r["block"], r["y"])
        y = r["y"] / np.linalg.norm(r["y"])
        print(spec, k, "bind", res["binding"][k], r["binding"], "dt+", (res["t_plus"][k] - r["t_plus"]) / r["t_plus"],
              "dt-", (res["t_minus"][k] - r["t_minus"]) / abs(r["t_minus"]), "cos_w", float(res["normal"][k] @ w),
              "cos_y", abs(float(res["kernel"][k] @ y)))
