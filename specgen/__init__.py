"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no chords, normals, walks or
estimators): it only builds LMI instances and seeded vectors.  Both `oracle/`
and `paper_2010_03817_b200/` consume its outputs; neither imports the other.

Instance recipes:

* ``rand_cube(n, m, seed)`` -- BASELINE.json configs 0/2/3/4: A0 = I_m,
  A_i symmetric with iid N(0, 1/m) entries on and above the diagonal
  (order i = 1..n, row r, column c >= r), plus the cube block -1 <= x_i <= 1.
  numpy PCG64 (`default_rng(seed)`), instance seed = config index.
* ``elliptope(k)`` -- config 1: n = k(k-1)/2 coordinates (j,l), j<l in
  lexicographic order, A0 = I_k, A_(jl) = E_jl + E_lj, no cube block.
* ``ball(n)`` -- arrow LMI [[I_n, x], [x^T, 1]] >= 0  <=>  |x| <= 1 (m = n+1).
* ``cube_dense(n)`` -- the cube [-1,1]^n as a *dense* diagonal LMI, m = 2n,
  slots (1 - x_i), (1 + x_i).
* ``paper_example()`` -- PAPER.md Appendix B with the lower
  blocks of A1, A2 read as -Q~ and the missing A1[0][5] entry read as 0
  (reading R1).
* ``paper_random(n, m, seed)`` -- the paper's generator:
  A0 = Z Z^T + I, A_i = blockdiag(Q~, -Q~), Q~ = Q + Q^T.
* ``objective(n, seed)`` -- c ~ N(0, I) normalised (config 3 / HMC).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass
class Instance:
    """An LMI F(x) = A[0] + sum_i x_i A[i] (A has shape (n+1, m, m)) and an
    optional cube block lo <= x <= hi."""

    name: str
    A: np.ndarray  # (n+1, m, m) float64, symmetric
    lo: Optional[np.ndarray] = None  # (n,) or None
    hi: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return self.A.shape[0] - 1

    @property
    def m(self) -> int:
        return self.A.shape[1]


def rand_cube(n: int, m: int, seed: int, scale: float = 1.0, cube: bool = True) -> Instance:
    rng = np.random.default_rng(seed)
    A = np.zeros((n + 1, m, m))
    A[0] = np.eye(m)
    iu = np.triu_indices(m)
    sd = 1.0 / np.sqrt(m)
    for i in range(1, n + 1):
        vals = rng.standard_normal(len(iu[0])) * sd * scale
        T = np.zeros((m, m))
        T[iu] = vals
        A[i] = T + np.triu(T, 1).T
    lo = -np.ones(n) if cube else None
    hi = np.ones(n) if cube else None
    return Instance(f"rand_cube_n{n}_m{m}_s{seed}", A, lo, hi)


def elliptope(k: int) -> Instance:
    pairs = [(j, l) for j in range(k) for l in range(j + 1, k)]
    n = len(pairs)
    A = np.zeros((n + 1, k, k))
    A[0] = np.eye(k)
    for i, (j, l) in enumerate(pairs, start=1):
        A[i, j, l] = 1.0
        A[i, l, j] = 1.0
    return Instance(f"elliptope_k{k}", A)


def ball(n: int) -> Instance:
    m = n + 1
    A = np.zeros((n + 1, m, m))
    A[0] = np.eye(m)
    for i in range(1, n + 1):
        A[i, i - 1, n] = 1.0
        A[i, n, i - 1] = 1.0
    return Instance(f"ball_n{n}", A)


def cube_dense(n: int) -> Instance:
    m = 2 * n
    A = np.zeros((n + 1, m, m))
    A[0] = np.eye(m)
    for i in range(1, n + 1):
        A[i, 2 * (i - 1), 2 * (i - 1)] = -1.0
        A[i, 2 * (i - 1) + 1, 2 * (i - 1) + 1] = 1.0
    return Instance(f"cube_dense_n{n}", A)


def cube_only(n: int) -> Instance:
    """Cube [-1,1]^n with a trivial 1x1 dense block F = 1 (never binding)."""
    A = np.zeros((n + 1, 1, 1))
    A[0, 0, 0] = 1.0
    return Instance(f"cube_only_n{n}", A, -np.ones(n), np.ones(n))


_A0_EX = [
    [16.7, 3.7, 12.3, 8.7, 5.1, 10.4],
    [3.7, 9.4, 2.3, 4.0, -2.3, -1.0],
    [12.3, 2.3, 26.8, 18.7, 7.1, 16.7],
    [8.7, 4.0, 18.7, 20.0, 3.7, 12.3],
    [5.1, -2.3, 7.1, 3.7, 6.1, 5.4],
    [10.4, -1.0, 16.7, 12.3, 5.4, 18.7],
]
_Q1_EX = [[0.5, -0.4, 2.7], [-0.4, 1.4, -0.2], [2.7, -0.2, 1.7]]
_Q2_EX = [[2.6, -0.1, 3.0], [-0.1, 1.0, -0.1], [3.0, -0.1, -1.0]]


def paper_example() -> Instance:
    """PAPER.md Appendix B, lower blocks -Q~ (reading R1)."""
    A = np.zeros((3, 6, 6))
    A[0] = np.array(_A0_EX)
    for i, Q in ((1, _Q1_EX), (2, _Q2_EX)):
        Q = np.array(Q)
        A[i, :3, :3] = Q
        A[i, 3:, 3:] = -Q
    return Instance("paper_appendix_b", A)


def paper_random(n: int, m: int, seed: int) -> Instance:
    if m % 2:
        raise ValueError("paper generator needs even m")
    rng = np.random.default_rng(seed)
    Z = rng.uniform(0.0, 1.0, (m, m))
    A = np.zeros((n + 1, m, m))
    A[0] = Z @ Z.T + np.eye(m)
    h = m // 2
    for i in range(1, n + 1):
        Q = rng.uniform(-1.0, 1.0, (h, h))
        Qt = Q + Q.T
        A[i, :h, :h] = Qt
        A[i, h:, h:] = -Qt
    return Instance(f"paper_S{n}_{m}_s{seed}", A)


def objective(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(10_000 + seed)
    c = rng.standard_normal(n)
    return c / np.linalg.norm(c)


def unit_vectors(count: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(20_000 + seed)
    g = rng.standard_normal((count, n))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def uniforms(count: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    rng = np.random.default_rng(30_000 + seed)
    return rng.uniform(lo, hi, count)


# BASELINE.json configs (instance seed = config index)
def config_instance(idx: int) -> Instance:
    if idx == 0:
        return rand_cube(10, 10, 0)
    if idx == 1:
        return elliptope(20)
    if idx == 2:
        return rand_cube(40, 40, 2)
    if idx == 3:
        return rand_cube(100, 100, 3)
    if idx == 4:
        return rand_cube(200, 200, 4)
    raise ValueError(idx)
