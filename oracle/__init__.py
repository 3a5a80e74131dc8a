"""CPU oracle for arXiv 2010.03817 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2010_03817_b200`` (the CUDA product path) and
neither imports the other; both consume inputs from ``specgen``.

The arithmetic lives in ``oracle.c`` (plain C99, fp64, no BLAS, built with
``-O2 -ffp-contract=off -fno-fast-math``); this module is the ctypes binding
plus the estimator drivers that follow PAPER.md step by step:

* ``chord`` / ``normal`` / ``reflect`` -- Alg. 2, Lemma 3
  (P:587-651), Alg. 3, lemma:gradient,
  eq:reflection, with the Schur deflation of DESIGN.md R6 for
  segments that start on the boundary.
* ``walk`` / ``trace`` -- Billiard walk (Alg. 5) and HMC-r
  (Alg. 6, eq:boltz_ode P:1440-1446).
* ``volume`` -- ball-phase MMC (eq:mmc_vol P:1291-1306, telescoping product
  P:1246-1259) with the schedule reading R11-R14.
* ``expectation`` -- Monte-Carlo mean.

Parity pins for every function are in ``tests/test_oracle_*.py``; see
DESIGN.md "Oracle pins".  Functions without an independent pin say
"parity unpinned" in their docstring.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")

INF = float("inf")
BILLIARD, HMC, HNR, CHNR, CHMC = 0, 1, 2, 3, 4  # HnR: Alg. 4; CHnR: P:985-996; CHMC: P:1146-1158
POT_LINEAR, POT_GAUSS, POT_LOGCOSH = 0, 1, 2
TAG_WALK = 0 << 28
TAG_VOLUME = 1 << 28
TAG_PILOT = 3 << 28


def build(force: bool = False) -> str:
    """Compile oracle.c into liborc.so (plain gcc, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = [
            "gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
            "-D_POSIX_C_SOURCE=200809L", "-pthread", "-o", _LIB + ".tmp", _SRC, "-lm",
        ]
        subprocess.check_call(cmd, cwd=_HERE)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None
_dp = C.POINTER(C.c_double)


class _ChordRes(C.Structure):
    _fields_ = [
        ("t_plus", C.c_double), ("t_minus", C.c_double), ("binding", C.c_int),
        ("degenerate", C.c_int), ("outward", C.c_int), ("theta_max", C.c_double),
        ("theta_2", C.c_double), ("ylen", C.c_int), ("y", C.c_double * (1024 + 8)),
    ]


class _Stats(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("calls", "reflections", "rejects", "degenerates", "steps", "failures")]


class _WalkParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("seed", C.c_uint64), ("tag", C.c_uint32), ("steps", C.c_int64),
        ("L", C.c_double), ("rho", C.c_int64), ("T", C.c_double), ("c", _dp),
        ("pot", C.c_int), ("mu", _dp), ("sigma", C.c_double), ("q", C.c_int), ("h", C.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        l = C.CDLL(build())
        l.orc_lmi_create.restype = C.c_void_p
        l.orc_lmi_create.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.c_double, C.c_int]
        l.orc_lmi_destroy.argtypes = [C.c_void_p]
        l.orc_lmi_nblocks.argtypes = [C.c_void_p]
        l.orc_lmi_block_size.argtypes = [C.c_void_p, C.c_int]
        l.orc_eval_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        l.orc_dir_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        l.orc_cholesky.argtypes = [C.c_int, _dp, _dp]
        l.orc_jacobi.argtypes = [C.c_int, _dp, _dp, _dp]
        l.orc_philox4x32_10.argtypes = [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        l.orc_u01.restype = C.c_double
        l.orc_u01.argtypes = [C.c_uint32, C.c_uint32]
        l.orc_step_draws.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _dp, _dp]
        l.orc_step_uniforms.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, _dp, _dp]
        l.orc_chord.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_int, _dp, C.POINTER(_ChordRes)]
        l.orc_normal.argtypes = [C.c_void_p, C.c_int, _dp, C.c_int, _dp]
        l.orc_reflect.argtypes = [C.c_int, _dp, _dp, _dp]
        l.orc_membership.argtypes = [C.c_void_p, _dp]
        l.orc_walk.argtypes = [C.c_void_p, C.POINTER(_WalkParams), C.c_int64, C.c_int64, _dp, C.c_int, _dp,
                               C.POINTER(_Stats), C.c_int]
        l.orc_trace.argtypes = [C.c_void_p, C.POINTER(_WalkParams), C.c_int64, _dp, C.c_int64, _dp, _dp, _dp,
                                _dp, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        l.orc_trace_stats.argtypes = [C.c_void_p, C.POINTER(_WalkParams), C.c_int64, _dp, C.c_int64, _dp, _dp,
                                      _dp, _dp, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(_Stats)]
        l.orc_replay.argtypes = [C.c_void_p, C.POINTER(_WalkParams), C.c_int64, _dp, C.c_int64, _dp,
                                 C.POINTER(C.c_int64)]
        l.orc_qep_root.argtypes = [C.c_int, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp]
        l.orc_hmc_chord.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp,
                                    C.POINTER(_ChordRes)]
        l.orc_colloc_basis.argtypes = [C.c_int, _dp, _dp]
        l.orc_colloc_poly.argtypes = [C.c_int, C.POINTER(_WalkParams), _dp, _dp, C.c_double, _dp]
        l.orc_pep_root.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp, C.c_double, _dp, _dp]
        l.orc_colloc_chord.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp,
                                       C.POINTER(_ChordRes)]
        _lib = l
    return _lib


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _arr(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class Lmi:
    """F(x) = blockdiag(dense F_0(x), cube blocks, ball arrow block) (eq:lmi P:70-75)."""

    def __init__(self, inst, ball_c=None, ball_r: float = 0.0, literal: bool = False, cube: bool = True):
        self.inst = inst
        self.n, self.m = inst.n, inst.m
        self._A = _arr(inst.A)
        lo = _arr(inst.lo) if (cube and inst.lo is not None) else None
        hi = _arr(inst.hi) if (cube and inst.hi is not None) else None
        bc = _arr(ball_c) if ball_c is not None else None
        self.has_cube = lo is not None
        self.has_ball = bc is not None
        self.ball_c, self.ball_r = bc, float(ball_r)
        self._h = lib().orc_lmi_create(self.n, self.m, _p(self._A), _p(lo), _p(hi), _p(bc), float(ball_r),
                                       1 if literal else 0)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_lmi_destroy(self._h)
            self._h = None

    @property
    def nblocks(self) -> int:
        return lib().orc_lmi_nblocks(self._h)

    def block_size(self, b: int) -> int:
        return lib().orc_lmi_block_size(self._h, b)

    def eval_block(self, b: int, x) -> np.ndarray:
        s = self.block_size(b)
        out = np.zeros((s, s))
        lib().orc_eval_block(self._h, b, _p(_arr(x)), _p(out))
        return out

    def dir_block(self, b: int, v) -> np.ndarray:
        s = self.block_size(b)
        out = np.zeros((s, s))
        lib().orc_dir_block(self._h, b, _p(_arr(v)), _p(out))
        return out

    def binding_code(self, b: int) -> int:
        """ABI binding id: 0 dense, 1+2i cube upper, 2+2i cube lower, -1 ball."""
        if self.has_ball and b == self.nblocks - 1:
            return -1
        return b


def cholesky(A) -> Optional[np.ndarray]:
    A = _arr(A)
    m = A.shape[0]
    L = np.zeros_like(A)
    return None if lib().orc_cholesky(m, _p(A), _p(L)) else L


def jacobi(A):
    A = _arr(A)
    m = A.shape[0]
    ev = np.zeros(m)
    V = np.zeros((m, m))
    lib().orc_jacobi(m, _p(A), _p(ev), _p(V))
    return ev, V


def philox(ctr, key) -> np.ndarray:
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def u01(a: int, b: int) -> float:
    return lib().orc_u01(a, b)


def step_draws(seed: int, tag: int, chain: int, step: int, n: int):
    g = np.zeros(n)
    eta = C.c_double()
    lib().orc_step_draws(seed, tag, chain, step, n, _p(g), C.byref(eta))
    return g, eta.value


def step_uniforms(seed: int, tag: int, chain: int, step: int, n: int):
    """(eta, u2): the two doubles of Philox block ceil(n/2) of a step (W-CHnR: j = floor(u2 n))."""
    eta, u2 = C.c_double(), C.c_double()
    lib().orc_step_uniforms(seed, tag, chain, step, n, C.byref(eta), C.byref(u2))
    return eta.value, u2.value


def chord(lmi: Lmi, x, v, F0=None, bound: int = -1, u=None) -> dict:
    """Boundary oracle on the line x + t v (Alg. 2 + Lemma 3; deflation R6)."""
    r = _ChordRes()
    x, v = _arr(x), _arr(v)
    F0a = _arr(F0) if F0 is not None else None
    ua = _arr(u) if u is not None else None
    rc = lib().orc_chord(lmi._h, _p(x), _p(F0a), None, _p(v), int(bound), _p(ua), C.byref(r))
    if rc:
        raise ValueError(f"orc_chord failed rc={rc} (x not interior?)")
    return dict(t_plus=r.t_plus, t_minus=r.t_minus, block=r.binding, binding=lmi.binding_code(r.binding)
                if r.binding >= 0 else None, degenerate=bool(r.degenerate), outward=bool(r.outward),
                theta_max=r.theta_max, theta_2=r.theta_2, y=np.array(r.y[: r.ylen]))


def normal(lmi: Lmi, block: int, y) -> Optional[np.ndarray]:
    y = _arr(y)
    w = np.zeros(lmi.n)
    rc = lib().orc_normal(lmi._h, block, _p(y), len(y), _p(w))
    return None if rc else w


def reflect(u, w) -> np.ndarray:
    u, w = _arr(u), _arr(w)
    s = np.zeros_like(u)
    lib().orc_reflect(len(u), _p(u), _p(w), _p(s))
    return s


def membership(lmi: Lmi, x) -> bool:
    return bool(lib().orc_membership(lmi._h, _p(_arr(x))))


def qep_root(B0, B1, B2, u=None):
    """First positive root of det(B0 + t B1 + t^2 B2) (companion + Francis QR)."""
    B0, B1, B2 = _arr(B0), _arr(B1), _arr(B2)
    mb = B0.shape[0]
    tp = C.c_double()
    y = np.zeros(mb)
    ua = _arr(u) if u is not None else None
    rc = lib().orc_qep_root(mb, _p(B0), _p(B1), _p(B2), 1 if u is not None else 0, _p(ua), C.byref(tp), _p(y))
    if rc:
        raise ValueError(f"qep_root rc={rc}")
    return tp.value, y


def hmc_chord(lmi: Lmi, x, v, c, T, F0=None, bound=-1, u=None) -> dict:
    r = _ChordRes()
    x, v, c = _arr(x), _arr(v), _arr(c)
    F0a = _arr(F0) if F0 is not None else None
    ua = _arr(u) if u is not None else None
    rc = lib().orc_hmc_chord(lmi._h, _p(x), _p(F0a), _p(v), _p(c), float(T), int(bound), _p(ua), C.byref(r))
    if rc:
        raise ValueError(f"hmc_chord rc={rc}")
    return dict(t_plus=r.t_plus, block=r.binding, outward=bool(r.outward), y=np.array(r.y[: r.ylen]))


def _params(kind, seed, tag, steps, L, rho, T=1.0, c=None, colloc=None):
    """colloc (kind CHMC): dict(pot=POT_*, mu=array or None, sigma=float, q=int, h=float)."""
    p = _WalkParams()
    p.kind, p.seed, p.tag, p.steps, p.L, p.rho, p.T = kind, seed, tag, steps, float(L), rho, float(T)
    keep = _arr(c) if c is not None else None
    p.c = _p(keep)
    keep_mu = None
    if colloc is not None:
        p.pot = int(colloc.get("pot", POT_GAUSS))
        keep_mu = _arr(colloc["mu"]) if colloc.get("mu") is not None else None
        p.mu = _p(keep_mu)
        p.sigma = float(colloc.get("sigma", 1.0))
        p.q = int(colloc.get("q", 3))
        p.h = float(colloc["h"])
    return p, (keep, keep_mu)


def colloc_basis(q: int):
    """Chebyshev nodes of [0, 1] and Lagrange monomial coefficients lcoef[j, k] (R33)."""
    nodes = np.zeros(q)
    lc = np.zeros((q, q))
    if lib().orc_colloc_basis(q, _p(nodes), _p(lc)):
        raise ValueError("q out of range")
    return nodes, lc


def colloc_poly(x0, v0, h: float, colloc: dict, c=None, T: float = 1.0):
    """Collocation polynomial of p'' = -grad f on [0, h]: coef[k] = t^k
    coefficient (q+2 rows), and the Picard iterations used (negative: not converged)."""
    x0, v0 = _arr(x0), _arr(v0)
    n = x0.shape[0]
    p, keep = _params(CHMC, 0, 0, 1, 1.0, 0, T, c, colloc)
    coef = np.zeros((p.q + 2, n))
    it = lib().orc_colloc_poly(n, C.byref(p), _p(x0), _p(v0), float(h), _p(coef))
    return coef, it


def pep_root(Bs, tmax: float = INF, u=None):
    """First root in (0, tmax] of det(sum_k t^k B_k) (degree-d companion + Francis QR);
    +inf if none.  u: unit kernel vector of B_0 (boundary start).  Returns (t_plus, kernel
    vector); raises on rc != 0 (2: B_0 not PD, 3: outward)."""
    B = _arr(np.stack([_arr(b) for b in Bs]))
    d = B.shape[0] - 1
    mb = B.shape[1]
    tp = C.c_double()
    y = np.zeros(mb)
    ua = _arr(u) if u is not None else None
    rc = lib().orc_pep_root(mb, d, _p(B), 1 if u is not None else 0, _p(ua), float(tmax), C.byref(tp), _p(y))
    if rc:
        raise ValueError(f"pep_root rc={rc}")
    return tp.value, y


def colloc_chord(lmi: Lmi, coef, tmax: float, F0=None, bound: int = -1, u=None) -> dict:
    """Chord of the curve sum_k coef[k] t^k over every block, t in (0, tmax]."""
    r = _ChordRes()
    coef = _arr(coef)
    d = coef.shape[0] - 1
    F0a = _arr(F0) if F0 is not None else None
    ua = _arr(u) if u is not None else None
    rc = lib().orc_colloc_chord(lmi._h, _p(F0a), _p(coef), d, float(tmax), int(bound), _p(ua), C.byref(r))
    if rc:
        raise ValueError(f"colloc_chord rc={rc}")
    return dict(t_plus=r.t_plus, block=r.binding, outward=bool(r.outward), y=np.array(r.y[: r.ylen]))


def walk(lmi: Lmi, kind: int, seed: int, chain_begin: int, chain_end: int, steps: int, L: float, rho: int,
         x0=None, T: float = 1.0, c=None, tag: int = TAG_WALK, nthreads: int = 0, colloc=None):
    """Run chains [chain_begin, chain_end) (global ids key the RNG). Returns (final_x, stats)."""
    n = lmi.n
    if x0 is None:
        x0 = np.zeros(n)
    x0 = _arr(x0)
    stride = 0 if x0.ndim == 1 else n
    p, keep = _params(kind, seed, tag, steps, L, rho, T, c, colloc)
    out = np.zeros((chain_end - chain_begin, n))
    st = _Stats()
    if nthreads <= 0:
        nthreads = os.cpu_count() or 1
    rc = lib().orc_walk(lmi._h, C.byref(p), chain_begin, chain_end, _p(x0), stride, _p(out), C.byref(st),
                        nthreads)
    if rc:
        raise ValueError(f"orc_walk rc={rc}")
    return out, {k: getattr(st, k) for k, _ in _Stats._fields_}


def trace(lmi: Lmi, kind: int, seed: int, chain: int, steps: int, L: float, rho: int, max_refl: int,
          x0=None, T: float = 1.0, c=None, tag: int = TAG_WALK, stop: bool = False, colloc=None) -> dict:
    """First max_refl reflections of one chain.  stop=True ends the walk right after the last
    record (orc_trace; calls = None), else the step of the last record is completed
    (orc_trace_stats; calls = every oracle call made)."""
    n = lmi.n
    x0 = _arr(np.zeros(n) if x0 is None else x0)
    p, keep = _params(kind, seed, tag, steps, L, rho, T, c, colloc)
    hit = np.zeros((max_refl, n))
    t = np.zeros(max_refl)
    w = np.zeros((max_refl, n))
    va = np.zeros((max_refl, n))
    bind = np.zeros(max_refl, dtype=np.int32)
    nrec = C.c_int64()
    st = _Stats()
    if stop:
        rc = lib().orc_trace(lmi._h, C.byref(p), chain, _p(x0), max_refl, _p(hit), _p(t), _p(w), _p(va),
                             bind.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nrec))
    else:
        rc = lib().orc_trace_stats(lmi._h, C.byref(p), chain, _p(x0), max_refl, _p(hit), _p(t), _p(w), _p(va),
                                   bind.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(nrec), C.byref(st))
    if rc:
        raise ValueError(f"orc_trace rc={rc}")
    k = nrec.value
    # calls: every boundary-oracle call of the walk (it finishes the step of the last record)
    return dict(hit_x=hit[:k], t=t[:k], w=w[:k], v_after=va[:k], binding=bind[:k],
                calls=None if stop else int(st.calls))


def replay(lmi: Lmi, kind: int, seed: int, chain: int, steps: int, L: float, rho: int, max_calls: int,
           x0=None, T: float = 1.0, c=None, tag: int = TAG_WALK, colloc=None):
    """x of one chain after exactly max_calls chord calls (GPU state after that many rounds)."""
    n = lmi.n
    x0 = _arr(np.zeros(n) if x0 is None else x0)
    p, keep = _params(kind, seed, tag, steps, L, rho, T, c, colloc)
    x = np.zeros(n)
    calls = C.c_int64()
    rc = lib().orc_replay(lmi._h, C.byref(p), chain, _p(x0), max_calls, _p(x), C.byref(calls))
    if rc:
        raise ValueError(f"orc_replay rc={rc}")
    return x, calls.value


def ball_volume(n: int, r: float = 1.0) -> float:
    """omega_n r^n = pi^(n/2) / Gamma(n/2+1) r^n."""
    return math.exp(0.5 * n * math.log(math.pi) - math.lgamma(0.5 * n + 1) + n * math.log(r))


# ---------------------------------------------------------------------------
# Estimators -- orchestration over the C oracle
# ---------------------------------------------------------------------------
PURPOSE_VOLUME, PURPOSE_PILOT = 1, 3


def vol_tag(purpose: int, phase: int, ball: bool, attempt: int = 0) -> int:
    """Philox counter word 3: purpose in bits 28-31, (attempt, phase, walk/ball) below."""
    return (purpose << 28) | (attempt << 20) | (phase << 1) | (1 if ball else 0)


def ball_samples(seed: int, tag: int, begin: int, count: int, n: int, c0, r: float) -> np.ndarray:
    """Exact uniform samples of B(c0, r): x = c0 + r eta^(1/n) g/|g| with the step-draw
    layout of O7 (g from blocks 0..ceil(n/2)-1, eta from block ceil(n/2)), sample j at
    counter (block, step 0, chain j, tag)."""
    X = np.empty((count, n))
    for k in range(count):
        g, eta = step_draws(seed, tag, begin + k, 0, n)
        X[k] = np.asarray(c0) + r * eta ** (1.0 / n) * g / np.linalg.norm(g)
    return X


def volume(inst, eps: float, seed: int, N: int, W: int = 10, burn: int = 20, L: float = None, rho: int = None,
           rho_star: float = 0.325, q_stop: float = 0.25, max_phases: int = 64, max_growth: int = 16,
           nthreads: int = 0) -> dict:
    """Ball-phase multiphase Monte Carlo volume (eq:mmc_vol P:1291-1300, telescoping
    product P:1246-1259; schedule = DESIGN.md readings R11-R14):

    pilot   : S_0 = S; billiard samples of S_i (phase 0 burned in from c0 = 0);
              r_{i+1} = rho*-quantile of |x - c0|; stop once q(r_{i+1}) =
              P_{U(B(r_{i+1}))}[x in S] >= q_stop (exact ball sampling + membership).
    estimate: fresh walks of S_i = S cap B(r_i), warm-started from the previous
              phase's points inside B(r_i) (resampled in chain order);
              rho_i = #{|x - c0| <= r_{i+1}} / N;  q = membership fraction of N
              exact samples of B(r_k);  vol = omega_n r_k^n q / prod rho_i.
    sigma_rel^2 = sum (1 - rho)/(N rho) + (1 - q)/(N q); N doubles (fresh tags)
    until sigma_rel <= eps/2 or N reaches max_growth * N."""
    n = inst.n
    L = 2.0 * math.sqrt(n) if L is None else L
    rho = 10 * n if rho is None else rho
    c0 = np.zeros(n)
    full = Lmi(inst)

    def walk_phase(r, X0, steps, tag, count):
        lmi = full if r is None else Lmi(inst, ball_c=c0, ball_r=r)
        X, st = walk(lmi, BILLIARD, seed, 0, count, steps, L, rho, x0=X0, tag=tag, nthreads=nthreads)
        return X, st

    def q_of(r, tag, count):
        B = ball_samples(seed, tag, 0, count, n, c0, r)
        return float(np.mean([membership(full, b) for b in B]))

    def resample(X, r, count):
        # strictly inside B(r): the pilot's quantile point itself lies on the sphere
        inside = X[np.linalg.norm(X - c0, axis=1) < r]
        idx = np.arange(count) % len(inside)
        return warm(inside[idx])

    def warm(X):
        # DESIGN.md R24: a warm start re-forms F(x); an end point within rounding of
        # the boundary is contracted towards the interior point c0 by 2^-40
        return c0 + (1.0 - 2.0 ** -40) * (X - c0)

    calls = 0
    # ---- pilot: radii
    radii = [None]
    X = np.zeros((N, n))
    X, st = walk_phase(None, X, burn, vol_tag(PURPOSE_PILOT, 0, False), N)
    calls += st["calls"]
    burned = X.copy()
    qs = []
    for i in range(max_phases):
        d = np.sort(np.linalg.norm(X - c0, axis=1))
        r_next = float(d[max(0, int(math.ceil(rho_star * N)) - 1)])
        q = q_of(r_next, vol_tag(PURPOSE_PILOT, i, True), N)
        radii.append(r_next)
        qs.append(q)
        if q >= q_stop:
            break
        X, st = walk_phase(r_next, resample(X, r_next, N), W, vol_tag(PURPOSE_PILOT, i + 1, False), N)
        calls += st["calls"]
    k = len(radii) - 1
    # ---- estimation
    attempt, Ne = 0, N
    while True:
        X = warm(burned if Ne == N else burned[np.arange(Ne) % N])
        ratios = []
        for i in range(k):
            X, st = walk_phase(radii[i], X, W, vol_tag(PURPOSE_VOLUME, i, False, attempt), Ne)
            calls += st["calls"]
            inside = np.linalg.norm(X - c0, axis=1) <= radii[i + 1]
            ratios.append(float(np.mean(inside)))
            X = resample(X, radii[i + 1], Ne)
        q = q_of(radii[k], vol_tag(PURPOSE_VOLUME, k, True, attempt), Ne)
        ratios_a = np.array(ratios)
        var = float(np.sum((1 - ratios_a) / (Ne * ratios_a)) + (1 - q) / (Ne * q))
        sig = math.sqrt(var)
        if sig <= eps / 2 or Ne >= max_growth * N:
            break
        attempt += 1
        Ne *= 2
    logv = math.log(ball_volume(n, radii[k])) + math.log(q) - float(np.sum(np.log(ratios_a)))
    return dict(volume=math.exp(logv), log_volume=logv, std_rel=sig, phases=k, radii=radii[1:],
                ratios=ratios, q=q, chains=Ne, calls=calls)


def expectation(inst, f_id: str, seed: int, chains: int, steps: int, L: float, rho: int, T: float = None,
                c=None, b1: float = None, b2: float = None, nthreads: int = 0) -> dict:
    """E[f] over the chains' end points (reading R18): uniform law by the
    billiard walk (T is None) or exp(-c.x/T) by HMC-r.  f in {"linear_c": c.x,
    "sqnorm": |x|^2, "halfspace_union": 1(c.x <= b1 or c.x >= b2)}.
    stderr = sample sd / sqrt(chains) (O9)."""
    lmi = Lmi(inst)
    kind = BILLIARD if T is None else HMC
    X, st = walk(lmi, kind, seed, 0, chains, steps, L, rho, T=1.0 if T is None else T, c=c, nthreads=nthreads)
    if f_id == "linear_c":
        vals = X @ np.asarray(c)
    elif f_id == "sqnorm":
        vals = np.sum(X * X, axis=1)
    elif f_id == "halfspace_union":
        cx = X @ np.asarray(c)
        vals = ((cx <= b1) | (cx >= b2)).astype(float)
    else:
        raise ValueError(f_id)
    return dict(est=float(vals.mean()), stderr=float(vals.std(ddof=1) / math.sqrt(chains)), calls=st["calls"])


def sdp_anneal(inst, c, kind: int, chains: int, iters: int, walk_len: int = 1, burn: int = 10, T0: float = 0.0,
               L: float = 0.0, rho: int = None, seed: int = 0, f_target: float = None, eps: float = 0.05,
               nthreads: int = 0) -> dict:
    """min c^T x over S (eq:sdp P:1406) by simulated annealing (sec:optimization P:1408-1434):
    uniform start points by the billiard walk from 0 (`burn` steps), T_0 = R = the
    largest |x| among them (S within R B_n) unless given, T_{i+1} = T_i (1 - 1/sqrt(n)),
    `walk_len` steps of `kind` (HMC: Alg. 6 with tau = L, default R; HNR / CHNR: Hit-and-Run with
    the Boltzmann pi_l) per temperature from each chain's previous point; best = the smallest
    c^T x seen.  Stops early once best - f_target <= eps |f_target|.  The cooling
    stops at T_0 2^-20 (R30: the chord ends' accuracy near a face bounds how close to the
    boundary the law can be followed).
    Tags: purpose 4, phase = temperature index + 1 (the start walk: phase 0)."""
    n = inst.n
    c = np.asarray(c, dtype=np.float64)
    rho = 10 * n if rho is None else rho
    lmi = Lmi(inst)
    X, st = walk(lmi, BILLIARD, seed, 0, chains, burn, 2.0 * math.sqrt(n), rho, tag=4 << 28, nthreads=nthreads)
    calls = st["calls"]
    R = float(np.max(np.linalg.norm(X, axis=1)))
    f = X @ c
    best = float(f.min())
    bx = X[int(np.argmin(f))].copy()
    T = T0 if T0 > 0 else R
    T0f = T
    Lh = L if L > 0 else R
    cool = 1.0 - 1.0 / math.sqrt(n)
    hist = []
    it = 0
    while it < iters:
        X, st = walk(lmi, kind, seed, 0, chains, walk_len, Lh, rho, x0=X, T=T, c=c, tag=(4 << 28) | (it + 1),
                     nthreads=nthreads)
        calls += st["calls"]
        f = X @ c
        if f.min() < best:
            best = float(f.min())
            bx = X[int(np.argmin(f))].copy()
        hist.append(best)
        T = max(T * cool, T0f * 2.0 ** -20)  # cooling floor (R30)
        it += 1
        if f_target is not None and best - f_target <= eps * abs(f_target):
            break
    return dict(best=best, best_x=bx, history=hist, iters=it, T0=T0 if T0 > 0 else R, L=Lh, calls=calls,
                last_min=float(f.min()))
