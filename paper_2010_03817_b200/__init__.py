"""B200-native batched spectrahedron boundary oracle (arXiv 2010.03817).

Thin ctypes binding over ``libspecwalk.so`` (C-ABI: ``include/specwalk.h``).
Argument marshalling only: every step of the hot path runs in the CUDA
kernels of ``csrc/``.  There is no CPU fallback: if the extension or a CUDA
device is missing, every entry point raises.

Names follow the paper: ``boundary_oracle`` = INTERSECTION +
REFLECTION normal (Alg. 2/3), ``walk_sample`` = Billiard walk (Alg. 5) /
HMC-r (Alg. 6), ``walk_trace`` = the first reflections of given chains.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import _build

_lib = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)

SPEC_OK = 0
ERRORS = {1: "EINVAL", 2: "EPRECOND", 3: "ERUNTIME", 4: "ECUDA", 5: "ENOMEM", 6: "EUNBOUNDED"}
BILLIARD, HMC, HNR, CHNR, CHMC = 0, 1, 2, 3, 4  # Alg. 5, Alg. 6, Alg. 4, W-CHnR,
#                                                collocation HMC-r
POT_LINEAR, POT_GAUSS, POT_LOGCOSH = 0, 1, 2
BIND_DENSE, BIND_BALL, BIND_NONE = 0, -1, -2

# the symbols include/specwalk.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "spec_last_error", "spec_create", "spec_destroy", "spec_set_objective", "spec_set_ball", "boundary_oracle",
    "boundary_oracle_dev", "walk_sample", "walk_sample_dev", "walk_trace", "spec_sync", "spec_stream",
    "spec_kernel_launches", "walk_begin", "walk_rounds", "walk_end", "spec_walk_stats_now", "spec_kernel_timing",
    "spec_kernel_times", "hmc_oracle", "spec_set_comm", "volume", "expectation", "spec_k2_phase_times",
    "spec_lanczos_iterations", "sdp_anneal", "spec_k2_config", "spec_set_potential", "chmc_oracle",
    "spec_chmc_counters",
)
F_LINEAR_C, F_SQNORM, F_HALFSPACE_UNION = 0, 1, 2
MAX_PHASES = 64

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_double))


class Comm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("rank", C.c_int), ("world", C.c_int), ("allgather_f64", ALLGATHER_FN)]


class VolumeOpts(C.Structure):
    _fields_ = [("walk_len", C.c_int64), ("burn", C.c_int64), ("L", C.c_double), ("rho", C.c_int64),
                ("rho_star", C.c_double), ("q_stop", C.c_double), ("max_phases", C.c_int), ("max_growth", C.c_int)]


class VolumeReport(C.Structure):
    _fields_ = [("volume", C.c_double), ("log_volume", C.c_double), ("std_rel", C.c_double), ("q", C.c_double),
                ("phases", C.c_int), ("chains", C.c_int64), ("calls", C.c_int64), ("device_ms", C.c_double),
                ("radii", C.c_double * MAX_PHASES), ("ratios", C.c_double * MAX_PHASES)]


class ExpectParams(C.Structure):
    _fields_ = [("chains", C.c_int64), ("steps", C.c_int64), ("L", C.c_double), ("rho", C.c_int64),
                ("b1", C.c_double), ("b2", C.c_double)]


class SdpParams(C.Structure):
    _fields_ = [("kind", C.c_int), ("chains", C.c_int64), ("iters", C.c_int64), ("walk_len", C.c_int64),
                ("burn", C.c_int64), ("T0", C.c_double), ("L", C.c_double), ("rho", C.c_int64), ("seed", C.c_uint64),
                ("f_target", C.c_double), ("eps", C.c_double)]


class SdpReport(C.Structure):
    _fields_ = [("best", C.c_double), ("last_min", C.c_double), ("T0", C.c_double), ("T_final", C.c_double),
                ("L", C.c_double), ("iters", C.c_int64), ("calls", C.c_int64), ("device_ms", C.c_double)]


class SpecError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class WalkParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("chain_begin", C.c_int64), ("chains", C.c_int64), ("steps", C.c_int64),
        ("L", C.c_double), ("rho", C.c_int64), ("seed", C.c_uint64), ("tag", C.c_uint32), ("T", C.c_double),
        ("q", C.c_int), ("h", C.c_double),
    ]


class WalkStats(C.Structure):
    _fields_ = [
        ("calls", C.c_int64), ("reflections", C.c_int64), ("rejects", C.c_int64), ("degenerates", C.c_int64),
        ("failures", C.c_int64), ("steps", C.c_int64), ("rounds", C.c_int64), ("device_ms", C.c_double),
        ("capped", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libspecwalk.so (building it with nvcc if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    alt = os.environ.get("SPECWALK_LIB")  # A/B measurements: an alternative in-tree build of the same ABI
    if alt:
        l = C.CDLL(alt)
    else:
        if build_if_missing and _build.needs_build():
            _build.build()
        if not os.path.exists(_build.LIB):
            raise ImportError(f"libspecwalk.so not built at {_build.LIB}")
        l = C.CDLL(_build.LIB)
    l.spec_last_error.restype = C.c_char_p
    l.spec_create.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int, C.POINTER(C.c_void_p)]
    l.spec_destroy.argtypes = [C.c_void_p]
    l.spec_set_objective.argtypes = [C.c_void_p, _dp]
    l.spec_set_ball.argtypes = [C.c_void_p, _dp, C.c_double]
    l.boundary_oracle.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
    l.boundary_oracle_dev.argtypes = [C.c_void_p, C.c_int64] + [C.c_void_p] * 8
    l.walk_sample.argtypes = [C.c_void_p, C.POINTER(WalkParams), _dp, C.c_int, _dp, _dp, _dp, C.POINTER(WalkStats)]
    l.walk_sample_dev.argtypes = [C.c_void_p, C.POINTER(WalkParams), C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.POINTER(WalkStats)]
    l.walk_trace.argtypes = [C.c_void_p, C.POINTER(WalkParams), _lp, C.c_int64, C.c_int64, _dp, _dp, _dp, _dp, _ip,
                             _lp]
    l.spec_sync.argtypes = [C.c_void_p]
    l.spec_stream.argtypes = [C.c_void_p]
    l.spec_stream.restype = C.c_void_p
    l.spec_kernel_launches.argtypes = [C.c_void_p]
    l.spec_kernel_launches.restype = C.c_int64
    l.walk_begin.argtypes = [C.c_void_p, C.POINTER(WalkParams), C.c_void_p, C.c_int]
    l.walk_rounds.argtypes = [C.c_void_p, C.c_int64, _lp]
    l.walk_end.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(WalkStats)]
    l.spec_walk_stats_now.argtypes = [C.c_void_p, C.POINTER(WalkStats)]
    l.spec_kernel_timing.argtypes = [C.c_void_p, C.c_int]
    l.spec_kernel_times.argtypes = [C.c_void_p, _dp, _lp, _lp]
    l.spec_k2_phase_times.argtypes = [C.c_void_p, _dp]
    l.spec_lanczos_iterations.argtypes = [C.c_void_p, C.c_int, _dp, _lp]
    l.spec_k2_config.argtypes = [C.c_void_p]
    l.spec_k2_config.restype = C.c_char_p
    l.sdp_anneal.argtypes = [C.c_void_p, C.POINTER(SdpParams), _dp, _dp, C.POINTER(SdpReport)]
    l.hmc_oracle.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp, _ip]
    l.chmc_oracle.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, C.c_int, C.c_double, _dp, _dp, _dp, _ip]
    l.spec_set_potential.argtypes = [C.c_void_p, C.c_int, _dp, C.c_double]
    l.spec_chmc_counters.argtypes = [C.c_void_p, C.c_int, _lp]
    l.spec_set_comm.argtypes = [C.c_void_p, C.POINTER(Comm)]
    l.volume.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_int64, C.POINTER(VolumeOpts),
                         C.POINTER(VolumeReport)]
    l.expectation.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.POINTER(ExpectParams), _dp, _dp]
    _lib = l
    return l


def _check(rc: int):
    if rc != SPEC_OK:
        raise SpecError(rc, _lib.spec_last_error().decode())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


class Spectrahedron:
    """A spectrahedron S = {x : A0 + sum x_i A_i >= 0} (eq:lmi P:70-75), with an
    optional cube block lo <= x <= hi, resident on one GPU."""

    def __init__(self, A, lo=None, hi=None, device: int = -1):
        l = load()
        A = _f64(A)
        if A.ndim != 3 or A.shape[1] != A.shape[2]:
            raise ValueError("A must have shape (n+1, m, m)")
        self.n, self.m = A.shape[0] - 1, A.shape[1]
        self._lo = _f64(lo) if lo is not None else None
        self._hi = _f64(hi) if hi is not None else None
        h = C.c_void_p()
        _check(l.spec_create(self.n, self.m, _p(A), _p(self._lo), _p(self._hi), device, C.byref(h)))
        self._h = h

    @classmethod
    def from_instance(cls, inst, device: int = -1):
        return cls(inst.A, inst.lo, inst.hi, device)

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.spec_destroy(self._h)
            self._h = None

    __del__ = close

    def set_objective(self, c):
        _check(_lib.spec_set_objective(self._h, _p(_f64(c))))

    def set_potential(self, pot: int, mu=None, scale: float = 1.0):
        """Potential f of exp(-f) for collocation HMC-r (POT_LINEAR: c^T x / scale with the
        objective; POT_GAUSS: |x - mu|^2 / 2 scale^2; POT_LOGCOSH: sum log cosh((x - mu) / scale))."""
        _check(_lib.spec_set_potential(self._h, int(pot), _p(_f64(mu)) if mu is not None else None, float(scale)))

    def set_ball(self, center, radius: float):
        _check(_lib.spec_set_ball(self._h, _p(_f64(center)) if center is not None else None, float(radius)))

    def set_comm(self, allgather, rank: int, world: int):
        """Multi-rank reductions: allgather(local: np.ndarray) -> np.ndarray (rank order).
        None removes it (single rank)."""
        if allgather is None:
            self._comm_keep = None
            _check(_lib.spec_set_comm(self._h, None))
            return

        def cb(user, inp, n_local, out):
            try:
                loc = np.ctypeslib.as_array(inp, shape=(n_local,)).copy()
                glob = np.asarray(allgather(loc), dtype=np.float64).reshape(-1)
                np.ctypeslib.as_array(out, shape=(n_local * world,))[:] = glob
                return 0
            except Exception:  # pragma: no cover - surfaced as ECUDA by the library
                return 1

        fn = ALLGATHER_FN(cb)
        comm = Comm(None, rank, world, fn)
        self._comm_keep = (fn, comm)
        _check(_lib.spec_set_comm(self._h, C.byref(comm)))

    def volume(self, eps: float, seed: int, chains_per_phase: int, walk_len: int = 0, burn: int = 0,
               L: float = 0.0, rho: int = 0, rho_star: float = 0.0, q_stop: float = 0.0, max_phases: int = 0,
               max_growth: int = 0) -> dict:
        """Ball-phase MMC volume (eq:mmc_vol P:1291-1300)."""
        o = VolumeOpts(walk_len, burn, float(L), rho, float(rho_star), float(q_stop), max_phases, max_growth)
        r = VolumeReport()
        _check(_lib.volume(self._h, float(eps), seed, chains_per_phase, C.byref(o), C.byref(r)))
        k = r.phases
        return dict(volume=r.volume, log_volume=r.log_volume, std_rel=r.std_rel, q=r.q, phases=k, chains=r.chains,
                    calls=r.calls, device_ms=r.device_ms, radii=list(r.radii[:k]), ratios=list(r.ratios[:k]))

    def expectation(self, f_id: int, T: float, seed: int, chains: int, steps: int, L: float, rho: int,
                    b1: float = 0.0, b2: float = 0.0) -> dict:
        """E[f] over chain end points; T <= 0 or inf: uniform (billiard)."""
        p = ExpectParams(chains, steps, float(L), rho, float(b1), float(b2))
        est, se = C.c_double(), C.c_double()
        _check(_lib.expectation(self._h, f_id, float(T), seed, C.byref(p), C.byref(est), C.byref(se)))
        return dict(est=est.value, stderr=se.value)

    def sdp_anneal(self, kind: int, chains: int, iters: int, seed: int = 0, walk_len: int = 0, burn: int = 0,
                   T0: float = 0.0, L: float = 0.0, rho: int = 0, f_target: Optional[float] = None,
                   eps: float = 0.0) -> dict:
        """min c^T x over S by simulated annealing (eq:sdp P:1406, sec:optimization P:1408-1434)."""
        p = SdpParams(kind, chains, iters, walk_len, burn, float(T0), float(L), rho, seed,
                      float("nan") if f_target is None else float(f_target), float(eps))
        bx = np.empty(self.n)
        hist = np.full(iters, np.nan)
        r = SdpReport()
        _check(_lib.sdp_anneal(self._h, C.byref(p), _p(bx), _p(hist), C.byref(r)))
        return dict(best=r.best, best_x=bx, history=hist[: r.iters], iters=r.iters, T0=r.T0, T_final=r.T_final,
                    L=r.L, calls=r.calls, device_ms=r.device_ms, last_min=r.last_min)

    def k2_config(self) -> str:
        return _lib.spec_k2_config(self._h).decode()

    def kernel_launches(self) -> int:
        return int(_lib.spec_kernel_launches(self._h))

    def stream(self) -> int:
        return int(_lib.spec_stream(self._h) or 0)

    def sync(self):
        _check(_lib.spec_sync(self._h))

    # -------------------------------------------------------------- oracle
    def boundary_oracle(self, x, v, u=None, want_kernel: bool = False) -> dict:
        x, v = _f64(x), _f64(v)
        if x.ndim == 1:
            x, v = x[None], v[None]
        B = x.shape[0]
        ua = _f64(u).reshape(B, self.m) if u is not None else None
        tm, tp = np.empty(B), np.empty(B)
        nrm = np.empty((B, self.n))
        ker = np.empty((B, self.m)) if want_kernel else None
        bind = np.empty(B, dtype=np.int32)
        _check(_lib.boundary_oracle(self._h, B, _p(x), _p(v), _p(ua), _p(tm), _p(tp), _p(nrm), _p(ker),
                                    bind.ctypes.data_as(_ip)))
        out = dict(t_minus=tm, t_plus=tp, normal=nrm, binding=bind)
        if want_kernel:
            out["kernel"] = ker
        return out

    def hmc_oracle(self, x, v, T: float, u=None, want_kernel: bool = False) -> dict:
        """Reflective-HMC chord on x + v t - c t^2 / (2T) (Alg. 6, eq:boltz_ode)."""
        x, v = _f64(x), _f64(v)
        if x.ndim == 1:
            x, v = x[None], v[None]
        B = x.shape[0]
        ua = _f64(u).reshape(B, self.m) if u is not None else None
        tp = np.empty(B)
        nrm = np.empty((B, self.n))
        ker = np.empty((B, self.m)) if want_kernel else None
        bind = np.empty(B, dtype=np.int32)
        _check(_lib.hmc_oracle(self._h, B, _p(x), _p(v), _p(ua), float(T), _p(tp), _p(nrm), _p(ker),
                               bind.ctypes.data_as(_ip)))
        out = dict(t_plus=tp, normal=nrm, binding=bind)
        if want_kernel:
            out["kernel"] = ker
        return out

    def chmc_oracle(self, x, v, q: int, h: float, u=None, want_kernel: bool = False) -> dict:
        """One collocation-HMC segment per line: first boundary hit in (0, h] (+inf: none)."""
        x, v = _f64(x), _f64(v)
        if x.ndim == 1:
            x, v = x[None], v[None]
        B = x.shape[0]
        ua = _f64(u).reshape(B, self.m) if u is not None else None
        tp = np.empty(B)
        nrm = np.empty((B, self.n))
        ker = np.empty((B, self.m)) if want_kernel else None
        bind = np.empty(B, dtype=np.int32)
        _check(_lib.chmc_oracle(self._h, B, _p(x), _p(v), _p(ua), int(q), float(h), _p(tp), _p(nrm), _p(ker),
                                bind.ctypes.data_as(_ip)))
        out = dict(t_plus=tp, normal=nrm, binding=bind)
        if want_kernel:
            out["kernel"] = ker
        return out

    def boundary_oracle_dev(self, x, v, u, t_minus, t_plus, normal, kernel, binding):
        """Device-pointer variant: arguments are torch CUDA tensors (or None for u / kernel)."""
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        _check(_lib.boundary_oracle_dev(self._h, x.shape[0], ptr(x), ptr(v), ptr(u), ptr(t_minus), ptr(t_plus),
                                        ptr(normal), ptr(kernel), ptr(binding)))

    # -------------------------------------------------------------- walks
    @staticmethod
    def _params(kind, chains, steps, L, rho, seed, chain_begin=0, tag=0, T=None, q=3, h=0.0) -> WalkParams:
        if T is None:  # HMC: T = 1; Hit-and-Run: the uniform law (T = inf); ignored by the billiard
            T = 1.0 if kind == HMC else float("inf")
        p = WalkParams()
        p.kind, p.chain_begin, p.chains, p.steps = kind, chain_begin, chains, steps
        p.L, p.rho, p.seed, p.tag, p.T = float(L), rho, seed, tag, float(T)
        p.q, p.h = int(q), float(h)
        return p

    def walk_sample(self, chains: int, steps: int, L: float, rho: int, seed: int, kind: int = BILLIARD,
                    x0=None, chain_begin: int = 0, tag: int = 0, T: Optional[float] = None, final: bool = True,
                    q: int = 3, h: float = 0.0) -> dict:
        p = self._params(kind, chains, steps, L, rho, seed, chain_begin, tag, T, q, h)
        per_chain = 0
        x0a = None
        if x0 is not None:
            x0a = _f64(x0)
            per_chain = 1 if x0a.ndim == 2 else 0
        sx = np.empty(self.n)
        sxx = np.empty(self.n * (self.n + 1) // 2)
        fx = np.empty((chains, self.n)) if final else None
        st = WalkStats()
        _check(_lib.walk_sample(self._h, C.byref(p), _p(x0a), per_chain, _p(sx), _p(sxx), _p(fx), C.byref(st)))
        return dict(sum_x=sx, sum_xx=sxx, final_x=fx, stats=st.as_dict())

    def walk_sample_dev(self, chains: int, steps: int, L: float, rho: int, seed: int, kind: int = BILLIARD,
                        x0=None, sum_x=None, sum_xx=None, final_x=None, chain_begin: int = 0, tag: int = 0,
                        T: Optional[float] = None, q: int = 3, h: float = 0.0) -> dict:
        p = self._params(kind, chains, steps, L, rho, seed, chain_begin, tag, T, q, h)
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        per_chain = 1 if (x0 is not None and x0.dim() == 2) else 0
        st = WalkStats()
        _check(_lib.walk_sample_dev(self._h, C.byref(p), ptr(x0), per_chain, ptr(sum_x), ptr(sum_xx),
                                    ptr(final_x), C.byref(st)))
        return st.as_dict()

    # resumable walk: begin / rounds / end (device buffers are torch CUDA tensors)
    def walk_begin(self, chains: int, steps: int, L: float, rho: int, seed: int, kind: int = BILLIARD, x0=None,
                   chain_begin: int = 0, tag: int = 0, T: Optional[float] = None, q: int = 3, h: float = 0.0):
        p = self._params(kind, chains, steps, L, rho, seed, chain_begin, tag, T, q, h)
        ptr = None if x0 is None else C.c_void_p(x0.data_ptr())
        per_chain = 1 if (x0 is not None and x0.dim() == 2) else 0
        _check(_lib.walk_begin(self._h, C.byref(p), ptr, per_chain))

    def walk_rounds(self, max_rounds: int) -> int:
        active = C.c_int64()
        _check(_lib.walk_rounds(self._h, max_rounds, C.byref(active)))
        return active.value

    def walk_end(self, sum_x=None, sum_xx=None, final_x=None) -> dict:
        ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        st = WalkStats()
        _check(_lib.walk_end(self._h, ptr(sum_x), ptr(sum_xx), ptr(final_x), C.byref(st)))
        return st.as_dict()

    def walk_stats_now(self) -> dict:
        st = WalkStats()
        _check(_lib.spec_walk_stats_now(self._h, C.byref(st)))
        return st.as_dict()

    def kernel_timing(self, enable: bool):
        _check(_lib.spec_kernel_timing(self._h, 1 if enable else 0))

    def kernel_times(self) -> dict:
        ms = (C.c_double * 4)()
        cnt = (C.c_int64 * 4)()
        items = C.c_int64()
        _check(_lib.spec_kernel_times(self._h, ms, cnt, C.byref(items)))
        names = ("K1_av_gemm", "K2_chord", "K3_normal_gemm", "K4_reflect")
        k2 = (C.c_double * 3)()
        _check(_lib.spec_k2_phase_times(self._h, k2))
        return dict(ms={k: ms[i] for i, k in enumerate(names)}, launches={k: cnt[i] for i, k in enumerate(names)},
                    k2_items=items.value,
                    k2_phases_ms=dict(K2a_factor=k2[0], K2b_lanczos=k2[1], K2c_tail=k2[2]))

    def chmc_counters(self, reset: bool = True) -> dict:
        """Collocation HMC-r device counters since the last reset."""
        out = np.zeros(4, dtype=np.int64)
        _check(_lib.spec_chmc_counters(self._h, 1 if reset else 0, out.ctypes.data_as(_lp)))
        return dict(picard=int(out[0]), segments=int(out[1]), unconverged=int(out[2]), congruences=int(out[3]))

    def lanczos_iterations(self, reset: bool = True) -> dict:
        """Device-counted Lanczos iterations per extreme-eigenvalue solve since the last reset."""
        mj, ns = C.c_double(), C.c_int64()
        _check(_lib.spec_lanczos_iterations(self._h, 1 if reset else 0, C.byref(mj), C.byref(ns)))
        return dict(mean_j=mj.value, solves=ns.value)

    def walk_trace(self, chain_ids, steps: int, L: float, rho: int, seed: int, max_refl: int,
                   kind: int = BILLIARD, T: Optional[float] = None, q: int = 3, h: float = 0.0) -> list:
        """First max_refl reflections of the given global chain ids (parity entry)."""
        ids = np.ascontiguousarray(np.asarray(chain_ids, dtype=np.int64))
        k = len(ids)
        p = self._params(kind, k, steps, L, rho, seed, 0, 0, T, q, h)
        n = self.n
        hit = np.zeros((k, max_refl, n))
        t = np.zeros((k, max_refl))
        w = np.zeros((k, max_refl, n))
        va = np.zeros((k, max_refl, n))
        bind = np.zeros((k, max_refl), dtype=np.int32)
        nrec = np.zeros(k, dtype=np.int64)
        _check(_lib.walk_trace(self._h, C.byref(p), ids.ctypes.data_as(_lp), k, max_refl, _p(hit), _p(t), _p(w),
                               _p(va), bind.ctypes.data_as(_ip), nrec.ctypes.data_as(_lp)))
        return [dict(hit_x=hit[i, : nrec[i]], t=t[i, : nrec[i]], w=w[i, : nrec[i]], v_after=va[i, : nrec[i]],
                     binding=bind[i, : nrec[i]]) for i in range(k)]
