"""Python mirror of the reference ``atfmm`` public API (proj/include/fmm/*.hpp).

Thin ctypes layer over ``libfmm.so`` (C ABI ``include/fmm_host.h``): the C++
host library keeps the pyramid, the connectivity, the engine and the
autotuner; the near field (and optionally M2L) runs on the B200 through
``BackendKind.cuda``.  Names, argument meaning and errors follow the
reference so the parity tests read like its own tests:

=========================  ==========================================
reference (C++)            here
=========================  ==========================================
SourceSet / EvalSet        :class:`SourceSet` / :class:`EvalSet` (complex128)
build_pyramid + _connect.  :class:`Tree` (geometry.hpp:59-74)
NearFieldBackend run       :meth:`Tree.nearfield` (backend.hpp:48-63)
FmmConfig / FmmEngine      :class:`FmmConfig` / :class:`FmmEngine` (engine.hpp:14-118)
Controller::step           :func:`controller_run` (autotune.hpp:73-121)
sims vortex driver         :func:`vortex_run` (sims.hpp:15-36)
exceptions (types.hpp)     :class:`InvalidParameter` ... :class:`BackendError`
=========================  ==========================================
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native

# ------------------------------------------------------------------ errors --


class InvalidParameter(ValueError):
    pass


class InvalidInput(ValueError):
    pass


class SingularConfiguration(RuntimeError):
    pass


class BackendError(RuntimeError):
    pass


class InvalidState(RuntimeError):
    pass


_ERR = {1: InvalidParameter, 2: InvalidInput, 3: SingularConfiguration, 4: BackendError,
        5: InvalidState}

KERNEL = {"harmonic": 0, "logarithmic": 1, "log": 1}
SMOOTHER = {"none": 0, "gaussian": 1, "plummer": 2}
BACKEND = {"serial": 0, "pool": 1, "throttled": 2, "cuda": 3}
PRULE = {"formula": 0, "table": 1}
TUNER = {"none": 0, "at1": 1, "at2": 2, "at3a": 3, "at3b": 4}

_lib = None
_dp = C.POINTER(C.c_double)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def host_lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_native.HOST_LIB):
            raise _native.NativeLibraryMissing(f"{_native.HOST_LIB} not built")
        lib = C.CDLL(_native.HOST_LIB)
        vp = C.c_void_p
        lib.fmmh_last_error.restype = C.c_char_p
        lib.fmmh_last_status.restype = C.c_int
        lib.fmmh_make_distribution.argtypes = [C.c_int, C.c_int64, C.c_uint64, vp, vp]
        lib.fmmh_make_distribution.restype = None
        lib.fmmh_tree_build.argtypes = [vp, vp, C.c_int64, vp, vp, C.c_int64, C.c_int, C.c_double,
                                        C.c_int]
        lib.fmmh_tree_build.restype = vp
        lib.fmmh_tree_free.argtypes = [vp]
        lib.fmmh_tree_free.restype = None
        lib.fmmh_tree_nboxes.argtypes = [vp, C.c_int]
        lib.fmmh_tree_nboxes.restype = C.c_int64
        lib.fmmh_tree_boxes.argtypes = [vp, C.c_int, vp, vp]
        lib.fmmh_tree_boxes.restype = None
        lib.fmmh_tree_perm.argtypes = [vp, vp, vp]
        lib.fmmh_tree_perm.restype = None
        lib.fmmh_tree_nnz.argtypes = [vp, C.c_int, C.c_int]
        lib.fmmh_tree_nnz.restype = C.c_int64
        lib.fmmh_tree_lists.argtypes = [vp, C.c_int, C.c_int, vp, vp]
        lib.fmmh_tree_lists.restype = None
        lib.fmmh_tree_nearfield.argtypes = [vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                            C.c_double, C.c_int, vp, C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_double)]
        lib.fmmh_engine_create.argtypes = [vp, vp, vp, C.c_int]
        lib.fmmh_engine_create.restype = vp
        lib.fmmh_engine_set_config.argtypes = [vp, vp, vp, vp, C.c_int]
        lib.fmmh_engine_evaluate.argtypes = [vp, vp, vp, C.c_int64, vp, vp, C.c_int64, vp, vp, vp,
                                             C.POINTER(C.c_int)]
        lib.fmmh_engine_free.argtypes = [vp]
        lib.fmmh_engine_free.restype = None
        lib.fmmh_controller_run.argtypes = [C.c_int, vp, vp, C.c_double, C.c_int, C.c_uint64,
                                            C.c_int64, vp, vp, vp]
        lib.fmmh_vortex_run.argtypes = [C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64, vp, vp, vp, C.c_int, vp, vp]
        lib.fmmh_m2l_add.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp]
        lib.fmmh_p2m.argtypes = [C.c_int, C.c_int, vp, vp, vp, C.c_int64, vp]
        lib.fmmh_choose_p.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        lib.fmmh_estimate_cost.argtypes = [C.c_double, C.c_int, C.c_double, C.c_int, vp]
        lib.fmmh_p2p_direct.argtypes = [vp, vp, C.c_int64, vp, vp, C.c_int64, C.c_int, C.c_int,
                                        C.c_double, vp]
        _lib = lib
    return _lib


def _raise(rc):
    if rc:
        msg = host_lib().fmmh_last_error().decode()
        raise _ERR.get(rc, RuntimeError)(msg)


def _c2(a) -> np.ndarray:
    """complex array -> contiguous (n, 2) float64 view/copy."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a.view(np.float64).reshape(-1, 2)


# ------------------------------------------------------------ value types --
@dataclass
class SourceSet:
    z: np.ndarray
    m: np.ndarray

    def __post_init__(self):
        self.z = np.ascontiguousarray(self.z, dtype=np.complex128)
        self.m = np.ascontiguousarray(self.m, dtype=np.complex128)

    def size(self):
        return len(self.z)


@dataclass
class EvalSet:
    y: np.ndarray
    source_id: np.ndarray | None = None

    def __post_init__(self):
        self.y = np.ascontiguousarray(self.y, dtype=np.complex128)
        if self.source_id is not None:
            self.source_id = np.ascontiguousarray(self.source_id, dtype=np.int64)

    def size(self):
        return len(self.y)

    @staticmethod
    def self_of(s: SourceSet) -> "EvalSet":
        return EvalSet(s.z.copy(), np.arange(s.size(), dtype=np.int64))

    @staticmethod
    def at(points) -> "EvalSet":
        return EvalSet(np.asarray(points, dtype=np.complex128))


def make_distribution(kind: str | int, n: int, seed: int) -> SourceSet:
    """Reference-generator inputs (tools/atfmm.cpp:70-86, tests/test_util.hpp:10-23)."""
    kinds = {"uniform": 0, "line": 1, "gauss8": 2, "random": 3, "positive": 4}
    k = kinds[kind] if isinstance(kind, str) else int(kind)
    z = np.empty(n, dtype=np.complex128)
    m = np.empty(n, dtype=np.complex128)
    host_lib().fmmh_make_distribution(k, n, seed, _p(z), _p(m))
    return SourceSet(z, m)


# ------------------------------------------------------------------- tree --
class Tree:
    """Pyramid + connectivity built by the host library (bit-exact)."""

    def __init__(self, sources: SourceSet, evals: EvalSet, n_levels: int, theta: float,
                 threads: int = 1):
        lib = host_lib()
        self.sources, self.evals = sources, evals
        ne = evals.size()
        y = evals.y if ne else None
        h = lib.fmmh_tree_build(_p(sources.z), _p(sources.m), sources.size(), _p(y),
                                _p(evals.source_id) if ne else None, ne, n_levels, theta, threads)
        if not h:
            _raise(lib.fmmh_last_status())
        self.h = h
        self.n_levels = n_levels
        self.perm = np.empty(sources.size(), dtype=np.uint32)
        eperm = np.empty(max(ne, 1), dtype=np.uint32)
        lib.fmmh_tree_perm(h, _p(self.perm), _p(eperm))
        self.eval_perm = eperm[:ne]
        self.boxes_f, self.boxes_u, self.strong, self.weak = [], [], [], []
        for lvl in range(n_levels):
            nb = lib.fmmh_tree_nboxes(h, lvl)
            f = np.empty((nb, 5))
            u = np.empty((nb, 4), dtype=np.uint32)
            lib.fmmh_tree_boxes(h, lvl, _p(f), _p(u))
            self.boxes_f.append(f)
            self.boxes_u.append(u)
            for weak, dst in ((0, self.strong), (1, self.weak)):
                nnz = lib.fmmh_tree_nnz(h, lvl, weak)
                off = np.empty(nb + 1, dtype=np.uint32)
                idx = np.empty(max(nnz, 1), dtype=np.uint32)
                lib.fmmh_tree_lists(h, lvl, weak, _p(off), _p(idx))
                dst.append((off, idx[:nnz]))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                host_lib().fmmh_tree_free(self.h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def leaf_csr(self):
        """(pt_off, ev_off, strong_off, strong_idx) of the finest level."""
        u = self.boxes_u[-1]
        pt_off = np.concatenate([u[:, 0], u[-1:, 1]]).astype(np.uint32)
        ev_off = np.concatenate([u[:, 2], u[-1:, 3]]).astype(np.uint32)
        off, idx = self.strong[-1]
        return pt_off, ev_off, off, idx

    def permuted(self):
        """Level-permuted (z, m, y, sid) as (n,2) float arrays (engine.cpp:227-241)."""
        zp = _c2(self.sources.z)[self.perm]
        mp = _c2(self.sources.m)[self.perm]
        yp = _c2(self.evals.y)[self.eval_perm] if self.evals.size() else np.zeros((0, 2))
        sid = None if self.evals.source_id is None else self.evals.source_id[self.eval_perm]
        return zp, mp, yp, sid

    def nearfield(self, backend="serial", *, kernel="harmonic", smoother="none", delta=0.0,
                  threads=1, devices=(0,), exact=False):
        """Run one NearFieldBackend over the finest level.  Returns
        (near potentials in permuted eval order (complex), pair_evals, seconds)."""
        ne = self.evals.size()
        out = np.zeros(max(ne, 1), dtype=np.complex128)
        dev = np.asarray(devices, dtype=np.int32)
        pairs = C.c_uint64()
        secs = C.c_double()
        rc = host_lib().fmmh_tree_nearfield(self.h, BACKEND[backend], _p(dev), len(dev),
                                            int(exact), KERNEL[kernel], SMOOTHER[smoother],
                                            delta, threads, _p(out), C.byref(pairs),
                                            C.byref(secs))
        _raise(rc)
        return out[:ne], int(pairs.value), float(secs.value)


# ------------------------------------------------------------------ engine --
@dataclass
class FmmConfig:
    theta: float = 0.5
    n_levels: int = 4
    tol: float = 1e-6
    kernel: str = "harmonic"
    p_rule: str = "table"
    p_calibration: float = 1.0
    p_override: int = 0
    backend: str = "serial"
    throttle_latency_s: float = 0.002
    throttle_throughput: float = 1.0
    worker_threads: int = 1
    task_split_level: int = 2
    smoother: str = "none"
    delta: float = 0.0
    devices: tuple = (0,)
    exact: bool = False
    m2l_on_device: bool = False
    device_pipeline: bool = False
    device_tree: bool = False

    def pack(self):
        f = np.array([self.theta, self.tol, self.p_calibration, self.delta,
                      self.throttle_latency_s, self.throttle_throughput])
        i = np.array([self.n_levels, KERNEL[self.kernel], PRULE[self.p_rule], self.p_override,
                      BACKEND[self.backend], self.worker_threads, self.task_split_level,
                      SMOOTHER[self.smoother], int(self.exact), int(self.m2l_on_device),
                      int(self.device_pipeline), int(self.device_tree)],
                     dtype=np.int32)
        d = np.asarray(self.devices, dtype=np.int32)
        return f, i, d


TIMING_KEYS = ("t_partition", "t_p2m", "t_upward", "t_m2l", "t_p2p", "t_q", "t_total", "cpu_wait")
COUNTER_KEYS = ("p2p_pairs", "m2l_ops", "p2m_points", "l2p_points")


@dataclass
class EvalResult:
    potentials: np.ndarray
    timings: dict = field(default_factory=dict)
    counters: dict = field(default_factory=dict)
    p: int = 0


class FmmEngine:
    """``fmm::FmmEngine`` (engine.hpp:95-118) behind ``fmmh_engine_*``."""

    def __init__(self, cfg: FmmConfig):
        self.cfg = cfg
        f, i, d = cfg.pack()
        h = host_lib().fmmh_engine_create(_p(f), _p(i), _p(d), len(d))
        if not h:
            _raise(host_lib().fmmh_last_status())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            host_lib().fmmh_engine_free(self.h)
            self.h = None

    def set_config(self, cfg: FmmConfig):
        f, i, d = cfg.pack()
        _raise(host_lib().fmmh_engine_set_config(self.h, _p(f), _p(i), _p(d), len(d)))
        self.cfg = cfg

    def evaluate(self, sources: SourceSet, evals: EvalSet) -> EvalResult:
        ne = evals.size()
        out = np.zeros(max(ne, 1), dtype=np.complex128)
        tim = np.zeros(8)
        cnt = np.zeros(4, dtype=np.uint64)
        p = C.c_int()
        rc = host_lib().fmmh_engine_evaluate(
            self.h, _p(sources.z), _p(sources.m), sources.size(), _p(evals.y) if ne else None,
            _p(evals.source_id) if (ne and evals.source_id is not None) else None, ne, _p(out),
            _p(tim), _p(cnt), C.byref(p))
        _raise(rc)
        return EvalResult(out[:ne], dict(zip(TIMING_KEYS, tim.tolist())),
                          dict(zip(COUNTER_KEYS, [int(c) for c in cnt])), p.value)


# ------------------------------------------------------------ operators ----
def choose_p(rule: str, tol: float, theta: float, calibration: float = 1.0) -> int:
    p = host_lib().fmmh_choose_p(PRULE[rule], tol, theta, calibration)
    if p < 0:
        _raise(-p)
    return p


def estimate_cost(n, n_levels, theta, p):
    out = np.empty(4)
    _raise(host_lib().fmmh_estimate_cost(n, n_levels, theta, p, _p(out)))
    return dict(zip(("c_p2p", "c_m2l", "c_m2m", "c_p2m"), out.tolist()))


def m2l_add(p, kernel, src_center, coeffs, tgt_center, local):
    loc = np.ascontiguousarray(local, dtype=np.complex128).copy()
    sc = np.array([complex(src_center)], dtype=np.complex128)
    tc = np.array([complex(tgt_center)], dtype=np.complex128)
    co = np.ascontiguousarray(coeffs, dtype=np.complex128)
    _raise(host_lib().fmmh_m2l_add(p, KERNEL[kernel], _p(sc), _p(co), _p(tc), _p(loc)))
    return loc


def p2m(center, z, m, kernel, p):
    z = np.ascontiguousarray(z, dtype=np.complex128)
    m = np.ascontiguousarray(m, dtype=np.complex128)
    c = np.array([complex(center)], dtype=np.complex128)
    out = np.empty(p + 1, dtype=np.complex128)
    _raise(host_lib().fmmh_p2m(p, KERNEL[kernel], _p(c), _p(z), _p(m), len(z), _p(out)))
    return out


def p2p_direct(evals: EvalSet, sources: SourceSet, kernel="harmonic", smoother="none", delta=0.0):
    ne = evals.size()
    out = np.zeros(max(ne, 1), dtype=np.complex128)
    _raise(host_lib().fmmh_p2p_direct(
        _p(sources.z), _p(sources.m), sources.size(), _p(evals.y) if ne else None,
        _p(evals.source_id) if evals.source_id is not None and ne else None, ne, KERNEL[kernel],
        SMOOTHER[smoother], delta, _p(out)))
    return out[:ne]


# ------------------------------------------------------------- autotuner ---
@dataclass
class ControllerConfig:
    theta_min: float = 0.25
    theta_max: float = 0.8
    nl_min: int = 1
    nl_max: int = 10
    base_thetastep: float = 0.01
    theta_every: int = 2
    nl_every: int = 10
    filter_window: int = 3
    init_fiblength: int = 3
    max_fiblength: int = 12
    cap: float = 0.1

    def pack(self):
        f = np.array([self.theta_min, self.theta_max, self.base_thetastep, self.cap])
        i = np.array([self.nl_min, self.nl_max, self.theta_every, self.nl_every,
                      self.filter_window, self.init_fiblength, self.max_fiblength], dtype=np.int32)
        return f, i


def controller_run(tuner: str, cc: ControllerConfig, theta0: float, nl0: int, seed: int,
                   measurements: np.ndarray):
    """Feed (time, cpu_wait, has_wait) rows to Controller::step; returns
    (params[n,2] after each step, events[n,3] = proposed, dir, accepted)."""
    meas = np.ascontiguousarray(measurements, dtype=np.float64).reshape(-1, 3)
    n = len(meas)
    out = np.empty((n, 2))
    ev = np.empty((n, 3), dtype=np.int32)
    f, i = cc.pack()
    _raise(host_lib().fmmh_controller_run(TUNER[tuner], _p(f), _p(i), theta0, nl0, seed, n,
                                          _p(meas), _p(out), _p(ev)))
    return out, ev


def vortex_run(n: int, aspect: float, steps: int, cfg: FmmConfig, tuner="none", cap=0.1,
               seed=1, want_positions=False):
    """Vortex-sheet time stepping (config 5) with the observer->controller
    wiring of the reference CLI.  Returns (trace[steps, 8], positions|None)."""
    f, i, d = cfg.pack()
    trace = np.zeros((steps, 8))
    pos = np.empty(n, dtype=np.complex128) if want_positions else None
    _raise(host_lib().fmmh_vortex_run(n, aspect, steps, TUNER[tuner], cap, seed, _p(f), _p(i),
                                      _p(d), len(d), _p(trace), _p(pos)))
    return trace, pos
