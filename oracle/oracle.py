"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

Two libraries live under ``oracle/`` (built by ``make -C oracle``):

* ``liboracle.so``      — plain-C restatement (``fmm_oracle.c``) of the
  reference's near-field arithmetic (backend.cpp:41-89, expansion.cpp:78-92,
  188-269) and of libgcc's ``__divdc3``.  Always available (own sources).
* ``_ref/libfmmref.so`` — the unmodified reference library compiled from
  ``/root/reference/proj/src`` plus ``ref_shim.cpp``.  Built in the dev
  container (where ``/root/reference`` exists) and shipped as a binary to the
  GPU box; callers must tolerate its absence.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC = None
_REF = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def _nullable(ptr_t):
    """ndpointer that also accepts None."""

    def from_param(cls, obj):
        if obj is None:
            return None
        return ptr_t.from_param(obj)

    return type(ptr_t.__name__ + "_or_null", (ptr_t,), {"from_param": classmethod(from_param)})


_i64p_n = _nullable(_i64p)
_dp_n = _nullable(_dp)


def oracle_lib():
    global _ORC
    if _ORC is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        lib.orc_cdiv_batch.argtypes = [C.c_int64, _dp, _dp, C.c_int]
        lib.orc_kernel_term.argtypes = [C.c_int, _dp, _dp, _dp, _dp]
        lib.orc_smoother.argtypes = [C.c_int, C.c_double, C.c_double]
        lib.orc_smoother.restype = C.c_double
        lib.orc_nearfield.argtypes = [C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p, _dp, _dp, _dp,
                                      _i64p_n, C.c_int, C.c_int, C.c_double, C.c_uint32,
                                      C.c_uint32, _dp]
        lib.orc_nearfield.restype = C.c_uint64
        lib.orc_m2l_add.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        lib.orc_m2l_add.restype = C.c_int
        lib.orc_binomial.argtypes = [C.c_int, C.c_int]
        lib.orc_binomial.restype = C.c_double
        lib.orc_hypot.argtypes = [C.c_double, C.c_double]
        lib.orc_hypot.restype = C.c_double
        lib.orc_hypot_check.argtypes = [C.c_int64, _dp, _dp_n]
        lib.orc_hypot_check.restype = C.c_int64
        _ORC = lib
    return _ORC


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libfmmref.so"))


def ref_lib():
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libfmmref.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (reference not built here)")
        lib = C.CDLL(path)
        lib.fmmref_last_error.restype = C.c_char_p
        lib.fmmref_make_distribution.argtypes = [C.c_int, C.c_int64, C.c_uint64, _dp, _dp]
        lib.fmmref_tree_build.argtypes = [_dp, _dp, C.c_int64, _dp_n, _i64p_n, C.c_int64, C.c_int,
                                          C.c_double, C.c_int]
        lib.fmmref_tree_build.restype = C.c_void_p
        lib.fmmref_tree_free.argtypes = [C.c_void_p]
        lib.fmmref_tree_nboxes.argtypes = [C.c_void_p, C.c_int]
        lib.fmmref_tree_nboxes.restype = C.c_int64
        lib.fmmref_tree_boxes.argtypes = [C.c_void_p, C.c_int, _dp, _u32p]
        lib.fmmref_tree_perm.argtypes = [C.c_void_p, _u32p, _u32p]
        lib.fmmref_tree_nnz.argtypes = [C.c_void_p, C.c_int, C.c_int]
        lib.fmmref_tree_nnz.restype = C.c_int64
        lib.fmmref_tree_lists.argtypes = [C.c_void_p, C.c_int, C.c_int, _u32p, _u32p]
        lib.fmmref_tree_nearfield.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int,
                                              C.c_int, C.c_int64, C.c_int64, _dp_n,
                                              C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.fmmref_nf_create.argtypes = [C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p,
                                         C.c_uint32, C.c_uint32, _dp, _dp, _dp_n, _i64p_n]
        lib.fmmref_nf_create.restype = C.c_void_p
        lib.fmmref_nf_free.argtypes = [C.c_void_p]
        lib.fmmref_nf_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                      C.c_int64, C.c_int64, _dp_n, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_double)]
        lib.fmmref_evaluate.argtypes = [_dp, _dp, C.c_int64, _dp_n, _i64p_n, C.c_int64, _dp, _ip,
                                        _dp_n, _dp, _u64p, C.POINTER(C.c_int)]
        lib.fmmref_m2l_add.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
        lib.fmmref_p2m.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.c_int64, _dp]
        lib.fmmref_kernel_term_batch.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp, _dp]
        lib.fmmref_smoother_factor.argtypes = [C.c_int, C.c_double, C.c_double]
        lib.fmmref_smoother_factor.restype = C.c_double
        lib.fmmref_choose_p.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double]
        lib.fmmref_estimate_cost.argtypes = [C.c_double, C.c_int, C.c_double, C.c_int, _dp]
        lib.fmmref_controller_run.argtypes = [C.c_int, _dp, _ip, C.c_double, C.c_int, C.c_uint64,
                                              C.c_int64, _dp, _dp, _ip]
        _REF = lib
    return _REF


# --------------------------------------------------------------- restatement
def hypot_check(xy: np.ndarray):
    """(mismatches vs libm hypot/cabs, restated glibc hypot values) for pairs xy[n, 2]."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    out = np.empty(len(xy))
    bad = oracle_lib().orc_hypot_check(len(xy), xy, out)
    return int(bad), out


def cdiv(q: np.ndarray, native: bool = False) -> np.ndarray:
    """q: (n, 4) [a, b, c, d] -> (n, 2) of (a+ib)/(c+id) via restated __divdc3."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.empty((q.shape[0], 2))
    oracle_lib().orc_cdiv_batch(q.shape[0], q.ravel(), out.ravel(), int(native))
    return out


def nearfield(csr: "LeafCSR", zp, mp, yp, sidp, kernel=0, smoother=0, delta=0.0,
              leaf_begin=0, leaf_end=None):
    """Restated near_box over CSR leaves.  Returns (out[n_eval,2] permuted, pairs)."""
    n_leaves = len(csr.pt_off) - 1
    if leaf_end is None:
        leaf_end = n_leaves
    zp = np.ascontiguousarray(zp, dtype=np.float64).reshape(-1)
    mp = np.ascontiguousarray(mp, dtype=np.float64).reshape(-1)
    yp = np.ascontiguousarray(yp, dtype=np.float64).reshape(-1)
    out = np.zeros(yp.size, dtype=np.float64)
    sid = None if sidp is None else np.ascontiguousarray(sidp, dtype=np.int64)
    pairs = oracle_lib().orc_nearfield(n_leaves, csr.pt_off, csr.ev_off, csr.s_off, csr.s_idx,
                                       csr.perm, zp, mp, yp if yp.size else np.zeros(2), sid,
                                       kernel, smoother, delta, leaf_begin, leaf_end,
                                       out if out.size else np.zeros(2))
    return out.reshape(-1, 2), int(pairs)


def m2l_add(p, kernel, src_center, coeffs, tgt_center, local):
    local = np.ascontiguousarray(local, dtype=np.float64).copy()
    rc = oracle_lib().orc_m2l_add(p, kernel, np.ascontiguousarray(src_center, dtype=np.float64),
                                  np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1),
                                  np.ascontiguousarray(tgt_center, dtype=np.float64),
                                  local.reshape(-1))
    if rc == 3:
        raise ZeroDivisionError("m2l: target center coincides with source center")
    return local


@dataclass
class LeafCSR:
    pt_off: np.ndarray
    ev_off: np.ndarray
    s_off: np.ndarray
    s_idx: np.ndarray
    perm: np.ndarray


# ----------------------------------------------------------- compiled reference
def make_distribution(kind: int, n: int, seed: int):
    z = np.empty((n, 2))
    m = np.empty((n, 2))
    ref_lib().fmmref_make_distribution(kind, n, seed, z.ravel(), m.ravel())
    return z, m


@dataclass
class RefTree:
    """Pyramid + connectivity built by the compiled reference."""

    n_levels: int
    perm: np.ndarray
    eval_perm: np.ndarray
    boxes_f: list = field(default_factory=list)   # per level (nb, 5)
    boxes_u: list = field(default_factory=list)   # per level (nb, 4)
    strong: list = field(default_factory=list)    # per level (off, idx)
    weak: list = field(default_factory=list)
    handle: int | None = None

    def leaf_csr(self) -> LeafCSR:
        u = self.boxes_u[-1]
        pt_off = np.concatenate([u[:, 0], u[-1:, 1]]).astype(np.uint32)
        ev_off = np.concatenate([u[:, 2], u[-1:, 3]]).astype(np.uint32)
        off, idx = self.strong[-1]
        return LeafCSR(pt_off, ev_off, off, idx, self.perm)

    def free(self):
        if self.handle:
            ref_lib().fmmref_tree_free(self.handle)
            self.handle = None


def ref_tree(z, m, y, sid, n_levels, theta, threads=1, keep=False) -> RefTree:
    lib = ref_lib()
    z = np.ascontiguousarray(z, dtype=np.float64)
    m = np.ascontiguousarray(m, dtype=np.float64)
    ne = 0 if y is None else len(y)
    yv = None if y is None or ne == 0 else np.ascontiguousarray(y, dtype=np.float64).ravel()
    sv = None if sid is None else np.ascontiguousarray(sid, dtype=np.int64)
    h = lib.fmmref_tree_build(z.ravel(), m.ravel(), len(z), yv, sv, ne, n_levels, theta, threads)
    if not h:
        raise RuntimeError(lib.fmmref_last_error().decode())
    perm = np.empty(len(z), dtype=np.uint32)
    eperm = np.empty(max(ne, 1), dtype=np.uint32)
    lib.fmmref_tree_perm(h, perm, eperm)
    t = RefTree(n_levels, perm, eperm[:ne])
    for lvl in range(n_levels):
        nb = lib.fmmref_tree_nboxes(h, lvl)
        f = np.empty((nb, 5))
        u = np.empty((nb, 4), dtype=np.uint32)
        lib.fmmref_tree_boxes(h, lvl, f.ravel(), u.ravel())
        t.boxes_f.append(f)
        t.boxes_u.append(u)
        for weak, dst in ((0, t.strong), (1, t.weak)):
            nnz = lib.fmmref_tree_nnz(h, lvl, weak)
            off = np.empty(nb + 1, dtype=np.uint32)
            idx = np.empty(max(nnz, 1), dtype=np.uint32)
            lib.fmmref_tree_lists(h, lvl, weak, off, idx)
            dst.append((off, idx[:nnz]))
    if keep:
        t.handle = h
    else:
        lib.fmmref_tree_free(h)
    return t


def ref_nearfield(tree: RefTree, kernel=0, smoother=0, delta=0.0, parallel=False, threads=1,
                  leaf_begin=0, leaf_end=None, want_out=True):
    """Reference nearfield_run on a kept tree.  Returns (out permuted, pairs, seconds)."""
    assert tree.handle, "build the tree with keep=True"
    nleaf = len(tree.boxes_u[-1])
    if leaf_end is None:
        leaf_end = nleaf
    ne = len(tree.eval_perm)
    out = np.empty(max(ne, 1) * 2) if want_out else None
    pairs = C.c_uint64()
    secs = C.c_double()
    rc = ref_lib().fmmref_tree_nearfield(tree.handle, kernel, smoother, delta, int(parallel),
                                         threads, leaf_begin, leaf_end, out, C.byref(pairs),
                                         C.byref(secs))
    if rc:
        raise RuntimeError(ref_lib().fmmref_last_error().decode())
    return (None if out is None else out[: 2 * ne].reshape(-1, 2)), int(pairs.value), secs.value


class RefNearField:
    """The reference's own nearfield_run over CSR leaves (ref_shim.cpp
    fmmref_nf_*): the CPU baseline timed beside the device path."""

    def __init__(self, csr: LeafCSR, zp, mp, yp, sidp):
        self._keep = [np.ascontiguousarray(a) for a in (csr.pt_off, csr.ev_off, csr.s_off,
                                                        csr.s_idx, csr.perm)]
        zp = np.ascontiguousarray(zp, dtype=np.float64).reshape(-1)
        mp = np.ascontiguousarray(mp, dtype=np.float64).reshape(-1)
        yp = np.ascontiguousarray(yp, dtype=np.float64).reshape(-1)
        sid = None if sidp is None else np.ascontiguousarray(sidp, dtype=np.int64)
        self.n_eval = yp.size // 2
        self.h = ref_lib().fmmref_nf_create(len(csr.pt_off) - 1, *self._keep, zp.size // 2,
                                            self.n_eval, zp, mp, yp if yp.size else None, sid)

    def run(self, leaf_begin, leaf_end, *, kernel=0, smoother=0, delta=0.0, parallel=True,
            threads=1, want_out=False):
        out = np.empty(max(self.n_eval, 1) * 2) if want_out else None
        pairs = C.c_uint64()
        secs = C.c_double()
        rc = ref_lib().fmmref_nf_run(self.h, kernel, smoother, delta, int(parallel), threads,
                                     leaf_begin, leaf_end, out, C.byref(pairs), C.byref(secs))
        if rc:
            raise RuntimeError(ref_lib().fmmref_last_error().decode())
        return (None if out is None else out[: 2 * self.n_eval].reshape(-1, 2),
                int(pairs.value), secs.value)

    def close(self):
        if self.h:
            ref_lib().fmmref_nf_free(self.h)
            self.h = None


def ref_evaluate(z, m, y, sid, *, theta=0.5, tol=1e-6, n_levels=4, kernel=0, p_rule=1,
                 p_override=0, backend=0, threads=1, split=2, smoother=0, delta=0.0,
                 calibration=1.0):
    lib = ref_lib()
    z = np.ascontiguousarray(z, dtype=np.float64)
    m = np.ascontiguousarray(m, dtype=np.float64)
    ne = 0 if y is None else len(y)
    yv = None if ne == 0 else np.ascontiguousarray(y, dtype=np.float64).ravel()
    sv = None if sid is None else np.ascontiguousarray(sid, dtype=np.int64)
    cf = np.array([theta, tol, calibration, delta])
    ci = np.array([n_levels, kernel, p_rule, p_override, backend, threads, split, smoother],
                  dtype=np.int32)
    out = np.empty(max(ne, 1) * 2)
    tim = np.empty(8)
    cnt = np.empty(4, dtype=np.uint64)
    p = C.c_int()
    rc = lib.fmmref_evaluate(z.ravel(), m.ravel(), len(z), yv, sv, ne, cf, ci, out, tim, cnt,
                             C.byref(p))
    if rc:
        raise RuntimeError(f"rc={rc}: " + lib.fmmref_last_error().decode())
    return out[: 2 * ne].reshape(-1, 2), tim, cnt, p.value
