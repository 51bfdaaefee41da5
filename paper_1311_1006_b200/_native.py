"""ctypes bindings of the in-tree native libraries.

* ``libfmmcuda.so`` — the B200 near field behind the C ABI of
  ``include/fmm_cuda.h`` (``fmmcu_*``).
* ``libfmm.so``     — the C++ host library (``include/fmm/*.hpp``) and its
  flat C ABI for Python (``include/fmm_host.h``, ``fmmh_*``).

Both are built in-tree by ``__graft_entry__.build()`` (``make -C
paper_1311_1006_b200``).  Loading fails loudly if they are missing: there is
no CPU or PyTorch fallback for the device path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
CUDA_LIB = os.path.join(PKG, "libfmmcuda.so")
HOST_LIB = os.path.join(PKG, "libfmm.so")

FMMCU_OK = 0
FMMCU_EINVAL = 1
FMMCU_ECUDA = 2
FMMCU_ESINGULAR = 4
FMMCU_ENOMEM = 5
FMMCU_ESTATE = 6

KERNELS = {"harmonic": 0, "logarithmic": 1, "log": 1}
SMOOTHERS = {"none": 0, "gaussian": 1, "plummer": 2}
MODES = {"fast": 0, "exact": 1}

_cuda = None
_host = None


class FmmJob(C.Structure):
    """Mirror of ``fmmcu_fmm_job`` (include/fmm_cuda.h)."""

    _fields_ = [
        ("n_src", C.c_uint32),
        ("n_eval", C.c_uint32),
        ("src_z", C.c_void_p),
        ("src_m", C.c_void_p),
        ("eval_y", C.c_void_p),
        ("eval_sid", C.c_void_p),
        ("n_levels", C.c_int),
        ("theta", C.c_double),
        ("p", C.c_int),
        ("kernel", C.c_int),
        ("smoother", C.c_int),
        ("delta", C.c_double),
        ("out", C.c_void_p),
        ("inputs_consumed", C.c_void_p),
        ("inputs_consumed_arg", C.c_void_p),
    ]


class FmmStats(C.Structure):
    """Mirror of ``fmmcu_fmm_stats`` (include/fmm_cuda.h)."""

    _fields_ = [(n, C.c_uint64) for n in ("p2p_pairs", "m2l_ops", "p2m_points", "l2p_points")] + \
               [(n, C.c_double) for n in ("t_upload", "t_tree", "t_connect", "t_p2m_upward",
                                          "t_m2l", "t_p2p", "t_device", "t_total")] + \
               [("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("t_far_wait", C.c_double)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class NativeLibraryMissing(RuntimeError):
    pass


class FmmcuError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fmmcu error {code}: {msg}")
        self.code = code


def _as_pairs(a):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        return np.ascontiguousarray(a, dtype=np.complex128).view(np.float64).reshape(-1, 2)
    return np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 2)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


class P2PJob(C.Structure):
    """Mirror of ``fmmcu_p2p_job`` (include/fmm_cuda.h)."""

    _fields_ = [
        ("n_leaves", C.c_uint32),
        ("n_src", C.c_uint32),
        ("n_eval", C.c_uint32),
        ("pt_off", C.c_void_p),
        ("ev_off", C.c_void_p),
        ("strong_off", C.c_void_p),
        ("strong_idx", C.c_void_p),
        ("perm", C.c_void_p),
        ("src_z", C.c_void_p),
        ("src_m", C.c_void_p),
        ("eval_y", C.c_void_p),
        ("eval_sid", C.c_void_p),
        ("kernel", C.c_int),
        ("smoother", C.c_int),
        ("delta", C.c_double),
        ("mode", C.c_int),
        ("leaf_begin", C.c_uint32),
        ("leaf_end", C.c_uint32),
        ("out", C.c_void_p),
    ]


class M2LBuffers(C.Structure):
    """Mirror of ``fmmcu_m2l_buffers`` (include/fmm_cuda.h)."""
    _fields_ = [("centers", C.POINTER(C.c_double)), ("coeffs", C.POINTER(C.c_double)),
                ("out", C.POINTER(C.c_double)), ("target_box", C.POINTER(C.c_uint32)),
                ("weak_off", C.POINTER(C.c_uint32)), ("weak_idx", C.POINTER(C.c_uint32))]


class L2LJob(C.Structure):
    _fields_ = [("n_levels", C.c_int), ("level_base", C.c_void_p), ("target_of", C.c_void_p),
                ("finest_out", C.c_void_p)]


class M2LJob(C.Structure):
    """Mirror of ``fmmcu_m2l_job`` (include/fmm_cuda.h)."""

    _fields_ = [
        ("p", C.c_int),
        ("kernel", C.c_int),
        ("n_boxes", C.c_uint32),
        ("centers", C.c_void_p),
        ("coeffs", C.c_void_p),
        ("n_targets", C.c_uint32),
        ("target_box", C.c_void_p),
        ("weak_off", C.c_void_p),
        ("weak_idx", C.c_void_p),
        ("out", C.c_void_p),
    ]


CUDA_SYMBOLS = [
    "fmmcu_create", "fmmcu_destroy", "fmmcu_last_error", "fmmcu_device_count",
    "fmmcu_p2p_launch", "fmmcu_p2p_finish", "fmmcu_p2p_stage", "fmmcu_p2p_run_staged",
    "fmmcu_p2p_device_out", "fmmcu_p2p_bind_device_out", "fmmcu_p2p_copy_out", "fmmcu_p2p_pairs", "fmmcu_p2p_work_prefix", "fmmcu_set_stream",
    "fmmcu_synchronize", "fmmcu_m2l_launch", "fmmcu_m2l_finish", "fmmcu_kernel_launches",
    "fmmcu_fp64_peak", "fmmcu_last_transfer_bytes", "fmmcu_host_register", "fmmcu_host_unregister",
    "fmmcu_fmm_evaluate", "fmmcu_fmm_launch", "fmmcu_fmm_finish", "fmmcu_fmm_tree_level", "fmmcu_fmm_tree_perm", "fmmcu_fmm_tree_lists",
    "fmmcu_hypot_batch", "fmmcu_p2p_kernel_info",
    "fmmcu_p2p_out_ipc_handle", "fmmcu_p2p_bind_peer_out", "fmmcu_nccl_unique_id",
    "fmmcu_nccl_init", "fmmcu_nccl_gather_out", "fmmcu_m2l_host_buffers",
    "fmmcu_pin_host", "fmmcu_unpin_host", "fmmcu_tree_build", "fmmcu_m2l_downward",
]
IPC_HANDLE_BYTES = 64
NCCL_ID_BYTES = 128
FMMCU_ENCCL = 7


def cuda_lib():
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB):
            raise NativeLibraryMissing(f"{CUDA_LIB} not built (run __graft_entry__.build())")
        lib = C.CDLL(CUDA_LIB)
        vp = C.c_void_p
        lib.fmmcu_create.argtypes = [C.POINTER(vp), C.c_int]
        lib.fmmcu_destroy.argtypes = [vp]
        lib.fmmcu_destroy.restype = None
        lib.fmmcu_last_error.argtypes = [vp]
        lib.fmmcu_last_error.restype = C.c_char_p
        lib.fmmcu_device_count.argtypes = [C.POINTER(C.c_int)]
        lib.fmmcu_p2p_launch.argtypes = [vp, C.POINTER(P2PJob)]
        lib.fmmcu_p2p_finish.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.fmmcu_p2p_stage.argtypes = [vp, C.POINTER(P2PJob)]
        lib.fmmcu_p2p_run_staged.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_int,
                                             C.POINTER(C.c_int)]
        lib.fmmcu_p2p_device_out.argtypes = [vp, C.POINTER(C.c_void_p)]
        lib.fmmcu_p2p_bind_device_out.argtypes = [vp, vp]
        lib.fmmcu_p2p_copy_out.argtypes = [vp, vp, C.c_uint32, C.c_uint32]
        lib.fmmcu_p2p_pairs.argtypes = [vp, C.POINTER(C.c_uint64)]
        lib.fmmcu_p2p_work_prefix.argtypes = [vp, vp]
        lib.fmmcu_set_stream.argtypes = [vp, vp]
        lib.fmmcu_host_register.argtypes = [vp, vp, C.c_uint64]
        lib.fmmcu_host_unregister.argtypes = [vp, vp]
        lib.fmmcu_fmm_evaluate.argtypes = [vp, C.POINTER(FmmJob), C.POINTER(FmmStats)]
        lib.fmmcu_fmm_launch.argtypes = [vp, C.POINTER(FmmJob)]
        lib.fmmcu_fmm_finish.argtypes = [vp, vp, C.POINTER(FmmStats)]
        lib.fmmcu_fmm_tree_level.argtypes = [vp, C.c_int, C.POINTER(C.c_uint32), vp, vp]
        lib.fmmcu_fmm_tree_perm.argtypes = [vp, vp, vp]
        lib.fmmcu_fmm_tree_lists.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_uint64), vp, vp]
        lib.fmmcu_hypot_batch.argtypes = [vp, vp, C.c_uint32, vp]
        lib.fmmcu_p2p_kernel_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        lib.fmmcu_synchronize.argtypes = [vp]
        lib.fmmcu_m2l_launch.argtypes = [vp, C.POINTER(M2LJob)]
        lib.fmmcu_m2l_downward.argtypes = [vp, C.POINTER(L2LJob)]
        lib.fmmcu_m2l_finish.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        lib.fmmcu_m2l_host_buffers.argtypes = [vp, C.c_uint32, C.c_int, C.c_uint32, C.c_uint64,
                                               C.POINTER(M2LBuffers)]
        lib.fmmcu_kernel_launches.argtypes = [vp]
        lib.fmmcu_kernel_launches.restype = C.c_uint64
        lib.fmmcu_fp64_peak.argtypes = [vp, C.POINTER(C.c_double)]
        lib.fmmcu_last_transfer_bytes.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.fmmcu_p2p_out_ipc_handle.argtypes = [vp, vp]
        lib.fmmcu_p2p_bind_peer_out.argtypes = [vp, vp]
        lib.fmmcu_nccl_unique_id.argtypes = [vp]
        lib.fmmcu_nccl_init.argtypes = [vp, vp, C.c_int, C.c_int]
        lib.fmmcu_nccl_gather_out.argtypes = [vp, C.c_int, vp]
        _cuda = lib
    return _cuda


def device_count() -> int:
    n = C.c_int(0)
    cuda_lib().fmmcu_device_count(C.byref(n))
    return n.value


class CudaContext:
    """One ``fmmcu_ctx`` (one device).  Mirrors the reference's concurrent
    near-field backend protocol: ``launch`` returns at once, ``finish`` joins
    and reports ``(pair_evals, seconds)`` (backend.hpp:39-57)."""

    def __init__(self, device: int = 0):
        self.lib = cuda_lib()
        h = C.c_void_p()
        rc = self.lib.fmmcu_create(C.byref(h), device)
        self.h = h
        if rc != FMMCU_OK:
            msg = self.lib.fmmcu_last_error(h).decode() if h else "create failed"
            if h:
                self.lib.fmmcu_destroy(h)
            self.h = None
            raise FmmcuError(rc, msg)
        self._keep = None

    def close(self):
        if self.h:
            self.lib.fmmcu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != FMMCU_OK:
            raise FmmcuError(rc, self.lib.fmmcu_last_error(self.h).decode())

    # -- job construction --------------------------------------------------
    @staticmethod
    def make_job(pt_off, ev_off, s_off, s_idx, perm, zp, mp, yp, sidp, out, *, kernel=0,
                 smoother=0, delta=0.0, mode=0, leaf_begin=0, leaf_end=None):
        arrs = dict(
            pt_off=np.ascontiguousarray(pt_off, dtype=np.uint32),
            ev_off=np.ascontiguousarray(ev_off, dtype=np.uint32),
            s_off=np.ascontiguousarray(s_off, dtype=np.uint32),
            s_idx=np.ascontiguousarray(s_idx, dtype=np.uint32),
            perm=np.ascontiguousarray(perm, dtype=np.uint32),
            zp=np.ascontiguousarray(zp, dtype=np.float64),
            mp=np.ascontiguousarray(mp, dtype=np.float64),
            yp=np.ascontiguousarray(yp, dtype=np.float64),
            sidp=None if sidp is None else np.ascontiguousarray(sidp, dtype=np.int64),
        )
        nl = len(arrs["pt_off"]) - 1
        j = P2PJob()
        j.n_leaves = nl
        j.n_src = arrs["zp"].size // 2
        j.n_eval = arrs["yp"].size // 2
        j.pt_off = _ptr(arrs["pt_off"])
        j.ev_off = _ptr(arrs["ev_off"])
        j.strong_off = _ptr(arrs["s_off"])
        j.strong_idx = _ptr(arrs["s_idx"]) if arrs["s_idx"].size else None
        j.perm = _ptr(arrs["perm"])
        j.src_z = _ptr(arrs["zp"])
        j.src_m = _ptr(arrs["mp"])
        j.eval_y = _ptr(arrs["yp"]) if arrs["yp"].size else None
        j.eval_sid = _ptr(arrs["sidp"])
        j.kernel = kernel
        j.smoother = smoother
        j.delta = delta
        j.mode = mode
        j.leaf_begin = leaf_begin
        j.leaf_end = nl if leaf_end is None else leaf_end
        j.out = _ptr(out) if out is not None and out.size else None
        return j, arrs

    # -- reference-facing protocol -----------------------------------------
    def launch(self, job, keep):
        self._keep = keep
        self._check(self.lib.fmmcu_p2p_launch(self.h, C.byref(job)))

    def finish(self):
        pairs = C.c_uint64()
        secs = C.c_double()
        rc = self.lib.fmmcu_p2p_finish(self.h, C.byref(pairs), C.byref(secs))
        self._keep = None
        self._check(rc)
        return int(pairs.value), float(secs.value)

    # -- device-resident protocol ------------------------------------------
    def stage(self, job, keep):
        self._check(self.lib.fmmcu_p2p_stage(self.h, C.byref(job)))
        del keep

    def run_staged(self, leaf_begin, leaf_end, mode=0) -> int:
        n = C.c_int()
        self._check(self.lib.fmmcu_p2p_run_staged(self.h, leaf_begin, leaf_end, mode,
                                                  C.byref(n)))
        return n.value

    def device_out_ptr(self) -> int:
        p = C.c_void_p()
        self._check(self.lib.fmmcu_p2p_device_out(self.h, C.byref(p)))
        return p.value

    def bind_device_out(self, dptr: int | None):
        """Write potentials into caller-owned device memory (e.g. a torch tensor)."""
        self._check(self.lib.fmmcu_p2p_bind_device_out(self.h, C.c_void_p(dptr or 0)))

    def copy_out(self, n_eval: int, eval_begin: int = 0, eval_end: int | None = None):
        out = np.zeros((n_eval, 2))
        e1 = n_eval if eval_end is None else eval_end
        self._check(self.lib.fmmcu_p2p_copy_out(self.h, _ptr(out), eval_begin, e1))
        return out

    def pairs(self) -> int:
        v = C.c_uint64()
        self._check(self.lib.fmmcu_p2p_pairs(self.h, C.byref(v)))
        return int(v.value)

    def work_prefix(self, n_leaves) -> np.ndarray:
        out = np.empty(n_leaves + 1, dtype=np.uint64)
        self._check(self.lib.fmmcu_p2p_work_prefix(self.h, _ptr(out)))
        return out

    def set_stream(self, stream_handle: int | None):
        self._check(self.lib.fmmcu_set_stream(self.h, C.c_void_p(stream_handle or 0)))

    def host_register(self, arr: np.ndarray):
        """Page-lock a host array (cudaHostRegister) so D2H lands in it directly."""
        self._check(self.lib.fmmcu_host_register(self.h, arr.ctypes.data, arr.nbytes))

    def host_unregister(self, arr: np.ndarray):
        self._check(self.lib.fmmcu_host_unregister(self.h, arr.ctypes.data))

    # -- whole FMM evaluation on the device (fmmcu_fmm_*) -------------------
    def fmm_evaluate(self, z, m, y, sid, *, n_levels, theta, p, kernel=0, smoother=0, delta=0.0,
                     out=None):
        """One device FmmEngine::evaluate.  z, m: [n] complex (or [n,2] float);
        y: [ne] eval positions, sid: [ne] int64 source ids or None.
        Returns (potentials [ne] complex in original order, stats dict)."""
        zz = _as_pairs(z)
        mm = _as_pairs(m)
        yy = _as_pairs(y)
        ne = len(yy)
        if out is None:
            out = np.zeros(max(ne, 1), dtype=np.complex128)
        sidp = None if sid is None else np.ascontiguousarray(sid, dtype=np.int64)
        j = FmmJob()
        j.n_src = len(zz)
        j.n_eval = ne
        j.src_z = _ptr(zz)
        j.src_m = _ptr(mm)
        j.eval_y = _ptr(yy) if ne else None
        j.eval_sid = _ptr(sidp)
        j.n_levels = n_levels
        j.theta = theta
        j.p = p
        j.kernel = kernel
        j.smoother = smoother
        j.delta = delta
        j.out = _ptr(out) if ne else None
        st = FmmStats()
        self._check(self.lib.fmmcu_fmm_evaluate(self.h, C.byref(j), C.byref(st)))
        return out[:ne], st.as_dict()

    def fmm_tree(self, n_levels: int, n_src: int, n_eval: int):
        """Device pyramid + connectivity of the last fmm_evaluate, in the
        layout of fmm.Tree: (boxes_f, boxes_u, perm, eval_perm, strong, weak)."""
        bf, bu, strong, weak = [], [], [], []
        for lvl in range(n_levels):
            nb = C.c_uint32()
            self._check(self.lib.fmmcu_fmm_tree_level(self.h, lvl, C.byref(nb), None, None))
            f = np.zeros((nb.value, 5))
            u = np.zeros((nb.value, 4), dtype=np.uint32)
            self._check(self.lib.fmmcu_fmm_tree_level(self.h, lvl, C.byref(nb), _ptr(f), _ptr(u)))
            bf.append(f)
            bu.append(u)
            for weak_flag, dst in ((0, strong), (1, weak)):
                nnz = C.c_uint64()
                self._check(self.lib.fmmcu_fmm_tree_lists(self.h, lvl, weak_flag, C.byref(nnz),
                                                          None, None))
                off = np.zeros(nb.value + 1, dtype=np.uint32)
                idx = np.zeros(max(nnz.value, 1), dtype=np.uint32)
                self._check(self.lib.fmmcu_fmm_tree_lists(self.h, lvl, weak_flag, C.byref(nnz),
                                                          _ptr(off), _ptr(idx)))
                dst.append((off, idx[: nnz.value]))
        perm = np.zeros(n_src, dtype=np.uint32)
        eperm = np.zeros(max(n_eval, 1), dtype=np.uint32)
        self._check(self.lib.fmmcu_fmm_tree_perm(self.h, _ptr(perm), _ptr(eperm)))
        return bf, bu, perm, eperm[:n_eval], strong, weak

    def hypot(self, xy: np.ndarray) -> np.ndarray:
        xy = np.ascontiguousarray(xy, dtype=np.float64)
        out = np.zeros(len(xy))
        self._check(self.lib.fmmcu_hypot_batch(self.h, _ptr(xy), len(xy), _ptr(out)))
        return out

    def synchronize(self):
        self._check(self.lib.fmmcu_synchronize(self.h))

    def launches(self) -> int:
        return int(self.lib.fmmcu_kernel_launches(self.h))

    def transfer_bytes(self):
        h2d, d2h = C.c_uint64(), C.c_uint64()
        self._check(self.lib.fmmcu_last_transfer_bytes(self.h, C.byref(h2d), C.byref(d2h)))
        return int(h2d.value), int(d2h.value)

    def kernel_info(self):
        """(symmetric, evals_per_lane) of the staged fast work list."""
        sym, e = C.c_int(), C.c_int()
        self._check(self.lib.fmmcu_p2p_kernel_info(self.h, C.byref(sym), C.byref(e)))
        return bool(sym.value), int(e.value)

    # -- multi-GPU (include/fmm_cuda.h, fmm_multi.cu) ------------------------
    def out_ipc_handle(self) -> bytes:
        """Root rank: IPC handle of the staged output buffer."""
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        self._check(self.lib.fmmcu_p2p_out_ipc_handle(self.h, buf))
        return buf.raw

    def bind_peer_out(self, handle: bytes | None):
        """Other ranks: write the shard's potentials into the root's buffer."""
        if handle is None:
            self._check(self.lib.fmmcu_p2p_bind_peer_out(self.h, None))
            return
        buf = C.create_string_buffer(bytes(handle), IPC_HANDLE_BYTES)
        self._check(self.lib.fmmcu_p2p_bind_peer_out(self.h, buf))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(NCCL_ID_BYTES)
        rc = cuda_lib().fmmcu_nccl_unique_id(buf)
        if rc != FMMCU_OK:
            raise FmmcuError(rc, "ncclGetUniqueId failed (libnccl.so.2)")
        return buf.raw

    def nccl_init(self, uid: bytes, rank: int, world: int):
        buf = C.create_string_buffer(bytes(uid), NCCL_ID_BYTES)
        self._check(self.lib.fmmcu_nccl_init(self.h, buf, rank, world))

    def nccl_gather_out(self, root: int, eval_cuts):
        cuts = np.ascontiguousarray(eval_cuts, dtype=np.uint32)
        self._check(self.lib.fmmcu_nccl_gather_out(self.h, root, _ptr(cuts)))

    def fp64_peak(self) -> float:
        v = C.c_double()
        self._check(self.lib.fmmcu_fp64_peak(self.h, C.byref(v)))
        return float(v.value)

    # -- M2L ------------------------------------------------------------------
    def m2l(self, p, kernel, centers, coeffs, target_box, weak_off, weak_idx):
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        target_box = np.ascontiguousarray(target_box, dtype=np.uint32)
        weak_off = np.ascontiguousarray(weak_off, dtype=np.uint32)
        weak_idx = np.ascontiguousarray(weak_idx, dtype=np.uint32)
        nt = len(target_box)
        out = np.zeros((nt, p + 1, 2))
        j = M2LJob()
        j.p = p
        j.kernel = kernel
        j.n_boxes = centers.size // 2
        j.centers = _ptr(centers)
        j.coeffs = _ptr(coeffs)
        j.n_targets = nt
        j.target_box = _ptr(target_box) if nt else None
        j.weak_off = _ptr(weak_off)
        j.weak_idx = _ptr(weak_idx) if weak_idx.size else None
        j.out = _ptr(out) if nt else None
        self._check(self.lib.fmmcu_m2l_launch(self.h, C.byref(j)))
        ops = C.c_uint64()
        secs = C.c_double()
        self._check(self.lib.fmmcu_m2l_finish(self.h, C.byref(ops), C.byref(secs)))
        return out, int(ops.value), float(secs.value)

    def m2l_downward(self, p, kernel, centers, coeffs, target_box, weak_off, weak_idx,
                     level_base, target_of):
        """m2l() with the sums kept on the device, then fmmcu_m2l_downward:
        the finest level's locals ([boxes of the finest level, p+1, 2]; rows
        of boxes without a target slot are zero here)."""
        centers = np.ascontiguousarray(centers, dtype=np.float64)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        target_box = np.ascontiguousarray(target_box, dtype=np.uint32)
        weak_off = np.ascontiguousarray(weak_off, dtype=np.uint32)
        weak_idx = np.ascontiguousarray(weak_idx, dtype=np.uint32)
        level_base = np.ascontiguousarray(level_base, dtype=np.uint32)
        target_of = np.ascontiguousarray(target_of, dtype=np.int32)
        L = len(level_base) - 1
        nfin = int(level_base[L] - level_base[L - 1])
        out = np.zeros((nfin, p + 1, 2))
        j = M2LJob()
        j.p = p
        j.kernel = kernel
        j.n_boxes = centers.size // 2
        j.centers = _ptr(centers)
        j.coeffs = _ptr(coeffs)
        j.n_targets = len(target_box)
        j.target_box = _ptr(target_box) if len(target_box) else None
        j.weak_off = _ptr(weak_off)
        j.weak_idx = _ptr(weak_idx) if weak_idx.size else None
        j.out = None  # keep the sums on the device
        self._check(self.lib.fmmcu_m2l_launch(self.h, C.byref(j)))
        d = L2LJob()
        d.n_levels = L
        d.level_base = _ptr(level_base)
        d.target_of = _ptr(target_of)
        d.finest_out = _ptr(out)
        rc = self.lib.fmmcu_m2l_downward(self.h, C.byref(d))
        ops = C.c_uint64()
        secs = C.c_double()
        rc2 = self.lib.fmmcu_m2l_finish(self.h, C.byref(ops), C.byref(secs))
        self._check(rc)
        self._check(rc2)
        return out, int(ops.value)

    def m2l_pinned(self, p, kernel, centers, coeffs, target_box, weak_off, weak_idx):
        """m2l() through the context's page-locked buffers
        (fmmcu_m2l_host_buffers): inputs copied into them, DMA'd in place,
        sums D2H'd straight into the pinned out."""
        centers = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1)
        nb, nt = centers.size // 2, len(target_box)
        nnz = int(np.asarray(weak_off)[nt]) if nt else 0
        b = M2LBuffers()
        self._check(self.lib.fmmcu_m2l_host_buffers(self.h, nb, p, nt, nnz, C.byref(b)))
        view = lambda ptr, n: np.ctypeslib.as_array(ptr, shape=(n,))  # noqa: E731
        view(b.centers, 2 * nb)[:] = centers
        view(b.coeffs, coeffs.size)[:] = coeffs
        if nt:
            view(b.target_box, nt)[:] = target_box
            view(b.weak_off, nt + 1)[:] = weak_off
        if nnz:
            view(b.weak_idx, nnz)[:] = weak_idx
        j = M2LJob()
        j.p = p
        j.kernel = kernel
        j.n_boxes = nb
        vp = lambda ptr: C.cast(ptr, C.c_void_p)  # noqa: E731
        j.centers = vp(b.centers)
        j.coeffs = vp(b.coeffs)
        j.n_targets = nt
        j.target_box = vp(b.target_box) if nt else None
        j.weak_off = vp(b.weak_off)
        j.weak_idx = vp(b.weak_idx) if nnz else None
        j.out = vp(b.out) if nt else None
        self._check(self.lib.fmmcu_m2l_launch(self.h, C.byref(j)))
        ops = C.c_uint64()
        secs = C.c_double()
        self._check(self.lib.fmmcu_m2l_finish(self.h, C.byref(ops), C.byref(secs)))
        out = view(b.out, nt * (p + 1) * 2).reshape(nt, p + 1, 2).copy() if nt else \
            np.zeros((0, p + 1, 2))
        return out, int(ops.value), float(secs.value)


def p2p(ctx: CudaContext, pt_off, ev_off, s_off, s_idx, perm, zp, mp, yp, sidp, *, kernel=0,
        smoother=0, delta=0.0, mode=0, leaf_begin=0, leaf_end=None, out=None):
    """One synchronous near-field evaluation through the reference-facing
    protocol (launch + finish).  Returns (out[n_eval, 2] permuted, pairs, seconds)."""
    n_eval = np.asarray(yp).size // 2
    if out is None:
        out = np.zeros((n_eval, 2))
    job, keep = CudaContext.make_job(pt_off, ev_off, s_off, s_idx, perm, zp, mp, yp, sidp, out,
                                     kernel=kernel, smoother=smoother, delta=delta, mode=mode,
                                     leaf_begin=leaf_begin, leaf_end=leaf_end)
    ctx.launch(job, keep)
    pairs, secs = ctx.finish()
    return out, pairs, secs
