"""The drop-in binding, proven on the reference itself.

oracle/_ref/libfmmref_cuda.so is the reference library compiled from a
scratch copy of /root/reference/proj with the three edits of
integration/patch_reference.py (BackendKind::cuda, its string form, the
make_backend case) plus integration/cuda_backend_ref.cpp, a NearFieldBackend
written against the unmodified interface (backend.hpp:48-57) that calls
libfmmcuda.so through the C ABI.  These tests run the REFERENCE's
FmmEngine::evaluate (engine.cpp:208-347) with that backend.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import ROOT, normwise
from oracle import oracle as O

LIB = os.path.join(ROOT, "oracle", "_ref", "libfmmref_cuda.so")
pytestmark = pytest.mark.skipif(not os.path.exists(LIB), reason="patched reference not built")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64 = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def _lib():
    lib = C.CDLL(LIB)
    lib.refcu_evaluate.argtypes = [C.c_char_p, _dp, _dp, C.c_int64, _i64, _dp, _ip, _dp, _dp, _u64,
                                   C.c_char_p, C.c_int]
    lib.refcu_last_error.restype = C.c_char_p
    return lib


def ref_evaluate(backend, z, m, *, n_levels, theta=0.5, threads=8):
    lib = _lib()
    n = len(z)
    out = np.empty((n, 2))
    tim = np.empty(8)
    cnt = np.empty(4, dtype=np.uint64)
    name = C.create_string_buffer(16)
    rc = lib.refcu_evaluate(backend.encode(), np.ascontiguousarray(z), np.ascontiguousarray(m), n,
                            np.arange(n, dtype=np.int64), np.array([theta, 1e-6]),
                            np.array([n_levels, 1, threads], dtype=np.int32), out, tim, cnt, name,
                            16)
    return rc, out, tim, cnt, name.value.decode(), lib.refcu_last_error().decode()


def test_patched_reference_knows_cuda_and_keeps_cpu_backends():
    z, m = O.make_distribution(0, 5000, 3)
    rc, out_s, _, cnt_s, name, _ = ref_evaluate("serial", z, m, n_levels=4)
    assert rc == 0 and name == "serial"
    # the patched library's CPU path is the reference's: bitwise equal to the
    # unmodified reference build
    want, _, cnt, _ = O.ref_evaluate(z, m, z, np.arange(len(z), dtype=np.int64), n_levels=4,
                                     backend=0, threads=1)
    assert np.array_equal(out_s.view(np.uint64), want.view(np.uint64))
    assert cnt_s.tolist() == cnt.tolist()


def test_cuda_backend_without_gpu_is_a_backend_error():
    from paper_1311_1006_b200 import _native
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    z, m = O.make_distribution(0, 1000, 3)
    rc, _, _, _, name, err = ref_evaluate("cuda", z, m, n_levels=3)
    assert rc == 4, err  # BackendError from the backend constructor (fmmcu_create)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,L", [(0, 200_000, 7), (2, 200_000, 8), (3, 50_000, 5)])
def test_reference_engine_with_cuda_backend_matches_pool(kind, n, L):
    z, m = O.make_distribution(kind, n, 11)
    rc_p, out_p, _, cnt_p, _, err = ref_evaluate("pool", z, m, n_levels=L)
    assert rc_p == 0, err
    rc_c, out_c, tim_c, cnt_c, name, err = ref_evaluate("cuda", z, m, n_levels=L)
    assert rc_c == 0, err
    assert name == "cuda"
    assert cnt_c.tolist() == cnt_p.tolist()  # p2p_pairs, m2l_ops, p2m, l2p identical
    assert normwise(out_c, out_p) <= 1e-12
    assert tim_c[4] > 0.0 and tim_c[7] >= 0.0  # t_p2p from the backend; cpu_wait (concurrent)
