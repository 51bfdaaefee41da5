"""The C ABIs load and export every symbol their headers declare; without a
GPU the device path fails loudly (no silent CPU fallback)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT
from paper_1311_1006_b200 import _native, fmm as F


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b((?:fmmcu|fmmh)_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,lib", [("fmm_cuda.h", _native.CUDA_LIB),
                                        ("fmm_host.h", _native.HOST_LIB)])
def test_library_exports_every_declared_symbol(header, lib):
    names = _declared(header)
    assert len(names) > 10
    so = ctypes.CDLL(lib)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_python_binding_covers_cuda_abi():
    assert sorted(_native.CUDA_SYMBOLS) == _declared("fmm_cuda.h")


def test_native_built_for_sm100a():
    data = open(_native.CUDA_LIB, "rb").read()
    assert b"sm_100a" in data


def test_no_gpu_fails_loudly():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_native.FmmcuError) as ei:
        _native.CudaContext(0)
    assert ei.value.code == _native.FMMCU_ECUDA
    s = F.make_distribution("uniform", 100, 1)
    with pytest.raises(F.BackendError):
        F.FmmEngine(F.FmmConfig(backend="cuda")).evaluate(s, F.EvalSet.self_of(s))


def test_product_does_not_link_the_oracle():
    for lib in (_native.CUDA_LIB, _native.HOST_LIB):
        data = open(lib, "rb").read()
        assert b"liboracle" not in data and b"libfmmref" not in data and b"orc_" not in data
