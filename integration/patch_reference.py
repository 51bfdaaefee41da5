#!/usr/bin/env python3
"""Register the B200 near field in a scratch copy of the reference.

    patch_reference.py <reference proj dir> <scratch dir>

Copies proj/include and the six Eigen-free translation units of proj/src
(geometry, expansion, backend, engine, autotune, csv) into the
scratch dir -- never into the repository -- and applies the three edits
INTEGRATION.md §A describes, nothing else:

  include/fmm/backend.hpp:13     enum BackendKind gains `cuda`, and the factory
                                 hook make_cuda_backend() is declared;
  src/backend.cpp:15-29          backend_from_string / to_string know "cuda";
  src/backend.cpp:170-177        make_backend returns make_cuda_backend().

The hook is defined in integration/cuda_backend_ref.cpp (a NearFieldBackend
over libfmmcuda.so's C ABI).  Each edit asserts that the line it anchors on
exists exactly once, so a changed reference fails loudly instead of building
something else.
"""
import os
import shutil
import sys

SRCS = ("geometry", "expansion", "backend", "engine", "autotune", "csv")


def edit(path, anchor, new):
    text = open(path).read()
    if text.count(anchor) != 1:
        sys.exit(f"patch_reference: anchor not found exactly once in {path}: {anchor!r}")
    open(path, "w").write(text.replace(anchor, new))


def main():
    ref, dst = sys.argv[1], sys.argv[2]
    if os.path.exists(dst):
        shutil.rmtree(dst)
    shutil.copytree(os.path.join(ref, "include"), os.path.join(dst, "include"))
    os.makedirs(os.path.join(dst, "src"))
    for s in SRCS:
        shutil.copy(os.path.join(ref, "src", s + ".cpp"), os.path.join(dst, "src", s + ".cpp"))
    hpp = os.path.join(dst, "include", "fmm", "backend.hpp")
    cpp = os.path.join(dst, "src", "backend.cpp")
    edit(hpp, "enum class BackendKind { serial, pool, throttled };",
         "enum class BackendKind { serial, pool, throttled, cuda };")
    edit(hpp, "std::unique_ptr<NearFieldBackend> make_backend(BackendKind kind, ThrottleSettings ts = {});",
         "std::unique_ptr<NearFieldBackend> make_backend(BackendKind kind, ThrottleSettings ts = {});\n"
         "// B200 near field (integration/cuda_backend_ref.cpp, libfmmcuda.so)\n"
         "std::unique_ptr<NearFieldBackend> make_cuda_backend();")
    edit(cpp, '  if (s == "throttled") return BackendKind::throttled;',
         '  if (s == "throttled") return BackendKind::throttled;\n'
         '  if (s == "cuda") return BackendKind::cuda;')
    edit(cpp, '    case BackendKind::throttled: return "throttled";',
         '    case BackendKind::throttled: return "throttled";\n'
         '    case BackendKind::cuda: return "cuda";')
    edit(cpp, "    case BackendKind::throttled: return std::make_unique<ThrottledBackend>(ts);",
         "    case BackendKind::throttled: return std::make_unique<ThrottledBackend>(ts);\n"
         "    case BackendKind::cuda: return make_cuda_backend();")
    open(os.path.join(dst, ".patched"), "w").write("ok\n")


if __name__ == "__main__":
    main()
