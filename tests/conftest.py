"""Shared fixtures.  `-m "not gpu"` runs on any CPU box; `-m gpu` needs a B200.

The native libraries are built in-tree by __graft_entry__.build(); if they
are missing (fresh checkout) they are built here once per session with the
same make targets.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (large N)")


def _ensure_built():
    need = [os.path.join(ROOT, "paper_1311_1006_b200", "libfmmcuda.so"),
            os.path.join(ROOT, "paper_1311_1006_b200", "libfmm.so"),
            os.path.join(ROOT, "oracle", "liboracle.so")]
    if not all(os.path.exists(p) for p in need):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True)
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1311_1006_b200")], check=True)


_ensure_built()


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name)) as f:
        return {k: f[k] for k in f.files}


@pytest.fixture(scope="session")
def golden_trees():
    out = {}
    for path in sorted(glob.glob(os.path.join(GOLDEN, "tree_*.npz"))):
        name = os.path.basename(path)[5:-4]
        out[name] = load_golden(os.path.basename(path))
    return out


def golden_leaf_csr(d):
    L = int(d["n_levels"])
    u = d[f"boxes_u_{L - 1}"]
    pt_off = np.concatenate([u[:, 0], u[-1:, 1]]).astype(np.uint32)
    ev_off = np.concatenate([u[:, 2], u[-1:, 3]]).astype(np.uint32)
    return pt_off, ev_off, d[f"strong_off_{L - 1}"], d[f"strong_idx_{L - 1}"]


def golden_permuted(d):
    zp = d["z"][d["perm"]]
    mp = d["m"][d["perm"]]
    yp = d["y"][d["eval_perm"]]
    sid = d["sid"][d["eval_perm"]] if "sid" in d else None
    return zp, mp, yp, sid


def normwise(a, b):
    """max|a-b| / max|b| over complex values stored as (n,2)."""
    a = np.asarray(a).reshape(-1, 2)
    b = np.asarray(b).reshape(-1, 2)
    scale = np.abs(b[:, 0] + 1j * b[:, 1]).max() if len(b) else 1.0
    diff = np.abs((a[:, 0] - b[:, 0]) + 1j * (a[:, 1] - b[:, 1])).max() if len(b) else 0.0
    return diff / (scale if scale > 0 else 1.0)


def bitwise(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
