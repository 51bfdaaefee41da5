"""Pin the CPU oracle (oracle/fmm_oracle.c) before trusting it.

* its restatement of libgcc __divdc3 equals the compiler's own complex
  division on random and special inputs, and equals the reference's
  kernel_term (tests/golden/kernel_term.npz, expansion.cpp:90-92);
* its near field equals the reference nearfield_run bit for bit on every
  golden tree and kernel/smoother variant (backend.cpp:41-89), including the
  pair count;
* its m2l_add equals the reference bit for bit (expansion.cpp:188-269),
  including the long double branch.
"""
import numpy as np
import pytest

from conftest import bitwise, golden_leaf_csr, golden_permuted, load_golden
from oracle import oracle as O


def test_divdc3_matches_native_complex_division():
    rng = np.random.default_rng(0)
    n = 200_000
    q = np.empty((n, 4))
    q[:, :2] = rng.uniform(-1, 1, (n, 2))
    q[:, 2:] = rng.uniform(-1, 1, (n, 2)) * 10.0 ** rng.uniform(-300, 300, (n, 1))
    special = np.array([
        [1, 0, 0, 0], [0, 0, 0, 0], [np.inf, 1, 1, 1], [1, 1, np.inf, 0],
        [1e-310, 1e-310, 1e-300, 2e-300], [1e300, 1e300, 1e-300, 1e-300],
        [1, 2, 1e308, 1e308], [np.nan, 1, 1, 1], [1, 1, 1e-320, 0], [3, 4, 5, 6],
        [-0.0, 0.0, -1.0, 0.0], [1.0, -0.0, 0.0, -2.0],
    ])
    q = np.vstack([special, q])
    a = O.cdiv(q)
    b = O.cdiv(q, native=True)
    same = (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))
    assert same.all()


def test_kernel_term_golden():
    g = load_golden("kernel_term.npz")
    q = np.stack([-g["m"][:, 0], -g["m"][:, 1], g["y"][:, 0] - g["x"][:, 0],
                  g["y"][:, 1] - g["x"][:, 1]], 1)
    assert bitwise(O.cdiv(q), g["out"])


@pytest.mark.parametrize("variant", [(0, 0), (1, 0), (0, 1), (0, 2)])
def test_oracle_nearfield_equals_reference_golden(golden_trees, variant):
    k, s = variant
    for name, d in golden_trees.items():
        pt, ev, so, si = golden_leaf_csr(d)
        zp, mp, yp, sid = golden_permuted(d)
        csr = O.LeafCSR(pt, ev, so, si, d["perm"])
        out, pairs = O.nearfield(csr, zp, mp, yp, sid, kernel=k, smoother=s,
                                 delta=float(d[f"delta_k{k}_s{s}"]))
        assert pairs == int(d[f"pairs_k{k}_s{s}"]), name
        assert bitwise(out, d[f"near_k{k}_s{s}"]), name


def test_oracle_m2l_equals_reference_golden():
    g = load_golden("m2l_cases.npz")
    for i in range(int(g["count"])):
        p, kern = int(g[f"{i}_p"]), int(g[f"{i}_kernel"])
        got = O.m2l_add(p, kern, g[f"{i}_sc"], g[f"{i}_coeffs"], g[f"{i}_tc"], g[f"{i}_local0"])
        assert bitwise(got, g[f"{i}_local"]), (i, p, kern)


def test_oracle_m2l_singular():
    with pytest.raises(ZeroDivisionError):
        O.m2l_add(4, 0, np.array([1.0, 1.0]), np.ones((5, 2)), np.array([1.0, 1.0]),
                  np.zeros((5, 2)))


def test_oracle_pair_count_identity(golden_trees):
    """pair_evals = sum_leaves n_evals * |strong sources| - self hits."""
    d = golden_trees["rand2000_L4"]
    pt, ev, so, si = golden_leaf_csr(d)
    total = 0
    for t in range(len(pt) - 1):
        S = sum(int(pt[b + 1] - pt[b]) for b in si[so[t]:so[t + 1]])
        total += int(ev[t + 1] - ev[t]) * S
    assert total - len(d["z"]) == int(d["pairs_k0_s0"])


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
def test_oracle_vs_live_reference_random_trees():
    for kind, n, L, seed in [(0, 6000, 5, 11), (2, 8000, 6, 12), (3, 3000, 3, 13)]:
        z, m = O.make_distribution(kind, n, seed)
        sid = np.arange(n, dtype=np.int64)
        t = O.ref_tree(z, m, z, sid, L, 0.5, keep=True)
        ref, pairs, _ = O.ref_nearfield(t)
        csr = t.leaf_csr()
        out, opairs = O.nearfield(csr, z[t.perm], m[t.perm], z[t.eval_perm], sid[t.eval_perm])
        t.free()
        assert opairs == pairs
        assert bitwise(out, ref)


def test_hypot_restatement_matches_libm_and_cabs():
    """glibc 2.39 __hypot restated (oracle/fmm_oracle.c orc_hypot): bitwise
    equal to libm hypot() and cabs() -- the two entry points the reference
    uses for box radii and centre distances (geometry.cpp:13-19,100) -- over
    unit-square magnitudes, tiny ratios, subnormal/huge exponents and signs."""
    rng = np.random.default_rng(7)
    n = 400_000
    xy = rng.random((n, 2))
    xy[: n // 5] *= rng.random((n // 5, 1)) ** 8
    xy[n // 5: 2 * n // 5, 1] *= 1e-9
    ex = rng.integers(-1074, 1023, (n // 5, 2)).astype(float)
    xy[2 * n // 5: 3 * n // 5] = rng.random((n // 5, 2)) * 2.0 ** ex
    xy[3 * n // 5: 4 * n // 5] = (rng.random((n // 5, 2)) - 0.5) * 1e-3
    xy[4 * n // 5:] = rng.integers(-4, 5, (n - 4 * n // 5, 2)) * 0.125
    special = np.array([[0.0, 0.0], [-0.0, 0.0], [3.0, 4.0], [1e308, 1e308], [5e-324, 5e-324],
                        [2.0 ** 511, 1.0], [2.0 ** -460, 2.0 ** -460], [1.0, 2.0 ** -54]])
    bad, _ = O.hypot_check(np.vstack([xy, special]))
    assert bad == 0
