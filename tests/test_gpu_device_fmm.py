"""Device FMM pipeline parity (needs a B200): fmmcu_fmm_evaluate runs the whole
FmmEngine::evaluate on the GPU (include/fmm_cuda.h).

Bars:
  * glibc hypot restated on the device: bitwise equal to libm hypot;
  * device pyramid (boxes, ranges, perm, eval_perm) and connectivity (strong
    and weak lists, every level): bitwise equal to the host library, which
    is itself bit-exact with the compiled reference (tests/test_host_geometry.py);
  * potentials: <= 1e-12 * max|phi| (normwise) against the CPU evaluate()
    of the host library (reference semantics), counters identical.
"""
import numpy as np
import pytest

from paper_1311_1006_b200 import _native as N
from paper_1311_1006_b200 import fmm as F

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    c = N.CudaContext(0)
    yield c
    c.close()


def _lattice(n_side, aspect=0.25):
    g = np.arange(n_side) * (1.0 / n_side)
    z = (g[:, None] + 1j * g[None, :] * aspect).ravel()
    return F.SourceSet(z, np.full(len(z), 0.5j))


def _cases():
    yield "uniform20k_L5", F.make_distribution("uniform", 20_000, 1), None, 5, 0.5
    yield "gauss30k_L6", F.make_distribution("gauss8", 30_000, 3), None, 6, 0.5
    yield "line8k_L5_t065", F.make_distribution("line", 8_000, 4), None, 5, 0.65
    yield "lattice_ties_L6", _lattice(120), None, 6, 0.5
    s = F.make_distribution("random", 5_000, 5)
    yield "separate_evals_L4", s, F.EvalSet(F.make_distribution("random", 3_000, 6).z * 1.2 - 0.1), 4, 0.5
    yield "single_level", F.make_distribution("random", 700, 7), None, 1, 0.5
    yield "two_levels", F.make_distribution("random", 900, 8), None, 2, 0.4
    # self-evaluation shape (ids given, M == N) but not self-evaluation: the
    # pipeline's speculative self build must be discarded and redone
    s = F.make_distribution("uniform", 6_000, 9)
    perm = np.random.default_rng(9).permutation(6_000)
    yield "self_shape_permuted", s, F.EvalSet(s.z[perm], perm.astype(np.int64)), 5, 0.5
    yield "self_shape_moved", s, F.EvalSet(s.z + 1e-9, np.arange(6_000, dtype=np.int64)), 5, 0.5


def _evals(s, e):
    return F.EvalSet.self_of(s) if e is None else e


def test_device_hypot_matches_libm(ctx):
    rng = np.random.default_rng(3)
    n = 1_000_000
    xy = rng.random((n, 2))
    xy[: n // 4] *= rng.random((n // 4, 1)) ** 8
    ex = rng.integers(-1074, 1023, (n // 4, 2)).astype(float)
    xy[n // 4: n // 2] = rng.random((n // 4, 2)) * 2.0 ** ex
    xy[n // 2: 3 * n // 4] = (rng.random((n // 4, 2)) - 0.5) * 1e-3
    got = ctx.hypot(xy)
    want = np.hypot(xy[:, 0], xy[:, 1])
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_device_tree_bitwise_equal_to_host(ctx, case):
    name, s, e, L, theta = case
    e = _evals(s, e)
    host = F.Tree(s, e, L, theta, threads=4)
    ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=17)
    bf, bu, perm, eperm, strong, weak = ctx.fmm_tree(L, s.size(), e.size())
    for lvl in range(L):
        assert np.array_equal(bu[lvl], host.boxes_u[lvl]), (name, lvl, "ranges")
        assert np.array_equal(bf[lvl].view(np.uint64), host.boxes_f[lvl].view(np.uint64)), \
            (name, lvl, "geometry")
        for got, want in ((strong[lvl], host.strong[lvl]), (weak[lvl], host.weak[lvl])):
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), (name, lvl)
    assert np.array_equal(perm, host.perm)
    assert np.array_equal(eperm, host.eval_perm)


@pytest.mark.parametrize("kernel,smoother,delta", [("harmonic", "none", 0.0),
                                                   ("logarithmic", "none", 0.0),
                                                   ("harmonic", "gaussian", 0.01)])
@pytest.mark.parametrize("case", list(_cases())[:5] + list(_cases())[7:], ids=lambda c: c[0])
def test_device_potentials_match_cpu_evaluate(ctx, case, kernel, smoother, delta):
    name, s, e, L, theta = case
    e = _evals(s, e)
    cfg = F.FmmConfig(n_levels=L, theta=theta, kernel=kernel, smoother=smoother, delta=delta,
                      backend="pool", worker_threads=4)
    ref = F.FmmEngine(cfg).evaluate(s, e)
    got, st = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=ref.p,
                               kernel=N.KERNELS[kernel], smoother=N.SMOOTHERS[smoother],
                               delta=delta)
    scale = np.abs(ref.potentials).max()
    assert np.abs(got - ref.potentials).max() <= TOL * scale, name
    for k in ("p2p_pairs", "m2l_ops", "p2m_points", "l2p_points"):
        assert st[k] == ref.counters[k], (name, k)


def test_device_pipeline_is_deterministic_and_reusable(ctx):
    s = F.make_distribution("uniform", 50_000, 11)
    e = F.EvalSet.self_of(s)
    a, _ = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=6, theta=0.5, p=17)
    s2 = F.make_distribution("gauss8", 20_000, 12)
    ctx.fmm_evaluate(s2.z, s2.m, s2.z, None, n_levels=5, theta=0.5, p=17)
    b, _ = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=6, theta=0.5, p=17)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_device_pipeline_rejects_bad_input(ctx):
    s = F.make_distribution("random", 100, 1)
    z = s.z.copy()
    z[5] = np.nan
    with pytest.raises(N.FmmcuError):
        ctx.fmm_evaluate(z, s.m, s.z, None, n_levels=3, theta=0.5, p=17)
    with pytest.raises(N.FmmcuError):
        ctx.fmm_evaluate(s.z, s.m, s.z, None, n_levels=3, theta=1.5, p=17)
    with pytest.raises(N.FmmcuError):
        ctx.fmm_evaluate(s.z[:0], s.m[:0], s.z, None, n_levels=3, theta=0.5, p=17)


def test_device_pipeline_page_locked_io_is_identical(ctx):
    """Page-locked inputs are DMA'd in place (no staging) and a page-locked
    out receives the D2H directly; the potentials must not change."""
    s = F.make_distribution("uniform", 60_000, 13)
    e = F.EvalSet.self_of(s)
    a, _ = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=6, theta=0.5, p=17)
    out = np.zeros(len(e.y), dtype=np.complex128)
    arrs = (s.z, s.m, e.y, e.source_id, out)
    for x in arrs:
        ctx.host_register(x)
    try:
        b, _ = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=6, theta=0.5, p=17, out=out)
        # separate evals, page-locked y
        y = F.make_distribution("random", 7_000, 14).z
        ctx.host_register(y)
        try:
            c1, _ = ctx.fmm_evaluate(s.z, s.m, y, None, n_levels=6, theta=0.5, p=17)
        finally:
            ctx.host_unregister(y)
    finally:
        for x in arrs:
            ctx.host_unregister(x)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    c0, _ = ctx.fmm_evaluate(s.z, s.m, y.copy(), None, n_levels=6, theta=0.5, p=17)
    assert np.array_equal(c0.view(np.uint64), c1.view(np.uint64))


def test_engine_result_reuse_across_sizes():
    """The Python engine handle reuses its SourceSet/EvalSet/EvalResult
    storage (FmmEngine::evaluate_into); results must match fresh engines
    whether the problem size stays or changes between calls."""
    eng = F.FmmEngine(F.FmmConfig(n_levels=5, backend="cuda", device_pipeline=True))
    sets = [F.make_distribution("uniform", 30_000, 21), F.make_distribution("uniform", 30_000, 22),
            F.make_distribution("gauss8", 12_000, 23), F.make_distribution("uniform", 30_000, 21)]
    got = [eng.evaluate(s, F.EvalSet.self_of(s)).potentials.copy() for s in sets]
    for s, g in zip(sets, got):
        fresh = F.FmmEngine(F.FmmConfig(n_levels=5, backend="cuda", device_pipeline=True))
        want = fresh.evaluate(s, F.EvalSet.self_of(s)).potentials
        assert np.array_equal(g.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(got[0].view(np.uint64), got[3].view(np.uint64))


@pytest.mark.parametrize("env", ["FMMCU_CONN_SYNC", "FMMCU_CONN_TIGHT"])
def test_connectivity_paths_agree(ctx, env, monkeypatch):
    """The connectivity is built speculatively (all levels into guessed
    buffers, one count read at the end).  The per-level-read build
    (FMMCU_CONN_SYNC) and the overflow redo (FMMCU_CONN_TIGHT: guesses too
    small, so every build is redone) give bitwise the same lists."""
    for name, s, e, L, theta in list(_cases())[:4]:
        e = _evals(s, e)
        ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=17)
        want = ctx.fmm_tree(L, s.size(), e.size())
        monkeypatch.setenv(env, "1")
        ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=17)
        got = ctx.fmm_tree(L, s.size(), e.size())
        monkeypatch.delenv(env)
        for lvl in range(L):
            for g, w in ((got[4][lvl], want[4][lvl]), (got[5][lvl], want[5][lvl])):
                assert np.array_equal(g[0], w[0]) and np.array_equal(g[1], w[1]), (name, lvl)


@pytest.mark.parametrize("force_e", [None, "4", "5"])
def test_device_work_list_equals_host_work_list(ctx, force_e, monkeypatch):
    """The pipeline's P2P work list is built on the device from the finest
    CSR (p2p_worklist.cuh); FMMCU_HOST_WL=1 selects the host builder
    (build_worklist) over a downloaded CSR.  Same items in the same order, so
    the potentials are bitwise equal and the pair counts identical -- also
    where heavy leaves are split into strong-list chunks (few levels,
    clustered) and with the evals-per-lane choice forced either way."""
    if force_e:
        monkeypatch.setenv("FMMCU_P2P_E", force_e)
    cases = list(_cases())[:5] + [
        ("heavy_gauss_L3", F.make_distribution("gauss8", 40_000, 31), None, 3, 0.5),
        ("heavy_uniform_L2", F.make_distribution("uniform", 12_000, 32), None, 2, 0.5),
        # more than 32 strong entries per leaf: the mutual kernel's entry rounds
        ("rounds_uniform_t015", F.make_distribution("uniform", 50_000, 33), None, 6, 0.15),
        ("rounds_gauss_t02", F.make_distribution("gauss8", 50_000, 34), None, 6, 0.2)]
    for name, s, e, L, theta in cases:
        e = _evals(s, e)
        dev, sd = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=17)
        monkeypatch.setenv("FMMCU_HOST_WL", "1")
        host, sh = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=theta, p=17)
        monkeypatch.delenv("FMMCU_HOST_WL")
        assert np.array_equal(dev.view(np.uint64), host.view(np.uint64)), name
        assert sd["p2p_pairs"] == sh["p2p_pairs"], name


def test_device_tree_bitwise_equal_to_reference_golden(ctx, golden_trees):
    """The device pyramid and connectivity against the trees the REFERENCE
    built (tests/golden/tree_*.npz, make_golden.py over build_pyramid /
    build_connectivity, geometry.cpp:106-216) -- directly, not through the
    host library: box ranges, geometry, perm, eval_perm and the strong and
    weak lists of every level, bitwise."""
    for name, d in golden_trees.items():
        L, theta = int(d["n_levels"]), float(d["theta"])
        z = d["z"][:, 0] + 1j * d["z"][:, 1]
        m = d["m"][:, 0] + 1j * d["m"][:, 1]
        y = d["y"][:, 0] + 1j * d["y"][:, 1]
        sid = d["sid"] if "sid" in d else None
        ctx.fmm_evaluate(z, m, y, sid, n_levels=L, theta=theta, p=17)
        bf, bu, perm, eperm, strong, weak = ctx.fmm_tree(L, len(z), len(y))
        for lvl in range(L):
            assert np.array_equal(bu[lvl], d[f"boxes_u_{lvl}"]), (name, lvl, "ranges")
            assert np.array_equal(bf[lvl].view(np.uint64),
                                  d[f"boxes_f_{lvl}"].view(np.uint64)), (name, lvl, "geometry")
            for kind, got in (("strong", strong[lvl]), ("weak", weak[lvl])):
                assert np.array_equal(got[0], d[f"{kind}_off_{lvl}"]), (name, lvl, kind)
                assert np.array_equal(got[1], d[f"{kind}_idx_{lvl}"]), (name, lvl, kind)
        assert np.array_equal(perm, d["perm"]), name
        assert np.array_equal(eperm, d["eval_perm"]), name


def test_engine_handle_pinned_io_is_identical(ctx):
    """The engine handle page-locks its kept SourceSet / EvalSet / EvalResult
    (fmmcu_pin_host) once the cuda backend is in use, so the device pipeline
    DMAs inputs and potentials in place.  Results must be bitwise those of a
    plain fmm_evaluate, across repeated calls, a size change (the storage is
    unpinned before it reallocates) and a switch to the pool backend."""
    a = F.make_distribution("uniform", 1_200_000, 41)
    b = F.make_distribution("uniform", 1_500_000, 42)
    eng = F.FmmEngine(F.FmmConfig(n_levels=8, backend="cuda", device_pipeline=True))
    for s in (a, a, b, a):
        e = F.EvalSet.self_of(s)
        got = eng.evaluate(s, e).potentials
        want, _ = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=8, theta=0.5, p=17)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    eng.set_config(F.FmmConfig(n_levels=8, backend="pool", worker_threads=8))
    e = F.EvalSet.self_of(a)
    ref = eng.evaluate(a, e).potentials
    assert np.abs(ref - want).max() <= 1e-12 * np.abs(ref).max()
