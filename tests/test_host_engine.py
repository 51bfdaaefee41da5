"""Host engine + operators against the reference (CPU backends only).

Restates the reference's engine/expansion tests (proj/tests/test_engine.cpp,
test_expansion.cpp) and adds bitwise comparisons with the compiled
reference's FmmEngine::evaluate (golden fixtures + live when available)."""
import numpy as np
import pytest

from conftest import bitwise, load_golden, normwise
from oracle import oracle as O
from paper_1311_1006_b200 import fmm as F


def _sets(d):
    s = F.SourceSet(d["z"][:, 0] + 1j * d["z"][:, 1], d["m"][:, 0] + 1j * d["m"][:, 1])
    e = F.EvalSet(d["y"][:, 0] + 1j * d["y"][:, 1], d["sid"] if "sid" in d else None)
    return s, e


def direct(s, e, kernel="harmonic"):
    """Independent O(N^2) oracle (test_util.hpp:27-45) in numpy."""
    d = e.y[:, None] - s.z[None, :]
    if e.source_id is not None:
        d[np.arange(len(e.y)), e.source_id] = np.nan
    t = (-s.m[None, :] / d) if kernel == "harmonic" else s.m[None, :] * np.log(d)
    return np.nansum(t, axis=1)


@pytest.mark.parametrize("backend", ["serial", "pool"])
def test_evaluate_bitwise_vs_golden(golden_trees, backend):
    for name, d in golden_trees.items():
        s, e = _sets(d)
        eng = F.FmmEngine(F.FmmConfig(theta=float(d["theta"]), n_levels=int(d["n_levels"]),
                                      backend=backend, worker_threads=4))
        r = eng.evaluate(s, e)
        assert r.p == int(d["eval_p"])
        assert bitwise(F._c2(r.potentials), d["eval_pot"]), name
        assert [r.counters[k] for k in F.COUNTER_KEYS] == d["eval_counters"].tolist(), name


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("case", [(0, 20000, 6, "harmonic", "none", 0.0),
                                  (4, 5000, 5, "log", "none", 0.0),
                                  (0, 8000, 5, "harmonic", "gaussian", 2e-3),
                                  (0, 8000, 5, "harmonic", "plummer", 2e-3),
                                  (2, 30000, 7, "harmonic", "none", 0.0)])
def test_evaluate_bitwise_vs_live_reference(case):
    kind, n, L, kern, sm, delta = case
    s = F.make_distribution(kind, n, 5)
    e = F.EvalSet.self_of(s)
    r = F.FmmEngine(F.FmmConfig(n_levels=L, kernel=kern, smoother=sm, delta=delta, backend="pool",
                                worker_threads=8)).evaluate(s, e)
    ro, _, cnt, p = O.ref_evaluate(F._c2(s.z), F._c2(s.m), F._c2(e.y), e.source_id, n_levels=L,
                                   kernel=F.KERNEL[kern], smoother=F.SMOOTHER[sm], delta=delta,
                                   backend=1, threads=8)
    assert bitwise(F._c2(r.potentials), ro)
    assert [r.counters[k] for k in F.COUNTER_KEYS] == cnt.tolist()


def test_two_sources_one_eval_equal_direct_sum():
    s = F.SourceSet(np.array([0.1 + 0.2j, 0.8 + 0.9j]), np.array([1.5 - 0.5j, -2.0 + 0.25j]))
    e = F.EvalSet.at([0.4 + 0.55j])
    # std::complex division (libgcc __divdc3, restated in the oracle), summed in order
    q = np.stack([-s.m.real, -s.m.imag, (e.y[0] - s.z).real, (e.y[0] - s.z).imag], 1)
    t = O.cdiv(q)
    want = complex((0.0 + t[0, 0]) + t[1, 0], (0.0 + t[0, 1]) + t[1, 1])
    eng = F.FmmEngine(F.FmmConfig(n_levels=1))
    assert eng.evaluate(s, e).potentials[0] == want
    for nl in (2, 3, 4):
        eng.set_config(F.FmmConfig(n_levels=nl))
        got = eng.evaluate(s, e).potentials[0]
        assert abs(got - want) <= 1e-6 * abs(want)


def test_accuracy_grid_against_direct_sum():
    s = F.make_distribution("positive", 2048, 5)
    e = F.EvalSet.self_of(s)
    want = direct(s, e)
    scale = np.abs(want).max()
    for theta in (0.35, 0.5, 0.65):
        for nl in (2, 3, 4):
            r = F.FmmEngine(F.FmmConfig(theta=theta, n_levels=nl)).evaluate(s, e)
            assert np.abs(r.potentials - want).max() <= 10 * 1e-6 * scale


def test_log_kernel_real_part():
    s = F.make_distribution("positive", 1024, 6)
    e = F.EvalSet.self_of(s)
    want = direct(s, e, "log")
    r = F.FmmEngine(F.FmmConfig(kernel="log", n_levels=3)).evaluate(s, e)
    assert np.abs(r.potentials.real - want.real).max() <= 10 * 1e-6 * np.abs(want.real).max()


def test_backend_equivalence_bitwise():
    s = F.make_distribution("random", 800, 23)
    e = F.EvalSet.self_of(s)
    base = F.FmmEngine(F.FmmConfig(n_levels=3, worker_threads=2)).evaluate(s, e)
    for b in ("pool", "throttled"):
        got = F.FmmEngine(F.FmmConfig(n_levels=3, worker_threads=2, backend=b,
                                      throttle_latency_s=0.0)).evaluate(s, e)
        assert bitwise(F._c2(got.potentials), F._c2(base.potentials))
        assert got.counters["p2p_pairs"] == base.counters["p2p_pairs"]


def test_split_level_and_threads_independence():
    s = F.make_distribution("random", 600, 15)
    e = F.EvalSet.self_of(s)
    ref = F.FmmEngine(F.FmmConfig(n_levels=4, task_split_level=1)).evaluate(s, e)
    for split in (1, 2, 3):
        for thr in (1, 4, 8):
            got = F.FmmEngine(F.FmmConfig(n_levels=4, task_split_level=split,
                                          worker_threads=thr)).evaluate(s, e)
            assert bitwise(F._c2(got.potentials), F._c2(ref.potentials))
            assert got.counters["m2l_ops"] == ref.counters["m2l_ops"]


def test_work_counters():
    s = F.make_distribution("random", 256, 13)
    r = F.FmmEngine(F.FmmConfig(n_levels=1)).evaluate(s, F.EvalSet.self_of(s))
    assert r.counters["p2p_pairs"] == 256 * 255
    assert r.counters["m2l_ops"] == 0 and r.counters["p2m_points"] == 256


def test_all_strong_tree_has_no_m2l():
    z = []
    for qx in (0.0, 1.0):
        for qy in (0.0, 1.0):
            for dx in (0.001, 0.999):
                for dy in (0.001, 0.999):
                    z.append(complex(qx + dx, qy + dy))
    s = F.SourceSet(np.array(z), np.full(len(z), 1.0 + 0.5j))
    e = F.EvalSet.self_of(s)
    r = F.FmmEngine(F.FmmConfig(theta=0.9, p_override=8, n_levels=2)).evaluate(s, e)
    assert r.counters["m2l_ops"] == 0
    want = direct(s, e)
    assert np.abs(r.potentials - want).max() <= 1e-13 * np.abs(want).max()


def test_smoothed_near_field_through_evaluate():
    s = F.make_distribution("random", 300, 14)
    e = F.EvalSet.self_of(s)
    r = F.FmmEngine(F.FmmConfig(smoother="gaussian", delta=1e-3, n_levels=3)).evaluate(s, e)
    want = F.p2p_direct(e, s, "harmonic", "gaussian", 1e-3)
    assert np.abs(r.potentials - want).max() <= 2e-6 * np.abs(want).max()


def test_empty_eval_set_and_validation():
    s = F.make_distribution("random", 50, 11)
    assert F.FmmEngine(F.FmmConfig(n_levels=3)).evaluate(s, F.EvalSet(np.zeros(0, complex))).potentials.size == 0
    e = F.EvalSet.self_of(s)
    for bad in (dict(theta=1.5), dict(n_levels=0), dict(worker_threads=0)):
        with pytest.raises(F.InvalidParameter):
            F.FmmEngine(F.FmmConfig(**bad)).evaluate(s, e)
    with pytest.raises(F.InvalidInput):
        F.FmmEngine(F.FmmConfig()).evaluate(F.SourceSet(np.zeros(0, complex), np.zeros(0)), e)
    with pytest.raises(F.InvalidParameter):
        F.FmmEngine(F.FmmConfig(m2l_on_device=True)).evaluate(s, e)


def test_concurrent_timing_law_throttled():
    s = F.make_distribution("random", 3000, 8)
    r = F.FmmEngine(F.FmmConfig(n_levels=4, backend="throttled",
                                throttle_latency_s=0.02)).evaluate(s, F.EvalSet.self_of(s))
    t = r.timings
    assert t["cpu_wait"] >= 0.0
    assert t["t_total"] >= max(t["t_m2l"], t["t_p2p"])
    assert t["t_total"] >= max(t["t_m2l"], t["t_p2p"]) + t["t_q"] - 0.05 * t["t_total"]
    assert t["t_p2p"] >= 0.02


def test_synchronous_timings_add_up():
    s = F.make_distribution("random", 1500, 9)
    t = F.FmmEngine(F.FmmConfig(n_levels=3)).evaluate(s, F.EvalSet.self_of(s)).timings
    assert t["cpu_wait"] == 0.0
    assert t["t_total"] >= t["t_q"] + t["t_m2l"] + t["t_p2p"] - 0.02 * t["t_total"] - 1e-5


# ------------------------------------------------------------- operators --
def test_choose_p_and_estimate_cost():
    assert F.choose_p("table", 1e-6, 0.5) == 17
    assert F.choose_p("table", 1e-8, 0.65) == 39
    assert F.choose_p("table", 1e-6, 0.35) == 11
    assert F.choose_p("table", 1e-7, 0.6) == 28
    assert F.choose_p("formula", 1e-6, 0.5) == 19
    assert F.choose_p("formula", 0.9, 0.5) == 1
    for bad in ((0.0, 0.5), (1e-6, 1.5)):
        with pytest.raises(F.InvalidParameter):
            F.choose_p("formula", *bad)
    c = F.estimate_cost(1e6, 6, 0.5, 17)
    assert abs(c["c_p2p"] / 1.3806e10 - 1) < 1e-3 and abs(c["c_m2l"] / 1.2551e7 - 1) < 1e-3
    assert c["c_m2m"] == pytest.approx(4 / 3 * 1024 * 289, rel=1e-12)
    with pytest.raises(F.InvalidParameter):
        F.estimate_cost(1e6, 0, 0.5, 17)


def test_p2p_direct_known_answers():
    s = F.SourceSet(np.array([1 + 0j]), np.array([1 + 0j]))
    assert F.p2p_direct(F.EvalSet.at([0j]), s)[0] == 1 + 0j
    s2 = F.SourceSet(np.array([0j, 1 + 0j]), np.ones(2, complex))
    out = F.p2p_direct(F.EvalSet.self_of(s2), s2)
    assert abs(out[0] - 1) < 1e-15 and abs(out[1] + 1) < 1e-15
    with pytest.raises(F.InvalidInput):
        F.p2p_direct(F.EvalSet.at([0j]), F.SourceSet(np.array([np.inf + 0j]), np.ones(1)))


def test_m2l_host_matches_reference_golden_bitwise():
    g = load_golden("m2l_cases.npz")
    for i in range(int(g["count"])):
        p, kern = int(g[f"{i}_p"]), int(g[f"{i}_kernel"])
        sc = complex(*g[f"{i}_sc"])
        tc = complex(*g[f"{i}_tc"])
        co = g[f"{i}_coeffs"][:, 0] + 1j * g[f"{i}_coeffs"][:, 1]
        l0 = g[f"{i}_local0"][:, 0] + 1j * g[f"{i}_local0"][:, 1]
        got = F.m2l_add(p, ["harmonic", "log"][kern], sc, co, tc, l0)
        assert bitwise(F._c2(got), g[f"{i}_local"]), i


def test_m2l_singular_and_single_source_accuracy():
    with pytest.raises(F.SingularConfiguration):
        F.m2l_add(4, "harmonic", 1 + 1j, np.ones(5, complex), 1 + 1j, np.zeros(5, complex))
    for kern in ("harmonic", "log"):
        b = F.p2m(0.25 + 0.25j, np.array([0.3 + 0.25j]), np.array([1 + 0j]), kern, 17)
        loc = F.m2l_add(17, kern, 0.25 + 0.25j, b, 2.25 + 0.25j, np.zeros(18, complex))
        y = 2.25 + 0.25j + (0.2 - 0.15j)
        w = y - (2.25 + 0.25j)
        approx = sum(loc[k] * w ** k for k in range(18))
        exact = -1 / (y - (0.3 + 0.25j)) if kern == "harmonic" else np.log(y - (0.3 + 0.25j))
        assert abs(approx - exact) <= 1e-6 * max(1.0, abs(exact))


def test_normwise_helper():
    a = np.array([[1.0, 0.0], [0.0, 2.0]])
    assert normwise(a, a) == 0.0


def test_vortex_run_matches_a_python_euler_loop():
    """fmmh_vortex_run (sims::vortex_steps: the update also writes the next
    step's inputs) against a Python loop of engine evaluations with the same
    smoother and time step (pos += dt * conj(phi), m = gamma / (2 pi i)):
    bitwise equal positions after 3 steps (pool backend)."""
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0])
    from test_gpu_config5 import shear_layer
    n, aspect, steps = 2000, 8.0, 3
    cfg = dict(theta=0.5, n_levels=4, p_rule="formula", backend="pool", worker_threads=4)
    _, got = F.vortex_run(n, aspect, steps, F.FmmConfig(**cfg), want_positions=True)
    pos, gam, delta = shear_layer(n, aspect, 2.0 * aspect / n)
    rows = int(round(np.sqrt(n / aspect)))
    rows = max(2, rows - rows % 2)
    while n % rows:
        rows -= 2
    dt = 0.5 * 1.0 / rows
    m = gam * (complex(0.0, -1.0) / (2.0 * np.pi))
    eng = F.FmmEngine(F.FmmConfig(smoother="gaussian", delta=delta, **cfg))
    for _ in range(steps):
        s = F.SourceSet(pos, m)
        r = eng.evaluate(s, F.EvalSet.self_of(s))
        phi = r.potentials
        phi = phi[:, 0] + 1j * phi[:, 1] if phi.ndim == 2 else phi
        pos = pos + dt * np.conj(phi)
    assert np.array_equal(np.asarray(got).view(np.uint64), pos.view(np.uint64))
