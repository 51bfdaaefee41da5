"""End-to-end FmmEngine with the cuda backend (and device M2L) vs the reference.

* exact mode: the device near field is bitwise equal to the reference and the
  host far field is the same arithmetic, so evaluate() is bitwise equal to
  the reference FmmEngine::evaluate (golden fixtures) for harmonic/none;
* fast mode: <= 1e-12 normwise; counters identical;
* m2l_on_device: <= 1e-12 normwise; m2l_ops identical;
* the concurrent-backend contract: cpu_wait >= 0, t_p2p > 0.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import bitwise, normwise
from oracle import oracle as O
from paper_1311_1006_b200 import _native as N
from paper_1311_1006_b200 import fmm as F

pytestmark = pytest.mark.gpu


def _sets(d):
    s = F.SourceSet(d["z"][:, 0] + 1j * d["z"][:, 1], d["m"][:, 0] + 1j * d["m"][:, 1])
    e = F.EvalSet(d["y"][:, 0] + 1j * d["y"][:, 1], d["sid"] if "sid" in d else None)
    return s, e


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("m2l_dev", [False, True])
def test_engine_cuda_vs_reference_golden(golden_trees, exact, m2l_dev):
    for name, d in golden_trees.items():
        s, e = _sets(d)
        eng = F.FmmEngine(F.FmmConfig(theta=float(d["theta"]), n_levels=int(d["n_levels"]),
                                      backend="cuda", exact=exact, m2l_on_device=m2l_dev,
                                      worker_threads=4))
        r = eng.evaluate(s, e)
        got = F._c2(r.potentials)
        assert [r.counters[k] for k in F.COUNTER_KEYS] == d["eval_counters"].tolist(), name
        if exact and not m2l_dev:
            assert bitwise(got, d["eval_pot"]), name
        else:
            assert normwise(got, d["eval_pot"]) <= 1e-12, (name, normwise(got, d["eval_pot"]))
        t = r.timings
        assert t["cpu_wait"] >= 0.0 and t["t_p2p"] > 0.0


@pytest.mark.parametrize("case", [("uniform", 400_000, 8, "harmonic", "none", 0.0),
                                  ("gauss8", 200_000, 8, "harmonic", "none", 0.0),
                                  ("positive", 100_000, 7, "log", "none", 0.0),
                                  ("uniform", 100_000, 7, "harmonic", "gaussian", 2e-3)])
def test_engine_cuda_vs_cpu_engine(case):
    """The CPU pool engine is bitwise the reference (test_host_engine.py), so it
    is the reference here at sizes the golden files do not cover."""
    kind, n, L, kern, sm, delta = case
    s = F.make_distribution(kind, n, 17)
    e = F.EvalSet.self_of(s)
    base = dict(n_levels=L, kernel=kern, smoother=sm, delta=delta, worker_threads=16)
    ref = F.FmmEngine(F.FmmConfig(backend="pool", **base)).evaluate(s, e)
    for m2l_dev in (False, True):
        got = F.FmmEngine(F.FmmConfig(backend="cuda", m2l_on_device=m2l_dev, **base)).evaluate(s, e)
        assert got.counters == ref.counters
        a, b = F._c2(got.potentials), F._c2(ref.potentials)
        if kern == "log":  # only the real part of the log potential is branch-free
            a, b = a.copy(), b.copy()
            a[:, 1] = 0.0
            b[:, 1] = 0.0
        assert normwise(a, b) <= 1e-12


def test_device_m2l_matches_reference_operator():
    """Batched device M2L against the reference m2l_add (golden cases incl. the
    long double branch): each case is one target with one partner."""
    from conftest import load_golden
    g = load_golden("m2l_cases.npz")
    ctx = N.CudaContext(0)
    for i in range(int(g["count"])):
        p, kern = int(g[f"{i}_p"]), int(g[f"{i}_kernel"])
        centers = np.stack([g[f"{i}_tc"], g[f"{i}_sc"]])
        coeffs = np.stack([np.zeros((p + 1, 2)), g[f"{i}_coeffs"]])
        out, ops, _ = ctx.m2l(p, kern, centers, coeffs, np.array([0]), np.array([0, 1]),
                              np.array([1]))
        want = g[f"{i}_local"] - g[f"{i}_local0"]
        assert ops == 1
        assert normwise(out[0], want) <= 1e-12, (i, p, kern, normwise(out[0], want))
    ctx.close()


def test_device_m2l_pinned_buffers_equal_pageable():
    """fmmcu_m2l_host_buffers: the same job flattened into the context's
    page-locked buffers (DMA'd in place, sums D2H'd into the pinned out) gives
    bitwise the pageable-input result; the buffers are reused across sizes."""
    rng = np.random.default_rng(5)
    ctx = N.CudaContext(0)
    for nb, nt, p in ((3000, 2000, 17), (500, 400, 9), (5000, 4500, 17)):
        centers = rng.random((nb, 2))
        coeffs = rng.standard_normal((nb, p + 1, 2)) * 1e-3
        target_box = rng.choice(nb, nt, replace=False).astype(np.uint32)
        deg = rng.integers(0, 30, nt)
        weak_off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint32)
        weak_idx = rng.integers(0, nb, int(weak_off[-1])).astype(np.uint32)
        # no coincident centres: partners distinct from their target
        weak_idx = np.where(weak_idx == np.repeat(target_box, deg), (weak_idx + 1) % nb, weak_idx)
        a, oa, _ = ctx.m2l(p, 0, centers, coeffs, target_box, weak_off, weak_idx)
        b, ob, _ = ctx.m2l_pinned(p, 0, centers, coeffs, target_box, weak_off, weak_idx)
        assert oa == ob == int(weak_off[-1])
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    ctx.close()


def test_device_downward_pass_vs_restated_l2l():
    """fmmcu_m2l_downward on a 4-level toy pyramid (1 + 4 + 16 + 64 boxes,
    children of box i are 4i..4i+3 of the next level): every box of levels
    >= 1 except a few (no evals) is a target with random partners; the
    finest locals against local = l2l_add(parent) + own M2L sum restated in
    numpy (sum_k C(k,l) d^(k-l) a_k, expansion.cpp l2l_add), <= 1e-12
    normwise; a downward call without a keep-on-device launch is refused."""
    from math import comb
    rng = np.random.default_rng(7)
    p, L = 12, 4
    sizes = [4 ** l for l in range(L)]
    level_base = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    nb = int(level_base[-1])
    centers = np.zeros((nb, 2))
    for l in range(L):
        n = sizes[l]
        side = 2 ** l
        idx = np.arange(n)
        centers[level_base[l]:level_base[l + 1], 0] = (idx % side + 0.5) / side
        centers[level_base[l]:level_base[l + 1], 1] = (idx // side + 0.5) / side
    coeffs = rng.standard_normal((nb, p + 1, 2)) * 1e-2
    empty = set(int(x) for x in rng.choice(np.arange(level_base[3], nb), 6, replace=False))
    # a box without evals has children without evals
    is_t = np.zeros(nb, dtype=bool)
    is_t[level_base[1]:] = True
    for g in list(empty):
        is_t[g] = False
    targets = np.nonzero(is_t)[0].astype(np.uint32)
    target_of = np.full(nb, -1, dtype=np.int32)
    target_of[targets] = np.arange(len(targets))
    weak, off = [], [0]
    for g in targets:
        lvl = int(np.searchsorted(level_base, g, side="right") - 1)
        cand = np.arange(level_base[lvl], level_base[lvl + 1])
        cand = cand[np.abs(centers[cand] - centers[g]).max(axis=1) > 1.5 / 2 ** lvl]
        pick = rng.choice(cand, min(len(cand), 5), replace=False) if len(cand) else []
        weak.extend(sorted(int(x) for x in pick))
        off.append(len(weak))
    weak_off, weak_idx = np.array(off, dtype=np.uint32), np.array(weak, dtype=np.uint32)
    ctx = N.CudaContext(0)
    sums, _, _ = ctx.m2l(p, 0, centers, coeffs, targets, weak_off, weak_idx)
    fin, ops = ctx.m2l_downward(p, 0, centers, coeffs, targets, weak_off, weak_idx, level_base,
                                target_of)
    assert ops == len(weak_idx)
    s = sums[..., 0] + 1j * sums[..., 1]
    cz = centers[:, 0] + 1j * centers[:, 1]
    loc = {}
    for l in range(1, L):
        for i in range(sizes[l]):
            g = int(level_base[l]) + i
            if target_of[g] < 0:
                continue
            v = np.zeros(p + 1, dtype=complex)
            if l >= 2:
                pg = int(level_base[l - 1]) + i // 4
                a, d = loc[pg], cz[g] - cz[pg]
                for ll in range(p + 1):
                    v[ll] += sum(comb(k, ll) * d ** (k - ll) * a[k] for k in range(ll, p + 1))
            loc[g] = v + s[target_of[g]]
    got = fin[..., 0] + 1j * fin[..., 1]
    for i in range(sizes[L - 1]):
        g = int(level_base[L - 1]) + i
        if target_of[g] >= 0:
            assert np.abs(got[i] - loc[g]).max() <= 1e-12 * max(1.0, np.abs(loc[g]).max())
    with pytest.raises(N.FmmcuError) as ei:
        d = N.L2LJob()
        ctx._check(ctx.lib.fmmcu_m2l_downward(ctx.h, C.byref(d)))
    assert ei.value.code == 6  # FMMCU_ESTATE: no keep-on-device launch in flight
    ctx.close()


def test_device_m2l_singular_raises():
    ctx = N.CudaContext(0)
    centers = np.array([[0.5, 0.5], [0.5, 0.5]])
    coeffs = np.ones((2, 5, 2))
    with pytest.raises(N.FmmcuError) as ei:
        ctx.m2l(4, 0, centers, coeffs, np.array([0]), np.array([0, 1]), np.array([1]))
    assert ei.value.code == N.FMMCU_ESINGULAR
    ctx.close()


def test_vortex_sheet_steps_cuda_vs_pool():
    """Config-5 driver (Gaussian smoother, p from the formula, AT3b wiring) on a
    small sheet: device and CPU runs produce the same trajectory."""
    cfg = dict(n_levels=5, p_rule="formula", worker_threads=8)
    tr_c, pos_c = F.vortex_run(20_000, 8.0, 3, F.FmmConfig(backend="cuda", **cfg), tuner="none",
                               want_positions=True)
    tr_p, pos_p = F.vortex_run(20_000, 8.0, 3, F.FmmConfig(backend="pool", **cfg), tuner="none",
                               want_positions=True)
    assert np.array_equal(tr_c[:, 7], tr_p[:, 7])  # identical pair counts per step
    assert np.abs(pos_c - pos_p).max() <= 1e-12 * np.abs(pos_p).max()


def test_engine_device_pipeline_vs_reference_golden(golden_trees):
    """FmmConfig.device_pipeline: the whole evaluate() on the GPU against the
    reference's own evaluate() outputs (golden fixtures): counters identical,
    potentials <= 1e-12 normwise."""
    for name, d in golden_trees.items():
        s, e = _sets(d)
        eng = F.FmmEngine(F.FmmConfig(theta=float(d["theta"]), n_levels=int(d["n_levels"]),
                                      backend="cuda", device_pipeline=True))
        r = eng.evaluate(s, e)
        assert [r.counters[k] for k in F.COUNTER_KEYS] == d["eval_counters"].tolist(), name
        assert normwise(F._c2(r.potentials), d["eval_pot"]) <= 1e-12, name
        assert r.timings["t_total"] > 0 and r.timings["t_p2p"] > 0


@pytest.mark.parametrize("dist,n,L", [("uniform", 200_000, 7), ("gauss8", 200_000, 8)])
def test_engine_device_pipeline_vs_pool(dist, n, L):
    s = F.make_distribution(dist, n, 5)
    e = F.EvalSet.self_of(s)
    ref = F.FmmEngine(F.FmmConfig(n_levels=L, backend="pool", worker_threads=8)).evaluate(s, e)
    r = F.FmmEngine(F.FmmConfig(n_levels=L, backend="cuda", device_pipeline=True)).evaluate(s, e)
    assert r.counters == ref.counters
    assert np.abs(r.potentials - ref.potentials).max() <= 1e-12 * np.abs(ref.potentials).max()


def test_engine_device_pipeline_requires_cuda_backend():
    s = F.make_distribution("uniform", 1000, 1)
    with pytest.raises(F.InvalidParameter):
        F.FmmEngine(F.FmmConfig(n_levels=3, backend="pool", device_pipeline=True)).evaluate(
            s, F.EvalSet.self_of(s))


def test_m2l_table_reupload_across_fresh_engines(golden_trees):
    """the M2L binomial table and the far-field Pascal rows
    are uploaded on the consuming stream.  Fresh engines alternating theta
    (hence p: 0.3 -> p=25, 0.5 -> 17, 0.7 -> 39 by PRule::table) and kernel,
    in a shuffled order, must each match the pool engine on the same input."""
    rng = np.random.default_rng(7)
    items = list(golden_trees.items())
    runs = []
    for rep in range(3):
        for name, d in items:
            for theta in (0.3, 0.5, 0.7):
                runs.append((name, theta, bool(rep % 2)))
    rng.shuffle(runs)
    refs = {}
    for name, theta, pipe in runs[:40]:
        d = golden_trees[name]
        s, e = _sets(d)
        base = dict(theta=theta, n_levels=int(d["n_levels"]), worker_threads=4)
        key = (name, theta)
        if key not in refs:
            refs[key] = F.FmmEngine(F.FmmConfig(backend="pool", **base)).evaluate(s, e)
        ref = refs[key]
        extra = dict(device_pipeline=True) if pipe else dict(m2l_on_device=True)
        got = F.FmmEngine(F.FmmConfig(backend="cuda", **extra, **base)).evaluate(s, e)
        assert got.counters == ref.counters, (name, theta, pipe)
        err = normwise(F._c2(got.potentials), F._c2(ref.potentials))
        assert err <= 1e-12, (name, theta, pipe, err)


def test_device_pipeline_wait_signal_sign():
    """The device pipeline reports the reference's wait signal (engine.cpp:312)
    from device events: the far chain's idle tail before the P2P ends.  A
    shallow tree (thousands of points per leaf) is near-field bound -> wait
    > 0; a very deep one (< 1 point per leaf) is far-field bound -> wait 0."""
    s = F.make_distribution("uniform", 400_000, 9)
    e = F.EvalSet.self_of(s)
    shallow = F.FmmEngine(F.FmmConfig(n_levels=4, backend="cuda", device_pipeline=True))
    deep = F.FmmEngine(F.FmmConfig(n_levels=10, backend="cuda", device_pipeline=True))
    for _ in range(2):  # second call: warm allocations
        ws = shallow.evaluate(s, e).timings
        wd = deep.evaluate(s, e).timings
    assert ws["cpu_wait"] > 0.0, ws
    assert wd["cpu_wait"] == 0.0, wd
    assert ws["cpu_wait"] <= ws["t_total"]


def test_at3a_moves_levels_with_device_wait_signal():
    """AT3a (autotune.cpp:155) steers n_levels by the wait sign.  Starting far
    too shallow for 60k vortices (~3750 per leaf), the device pipeline's wait
    is positive, so AT3a must deepen the tree (the r1 hard-coded zero walked
    it the other way)."""
    cfg = F.FmmConfig(n_levels=3, p_rule="formula", backend="cuda", device_pipeline=True)
    tr, _ = F.vortex_run(60_000, 8.0, 25, cfg, tuner="at3a")
    assert (tr[:12, 4] > 0).all()  # near-bound: positive wait
    assert tr[-1, 6] > 3, tr[:, 6]


@pytest.mark.parametrize("dist,n,L", [("uniform", 300_000, 8), ("gauss8", 200_000, 8)])
def test_engine_cuda_multi_context_shards_vs_pool(dist, n, L):
    """CudaSettings.devices with several entries: the target leaves are split
    into pair-work-balanced ranges, one context each, every context uploading
    only its halo and writing its slice of the potentials; with three
    contexts on the one test GPU (devices=(0, 0, 0)) the result must match
    the CPU pool engine: identical counters, <= 1e-12 normwise."""
    s = F.make_distribution(dist, n, 21)
    e = F.EvalSet.self_of(s)
    base = dict(n_levels=L, worker_threads=8)
    ref = F.FmmEngine(F.FmmConfig(backend="pool", **base)).evaluate(s, e)
    for devs in ((0, 0), (0, 0, 0)):
        got = F.FmmEngine(F.FmmConfig(backend="cuda", devices=devs, **base)).evaluate(s, e)
        assert got.counters == ref.counters, devs
        assert normwise(F._c2(got.potentials), F._c2(ref.potentials)) <= 1e-12, devs


@pytest.mark.parametrize("m2l_dev", [False, True])
def test_hybrid_device_tree_equals_host_tree(golden_trees, m2l_dev):
    """FmmConfig.device_tree: the hybrid engine builds the pyramid and lists
    on the GPU (fmmcu_tree_build) and reads them back for the CPU far field.
    The device tree is bit-exact, and everything downstream is the same
    code, so the potentials are bitwise those of the host-tree hybrid, with
    equal counters -- golden trees (ties, separate evals, theta 0.65), a
    lattice with tied splits and a clustered set."""
    cases = [(_sets(d), int(d["n_levels"]), float(d["theta"])) for d in golden_trees.values()]
    g = np.arange(120) / 120.0
    lat = F.SourceSet((g[:, None] + 1j * g[None, :] * 0.25).ravel(), np.full(14400, 0.5j))
    cases.append(((lat, F.EvalSet.self_of(lat)), 6, 0.5))
    s = F.make_distribution("gauss8", 60_000, 7)
    cases.append(((s, F.EvalSet.self_of(s)), 6, 0.5))
    for (s, e), L, theta in cases:
        base = dict(n_levels=L, theta=theta, backend="cuda", m2l_on_device=m2l_dev,
                    worker_threads=8)
        a = F.FmmEngine(F.FmmConfig(**base)).evaluate(s, e)
        b = F.FmmEngine(F.FmmConfig(device_tree=True, **base)).evaluate(s, e)
        assert a.counters == b.counters
        assert np.array_equal(a.potentials.view(np.uint64), b.potentials.view(np.uint64))


def test_hybrid_device_downward_bitwise_equal_to_host_l2l(tmp_path):
    """The hybrid engine's device downward pass (fmmcu_m2l_downward, default)
    and its host L2L chain (FMM_HOST_L2L=1, read once per process, hence the
    subprocesses) give bitwise the same potentials: the device restates
    l2l_add's arithmetic operation for operation."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "from paper_1311_1006_b200 import fmm as F\n"
        "s = F.make_distribution('gauss8', 200000, 3); e = F.EvalSet.self_of(s)\n"
        "r = F.FmmEngine(F.FmmConfig(n_levels=7, backend='cuda', m2l_on_device=True,"
        " worker_threads=8)).evaluate(s, e)\n"
        "np.save(sys.argv[1], np.asarray(r.potentials))\n")
    out = {}
    for tag, extra in (("dev", {}), ("host", {"FMM_HOST_L2L": "1"})):
        path = str(tmp_path / f"{tag}.npy")
        env = {k: v for k, v in os.environ.items() if k != "FMM_HOST_L2L"}
        env.update(extra)
        subprocess.run([sys.executable, "-c", code, path], env=env, check=True, timeout=300)
        out[tag] = np.load(path)
    assert np.array_equal(out["dev"].view(np.uint64), out["host"].view(np.uint64))
