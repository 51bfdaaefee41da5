"""Device P2P parity (needs a B200).  Everything goes through the C ABI
(include/fmm_cuda.h) via paper_1311_1006_b200._native.

Bars:
  * pair_evals exactly equal to the reference counter;
  * exact mode (restated __divdc3, reference order): bitwise equal for the
    harmonic kernel without smoother;
  * fast FP64 mode: max|phi_gpu - phi_ref| <= 1e-12 * max|phi_ref|
    (normwise, test_util.hpp:47-57 convention) for every kernel/smoother.
"""
import numpy as np
import pytest

from conftest import bitwise, golden_leaf_csr, golden_permuted, normwise
from oracle import oracle as O
from paper_1311_1006_b200 import _native as N
from paper_1311_1006_b200 import fmm as F

pytestmark = pytest.mark.gpu
TOL_FP64 = 1e-12


@pytest.fixture(scope="module")
def ctx():
    c = N.CudaContext(0)
    yield c
    c.close()


def _run(ctx, pt, ev, so, si, perm, zp, mp, yp, sid, **kw):
    return N.p2p(ctx, pt, ev, so, si, perm, zp, mp, yp, sid, **kw)


@pytest.mark.parametrize("variant", [(0, 0), (1, 0), (0, 1), (0, 2)])
def test_golden_trees_fast_and_exact(ctx, golden_trees, variant):
    k, s = variant
    for name, d in golden_trees.items():
        pt, ev, so, si = golden_leaf_csr(d)
        zp, mp, yp, sid = golden_permuted(d)
        want = d[f"near_k{k}_s{s}"]
        delta = float(d[f"delta_k{k}_s{s}"])
        for mode in (0, 1):
            out, pairs, _ = _run(ctx, pt, ev, so, si, d["perm"], zp, mp, yp, sid, kernel=k,
                                 smoother=s, delta=delta, mode=mode)
            assert pairs == int(d[f"pairs_k{k}_s{s}"]), (name, mode)
            assert normwise(out, want) <= TOL_FP64, (name, mode, normwise(out, want))
            if mode == 1 and k == 0 and s == 0:
                assert bitwise(out, want), name


def _tree_case(kind, n, L, seed, self_eval=True, n_eval=None, theta=0.5):
    s = F.make_distribution(kind, n, seed)
    if self_eval:
        e = F.EvalSet.self_of(s)
    else:
        e = F.EvalSet(F.make_distribution("random", n_eval, seed + 1).z * 1.1 - 0.05)
    t = F.Tree(s, e, L, theta, threads=8)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    return t, (pt, ev, so, si, t.perm, zp, mp, yp, sid)


@pytest.mark.parametrize("case", [(0, 100_000, 6, 1), (0, 100_000, 7, 1), (2, 200_000, 7, 3),
                                  (1, 50_000, 6, 4), (3, 30_000, 5, 5)])
def test_random_trees_vs_oracle(ctx, case):
    kind, n, L, seed = case
    t, args = _tree_case(kind, n, L, seed)
    csr = O.LeafCSR(args[0], args[1], args[2], args[3], args[4])
    want, wpairs = O.nearfield(csr, *args[5:9])
    for mode in (0, 1):
        out, pairs, _ = _run(ctx, *args, mode=mode)
        assert pairs == wpairs
        if mode == 1:
            assert bitwise(out, want)
        else:
            assert normwise(out, want) <= TOL_FP64


def test_separate_eval_points_no_ids(ctx):
    t, args = _tree_case(0, 40_000, 6, 9, self_eval=False, n_eval=25_000)
    csr = O.LeafCSR(*args[:5])
    want, wpairs = O.nearfield(csr, *args[5:9])
    out, pairs, _ = _run(ctx, *args)
    assert pairs == wpairs
    assert normwise(out, want) <= TOL_FP64
    out, pairs, _ = _run(ctx, *args, mode=1)
    assert bitwise(out, want)


def test_lattice_layout_perm_differs_from_eval_perm(ctx):
    g = np.arange(120) * (1.0 / 120)
    z = (g[:, None] + 1j * g[None, :] * 0.25).ravel()
    s = F.SourceSet(z, np.full(len(z), 0.5j))
    e = F.EvalSet.self_of(s)
    t = F.Tree(s, e, 6, 0.5)
    assert not np.array_equal(t.perm, t.eval_perm)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    want, wpairs = O.nearfield(O.LeafCSR(pt, ev, so, si, t.perm), zp, mp, yp, sid, smoother=1,
                               delta=0.01)
    out, pairs, _ = _run(ctx, pt, ev, so, si, t.perm, zp, mp, yp, sid, smoother=1, delta=0.01)
    assert pairs == wpairs
    assert normwise(out, want) <= TOL_FP64


def test_single_box_equals_direct_sum(ctx):
    t, args = _tree_case(3, 3000, 1, 10)
    want, wpairs = O.nearfield(O.LeafCSR(*args[:5]), *args[5:9])
    out, pairs, _ = _run(ctx, *args)
    assert pairs == 3000 * 2999 == wpairs
    assert normwise(out, want) <= TOL_FP64


def test_empty_eval_set_and_empty_leaves(ctx):
    s = F.make_distribution("random", 500, 3)
    t = F.Tree(s, F.EvalSet(np.zeros(0, complex)), 3, 0.5)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    out, pairs, _ = _run(ctx, pt, ev, so, si, t.perm, zp, mp, yp, None)
    assert pairs == 0 and out.size == 0
    # evals concentrated in a corner: most leaves have no evals
    e = F.EvalSet(0.01 * F.make_distribution("random", 50, 4).z)
    t = F.Tree(s, e, 4, 0.5)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    assert (np.diff(ev.astype(np.int64)) == 0).sum() > 0
    want, wp = O.nearfield(O.LeafCSR(pt, ev, so, si, t.perm), zp, mp, yp, None)
    out, pairs, _ = _run(ctx, pt, ev, so, si, t.perm, zp, mp, yp, None)
    assert pairs == wp and normwise(out, want) <= TOL_FP64


def test_heavy_leaves_are_split_and_reduced(ctx):
    """Clustered input with a deep tree: strong lists of thousands of leaves
     exercise the chunked work list and its fixed-order reduction."""
    t, args = _tree_case(2, 300_000, 8, 3)
    so = args[2]
    assert np.diff(so.astype(np.int64)).max() > 1000
    want, wpairs = O.nearfield(O.LeafCSR(*args[:5]), *args[5:9])
    out, pairs, _ = _run(ctx, *args)
    assert pairs == wpairs
    assert normwise(out, want) <= TOL_FP64
    out2, _, _ = _run(ctx, *args)
    assert bitwise(out, out2)  # deterministic


@pytest.mark.parametrize("ordered", [True, False])
def test_leaf_shards_compose_to_the_full_result(ctx, ordered, monkeypatch):
    """Leaf-range launches compose to the whole job: bitwise with the ordered
    list; with the mutual kernel (FMMCU_E2E_SYM=1) pairs across a shard cut
    run ordered, so the bar is 1e-12 normwise -- and exact pair counts."""
    if ordered:
        monkeypatch.setenv("FMMCU_NO_SYM", "1")
    else:
        monkeypatch.setenv("FMMCU_E2E_SYM", "1")
    t, args = _tree_case(0, 120_000, 7, 12)
    full, pairs_full, _ = _run(ctx, *args)
    nl = len(args[0]) - 1
    cuts = [0, nl // 3, nl // 2, nl]
    acc = np.zeros_like(full)
    tot = 0
    for a, b in zip(cuts[:-1], cuts[1:]):
        out, pairs, _ = _run(ctx, *args, leaf_begin=a, leaf_end=b)
        e0, e1 = int(args[1][a]), int(args[1][b])
        acc[e0:e1] = out[e0:e1]
        tot += pairs
    assert tot == pairs_full
    if ordered:
        assert bitwise(acc, full)
    else:
        assert normwise(acc, full) <= TOL_FP64


def test_staged_device_path_matches_launch(ctx):
    t, args = _tree_case(0, 200_000, 7, 2)
    full, pairs_full, _ = _run(ctx, *args)
    job, keep = N.CudaContext.make_job(*args, None)
    ctx.stage(job, keep)
    nl = len(args[0]) - 1
    n = ctx.run_staged(0, nl)
    assert n >= 1
    assert ctx.pairs() == pairs_full
    # self-evaluation: the staged path runs the mutual (symmetric) kernel
    staged = ctx.copy_out(len(full))
    assert normwise(staged, full) <= TOL_FP64
    # potentials written straight into a torch-owned device tensor
    import torch
    buf = torch.zeros(full.size, dtype=torch.float64, device="cuda:0")
    torch.cuda.synchronize()
    ctx.bind_device_out(buf.data_ptr())
    ctx.run_staged(0, nl)
    ctx.synchronize()
    ctx.bind_device_out(None)
    assert bitwise(buf.cpu().numpy().reshape(full.shape), staged)


def test_linearity_at_scale(ctx):
    """Size-independent property at 2M: doubling every strength doubles every
    potential exactly (2x is exact in binary FP), fast mode."""
    t, args = _tree_case(0, 2_000_000, 9, 4)
    out1, p1, _ = _run(ctx, *args)
    args2 = list(args)
    args2[6] = args[6] * 2.0
    out2, p2, _ = _run(ctx, *args2)
    assert p1 == p2
    assert bitwise(out2, 2.0 * out1)
    # spot-check 200 target leaves against the oracle
    nl = len(args[0]) - 1
    rng = np.random.default_rng(0)
    csr = O.LeafCSR(*args[:5])
    for lb in rng.choice(nl, 20, replace=False):
        w, _ = O.nearfield(csr, *args[5:9], leaf_begin=int(lb), leaf_end=int(lb) + 1)
        e0, e1 = int(args[1][lb]), int(args[1][lb + 1])
        assert normwise(out1[e0:e1], w[e0:e1]) <= TOL_FP64


def test_sliced_launch_direct_into_registered_output(ctx):
    """n_eval > 2^20: the launch runs 8 pair-balanced leaf slices whose D2H
    overlaps the next slice.  Staged and page-locked (direct DMA) outputs,
    and the device-resident path agree bitwise, a shard spanning slices to
    1e-12 (its cross-cut pairs run ordered)."""
    t, args = _tree_case(0, 1_500_000, 8, 6)
    staged, p_staged, _ = _run(ctx, *args)
    host = np.full_like(staged, np.nan)
    ctx.host_register(host)
    try:
        out, p_direct, _ = _run(ctx, *args, out=host)
    finally:
        ctx.host_unregister(host)
    assert out is host and p_direct == p_staged
    assert bitwise(host, staged)
    nl = len(args[0]) - 1
    a, b = nl // 5, nl - nl // 7
    part, _, _ = _run(ctx, *args, leaf_begin=a, leaf_end=b)
    e0, e1 = int(args[1][a]), int(args[1][b])
    # (mutual kernel: pairs across the shard cut run ordered -> 1e-12, not bitwise)
    assert normwise(part[e0:e1], staged[e0:e1]) <= TOL_FP64
    job, keep = N.CudaContext.make_job(*args, None)
    ctx.stage(job, keep)
    ctx.run_staged(0, nl)
    assert ctx.pairs() == p_staged
    assert normwise(ctx.copy_out(len(staged)), staged) <= TOL_FP64
    csr = O.LeafCSR(*args[:5])
    for lb in (0, nl // 2, nl - 1):
        w, _ = O.nearfield(csr, *args[5:9], leaf_begin=lb, leaf_end=lb + 1)
        e0, e1 = int(args[1][lb]), int(args[1][lb + 1])
        assert normwise(staged[e0:e1], w[e0:e1]) <= TOL_FP64


def test_page_locked_inputs_take_the_dma_path(ctx):
    """Page-locked z / m: the launch DMAs them as-is and packs the records on
    the device; results bitwise equal to the staged-copy path, and for a
    layout that is not self-evaluation (separate evals) too."""
    for self_eval in (True, False):
        t, args = _tree_case(0, 1_200_000, 8, 21, self_eval=self_eval, n_eval=700_000)
        want, pw, _ = _run(ctx, *args)
        zp = np.ascontiguousarray(args[5]).copy()
        mp = np.ascontiguousarray(args[6]).copy()
        out = np.zeros_like(want)
        for a in (zp, mp, out):
            ctx.host_register(a)
        try:
            a2 = list(args)
            a2[5], a2[6] = zp, mp
            got, pg, _ = _run(ctx, *a2, out=out)
        finally:
            for a in (zp, mp, out):
                ctx.host_unregister(a)
        assert pg == pw
        assert bitwise(got, want)


def test_one_array_for_both_positions(ctx):
    """Self-evaluation with page-locked inputs and one array passed as both
    src_z and eval_y: the per-chunk self check then reads only the ids.  The
    result is bitwise the separate-array result; with ids that do not match
    the sources (a shuffled sid) the chunks fall back to uploaded evals and
    still match the separate-array launch."""
    t, args = _tree_case(0, 1_200_000, 8, 23, self_eval=True)
    zp = np.ascontiguousarray(args[5]).copy()
    mp = np.ascontiguousarray(args[6]).copy()
    for a in (zp, mp):
        ctx.host_register(a)
    try:
        for shuffle in (False, True):
            a2 = list(args)
            a2[5], a2[6] = zp, mp
            if shuffle:
                sid = np.asarray(a2[8]).copy()
                sid[:1000] = np.roll(sid[:1000], 1)
                a2[8] = sid
            a2[7] = zp.copy()
            want, pw, _ = _run(ctx, *a2)
            a2[7] = zp  # the same array for both positions
            got, pg, _ = _run(ctx, *a2)
            assert pg == pw
            assert bitwise(got, want)
    finally:
        for a in (zp, mp):
            ctx.host_unregister(a)


@pytest.mark.parametrize("case", [(0, 200_000, 7, 31, 0), (0, 150_000, 7, 32, 1),
                                  (2, 200_000, 7, 33, 0), (3, 60_000, 6, 34, 2)])
def test_symmetric_kernel_vs_oracle(ctx, case):
    """Self-evaluation through the staged path runs the mutual kernel
    (p2p_sym.cuh): each leaf pair once, contributions reduced in a fixed
    order.  Pair counts exact, potentials <= 1e-12 normwise of the oracle,
    deterministic, and a leaf-range job (ordered runs outside the range)."""
    kind, n, L, seed, sm = case
    t, args = _tree_case(kind, n, L, seed)
    delta = 0.01 if sm else 0.0
    csr = O.LeafCSR(*args[:5])
    want, wpairs = O.nearfield(csr, *args[5:9], smoother=sm, delta=delta)
    nl = len(args[0]) - 1
    outs = []
    for rep in range(2):
        job, keep = N.CudaContext.make_job(*args, None, smoother=sm, delta=delta)
        ctx.stage(job, keep)
        ctx.run_staged(0, nl)
        assert ctx.pairs() == wpairs
        outs.append(ctx.copy_out(len(want)))
    assert normwise(outs[0], want) <= TOL_FP64
    assert bitwise(outs[0], outs[1])
    # a leaf range: partners outside it run as ordered pairs
    a, b = nl // 4, nl - nl // 3
    job, keep = N.CudaContext.make_job(*args, None, smoother=sm, delta=delta,
                                       leaf_begin=a, leaf_end=b)
    ctx.stage(job, keep)
    ctx.run_staged(a, b)
    part = ctx.copy_out(len(want))
    e0, e1 = int(args[1][a]), int(args[1][b])
    assert normwise(part[e0:e1], want[e0:e1]) <= TOL_FP64
    # a symmetric list staged for [a, b) must refuse another range (its
    # contribution slots only cover pairs inside [a, b)); an ordinary list
    # (a leaf of the range with more than 256 entries once its in-range lower
    # partners are dropped: the clustered case) runs any range exactly
    so, si = args[2], args[3]
    most = max(int(((r < a) | (r >= i)).sum()) for i in range(a, b)
               for r in [si[so[i]:so[i + 1]]])
    sym, _ = ctx.kernel_info()
    assert sym == (most <= 256)
    if sym:
        with pytest.raises(N.FmmcuError) as ei:
            ctx.run_staged(0, nl)
        assert ei.value.code == 6  # FMMCU_ESTATE
    else:
        ctx.run_staged(0, nl)
        assert ctx.pairs() == wpairs
        assert normwise(ctx.copy_out(len(want)), want) <= TOL_FP64
    # uniform inputs always take the mutual kernel
    if kind == 0:
        assert sym


@pytest.mark.parametrize("case", [(0, 50_000, 6, 0.15, 0, 35), (1, 50_000, 6, 0.2, 1, 36),
                                  (0, 50_000, 6, 0.15, 2, 37)])
def test_symmetric_kernel_entry_rounds(ctx, case):
    """Leaves with more than 32 strong entries (small theta, or the
    non-uniform distribution) run the mutual kernel's entry-round
    instantiation (p2p_sym.cuh ROUNDS: 32 entries per round over the same
    evals, chunks continuing across rounds).  Pair counts exact, <= 1e-12
    normwise of the oracle, deterministic; the launch path (ordered device
    work list) agrees to the same bar."""
    kind, n, L, theta, sm, seed = case
    t, args = _tree_case(kind, n, L, seed, theta=theta)
    so, si = args[2], args[3]
    upper = [int((si[so[i]:so[i + 1]] >= i).sum()) for i in range(len(so) - 1)]
    assert 32 < max(upper) <= 256  # the case exercises entry rounds
    delta = 0.01 if sm else 0.0
    csr = O.LeafCSR(*args[:5])
    want, wpairs = O.nearfield(csr, *args[5:9], smoother=sm, delta=delta)
    nl = len(args[0]) - 1
    outs = []
    for rep in range(2):
        job, keep = N.CudaContext.make_job(*args, None, smoother=sm, delta=delta)
        ctx.stage(job, keep)
        ctx.run_staged(0, nl)
        assert ctx.kernel_info()[0]
        assert ctx.pairs() == wpairs
        outs.append(ctx.copy_out(len(want)))
    assert normwise(outs[0], want) <= TOL_FP64
    assert bitwise(outs[0], outs[1])
    dev, pd, _ = _run(ctx, *args, smoother=sm, delta=delta)
    assert pd == wpairs
    assert normwise(dev, want) <= TOL_FP64


def test_invalid_jobs_fail_loudly(ctx):
    t, args = _tree_case(0, 1000, 3, 1)
    with pytest.raises(N.FmmcuError):
        _run(ctx, *args, kernel=7)
    with pytest.raises(N.FmmcuError):
        _run(ctx, *args, smoother=1, delta=0.0)
    bad = list(args)
    bad[3] = args[3].copy()
    bad[3][0] = 10**6
    with pytest.raises(N.FmmcuError):
        _run(ctx, *bad)
    with pytest.raises(N.FmmcuError):
        ctx.finish()


@pytest.mark.parametrize("pinned", [False, True])
def test_device_work_list_equals_host_work_list(ctx, pinned, monkeypatch):
    """fmmcu_p2p_launch builds its work list on the device (p2p_worklist.cuh)
    from the uploaded CSR, grouped by upload chunk; FMMCU_HOST_WL=1 selects
    the host builder.  Same items in the same order: bitwise equal potentials
    and equal pair counts for whole jobs, leaf shards (halo-only uploads) and
    split heavy leaves, with pageable and page-locked inputs."""
    # the ordered list on both sides (self-evaluation jobs would otherwise
    # take the grouped mutual list: test_launch_mutual_kernel_grouped)
    monkeypatch.setenv("FMMCU_NO_SYM", "1")
    cases = [_tree_case(0, 1_500_000, 8, 41)[1], _tree_case(2, 300_000, 8, 3)[1],
             _tree_case(3, 80_000, 6, 42, self_eval=False, n_eval=50_000)[1]]
    for args in cases:
        args = list(args)
        nl = len(args[0]) - 1
        reg = []
        if pinned:
            args[5] = np.ascontiguousarray(args[5]).copy()
            args[6] = np.ascontiguousarray(args[6]).copy()
            reg = [args[5], args[6]]
            for a in reg:
                ctx.host_register(a)
        try:
            for lb, le in ((0, nl), (nl // 5, nl // 2)):
                dev, pd, _ = _run(ctx, *args, leaf_begin=lb, leaf_end=le)
                monkeypatch.setenv("FMMCU_HOST_WL", "1")
                host, ph, _ = _run(ctx, *args, leaf_begin=lb, leaf_end=le)
                monkeypatch.delenv("FMMCU_HOST_WL")
                e0, e1 = int(args[1][lb]), int(args[1][le])
                assert pd == ph
                assert bitwise(dev[e0:e1], host[e0:e1])
        finally:
            for a in reg:
                ctx.host_unregister(a)


def test_launch_mutual_kernel_grouped(ctx, monkeypatch):
    """FMMCU_E2E_SYM=1: self-evaluation through fmmcu_p2p_launch (the e2e
    path) runs the mutual kernel on a list grouped by upload chunk
    (worklist_dev.cu, build_sym_worklist_dev with groups): pairs inside a
    group once, across groups ordered; each group's finalize stores its own
    chunk to device memory for a copy-engine D2H and the other leaves
    straight into the host output.  Against the ordered launch: equal pair
    counts, <= 1e-12 normwise; deterministic; page-locked and pageable
    inputs; more than 32 entries per leaf (entry rounds); and a job whose
    first ids match their sources but a later chunk does not falls back to
    the ordered list (bitwise equal to it)."""
    monkeypatch.setenv("FMMCU_E2E_SYM", "1")
    for kind, n, L, seed, theta in ((0, 2_500_000, 9, 51, 0.5), (0, 1_200_000, 8, 52, 0.2),
                                    (2, 1_500_000, 8, 53, 0.5)):
        t, args = _tree_case(kind, n, L, seed, theta=theta)
        args = list(args)
        for pinned in (False, True):
            reg = []
            if pinned:
                args[5] = np.ascontiguousarray(args[5]).copy()
                args[6] = np.ascontiguousarray(args[6]).copy()
                reg = [args[5], args[6]]
                for a in reg:
                    ctx.host_register(a)
            try:
                a1, p1, _ = _run(ctx, *args)
                sym, _ = ctx.kernel_info()
                a2, p2, _ = _run(ctx, *args)
                monkeypatch.setenv("FMMCU_NO_SYM", "1")
                want, pw, _ = _run(ctx, *args)
                monkeypatch.delenv("FMMCU_NO_SYM")
            finally:
                for a in reg:
                    ctx.host_unregister(a)
            if kind == 0:
                assert sym
            assert p1 == pw and p2 == pw
            assert bitwise(a1, a2)
            assert normwise(a1, want) <= TOL_FP64
    # fallback: the positions of one point in the second upload chunk moved
    t, args = _tree_case(0, 2_500_000, 9, 54)
    args = list(args)
    yp = np.array(args[7], copy=True)
    yp.reshape(-1)[2 * 1_600_000] += 1e-9
    args[7] = yp
    got, pg, _ = _run(ctx, *args)
    assert not ctx.kernel_info()[0]
    monkeypatch.setenv("FMMCU_NO_SYM", "1")
    want, pw, _ = _run(ctx, *args)
    monkeypatch.delenv("FMMCU_NO_SYM")
    assert pg == pw
    assert bitwise(got, want)
