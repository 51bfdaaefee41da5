"""Parity at the headline size (BASELINE config 4; needs a B200).

N = 10,000,000 uniform points (make_distribution seed 4), self-evaluation,
n_levels = 10 (262,144 leaves, 38-39 points each), theta = 0.5, harmonic,
no smoother: exactly the workload bench.py reports.  The full result cannot
be re-run on the CPU in test time, so (oracle/parity.py):

* the TOTAL pair count is checked exactly against the reference identity
  Σ_leaves n_evals·S − self hits evaluated over every leaf;
* the potentials are checked against the restated near_box (backend.cpp:41-89)
  on a stratified sample of >= 4096 target leaves: 64 evenly spread blocks of
  64 leaves, the first and last leaves, and a block straddling every cut of a
  2-, 4- and 8-way shard split;
* fast FP64 paths: <= 1e-12 normwise on the sample; the exact path: bitwise.

Paths: the staged mutual kernel (p2p_sym_kernel, the bench `value`), the
reference-facing C ABI launch/finish (the bench `e2e`), the bit-compatible
exact kernel, and an 8-way shard split run leaf range by leaf range (the
multi-GPU partition of bench.py, here on one device).
"""
import os

import numpy as np
import pytest

from oracle import parity as P
from paper_1311_1006_b200 import _native as N
from paper_1311_1006_b200 import fmm as F
from paper_1311_1006_b200.sharding import shard_cuts

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL_FP64 = 1e-12


@pytest.fixture(scope="module")
def c4():
    s = F.make_distribution("uniform", 10_000_000, 4)
    e = F.EvalSet.self_of(s)
    t = F.Tree(s, e, 10, 0.5, threads=os.cpu_count() or 8)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    perm = t.perm
    del t, s, e
    per_leaf = P.pair_identity(pt, ev, so, si, perm, sid)
    prefix = np.concatenate([[0], np.cumsum(per_leaf)])
    cuts = sorted({int(c) for w in (2, 4, 8) for c in shard_cuts(prefix, w)})
    blocks = P.leaf_blocks(len(pt) - 1, cuts=cuts, n_blocks=64, block=64)
    return dict(args=(pt, ev, so, si, perm, zp, mp, yp, sid), total=int(per_leaf.sum()),
                prefix=prefix, blocks=blocks, n_leaves=len(pt) - 1, n_eval=len(yp))


@pytest.fixture(scope="module")
def ctx():
    c = N.CudaContext(0)
    yield c
    c.close()


def _check(c4, got, bitwise=False):
    r = P.sampled_check(got, *c4["args"], blocks=c4["blocks"], bitwise=bitwise)
    assert r["leaves"] >= 4096
    assert r["pair_identity_ok"]
    return r


def test_sample_covers_edges_and_cuts(c4):
    b = c4["blocks"]
    assert b[0][0] == 0 and b[-1][1] == c4["n_leaves"]
    assert c4["n_leaves"] == 4 ** 9
    assert c4["total"] == 4954189552  # the bench's pairs/step (BENCH_r01)


def test_config4_staged_mutual_kernel(ctx, c4):
    job, keep = N.CudaContext.make_job(*c4["args"], None)
    ctx.stage(job, keep)
    sym, _ = ctx.kernel_info()
    assert sym, "config 4 (<= 32 strong entries per leaf) must take the mutual kernel"
    ctx.run_staged(0, c4["n_leaves"])
    assert ctx.pairs() == c4["total"]
    got = ctx.copy_out(c4["n_eval"])
    r = _check(c4, got)
    assert r["normwise"] <= TOL_FP64, r
    # deterministic: a second run is bitwise identical on the whole array
    ctx.run_staged(0, c4["n_leaves"])
    again = ctx.copy_out(c4["n_eval"])
    assert np.array_equal(got.view(np.uint64), again.view(np.uint64))


def test_config4_c_abi_launch_path(ctx, c4):
    pt, ev, so, si, perm, zp, mp, yp, sid = c4["args"]
    out, pairs, _ = N.p2p(ctx, pt, ev, so, si, perm, zp, mp, zp, sid)  # e2e: one array for y, z
    assert pairs == c4["total"]
    r = _check(c4, out)
    assert r["normwise"] <= TOL_FP64, r


def test_config4_grouped_mutual_launch(ctx, c4, monkeypatch):
    """FMMCU_E2E_SYM=1: the C-ABI launch with the mutual kernel on the list
    grouped by upload chunk (10 groups at 10M) and the split finalize."""
    monkeypatch.setenv("FMMCU_E2E_SYM", "1")
    pt, ev, so, si, perm, zp, mp, yp, sid = c4["args"]
    out, pairs, _ = N.p2p(ctx, pt, ev, so, si, perm, zp, mp, zp, sid)
    assert ctx.kernel_info()[0]
    assert pairs == c4["total"]
    r = _check(c4, out)
    assert r["normwise"] <= TOL_FP64, r


def test_config4_exact_mode_bitwise(ctx, c4):
    out, pairs, _ = N.p2p(ctx, *c4["args"], mode=1)
    assert pairs == c4["total"]
    r = _check(c4, out, bitwise=True)
    assert r["bit_mismatches"] == 0, r


def test_config4_eight_way_shards(ctx, c4):
    """The bench's 8-rank partition, one leaf range at a time: each shard's
    mutual work list covers only its range (partners outside it run as
    ordered pairs); the slices assembled together match the oracle and the
    shard pair counts add up to the total."""
    cuts = shard_cuts(c4["prefix"], 8)
    pt, ev = c4["args"][0], c4["args"][1]
    full = np.zeros((c4["n_eval"], 2))
    total = 0
    for r in range(8):
        a, b = int(cuts[r]), int(cuts[r + 1])
        job, keep = N.CudaContext.make_job(*c4["args"], None, leaf_begin=a, leaf_end=b)
        ctx.stage(job, keep)
        ctx.run_staged(a, b)
        total += ctx.pairs()
        e0, e1 = int(ev[a]), int(ev[b])
        full[e0:e1] = ctx.copy_out(c4["n_eval"], e0, e1)[e0:e1]
    assert total == c4["total"]
    r = _check(c4, full)
    assert r["normwise"] <= TOL_FP64, r
