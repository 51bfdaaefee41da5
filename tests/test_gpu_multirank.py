"""Multi-rank bench path on a one-GPU box.

bench.py under torchrun shards the target leaves by pair work
(sharding.shard_cuts), stages each rank's shard halo-only with its mutual
work list, and gathers the potentials into rank 0's buffer with peer stores
fused into the kernels (the root's output mapped over CUDA IPC); it reports
max-over-ranks time.  With FMM_BENCH_SHARED_GPU=1 every rank runs on cuda:0
(gloo for the host-side plumbing), so the whole path -- including the IPC
stores, whose result rank 0 compares with a one-context evaluation of every
leaf -- is exercised on the single GPU the test boxes have.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
@pytest.mark.parametrize("nproc", [2, 3])
def test_bench_multirank_shared_gpu(nproc):
    env = dict(os.environ, FMM_BENCH_SHARED_GPU="1", OMP_NUM_THREADS="2")
    port = 29700 + nproc
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(ROOT / "bench.py"), "--gpus", str(nproc), "--steps", "3", "--warmup", "3",
           "--points", "300000", "--levels", "7", "--no-fmm", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == nproc
    assert d["gather_check"]["ok"], d["gather_check"]
    assert d["gather_check"]["mode"] == "peer"
    assert d["parity"]["ok"], d["parity"]
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_halo_staging_uploads_only_the_shard():
    """fmmcu_p2p_stage with a leaf range uploads the sources its strong lists
    read (its leaves + a halo), not all of them, and the shard still matches
    the full-range result on its slice."""
    import numpy as np
    sys.path.insert(0, str(ROOT))
    from paper_1311_1006_b200 import _native as N
    from paper_1311_1006_b200 import fmm as F
    from paper_1311_1006_b200.sharding import leaf_work_prefix, shard_cuts
    s = F.make_distribution("uniform", 400_000, 5)
    t = F.Tree(s, F.EvalSet.self_of(s), 8, 0.5, threads=8)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    args = (pt, ev, so, si, t.perm, zp, mp, yp, sid)
    ctx = N.CudaContext(0)
    try:
        job, keep = N.CudaContext.make_job(*args, None)
        ctx.stage(job, keep)
        full_h2d, _ = ctx.transfer_bytes()
        ctx.run_staged(0, len(pt) - 1)
        want = ctx.copy_out(len(yp))
        cuts = shard_cuts(leaf_work_prefix(pt, ev, so, si), 8)
        a, b = int(cuts[3]), int(cuts[4])
        job, keep = N.CudaContext.make_job(*args, None, leaf_begin=a, leaf_end=b)
        ctx.stage(job, keep)
        part_h2d, _ = ctx.transfer_bytes()
        ctx.run_staged(a, b)
        e0, e1 = int(ev[a]), int(ev[b])
        got = ctx.copy_out(len(yp), e0, e1)[e0:e1]
        assert part_h2d < 0.4 * full_h2d, (part_h2d, full_h2d)
        err = np.abs(got - want[e0:e1]).max() / np.abs(want[e0:e1]).max()
        assert err <= 1e-12
    finally:
        ctx.close()


@pytest.mark.gpu
def test_nccl_single_rank_gather_is_identity():
    """The library's NCCL path on one rank (the only NCCL topology a one-GPU
    box allows): the communicator initialises and a gather to the root
    leaves the potentials unchanged."""
    import numpy as np
    sys.path.insert(0, str(ROOT))
    from paper_1311_1006_b200 import _native as N
    from paper_1311_1006_b200 import fmm as F
    s = F.make_distribution("uniform", 50_000, 6)
    t = F.Tree(s, F.EvalSet.self_of(s), 6, 0.5, threads=8)
    zp, mp, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    ctx = N.CudaContext(0)
    try:
        job, keep = N.CudaContext.make_job(pt, ev, so, si, t.perm, zp, mp, yp, sid, None)
        ctx.stage(job, keep)
        ctx.run_staged(0, len(pt) - 1)
        want = ctx.copy_out(len(yp))
        ctx.nccl_init(N.CudaContext.nccl_unique_id(), 0, 1)
        ctx.nccl_gather_out(0, np.array([0, len(yp)], dtype=np.uint32))
        ctx.synchronize()
        assert np.array_equal(ctx.copy_out(len(yp)).view(np.uint64), want.view(np.uint64))
    finally:
        ctx.close()
