"""Multi-rank bench path on a one-GPU box.

bench.py under torchrun shards the target leaves by pair work
(sharding.shard_cuts), re-stages each rank's mutual work list for its leaf
range, gathers the potentials and reports max-over-ranks time.  With
FMM_BENCH_SHARED_GPU=1 every rank runs on cuda:0 with gloo collectives, so the
whole path -- including the gathered result, which rank 0 compares with a
one-rank evaluation of every leaf -- is exercised on the single GPU the test
boxes have.
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
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0
