"""Multi-rank near-field sharding on CPU: world_size 2 over gloo.

Each rank evaluates its work-balanced leaf range with the CPU oracle (the
GPU kernel is covered by test_gpu_p2p.py::test_leaf_shards_compose...), the
slices go to the root with gather_slices_to_root -- the send/recv pattern the
library's fmmcu_nccl_gather_out issues as one NCCL group -- and the assembled
array must equal the unsharded oracle result bit for bit.  World sizes 2 and
3 (an odd split leaves one rank with a short or empty slice)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from paper_1311_1006_b200.sharding import (eval_slices, gather_slices_to_root, leaf_work_prefix,
                                           shard_cuts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case():
    import sys
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_1311_1006_b200 import fmm as F
    s = F.make_distribution("gauss8", 20_000, 3)
    t = F.Tree(s, F.EvalSet.self_of(s), 6, 0.5)
    zp, mp_, yp, sid = t.permuted()
    pt, ev, so, si = t.leaf_csr()
    csr = O.LeafCSR(pt, ev, so, si, t.perm)
    return O, csr, zp, mp_, yp, sid


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O, csr, zp, mp_, yp, sid = _case()
        nl = len(csr.pt_off) - 1
        work = np.zeros(nl + 1, dtype=np.uint64)
        for tl in range(nl):
            S = sum(int(csr.pt_off[b + 1] - csr.pt_off[b])
                    for b in csr.s_idx[csr.s_off[tl]:csr.s_off[tl + 1]])
            work[tl + 1] = work[tl] + int(csr.ev_off[tl + 1] - csr.ev_off[tl]) * S
        assert np.array_equal(work, leaf_work_prefix(csr.pt_off, csr.ev_off, csr.s_off, csr.s_idx))
        cuts = shard_cuts(work, world)
        slices = eval_slices(csr.ev_off, cuts)
        out, pairs = O.nearfield(csr, zp, mp_, yp, sid, leaf_begin=int(cuts[rank]),
                                 leaf_end=int(cuts[rank + 1]))
        full = torch.zeros(out.size, dtype=torch.float64)
        e0, e1 = slices[rank]
        full[2 * e0: 2 * e1] = torch.from_numpy(out.reshape(-1)[2 * e0: 2 * e1])
        gather_slices_to_root(full, slices, rank, root=0)
        tot = torch.tensor([pairs], dtype=torch.float64)
        dist.all_reduce(tot)
        if rank == 0:
            np.savez(result_path, full=full.numpy(), pairs=tot.item(), cuts=cuts, work=work)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_gather_equals_unsharded(tmp_path, world):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    res = np.load(path)
    O, csr, zp, mp_, yp, sid = _case()
    want, wpairs = O.nearfield(csr, zp, mp_, yp, sid)
    assert res["pairs"] == wpairs
    assert np.array_equal(res["full"].view(np.uint64), want.reshape(-1).view(np.uint64))
    # the split is balanced by pair work, not by leaf count
    cuts, work = res["cuts"], res["work"].astype(np.float64)
    parts = [work[cuts[r + 1]] - work[cuts[r]] for r in range(world)]
    assert (max(parts) - min(parts)) / work[-1] < 0.05


def test_shard_cuts_properties():
    rng = np.random.default_rng(1)
    w = np.concatenate([[0], np.cumsum(rng.integers(0, 1000, 5000))]).astype(np.uint64)
    for world in (1, 2, 3, 8):
        c = shard_cuts(w, world)
        assert c[0] == 0 and c[-1] == 5000 and np.all(np.diff(c) >= 0)
    # heavily skewed work: one huge leaf
    w = np.zeros(101, dtype=np.uint64)
    w[1:] = 1
    w[51:] += 10**6
    c = shard_cuts(np.cumsum(np.diff(w, prepend=0)), 4)
    assert c[-1] == 100 and np.all(np.diff(c) >= 0)
