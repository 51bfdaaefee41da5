"""Multi-GPU sharding of the near field: one process per GPU.

The near field shards naturally: a target leaf's potentials
depend only on its own evals and the sources of its strong list, so each
rank evaluates a contiguous range of finest-level leaves (Z-ordered median
cells, spatially compact) staging only the sources its strong lists read
(halo-only), and the only data
exchange is gathering the potential slices to the root.  Ranges are balanced
by pair work n_evals * |strong sources| (clustered strong lists vary 3000x),
not by leaf count.  The gather itself lives in the library
(include/fmm_cuda.h, csrc/fmm_multi.cu): fused into the kernels' stores over
NVLink (IPC-mapped root buffer), or one grouped NCCL send/recv of the
slices; gather_slices_to_root restates the latter for CPU tests.
"""
from __future__ import annotations

import numpy as np


def shard_cuts(work_prefix: np.ndarray, world: int) -> np.ndarray:
    """Leaf cut points [0 = c_0 <= c_1 <= ... <= c_world = n_leaves] so that
    rank r owns leaves [c_r, c_{r+1}) with ~1/world of the pair work.
    ``work_prefix`` is the inclusive prefix over leaves ([n_leaves + 1])."""
    work_prefix = np.asarray(work_prefix, dtype=np.float64)
    n_leaves = len(work_prefix) - 1
    total = work_prefix[-1]
    cuts = np.zeros(world + 1, dtype=np.int64)
    cuts[-1] = n_leaves
    for r in range(1, world):
        cuts[r] = int(np.searchsorted(work_prefix, total * r / world, side="left"))
        cuts[r] = min(max(cuts[r], cuts[r - 1]), n_leaves)
    return cuts


def eval_slices(ev_off: np.ndarray, cuts: np.ndarray):
    """[(e0, e1)] eval ranges owned by each rank (contiguous, nested ranges)."""
    ev_off = np.asarray(ev_off, dtype=np.int64)
    return [(int(ev_off[cuts[r]]), int(ev_off[cuts[r + 1]])) for r in range(len(cuts) - 1)]


def leaf_work_prefix(pt_off, ev_off, s_off, s_idx) -> np.ndarray:
    """Inclusive prefix [n_leaves + 1] of the per-leaf pair work
    n_evals * |strong sources| (before self-skips): the balance key of
    shard_cuts, from the leaf CSR alone (no staging needed)."""
    pt_off = np.asarray(pt_off, dtype=np.int64)
    s_off = np.asarray(s_off, dtype=np.int64)
    s_idx = np.asarray(s_idx, dtype=np.int64)
    npts = np.diff(pt_off)
    S = np.zeros(len(npts), dtype=np.int64)
    if len(s_idx):
        cs = np.concatenate([[0], np.cumsum(npts[s_idx])])
        S = cs[s_off[1:]] - cs[s_off[:-1]]
    work = np.diff(np.asarray(ev_off, dtype=np.int64)) * S
    return np.concatenate([[0], np.cumsum(work)]).astype(np.uint64)


def gather_slices_to_root(full, slices, rank: int, root: int = 0, group=None):
    """The gather the library does with one grouped ncclSend / ncclRecv
    (fmmcu_nccl_gather_out), restated over torch.distributed point-to-point
    so the protocol runs on gloo/CPU in tests: every rank sends its eval
    slice of ``full`` (flat float64, [2 n_eval]) to the root, which receives
    each slice in place at its own offset -- no padding, no staging copy."""
    import torch.distributed as dist

    world = len(slices)
    if rank == root:
        reqs = []
        for r in range(world):
            a, b = slices[r]
            if r == root or b == a:
                continue
            reqs.append(dist.irecv(full[2 * a: 2 * b], src=r, group=group))
        for q in reqs:
            q.wait()
    else:
        a, b = slices[rank]
        if b > a:
            dist.send(full[2 * a: 2 * b].contiguous(), dst=root, group=group)
    return full
