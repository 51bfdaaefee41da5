"""Multi-GPU sharding of the near field: one process per GPU.

The near field shards naturally: a target leaf's potentials
depend only on its own evals and the sources of its strong list, so each
rank evaluates a contiguous range of finest-level leaves (Z-ordered median
cells, spatially compact) with the sources replicated, and the only data
exchange is gathering the potential slices.  Ranges are balanced by pair
work n_evals * |strong sources| (clustered strong lists vary 3000x), not by
leaf count.  The gather is one NCCL all-gather of equal-size padded slices
over NVLink (torch.distributed), so every rank ends with the full potential
array in permuted eval order.
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


class PotentialGather:
    """All-gather of per-rank potential slices into the full array.

    ``full`` is a flat float64 tensor [2 * n_eval] (the rank writes its own
    slice in place, e.g. the kernel output bound with bind_device_out).  The
    pad buffers are allocated once so the gather is allocation-free inside a
    timed loop."""

    def __init__(self, slices, rank: int, full, group=None, via_host: bool = False):
        import torch

        self.slices = slices
        self.rank = rank
        self.world = len(slices)
        self.full = full
        self.group = group
        self.maxlen = max(1, max(e1 - e0 for e0, e1 in slices)) * 2
        # via_host: gloo test mode (several ranks sharing one GPU)
        dev = "cpu" if via_host else full.device
        self.send = torch.zeros(self.maxlen, dtype=full.dtype, device=dev)
        self.recv = torch.zeros(self.maxlen * self.world, dtype=full.dtype, device=dev)

    def bytes_moved(self) -> int:
        return int(self.recv.numel() * self.recv.element_size())

    def __call__(self):
        import torch.distributed as dist

        e0, e1 = self.slices[self.rank]
        n = (e1 - e0) * 2
        if n:
            self.send[:n].copy_(self.full[2 * e0: 2 * e1])
        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        for r, (a, b) in enumerate(self.slices):
            if r == self.rank or b == a:
                continue
            m = (b - a) * 2
            self.full[2 * a: 2 * b].copy_(self.recv[r * self.maxlen: r * self.maxlen + m],
                                          non_blocking=False)
        return self.full
