"""TEST INFRASTRUCTURE ONLY — sampled parity of a full-size near-field result.

At BASELINE config 4 (10M points, L = 10, 262,144 leaves) the CPU restatement
cannot re-run every leaf in the seconds a test or a bench line affords, so
the device result is checked on a stratified sample of target leaves:

* ``n_blocks`` contiguous blocks of ``block`` leaves spread evenly over the
  leaf range, plus blocks that start at leaf 0, end at the last leaf and
  straddle every shard cut a 2/4/8-way split puts in (``cuts``) -- the places
  where uint32 offsets, contribution slots and work-item bounds turn over;
* on each block, the restated ``near_box`` (backend.cpp:41-69, via
  ``oracle.nearfield``) gives the reference potentials and pair count;
* the pair identity ``Σ_leaves n_evals·S − self hits`` is
  evaluated in numpy over ALL leaves, so the device's total count is checked
  exactly, and per block it must equal the oracle's count.

Used only by tests/ and by bench.py's parity block (computed outside the
timed region, as the checker).
"""
from __future__ import annotations

import numpy as np

from . import oracle as O


def leaf_blocks(n_leaves: int, cuts=(), n_blocks: int = 64, block: int = 64):
    """Sorted, disjoint [(b0, b1)] leaf blocks: evenly spread strata, the first
    and last leaves, and a block centred on every interior cut."""
    block = max(1, min(block, n_leaves))
    starts = {0, n_leaves - block}
    if n_blocks > 0:
        for s in np.linspace(0, n_leaves - block, n_blocks).astype(np.int64):
            starts.add(int(s))
    for c in cuts:
        c = int(c)
        if 0 < c < n_leaves:
            starts.add(int(min(max(c - block // 2, 0), n_leaves - block)))
    out = []
    for s in sorted(starts):
        b0, b1 = s, s + block
        if out and b0 < out[-1][1]:
            out[-1] = (out[-1][0], max(out[-1][1], b1))
        else:
            out.append((b0, b1))
    return out


def pair_identity(pt_off, ev_off, s_off, s_idx, perm=None, sid=None):
    """Per-leaf reference pair count n_evals * |strong sources| - self hits
    (backend.cpp:53-62: a pair is counted before the g == 0 skip, and an
    eval skips its own source only when that source lies in a strong box)."""
    pt_off = np.asarray(pt_off, dtype=np.int64)
    ev_off = np.asarray(ev_off, dtype=np.int64)
    s_off = np.asarray(s_off, dtype=np.int64)
    s_idx = np.asarray(s_idx, dtype=np.int64)
    n = len(pt_off) - 1
    npts = np.diff(pt_off)
    nev = np.diff(ev_off)
    rows = np.diff(s_off)
    S = np.zeros(n, dtype=np.int64)
    if len(s_idx):
        cs = np.concatenate([[0], np.cumsum(npts[s_idx])])
        S = cs[s_off[1:]] - cs[s_off[:-1]]
    per_leaf = nev * S
    if sid is not None and len(sid):
        sid = np.asarray(sid, dtype=np.int64)
        perm = np.asarray(perm, dtype=np.int64)
        inv = np.empty(len(perm), dtype=np.int64)
        inv[perm] = np.arange(len(perm))
        has = sid >= 0
        e_leaf = np.repeat(np.arange(n), nev)[has]
        s_leaf = np.searchsorted(pt_off, inv[sid[has]], side="right") - 1
        strong_key = np.repeat(np.arange(n), rows) * n + s_idx
        hit = np.isin(e_leaf * n + s_leaf, strong_key)
        per_leaf = per_leaf - np.bincount(e_leaf[hit], minlength=n)
    return per_leaf


def sampled_check(got, pt, ev, so, si, perm, zp, mp, yp, sid, *, blocks, kernel=0,
                  smoother=0, delta=0.0, bitwise=False):
    """Compare ``got`` ([n_eval, 2] permuted order) with the oracle on the
    given leaf blocks.  Returns a dict with the normwise error over the
    sample (max|d| / max|ref| on the sample), the max per-point relative
    error, the number of leaves / evals / pairs checked, and (bitwise mode)
    the number of differing doubles."""
    csr = O.LeafCSR(pt, ev, so, si, perm)
    got = np.asarray(got).reshape(-1, 2)
    ev = np.asarray(ev, dtype=np.int64)
    per_leaf = pair_identity(pt, ev, so, si, perm, sid)
    num = 0.0
    den = 0.0
    rel = 0.0
    n_leaves = n_evals = pairs = mism = 0
    pair_ok = True
    for b0, b1 in blocks:
        want, wp = O.nearfield(csr, zp, mp, yp, sid, kernel=kernel, smoother=smoother,
                               delta=delta, leaf_begin=b0, leaf_end=b1)
        e0, e1 = int(ev[b0]), int(ev[b1])
        w = want[e0:e1]
        g = got[e0:e1]
        if int(per_leaf[b0:b1].sum()) != wp:
            pair_ok = False
        d = np.hypot(g[:, 0] - w[:, 0], g[:, 1] - w[:, 1])
        a = np.hypot(w[:, 0], w[:, 1])
        if len(d):
            num = max(num, float(d.max()))
            den = max(den, float(a.max()))
            rel = max(rel, float((d / np.maximum(a, 1e-300)).max()))
        if bitwise:
            mism += int(np.count_nonzero(g.view(np.uint64) != w.view(np.uint64)))
        n_leaves += b1 - b0
        n_evals += e1 - e0
        pairs += wp
    return {"normwise": num / den if den > 0 else num, "max_rel_err_point": rel,
            "leaves": n_leaves, "evals": n_evals, "pairs": pairs, "blocks": len(blocks),
            "pair_identity_ok": pair_ok, "bit_mismatches": mism if bitwise else None,
            "total_pairs_identity": int(per_leaf.sum())}
