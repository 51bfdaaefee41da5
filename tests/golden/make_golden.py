"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the dev container (needs /root/reference, built into
oracle/_ref/libfmmref.so by ``make -C oracle``):

    python tests/golden/make_golden.py

Every array comes straight out of the reference library (build_pyramid,
build_connectivity, nearfield_run, FmmEngine::evaluate, m2l_add,
kernel_term) through oracle/ref_shim.cpp; the fixtures are then checked in
so the GPU box (which has no /root/reference) can pin the oracle and the
product against them.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402

# (name, distribution kind, n_src, seed, n_levels, theta, separate eval count or None)
TREE_CASES = [
    ("rand2000_L4", 3, 2000, 42, 4, 0.5, None),
    ("unif1500_ev700_L4", 0, 1500, 5, 4, 0.5, 700),
    ("gauss4000_L5", 2, 4000, 3, 5, 0.5, None),
    ("line3000_L5_t065", 1, 3000, 8, 5, 0.65, None),
    ("pos1024_L1", 4, 1024, 13, 1, 0.5, None),
]
# near-field variants per tree: (kernel, smoother, delta)
NF_VARIANTS = [(0, 0, 0.0), (1, 0, 0.0), (0, 1, 1e-2), (0, 2, 2e-2)]


def tree_fixture(name, kind, n, seed, L, theta, n_eval):
    z, m = O.make_distribution(kind, n, seed)
    if n_eval is None:
        y, sid = z.copy(), np.arange(n, dtype=np.int64)
    else:
        yz, _ = O.make_distribution(3, n_eval, seed + 1000)
        y, sid = yz * 1.4 - 0.2, None  # spills outside the source box
    t = O.ref_tree(z, m, y, sid, L, theta, keep=True)
    d = dict(z=z, m=m, y=y, n_levels=L, theta=theta, perm=t.perm, eval_perm=t.eval_perm)
    if sid is not None:
        d["sid"] = sid
    for lvl in range(L):
        d[f"boxes_f_{lvl}"] = t.boxes_f[lvl]
        d[f"boxes_u_{lvl}"] = t.boxes_u[lvl]
        d[f"strong_off_{lvl}"], d[f"strong_idx_{lvl}"] = t.strong[lvl]
        d[f"weak_off_{lvl}"], d[f"weak_idx_{lvl}"] = t.weak[lvl]
    for k, s, dl in NF_VARIANTS:
        out, pairs, _ = O.ref_nearfield(t, kernel=k, smoother=s, delta=dl)
        d[f"near_k{k}_s{s}"] = out
        d[f"pairs_k{k}_s{s}"] = np.uint64(pairs)
        d[f"delta_k{k}_s{s}"] = dl
    t.free()
    # end-to-end evaluate (serial backend, table p) for the harmonic kernel
    pot, tim, cnt, p = O.ref_evaluate(z, m, y, sid, theta=theta, n_levels=L, kernel=0)
    d["eval_pot"] = pot
    d["eval_counters"] = cnt
    d["eval_p"] = p
    np.savez_compressed(os.path.join(HERE, f"tree_{name}.npz"), **d)
    print("wrote", name, "pairs", d["pairs_k0_s0"], "p", p)


def m2l_fixture():
    rng = np.random.default_rng(1311)
    rows = []
    # the small scale sends m2l_add down its long double branch
    # ((p+2) log10|w| >= 250) while the local coefficients stay finite
    small = {8: 1e-30, 17: 1e-15, 19: 1e-15, 30: 3e-9}
    for p in (8, 17, 19, 30):
        for kernel in (0, 1):
            for scale in (1.0, small[p]):
                sc = rng.uniform(-1, 1, 2) * scale
                tc = rng.uniform(-1, 1, 2) * scale + np.array([3.0, 0.5]) * scale
                coeffs = rng.uniform(-1, 1, (p + 1, 2)) * (0.4 * scale) ** np.arange(p + 1)[:, None]
                local0 = rng.uniform(-1, 1, (p + 1, 2))
                local = local0.copy()
                O.ref_lib().fmmref_m2l_add(p, kernel, sc, coeffs.ravel().copy(), tc, local.ravel())
                rows.append(dict(p=p, kernel=kernel, sc=sc, tc=tc, coeffs=coeffs, local0=local0,
                                 local=local))
    d = {}
    for i, r in enumerate(rows):
        for key, v in r.items():
            d[f"{i}_{key}"] = v
    d["count"] = len(rows)
    np.savez_compressed(os.path.join(HERE, "m2l_cases.npz"), **d)
    print("wrote m2l_cases", len(rows))


def divide_fixture():
    rng = np.random.default_rng(7)
    n = 4000
    y = rng.uniform(0, 1, (n, 2))
    x = y + rng.uniform(-1, 1, (n, 2)) * 10.0 ** rng.uniform(-9, 0, (n, 1))
    m = rng.uniform(-1, 1, (n, 2))
    special = np.array([
        [0.0, 0.0, 1.0, 0.0, 1.0, 0.0],          # -1/(0-1) = 1
        [0.0, 0.0, 1e-300, 2e-300, 1.0, 1.0],    # tiny separation
        [1e300, 1e300, 0.0, 0.0, 1.0, -1.0],     # huge separation
        [0.5, 0.5, 0.5, 0.5 + 1e-310, 1.0, 0.0],  # subnormal difference
    ])
    y = np.vstack([special[:, 0:2], y])
    x = np.vstack([special[:, 2:4], x])
    m = np.vstack([special[:, 4:6], m])
    out = np.empty_like(y)
    O.ref_lib().fmmref_kernel_term_batch(0, len(y), y.ravel(), x.ravel(), m.ravel(), out.ravel())
    np.savez_compressed(os.path.join(HERE, "kernel_term.npz"), y=y, x=x, m=m, out=out)
    print("wrote kernel_term", len(y))


def controller_fixture():
    rng = np.random.default_rng(3)
    d = {}
    cases = 0
    for kind in range(5):
        for trial in range(3):
            n = 400
            t = 1.0 + 0.2 * rng.random(n) + np.linspace(0, 0.1, n)
            w = np.where(rng.random(n) < 0.5, 0.01 * rng.random(n), 0.0)
            hw = float(trial % 2)
            meas = np.stack([t, w, np.full(n, hw)], 1)
            cf = np.array([0.25, 0.8, 0.01, 0.1 if trial < 2 else 0.02])
            ci = np.array([1, 10, 2, 10 if trial != 1 else 5, 3, 3, 12], dtype=np.int32)
            out = np.empty((n, 2))
            ev = np.empty((n, 3), dtype=np.int32)
            rc = O.ref_lib().fmmref_controller_run(kind, cf, ci, 0.5, 5, 100 + trial, n, meas.ravel(),
                                                   out.ravel(), ev.ravel())
            assert rc == 0
            key = f"{cases}"
            d[key + "_kind"] = kind
            d[key + "_seed"] = 100 + trial
            d[key + "_cf"] = cf
            d[key + "_ci"] = ci
            d[key + "_meas"] = meas
            d[key + "_out"] = out
            d[key + "_ev"] = ev
            cases += 1
    d["count"] = cases
    np.savez_compressed(os.path.join(HERE, "controller.npz"), **d)
    print("wrote controller", cases)


if __name__ == "__main__":
    if not O.ref_available():
        sys.exit("oracle/_ref/libfmmref.so missing: run `make -C oracle` in the dev container")
    for case in TREE_CASES:
        tree_fixture(*case)
    m2l_fixture()
    divide_fixture()
    controller_fixture()
