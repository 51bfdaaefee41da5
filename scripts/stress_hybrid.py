"""Stress for the round-1 intermittent hybrid failure (0.14 normwise on a
golden case with fast P2P + m2l_on_device): every golden tree through fresh
FmmEngine(cuda) instances, exact/fast x host/device M2L, in a shuffled order
per round, N rounds; also a 1.2M-point page-locked launch to exercise the
two-stream grouped kernels.  Prints the worst error per configuration."""
import glob
import os
import sys

import numpy as np

ROOT = __file__.rsplit("/scripts/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden, normwise  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 20
names = sorted(os.path.basename(p) for p in glob.glob(os.path.join(ROOT, "tests/golden/tree_*.npz")))
gold = {n: load_golden(n) for n in names}
rng = np.random.default_rng(0)
worst = {}
fails = 0
for r in range(rounds):
    jobs = [(n, ex, md) for n in names for ex in (True, False) for md in (False, True)]
    rng.shuffle(jobs)
    for n, ex, md in jobs:
        d = gold[n]
        s = F.SourceSet(d["z"][:, 0] + 1j * d["z"][:, 1], d["m"][:, 0] + 1j * d["m"][:, 1])
        e = F.EvalSet(d["y"][:, 0] + 1j * d["y"][:, 1], d["sid"] if "sid" in d else None)
        eng = F.FmmEngine(F.FmmConfig(theta=float(d["theta"]), n_levels=int(d["n_levels"]),
                                      backend="cuda", exact=ex, m2l_on_device=md,
                                      worker_threads=4))
        got = F._c2(eng.evaluate(s, e).potentials)
        err = normwise(got, d["eval_pot"])
        k = (n, ex, md)
        worst[k] = max(worst.get(k, 0.0), err)
        if err > 1e-12:
            fails += 1
            print(f"FAIL round {r}: {k} err {err:.3e}", flush=True)
for k, v in sorted(worst.items()):
    print(k, f"{v:.2e}")
print(f"rounds {rounds}, failures {fails}", flush=True)
