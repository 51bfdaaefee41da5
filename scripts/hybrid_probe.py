"""Hybrid FmmEngine (host tree + far field, device P2P + batched M2L) at N
(default 10M): per-phase timings of a few evaluations.  Not a benchmark."""
import argparse
import os
import sys
import time

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import fmm as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--levels", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--device-tree", action="store_true")
ap.add_argument("--host-m2l", action="store_true")
a = ap.parse_args()
s = F.make_distribution("uniform", a.n, 4)
e = F.EvalSet.self_of(s)
eng = F.FmmEngine(F.FmmConfig(n_levels=a.levels, backend="cuda", m2l_on_device=not a.host_m2l,
                              device_tree=a.device_tree, worker_threads=os.cpu_count()))
for r in range(a.reps):
    t0 = time.perf_counter()
    res = eng.evaluate(s, e)
    print(f"rep {r}: wall {time.perf_counter() - t0:.3f} s  " +
          " ".join(f"{k}={1e3 * v:.1f}ms" for k, v in res.timings.items()), flush=True)
