"""Device-pipeline FMM at N (default 10M): per-call timings and stats, for
tracing (FMMCU_TRACE=1) and ncu launch lists.  Not a benchmark."""
import argparse
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--levels", type=int, default=10)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dist", default="uniform")
ap.add_argument("--register", action="store_true", help="page-lock inputs and output once")
a = ap.parse_args()
s = F.make_distribution(a.dist, a.n, 4)
e = F.EvalSet.self_of(s)
ctx = N.CudaContext(0)
out = np.zeros(a.n, dtype=np.complex128)
if a.register:
    for arr in (s.z, s.m, e.y, e.source_id, out):
        ctx.host_register(arr)
ref = None
for r in range(a.reps):
    t0 = time.perf_counter()
    out, st = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=a.levels, theta=0.5, p=17,
                               out=out)
    if ref is None:
        ref = out.copy()
    elif not np.array_equal(ref, out):
        print("MISMATCH between reps", flush=True)
    t1 = time.perf_counter()
    print(f"rep {r}: wall {1e3 * (t1 - t0):.2f} ms  " +
          " ".join(f"{k}={1e3 * v:.2f}ms" for k, v in st.items() if k.startswith("t_")), flush=True)
if a.register:
    for arr in (s.z, s.m, e.y, e.source_id, out):
        ctx.host_unregister(arr)
ctx.close()
totals = []
eng = F.FmmEngine(F.FmmConfig(n_levels=a.levels, backend="cuda", device_pipeline=True))
for r in range(a.reps):
    t0 = time.perf_counter()
    res = eng.evaluate(s, e)
    t1 = time.perf_counter()
    totals.append(res.timings["t_total"])
    print(f"engine rep {r}: wall {1e3 * (t1 - t0):.2f} ms  t_total {1e3 * res.timings['t_total']:.2f} ms",
          flush=True)
if len(totals) > 2:
    t = sorted(totals[1:])
    print(f"engine t_total over reps 1..: median {1e3 * t[len(t) // 2]:.2f} ms, "
          f"min {1e3 * t[0]:.2f}, max {1e3 * t[-1]:.2f}", flush=True)
