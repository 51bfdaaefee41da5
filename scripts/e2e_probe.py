"""e2e P2P launch at config 4 (10M uniform, L = 10): fmmcu_p2p_launch +
finish with page-locked host buffers, per-call wall times; FMMCU_TRACE=1
prints the chunk / group timeline.  Not a benchmark (bench.py is)."""
import argparse
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--levels", type=int, default=10)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--pageable-out", action="store_true",
                help="leave the output pageable (device buffer + copy in finish)")
a = ap.parse_args()
s = F.make_distribution("uniform", a.n, 4)
e = F.EvalSet.self_of(s)
t = F.Tree(s, e, a.levels, 0.5, threads=16)
zp, mp, yp, sid = t.permuted()
pt, ev, so, si = t.leaf_csr()
ctx = N.CudaContext(0)
out = np.zeros((len(zp), 2))
for arr in ((zp, mp, pt, ev, so, si) if a.pageable_out else (out, zp, mp, pt, ev, so, si)):
    ctx.host_register(arr)
ts = []
for r in range(3 if a.reps > 2 else 0):  # split: make_job / launch / finish
    t0 = time.perf_counter()
    job, keep = N.CudaContext.make_job(pt, ev, so, si, t.perm, zp, mp, zp, sid, out)
    t1 = time.perf_counter()
    ctx.launch(job, keep)
    t2 = time.perf_counter()
    pairs, secs = ctx.finish()
    t3 = time.perf_counter()
    print(f"split: make_job {1e3 * (t1 - t0):.3f} ms, launch {1e3 * (t2 - t1):.3f} ms, "
          f"finish {1e3 * (t3 - t2):.3f} ms, busy {1e3 * secs:.3f} ms", flush=True)
for r in range(a.reps):
    t0 = time.perf_counter()
    _, pairs, secs = N.p2p(ctx, pt, ev, so, si, t.perm, zp, mp, zp, sid, out=out)
    ts.append(time.perf_counter() - t0)
    print(f"rep {r}: wall {1e3 * ts[-1]:.3f} ms, busy {1e3 * secs:.3f} ms, pairs {pairs}", flush=True)
print(f"median wall {1e3 * statistics.median(ts[1:]):.3f} ms", flush=True)
