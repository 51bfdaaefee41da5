"""Per-rank work of the N-GPU near field, measured on one B200: the config-4
job (10M uniform, L = 10) cut into N work-balanced leaf shards exactly as
bench.py --gpus N cuts it; each shard staged halo-only in its own context
(what one rank uploads) and its kernels timed alone with CUDA events
(median of reps).  max over shards = the strong-scaling step of N ranks
before the gather; the gather costs are reported from the shard sizes.
Prints one JSON line.  A projection from 1-GPU measurements, not a
multi-GPU measurement."""
import argparse
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
import torch  # noqa: E402

from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402
from paper_1311_1006_b200.sharding import eval_slices, leaf_work_prefix, shard_cuts  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10_000_000)
ap.add_argument("--levels", type=int, default=10)
ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
s = F.make_distribution("uniform", a.n, 4)
e = F.EvalSet.self_of(s)
t = F.Tree(s, e, a.levels, 0.5, threads=16)
zp, mp, yp, sid = t.permuted()
pt, ev, so, si = t.leaf_csr()
nl = len(pt) - 1
prefix = leaf_work_prefix(pt, ev, so, si)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
res = {}
for world in a.ranks:
    cuts = shard_cuts(prefix, world)
    sl = eval_slices(ev, cuts)
    per = []
    for r in range(world):
        lb, le = int(cuts[r]), int(cuts[r + 1])
        ctx = N.CudaContext(0)
        ctx.set_stream(stream.cuda_stream)
        job, keep = N.CudaContext.make_job(pt, ev, so, si, t.perm, zp, mp, zp, sid, None,
                                           leaf_begin=lb, leaf_end=le)
        ctx.stage(job, keep)
        staged_h2d, _ = ctx.transfer_bytes()
        for _ in range(3):
            ctx.run_staged(lb, le)
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.run_staged(lb, le)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        pairs = ctx.pairs()
        per.append({"leaves": [lb, le], "ms": statistics.median(ms), "pairs": pairs,
                    "slice_bytes": 16 * (sl[r][1] - sl[r][0]), "staged_h2d": staged_h2d})
        ctx.close()
    kmax = max(p["ms"] for p in per)
    root_recv = sum(p["slice_bytes"] for i, p in enumerate(per) if i != 0)
    res[world] = {"kernel_ms_max": kmax, "kernel_ms_min": min(p["ms"] for p in per),
                  "pairs_total": sum(p["pairs"] for p in per),
                  "root_receive_bytes": root_recv,
                  "shards": per}
    print(f"N={world}: kernel max {kmax:.3f} ms, min {res[world]['kernel_ms_min']:.3f} ms, "
          f"root receives {root_recv / 1e6:.1f} MB", flush=True)
base = res[min(res)]["kernel_ms_max"]
for w, r in res.items():
    r["kernel_speedup_vs_1"] = base / r["kernel_ms_max"]
print(json.dumps({"n": a.n, "levels": a.levels, "per_world": res}))
