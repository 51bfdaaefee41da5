"""Small cases of every device path for compute-sanitizer runs (memcheck,
racecheck, synccheck, initcheck): ordered / mutual / exact P2P through the
C ABI, the overlapped launch, the staged path, batched M2L, the device
pipeline (mutual and ordered lists) and the device tree.  Not a benchmark."""
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

s = F.make_distribution("uniform", 6000, 1)
e = F.EvalSet.self_of(s)
t = F.Tree(s, e, 4, 0.5, threads=4)
zp, mp, yp, sid = t.permuted()
pt, ev, so, si = t.leaf_csr()
ctx = N.CudaContext(0)
for mode in (0, 1):
    N.p2p(ctx, pt, ev, so, si, t.perm, zp, mp, yp, sid, mode=mode)
job, keep = N.CudaContext.make_job(pt, ev, so, si, t.perm, zp, mp, yp, sid, None)
ctx.stage(job, keep)
ctx.run_staged(0, len(pt) - 1)
ctx.synchronize()
ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=4, theta=0.5, p=8)
os.environ["FMMCU_PIPE_ORDERED"] = "1"
ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=4, theta=0.5, p=8)
ctx.close()
r = F.FmmEngine(F.FmmConfig(n_levels=4, backend="cuda", m2l_on_device=True, device_tree=True,
                            worker_threads=4)).evaluate(s, e)
print("sanitize smoke ok", r.counters)
