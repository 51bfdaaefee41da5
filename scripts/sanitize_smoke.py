"""Small cases of every device path for compute-sanitizer runs (memcheck,
racecheck, synccheck, initcheck): ordered / mutual / exact P2P through the
C ABI, the overlapped launch (ordered, and the grouped mutual list when
FMMCU_CHUNK is set), the staged path, the mutual kernel's entry rounds,
batched M2L, the device pipeline (mutual and ordered lists) and the device
tree.  Not a benchmark."""
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
# entry rounds (> 32 strong entries per leaf: small theta) through the
# staged mutual kernel and the pipeline
t2 = F.Tree(s, e, 4, 0.15, threads=4)
z2, m2, y2, sid2 = t2.permuted()
p2, e2, so2, si2 = t2.leaf_csr()
job, keep = N.CudaContext.make_job(p2, e2, so2, si2, t2.perm, z2, m2, y2, sid2, None, smoother=1,
                                   delta=0.01)
ctx.stage(job, keep)
ctx.run_staged(0, len(p2) - 1)
ctx.synchronize()
ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=4, theta=0.15, p=8)
# grouped mutual list in the overlapped launch (FMMCU_CHUNK=16384 in the
# environment: three upload groups at 40k sources), page-locked inputs
if os.environ.get("FMMCU_CHUNK"):
    os.environ["FMMCU_E2E_SYM"] = "1"
    s3 = F.make_distribution("uniform", 40_000, 3)
    t3 = F.Tree(s3, F.EvalSet.self_of(s3), 5, 0.5, threads=4)
    z3, m3, y3, sid3 = t3.permuted()
    p3, e3, so3, si3 = t3.leaf_csr()
    zr, mr = np.ascontiguousarray(z3).copy(), np.ascontiguousarray(m3).copy()
    for a in (zr, mr):
        ctx.host_register(a)
    N.p2p(ctx, p3, e3, so3, si3, t3.perm, zr, mr, zr, sid3)
    assert ctx.kernel_info()[0]
    for a in (zr, mr):
        ctx.host_unregister(a)
    N.p2p(ctx, p3, e3, so3, si3, t3.perm, z3, m3, y3, sid3)
    del os.environ["FMMCU_E2E_SYM"]
os.environ["FMMCU_PIPE_ORDERED"] = "1"
ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=4, theta=0.5, p=8)
ctx.close()
r = F.FmmEngine(F.FmmConfig(n_levels=4, backend="cuda", m2l_on_device=True, device_tree=True,
                            worker_threads=4)).evaluate(s, e)
print("sanitize smoke ok", r.counters)
