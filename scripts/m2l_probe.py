"""Device-pipeline M2L timing probe (FMMCU_M2L=old|thread|warp selects the
kernel): per case, the far-stream M2L(+L2L) span and the potentials' checksum
so the variants can be compared."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

ctx = N.CudaContext(0)
cases = [("uniform", 10_000_000, 10, 17), ("gauss8", 1_000_000, 8, 19), ("gauss8", 1_000_000, 8, 17),
         ("uniform", 1_000_000, 9, 19), ("uniform", 1_000_000, 9, 17)]
for kind, n, L, p in cases:
    s = F.make_distribution(kind, n, 3)
    e = F.EvalSet.self_of(s)
    for rep in range(2):
        out, st = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=0.5, p=p)
    print(kind, n, L, p, "m2l_ops", st["m2l_ops"], "t_m2l %.3f ms" % (1e3 * st["t_m2l"]),
          "t_p2p %.3f ms" % (1e3 * st["t_p2p"]), "sum %.15e %.15e" % (out.real.sum(), out.imag.sum()),
          flush=True)
