"""Potentials of the device pipeline at 10M/L10 (p=17, harmonic) and 1M/L8
gauss8 (p=19) to an .npy file (FMMCU_M2L_OLD selects the M2L kernel)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import _native as N  # noqa: E402
from paper_1311_1006_b200 import fmm as F  # noqa: E402

ctx = N.CudaContext(0)
outs = []
for kind, n, L, p, kern in (("uniform", 10_000_000, 10, 17, 0), ("gauss8", 1_000_000, 8, 19, 0),
                            ("positive", 1_000_000, 8, 17, 1)):
    s = F.make_distribution(kind, n, 4)
    e = F.EvalSet.self_of(s)
    out, st = ctx.fmm_evaluate(s.z, s.m, e.y, e.source_id, n_levels=L, theta=0.5, p=p,
                               kernel=kern)
    o = np.zeros(10_000_000, dtype=np.complex128)
    o[:n] = out.real if kern else out
    outs.append(o)
    print(kind, n, L, p, {k: round(1e3 * v, 3) for k, v in st.items() if k.startswith("t_")})
np.save(sys.argv[1], np.stack(outs))
