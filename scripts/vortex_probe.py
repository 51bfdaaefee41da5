"""Config 5 probe: vortex sheet N=2M, aspect 8, gaussian smoother, p by the
formula rule, AT3b tuner (cap 0.1), device pipeline vs hybrid."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import fmm as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
for name, kw in (("device_pipeline", dict(device_pipeline=True)),
                 ("hybrid", dict(m2l_on_device=True))):
    cfg = F.FmmConfig(theta=0.5, n_levels=9, p_rule="formula", backend="cuda", worker_threads=16,
                      **kw)
    st = steps if name == "device_pipeline" else min(steps, 5)
    t0 = time.perf_counter()
    tr, _ = F.vortex_run(n, 8.0, st, cfg, tuner="at3b", cap=0.1, seed=1)
    wall = time.perf_counter() - t0
    print(f"{name}: {st} steps wall {wall:.2f} s, mean t_total {1e3 * tr[:, 0].mean():.2f} ms, "
          f"median {1e3 * np.median(tr[:, 0]):.2f} ms, last theta {tr[-1, 5]:.3f} L {int(tr[-1, 6])}, "
          f"pairs/step {tr[-1, 7]:.3e}", flush=True)
