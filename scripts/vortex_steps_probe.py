"""Config-5 step-time distribution (device pipeline, AT3b): wall, sum of
t_total, the slowest steps.  Not a benchmark."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import fmm as F  # noqa: E402

tuner = sys.argv[1] if len(sys.argv) > 1 else "at3b"
cfg = F.FmmConfig(theta=0.5, n_levels=9, p_rule="formula", backend="cuda", worker_threads=16,
                  device_pipeline=True)
t0 = time.perf_counter()
tr, _ = F.vortex_run(2_000_000, 8.0, 100, cfg, tuner=tuner, cap=0.1, seed=1)
wall = time.perf_counter() - t0
t = tr[:, 0] * 1e3
print(f"{tuner}: wall {wall:.2f} s, sum t_total {t.sum() / 1e3:.2f} s, median {np.median(t):.2f} ms, "
      f"slowest {np.sort(t)[-6:].round(1).tolist()} at steps {np.argsort(t)[-6:].tolist()}, "
      f"L {sorted(set(tr[:, 6].astype(int).tolist()))}", flush=True)
