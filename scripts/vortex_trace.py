"""A few config-5 steps (2M vortex sheet, device pipeline, no tuner) under
FMMCU_TRACE: device timelines of the evaluations.  Not a benchmark."""
import sys

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from paper_1311_1006_b200 import fmm as F  # noqa: E402

cfg = F.FmmConfig(theta=0.5, n_levels=9, p_rule="formula", backend="cuda", worker_threads=16,
                  device_pipeline=True)
tr, _ = F.vortex_run(2_000_000, 8.0, 6, cfg, tuner="none", seed=1)
print("t_total ms:", (tr[:, 0] * 1e3).round(2).tolist())
