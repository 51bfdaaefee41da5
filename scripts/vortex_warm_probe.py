import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1311_1006_b200 import fmm as F
# warm the process as bench does (a device-pipeline evaluate first)
s = F.make_distribution("uniform", 1_000_000, 1); e = F.EvalSet.self_of(s)
F.FmmEngine(F.FmmConfig(n_levels=8, backend="cuda", device_pipeline=True)).evaluate(s, e)
for tuner in ("at3b", "at3a", "at3b"):
    cfg = F.FmmConfig(theta=0.5, n_levels=9, p_rule="formula", backend="cuda", device_pipeline=True, worker_threads=16)
    t0 = time.perf_counter()
    tr, _ = F.vortex_run(2_000_000, 8.0, 100, cfg, tuner=tuner, cap=0.1, seed=1)
    wall = time.perf_counter() - t0
    t = tr[:, 0] * 1e3
    print(f"{tuner}: wall {wall:.3f} s sum {t.sum()/1e3:.3f} s first {t[:4].round(1).tolist()} slowest {np.sort(t)[-5:].round(1).tolist()} at {np.argsort(t)[-5:].tolist()}", flush=True)
