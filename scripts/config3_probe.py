import os, sys, statistics
sys.path.insert(0, "/root/repo")
from paper_1311_1006_b200 import fmm as F
for kind, L in (("gauss8", 7), ("uniform", 9)):
    s = F.make_distribution(kind, 1_000_000, 4); e = F.EvalSet.self_of(s)
    eng = F.FmmEngine(F.FmmConfig(n_levels=L, backend="cuda", device_pipeline=True))
    t = [eng.evaluate(s, e).timings["t_total"] for _ in range(7)][1:]
    print(kind, os.environ.get("FMMCU_CONN_SYNC"), "median %.2f ms min %.2f" % (1e3 * statistics.median(t), 1e3 * min(t)), flush=True)
