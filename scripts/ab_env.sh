#!/bin/bash
# A/B of a run-time switch on the bench: runs bench.py (extra args in BARGS)
# once per setting in AB ("-" = unset), JSON lines into gpurun_out/${TAG}_ab_<i>.json
set -u
mkdir -p gpurun_out
TAG=${TAG:-ab}
i=0
for setting in ${AB:-"-"}; do
  if [ "$setting" = "-" ]; then
    timeout 900 python bench.py ${BARGS:-} > gpurun_out/${TAG}_ab_${i}.json 2> gpurun_out/${TAG}_ab_${i}.err
  else
    env $setting timeout 900 python bench.py ${BARGS:-} > gpurun_out/${TAG}_ab_${i}.json 2> gpurun_out/${TAG}_ab_${i}.err
  fi
  echo "ab $i ($setting) exit $?"
  python - "$i" "$setting" <<'PY'
import json, sys
i, s = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/{__import__('os').environ.get('TAG','ab')}_ab_{i}.json").read().strip().splitlines()[-1])
except Exception as e:
    print("no json", e); sys.exit(0)
e2e = d.get("e2e") or {}
f = d.get("fmm_evals_per_sec") or {}
print(s, "value %.4g" % d["value"], "ms %.3f" % d["ms_per_step"], "e2e_ms", e2e.get("ms_per_step"),
      "fmm", f.get("value"), "t", (f.get("timings_s") or {}).get("t_total"),
      "c2", ((f.get("other_configs") or {}).get("config2_uniform_1M") or {}).get("t_total_ms"),
      "c3", ((f.get("other_configs") or {}).get("config3_gauss8_1M") or {}).get("t_total_ms"),
      "vortex", (f.get("config5_vortex") or {}).get("value"), "parity", (d.get("parity") or {}).get("ok"))
PY
  i=$((i+1))
done
