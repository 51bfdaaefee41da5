#!/bin/bash
# P2P kernel variant sweep on the bench workload (config 4); one summary line per variant.
#   VARIANTS="0 1 2" ES="4 5" bash scripts/variant_sweep.sh [bench args]
for e in ${ES:-4 5}; do
for v in ${VARIANTS:-0 1 2}; do
  FMMCU_P2P_E=$e FMMCU_P2P_VARIANT=$v python bench.py --no-e2e --no-fmm --no-cpu --steps 10 --warmup 3 "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('E', $e, 'variant', $v, 'Tpairs/s %.4f'%(d['value']/1e12), 'kernel_ms %.3f'%r['kernel_ms'], 'frac %.3f'%r['frac'], 'clk', d['clocks']['sm_mhz'])"
done
done
