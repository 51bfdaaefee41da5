#!/bin/bash
# One GPU call: parity tests, smoke, bench line, ncu launch list and one full
# capture of the dominant kernel. Everything lands in gpurun_out/ (scratch);
# summaries worth keeping are copied to profiles/ by hand.
#   STAGES="tests smoke bench launches full" (default: all)
set -u
mkdir -p gpurun_out
STAGES=${STAGES:-"tests smoke bench launches full"}
TAG=${TAG:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
for s in $STAGES; do
  case $s in
    tests)
      timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
      echo "pytest-gpu exit $?" ; tail -3 gpurun_out/${TAG}_pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
      echo "smoke exit $?"; tail -2 gpurun_out/${TAG}_smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
      echo "bench exit $?"; tail -c 600 gpurun_out/${TAG}_bench.json ;;
    refbench)
      timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_refbench.json 2>&1
      echo "refbench exit $?"; tail -c 400 gpurun_out/${TAG}_refbench.json ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/${TAG}_launches.csv \
        python bench.py --no-e2e --no-fmm --no-cpu --steps 3 --warmup 3 > gpurun_out/${TAG}_launches.log 2>&1
      echo "launches exit $?" ;;
    full)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KPAT:-p2p_warp_kernel} \
        -s ${KSKIP:-1} -c 1 -f -o gpurun_out/${TAG}_prof \
        python bench.py --no-e2e --no-fmm --no-cpu --steps 1 --warmup 3 > gpurun_out/${TAG}_full.log 2>&1
      echo "full exit $?"; tail -3 gpurun_out/${TAG}_full.log ;;
    *) echo "unknown stage $s" ;;
  esac
done
