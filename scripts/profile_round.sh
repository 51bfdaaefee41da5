#!/bin/bash
# ncu evidence for profiles/: launch list of the bench step, one full capture
# of the P2P kernel (bench workload) and of the device-pipeline M2L, plus a
# launch list of one device-pipeline evaluate.  TAG names the outputs.
set -u
TAG=${TAG:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --no-e2e --no-fmm --no-cpu --steps 3 --warmup 3 > gpurun_out/${TAG}_launches.log 2>&1
echo "launches $?"
ncu --set full --clock-control none --import-source on -k regex:${P2P_KPAT:-p2p_sym_kernel} -s 1 -c 1 -f \
  -o gpurun_out/${TAG}_p2p python bench.py --no-e2e --no-fmm --no-cpu --steps 1 --warmup 3 \
  > gpurun_out/${TAG}_p2p.log 2>&1
echo "p2p full $?"
ncu --set full --clock-control none --import-source on -k regex:${M2L_KPAT:-m2l_reg_kernel} -s 1 -c 1 -f \
  -o gpurun_out/${TAG}_m2l python scripts/fmm_pipeline_probe.py --reps 2 > gpurun_out/${TAG}_m2l.log 2>&1
echo "m2l full $?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_pipe_launches.csv \
  python scripts/fmm_pipeline_probe.py --reps 2 > /dev/null 2>&1
echo "pipe launches $?"
# summaries (the .ncu-rep files can exceed gpurun's 64 MiB return limit)
for k in p2p m2l; do
  ncu -i gpurun_out/${TAG}_${k}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_raw.csv 2>/dev/null
  ncu -i gpurun_out/${TAG}_${k}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${k}_sass.csv 2>/dev/null
  gzip -f gpurun_out/${TAG}_${k}_sass.csv
done
ls -la gpurun_out/
du -sh gpurun_out/*.ncu-rep
rm -f gpurun_out/${TAG}_m2l.ncu-rep gpurun_out/${TAG}_p2p.ncu-rep
true
