#!/bin/bash
# A/B of the device M2L kernels inside the 10M / L10 device pipeline (p=17)
# and the 2M-point vortex-like case (p=19): kernel times from an ncu launch
# list (gpu__time_duration, M2L kernels only), and potentials old vs new.
set -u
mkdir -p gpurun_out
TAG=${TAG:-m2l}
for v in 1 0; do
  FMMCU_M2L_OLD=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:m2l \
    --log-file gpurun_out/${TAG}_old${v}.csv python scripts/fmm_pipeline_probe.py --reps 2 \
    > gpurun_out/${TAG}_old${v}.log 2>&1
  echo "ncu old=$v $?"
  FMMCU_M2L_OLD=$v python scripts/m2l_dump.py gpurun_out/${TAG}_pot_old${v}.npy > gpurun_out/${TAG}_dump${v}.log 2>&1
  echo "dump old=$v $?"
done
TAG=$TAG python - <<'PY'
import numpy as np, csv, os
TAG = os.environ["TAG"]
a = np.load("gpurun_out/%s_pot_old1.npy" % TAG)
b = np.load("gpurun_out/%s_pot_old0.npy" % TAG)
for i in range(a.shape[0]):
    print("case", i, "normwise new vs old", np.abs(a[i] - b[i]).max() / np.abs(a[i]).max())
for v in (1, 0):
    rows = [r for r in csv.reader(open("gpurun_out/%s_old%d.csv" % (TAG, v))) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        print("old=%d" % v, r[ki][:60], r[vi])
PY
rm -f gpurun_out/${TAG}_pot_old*.npy
