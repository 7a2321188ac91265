#!/bin/bash
# ncu evidence for the phase-3 tile kernel (run from the repo root on the GPU box):
#  1. launch list of minplus_nt_kernel for one n=16384 solve;
#  2. --set full capture of the 7th long (phase-3b) launch.
set -e
mkdir -p gpurun_out
K=regex:minplus_nt_kernel
ncu -k $K --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/p3_list.csv python tools/p3_driver.py > gpurun_out/p3_list.log 2>&1
SKIP=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/p3_list.csv")) if len(r) > 5]
h = rows[0]; rows = rows[1:]
ki, vi = h.index("ID"), h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows]
long_ = [i for i, x in enumerate(t) if x > 0.8 * max(t)]
print(long_[6])
PY
)
echo "skip $SKIP" > gpurun_out/p3_skip.txt
ncu -k $K --launch-skip $SKIP --launch-count 1 --set full --clock-control none --import-source on \
  -o gpurun_out/p3_full -f python tools/p3_driver.py > gpurun_out/p3_full.log 2>&1
