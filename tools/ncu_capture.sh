#!/bin/bash
# ncu evidence for one kernel family (run from the repo root on the GPU box):
#   tools/ncu_capture.sh TAG KERNEL_REGEX -- driver command...
#  1. launch list (gpu__time_duration.sum) of KERNEL_REGEX over the driver command;
#  2. --set full capture of the 7th launch among those with the longest launch's grid
#     (a mid-solve phase-3b launch for the FW drivers); PICK=i chooses another (e.g. -2).
#     GRID="(126, 1, 1)" picks among the launches of that grid instead.
# Outputs: gpurun_out/TAG_list.csv, gpurun_out/TAG_full.ncu-rep
set -e
TAG=$1; K=$2; shift 2; [ "$1" = "--" ] && shift
mkdir -p gpurun_out
ncu -k "regex:$K" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_list.csv "$@" > gpurun_out/${TAG}_list.log 2>&1
SKIP=$(python - "$TAG" <<'PY'
import csv, os, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_list.csv")) if len(r) > 5]
h = rows[0]; rows = rows[1:]
vi, gi = h.index("Metric Value"), h.index("Grid Size")
t = [float(r[vi].replace(",", "")) for r in rows]
g = os.environ.get("GRID") or rows[t.index(max(t))][gi]
long_ = [i for i, r in enumerate(rows) if r[gi] == g]   # launches with the longest one's grid
import os
pick = int(os.environ.get("PICK", "6"))
print(long_[max(-len(long_), min(pick, len(long_) - 1))])
PY
)
echo "skip $SKIP" > gpurun_out/${TAG}_skip.txt
ncu -k "regex:$K" --launch-skip $SKIP --launch-count 1 --set full --clock-control none --import-source on \
  -o gpurun_out/${TAG}_full -f "$@" > gpurun_out/${TAG}_full.log 2>&1
