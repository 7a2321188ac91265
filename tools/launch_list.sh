#!/bin/bash
# Launch list of every kernel of a driver command (ncu, gpu__time_duration.sum), then the
# per-kernel share summary:  tools/launch_list.sh TAG -- driver command...
set -e
TAG=$1; shift; [ "$1" = "--" ] && shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv "$@" \
  > gpurun_out/${TAG}_launches.log 2>&1
python tools/ncu_summary.py launches gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launches.txt
