#!/bin/bash
# compute-sanitizer evidence: racecheck + synccheck on the FW tiers (shared-memory
# rings, barrier-free slot release, closures), memcheck on every kernel family including the
# odd-n floor-split R-Kleene and the fused peer-store paths (emulated ranks).
# usage (GPU box, repo root): tools/sanitize.sh TOOL CASE...   -> gpurun_out/san_TOOL_CASE.log
TOOL=$1; shift
mkdir -p gpurun_out
for CASE in "$@"; do
  timeout 900 compute-sanitizer --tool "$TOOL" --print-limit 50 --error-exitcode 99 \
    python tools/san_driver.py "$CASE" > "gpurun_out/san_${TOOL}_${CASE}.log" 2>&1
  echo "$TOOL $CASE exit=$?" | tee -a gpurun_out/san_summary.txt
done
