#!/bin/bash
# A/B of the blocked closure's phases (APSP_BLK_SKIP; results are wrong in the skipped runs):
# ncu launch times of block_close_blk over one continuous-fp32 n=4096 solve per variant.
mkdir -p gpurun_out
for SK in 0 1 2 4 8 14 15; do
  APSP_BLK_SKIP=$SK ncu -k regex:block_close_blk --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/close_ab_$SK.csv python tools/f32_profile_driver.py 4096 > /dev/null 2>&1
  python - "$SK" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/close_ab_{sys.argv[1]}.csv")) if len(r) > 5]
vi = rows[0].index("Metric Value")
t = [float(r[vi].replace(",", "")) / 1e3 for r in rows[1:]]
print(f"skip={sys.argv[1]:>2} launches={len(t)} mean={sum(t)/len(t):.1f} us first={t[0]:.1f} last={t[-1]:.1f}")
PY
done
