#!/bin/bash
# A/B of the grouped tile rasterisation (APSP_RASTER_G) on the bench workload (n=16384):
# device time per solve, then DRAM bytes, L2 hit rate and duration of one mid-solve phase-3b
# launch (ncu; the 7th long launch of the solve, as in tools/p3_capture.sh).
mkdir -p gpurun_out
for G in 1 8; do
  echo "APSP_RASTER_G=$G"; APSP_RASTER_G=$G python tools/small_n_driver.py 16384 0.1 5
done
ncu -k regex:minplus_nt_kernel --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/raster_list.csv python tools/p3_driver.py > /dev/null 2>&1
SKIP=$(python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/raster_list.csv")) if len(r) > 5]
h = rows[0]; rows = rows[1:]
vi = h.index("Metric Value")
t = [float(r[vi].replace(",", "")) for r in rows]
print([i for i, x in enumerate(t) if x > 0.8 * max(t)][6])
PY
)
echo "phase-3b launch index $SKIP"
for G in 1 8; do
  APSP_RASTER_G=$G ncu -k regex:minplus_nt_kernel --launch-skip $SKIP --launch-count 1 --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --csv python tools/p3_driver.py 2>/dev/null | grep -E "gpu__time|dram__bytes|lts__t_sector" | \
    awk -v g=$G -F'","' '{print "G=" g, $(NF-2), $(NF-1), $NF}'
done
