#!/bin/bash
# A/B of the fp32 rescan granularity (APSP_F32_FINE = fraction of FW rounds at 8-k granularity)
for F in 0 0.125 0.25 0.5 1; do
  echo "APSP_F32_FINE=$F"; APSP_F32_FINE=$F python tools/f32_timing.py 4096 | head -2
done
APSP_F32_FINE=0 python tools/f32_timing.py 8192 | head -1; python tools/f32_timing.py 8192 | head -1
