#!/bin/bash
# Two-deep lookahead (default) vs the one-deep schedule (APSP_NO_DEEP=1)
for N in 4096 6144 8192; do
  echo "u8 n=$N deep: $(python tools/small_n_driver.py $N 1.0 5 | sed 's/.*median //') | one-deep: $(APSP_NO_DEEP=1 python tools/small_n_driver.py $N 1.0 5 | sed 's/.*median //')"
done
echo "u16/w32 n=4096 rho=0.002 deep: $(python tools/small_n_driver.py 4096 0.002 5 | sed 's/.*median //') | one-deep: $(APSP_NO_DEEP=1 python tools/small_n_driver.py 4096 0.002 5 | sed 's/.*median //')"
echo "f32 continuous:"; python tools/f32_timing.py 4096 2>/dev/null | head -1; APSP_NO_DEEP=1 python tools/f32_timing.py 4096 2>/dev/null | head -1
python tools/f32_timing.py 8192 2>/dev/null | head -1; APSP_NO_DEEP=1 python tools/f32_timing.py 8192 2>/dev/null | head -1
