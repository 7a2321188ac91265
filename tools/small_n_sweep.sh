#!/bin/bash
# Small-n FW: blocked schedule (APSP_SQUARING_MAX_N=0) vs min-plus squaring (=2048) per size/density
for N in 256 512 1024 1536 2048; do
  for RHO in 0.002 0.01 0.1 1.0; do
    A=$(APSP_SQUARING_MAX_N=0 python tools/small_n_driver.py $N $RHO 10 | sed 's/.*median //')
    B=$(APSP_SQUARING_MAX_N=2048 python tools/small_n_driver.py $N $RHO 10 | sed 's/.*median //')
    echo "n=$N rho=$RHO blocked: $A | squaring: $B"
  done
done
