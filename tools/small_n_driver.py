#!/usr/bin/env python3
"""Small-n FW solves (the paper's n <= 1000 regime and the C5 small sizes) for timing and ncu.
usage: tools/small_n_driver.py n [rho] [reps]  -> prints the median device time of ap.solve"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402

n = int(sys.argv[1])
rho = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)).cuda()
ts = []
for i in range(reps + 5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ap.solve(h)
    e1.record()
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(e0.elapsed_time(e1))
print(f"n={n} rho={rho} tier={r.info["tier"]} it={r.info.get("iterations")} median {statistics.median(ts):.3f} ms min {min(ts):.3f} ms")
