#!/usr/bin/env python3
"""fw_classic(method="classic") (K1, pred bit-exact with the reference) device time at small n."""
import statistics, sys, time
import numpy as np
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
for n in (128, 256, 384, 448, 512):
    raw = ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int64)
    h = ap.CostMatrix(raw)
    ts = []
    for i in range(6):
        r = ap.fw_classic(h, method="classic")
        if i >= 1: ts.append(r.info["device_ms"])
    print(n, f"device {statistics.median(ts):.3f} ms", r.info["tier"], flush=True)
