#!/usr/bin/env python3
"""u8 FW device time with pivot block 128 vs 256 around the default switch (n=6144)."""
import statistics, sys
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
for n in (5120, 6144, 7168):
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.int32)).cuda()
    for blk in (128, 256):
        ts = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); r = ap.solve(h, block=blk); e1.record(); torch.cuda.synchronize()
            if i >= 3: ts.append(e0.elapsed_time(e1))
        print(n, blk, f"{statistics.median(ts):.3f} ms", flush=True)
