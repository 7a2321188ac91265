#!/usr/bin/env python3
"""R-Kleene (aligned, pred) device time by n and base threshold (A/B of its leaf schedule)."""
import statistics, sys
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
for n, thr in [(1024, 512), (2048, 1024), (4096, 1024), (8192, 2048)]:
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.int32)).cuda()
    ts = []
    for i in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=thr); e1.record()
        torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    print(n, thr, f"{statistics.median(ts):.2f} ms", r.info["tier"], flush=True)
