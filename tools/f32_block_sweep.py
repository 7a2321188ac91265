#!/usr/bin/env python3
"""Continuous-fp32 FW time by pivot block (A/B for the default block choice). usage: tools/f32_block_sweep.py n"""
import statistics, sys
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
n = int(sys.argv[1])
h = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, 1.0, 100, 7 + n))).cuda()
for blk in [0, 128, 256, 512]:
    ts = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = ap.solve(h, block=blk); e1.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    print(n, "block", blk, f"{statistics.median(ts):.2f} ms", r.info["block"], flush=True)
