#!/usr/bin/env python3
"""fp32-continuous / w32 FW device times at n=4096, 8192 (A/B with APSP_NO_PDL=1)."""
import statistics, sys
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
def t(h, **kw):
    ts = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = ap.solve(h, **kw); e1.record(); torch.cuda.synchronize()
        if i >= 2: ts.append(e0.elapsed_time(e1))
    return statistics.median(ts), r.info["tier"]
for n in (4096, 8192):
    hc = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, 1.0, 100, 7 + n))).cuda()
    hw = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.002, 100, 7 + n), np.int32)).cuda()
    print(n, "f32c %.2f ms %s" % t(hc), "| w32-ish %.2f ms %s" % t(hw), "| forced w32 dense %.2f ms %s" % t(
        torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.int32)).cuda(), tier="w32"), flush=True)
