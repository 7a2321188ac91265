#!/usr/bin/env python3
"""Are results tier-independent? Solve the same graph on every admissible forced tier (default
and 128 block) and compare distances and pred bitwise against the narrowest."""
import sys
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap
for n, rho, seed in [(300, 0.1, 1), (700, 0.05, 2), (1024, 0.03, 3), (1500, 0.02, 4), (3200, 0.02, 5)]:
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, seed), np.int32)).cuda()
    for blk in (0, 128):
        res = {}
        for t in ("u8", "u16", "w32", "i32"):
            try:
                r = ap.solve(h, block=blk, tier=t)
                res[t] = r
            except Exception as e:
                res[t] = None
        base = None
        line = []
        for t, r in res.items():
            if r is None:
                line.append(f"{t}:n/a"); continue
            if base is None:
                base = r; line.append(f"{t}:base"); continue
            line.append(f"{t}:{'same' if torch.equal(r.distances, base.distances) and torch.equal(r.index, base.index) else ('dist-same-pred-DIFF' if torch.equal(r.distances, base.distances) else 'DIFF')}")
        print(n, rho, "block", blk, " ".join(line), flush=True)
