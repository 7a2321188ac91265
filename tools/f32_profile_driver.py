#!/usr/bin/env python3
"""One continuous-weight fp32 solve (BASELINE C2 variant) for ncu captures.
usage: tools/f32_profile_driver.py n [algorithm] [block]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402

n = int(sys.argv[1])
alg = sys.argv[2] if len(sys.argv) > 2 else "fw_blocked"
block = int(sys.argv[3]) if len(sys.argv) > 3 else 0
hd = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, 1.0, 100, 7 + n))).cuda()
kw = {"track": "pred", "base_threshold": 512} if alg == "rkleene" else {"block": block}
ap.solve(hd, alg, **kw)
torch.cuda.synchronize()
