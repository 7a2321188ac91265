#!/usr/bin/env python3
"""Re-run one stress case step by step (debug helper): repro_case.py seed index"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
import paper_2310_03983_b200 as ap  # noqa: E402
from stress import rand_raw  # noqa: E402

seed, idx = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
for c in range(idx + 1):
    small = rng.random() < 0.7
    n = int(rng.integers(1, 700)) if small else int(rng.choice([2176, 2304, 2560, 3072]))
    raw, dens, wmax = rand_raw(rng, n)
print("case", n, dens, wmax, small, flush=True)
h = ap.CostMatrix(raw.copy(), _validated=True)
for name, fn in (("fw", lambda: ap.fw_classic(h)), ("classic", lambda: ap.fw_classic(h, method="classic")),
                 ("rk", lambda: ap.rkleene(h)),
                 ("rkpred", lambda: ap.rkleene(h, track="pred", split="aligned", base_threshold=128))):
    try:
        r = fn()
        print(name, "ok", r.info.get("tier"), flush=True)
    except Exception as e:
        print(name, "FAILED", type(e).__name__, e, flush=True)
        break
