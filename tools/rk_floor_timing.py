#!/usr/bin/env python3
"""Time the reference-parity R-Kleene (rkleene(h): floor split, via, base_threshold 64 -- the
reference's defaults, bit-exact via) at a few n."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["2048", "8192"])]:
    h = ap.CostMatrix(ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int64), _validated=True)
    ap.rkleene(h)
    t = time.perf_counter()
    r = ap.rkleene(h)
    dt = time.perf_counter() - t
    print(f"rkleene(h) floor/via thr=64 n={n}: {dt * 1e3:.1f} ms, device {r.info['device_ms']:.1f} ms, "
          f"tier {r.info['tier']}, launches {r.info['launches']}", flush=True)
