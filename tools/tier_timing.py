#!/usr/bin/env python3
"""Time fw_blocked / rkleene per value tier on generator graphs (one B200).

usage: tools/tier_timing.py n:rho:tier[:alg] ...   (tier auto|u8|u16|w32|i32|i64, alg fw|rk)
Prints one line per case: device ms (median of 3 after two warm-ups) and T upd/s.
"""

from __future__ import annotations

import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        parts = spec.split(":")
        n, rho, tier = int(parts[0]), float(parts[1]), parts[2]
        alg = parts[3] if len(parts) > 3 else "fw"
        h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)).cuda()
        kw = {} if tier == "auto" else {"tier": tier}
        if alg == "rk":
            fn = lambda: ap.solve(h, "rkleene", track="pred", split="aligned",  # noqa: E731
                                  base_threshold=min(1024, n // 2), **kw)
        else:
            fn = lambda: ap.solve(h, "fw_blocked", **kw)  # noqa: E731
        for _ in range(4):      # lazy module loading, pool growth, clock ramp from idle
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"n={n:6d} rho={rho:<6} {alg} tier={r.info['tier']:4s} block={r.info.get('block')} "
              f"{ms:9.2f} ms {n ** 3 / ms / 1e9:7.2f} T upd/s maxd={r.info['max_finite']}", flush=True)
        del h, r
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
