#!/usr/bin/env python3
"""FW device time per pivot block: tools/block_sweep.py n rho b1 b2 ... (median of 3 after 3 warm-ups).
rho prefixed with "c" (e.g. c1.0): continuous fp32 weights U[1,100) on the generator's mask
(the BASELINE C2 variant, as tools/f32_timing.py)."""

from __future__ import annotations

import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def main():
    n, cont = int(sys.argv[1]), sys.argv[2].startswith("c")
    rho = float(sys.argv[2].lstrip("c"))
    if cont:
        hn = ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.float32)
        rng = np.random.default_rng(n)
        fin = np.isfinite(hn) & (hn > 0)
        hn[fin] = rng.uniform(1.0, 100.0, size=int(fin.sum())).astype(np.float32)
    else:
        hn = ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)
    h = torch.from_numpy(hn).cuda()
    for b in map(int, sys.argv[3:]):
        fn = lambda: ap.solve(h, "fw_blocked", block=b)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"n={n} rho={sys.argv[2]} block={b}: {statistics.median(ts):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
