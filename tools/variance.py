#!/usr/bin/env python3
"""Repeat one solve and print every device time (run-to-run variance check).
usage: tools/variance.py n rho reps [alg]"""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def main():
    n, rho, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
    alg = sys.argv[4] if len(sys.argv) > 4 else "fw_blocked"
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)).cuda()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = ap.solve(h, alg)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"n={n} rho={rho} {alg} tier={r.info['tier']} block={r.info.get('block')} ms: "
          + " ".join(f"{t:.1f}" for t in ts) + f" | {clk}", flush=True)


if __name__ == "__main__":
    main()
