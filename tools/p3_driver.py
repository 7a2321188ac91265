#!/usr/bin/env python3
"""One blocked-FW solve at n=16384 (bench workload) for ncu captures of the phase-3 tile kernel.

usage (GPU box): ncu -k regex:minplus_nt_kernel ... python tools/p3_driver.py [n]
tools/p3_capture.sh picks a mid-solve phase-3b launch from a launch list and captures it."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int32)).cuda()
    s = ap.solve(h)
    torch.cuda.synchronize()
    print("tier", s.info["tier"], "block", s.info.get("block"), flush=True)


if __name__ == "__main__":
    main()
