#!/usr/bin/env python3
"""End-to-end time of the reference-facing Python API (numpy int64 CostMatrix in, frozen int64
ApspSolution out: pageable host memory both ways) at n (default 16384), against the
device-resident solve of the same matrix."""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    p = ap.GenParams(n, 0.1, 100, 7 + n)
    h = ap.CostMatrix(ap.dense_costs(p, np.int64), _validated=True)
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        s = ap.fw_classic(h)
        ts.append((time.perf_counter() - t) * 1e3)
    info = s.info if hasattr(s, "info") else {}
    print(f"fw_classic(CostMatrix int64) n={n}: ms " + " ".join(f"{x:.1f}" for x in ts)
          + f" | device {info.get('device_ms', float('nan')):.1f} ms, up {info.get('h2d_bytes_per_cell')} B/cell, "
          f"down {info.get('d2h_bytes_per_cell')} B/cell", flush=True)
    h32 = ap.dense_costs(p, np.int32)
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        ap.solve(h32)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"solve(numpy int32, pageable) n={n}: ms " + " ".join(f"{x:.1f}" for x in ts), flush=True)


if __name__ == "__main__":
    main()
