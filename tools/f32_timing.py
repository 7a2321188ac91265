#!/usr/bin/env python3
"""Continuous-weight fp32 timing (BASELINE C2 variant): the generator's mask with U[1,100) fp32
weights; FW and R-Kleene device time, and the max relative error against a float64 FW on a
row sample.  usage: tools/f32_timing.py n"""

from __future__ import annotations

import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402


def timed(fn):
    for _ in range(3):
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
    return statistics.median(ts), r


def main():
    n = int(sys.argv[1])
    h = ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.float32)
    rng = np.random.default_rng(n)
    fin = np.isfinite(h) & (h > 0)
    h[fin] = rng.uniform(1.0, 100.0, size=int(fin.sum())).astype(np.float32)
    hd = torch.from_numpy(h).cuda()
    ms, r = timed(lambda: ap.solve(hd, "fw_blocked"))
    print(f"n={n} fp32 continuous fw_blocked: {ms:.2f} ms ({n ** 3 / ms / 1e9:.2f} T upd/s) tier={r.info['tier']}")
    ms2, r2 = timed(lambda: ap.solve(hd, "rkleene", track="pred", split="aligned", base_threshold=1024))
    print(f"n={n} fp32 continuous rkleene: {ms2:.2f} ms ({n ** 3 / ms2 / 1e9:.2f} T upd/s)")
    # float64 reference on sampled rows: Dijkstra-free check via Bellman fixpoint on the
    # returned distances (row sample) plus rel error against float64 relaxation of the same
    D = r.distances.double()
    H = hd.double()
    rows = torch.arange(0, n, max(1, n // 16), device=hd.device)
    best = torch.full((len(rows), n), float("inf"), dtype=torch.float64, device=hd.device)
    for k0 in range(0, n, 512):
        best = torch.minimum(best, (D[rows, k0:k0 + 512].unsqueeze(2) + H[k0:k0 + 512].unsqueeze(0)).amin(1))
    best[torch.arange(len(rows)), rows] = 0
    rel = ((D[rows] - best).abs() / best.clamp(min=1)).max().item()
    print(f"max rel deviation of the Bellman fixpoint on {len(rows)} rows: {rel:.2e}; "
          f"rkleene == fw: {bool(torch.allclose(r.distances, r2.distances, rtol=1e-5))}")


if __name__ == "__main__":
    main()
