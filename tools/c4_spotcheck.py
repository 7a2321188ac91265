#!/usr/bin/env python3
"""BASELINE config 4 on one GPU: n=32768 generator graph (rho=0.1, int32), blocked FW with
predecessors, then an independent spot check of sampled source rows against scipy's Dijkstra
 and the predecessor-tree certificate on the same rows.

usage: tools/c4_spotcheck.py [n] [rows]      (defaults 32768, 8)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402
from paper_2310_03983_b200.core import INF32  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    t = time.perf_counter()
    h = ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int32)
    print(f"generated n={n} in {time.perf_counter() - t:.1f}s", flush=True)
    hd = torch.from_numpy(h).cuda()
    r = ap.solve(hd, "fw_blocked")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = ap.solve(hd, "fw_blocked")
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"fw_blocked n={n}: {ms:.1f} ms ({n ** 3 / ms / 1e9:.2f} T upd/s) tier={r.info['tier']} "
          f"block={r.info['block']}", flush=True)
    rng = np.random.default_rng(n)
    rows = np.sort(rng.choice(n, size=nrows, replace=False))
    dist_rows = r.distances[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.int64)
    pred_rows = r.index[torch.from_numpy(rows).cuda()].cpu().numpy().astype(np.int64)
    del r, hd
    torch.cuda.empty_cache()
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra

    fin = (h != INF32)
    np.fill_diagonal(fin, False)
    ii, jj = np.nonzero(fin)
    g = csr_matrix((h[ii, jj].astype(np.float64), (ii, jj)), shape=(n, n))
    del ii, jj, fin
    t = time.perf_counter()
    ref = dijkstra(g, directed=True, indices=rows)
    print(f"scipy dijkstra on {nrows} rows: {time.perf_counter() - t:.1f}s", flush=True)
    ref_i = np.where(np.isinf(ref), INF32, ref).astype(np.int64)
    ok_dist = np.array_equal(ref_i, dist_rows)
    # predecessor certificate on the sampled rows: d[s][p] + w[p][j] == d[s][j] for every
    # reachable j != s (pred rows point at a real last hop of a shortest path)
    ok_pred = True
    for a, s in enumerate(rows):
        d = dist_rows[a]
        p = pred_rows[a]
        reach = (d != INF32) & (np.arange(n) != s)
        pj = p[reach]
        if (pj < 0).any():
            ok_pred = False
            break
        jj = np.nonzero(reach)[0]
        if not np.array_equal(d[pj] + h[pj, jj].astype(np.int64), d[jj]):
            ok_pred = False
            break
    print(f"rows {rows.tolist()}: distances == scipy dijkstra: {ok_dist}; pred last-hop certificate: {ok_pred}",
          flush=True)
    if not (ok_dist and ok_pred):
        sys.exit(1)


if __name__ == "__main__":
    main()
