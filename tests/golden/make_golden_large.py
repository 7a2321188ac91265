"""Record sha256 digests of the REFERENCE's own results at BASELINE's stated sizes.

Run in the build container only (the reference is not on the GPU box); it takes ~40 min on
8 cores:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_large.py [c2] [c3] [c16k]

It imports apsp 0.1.0 read-only from /root/reference/pkg/src and runs, on the reference's own
generator output (`generate` -> `cost_matrix_from_graph`):

* c2   BASELINE config 2: GenParams(4096, 1.0, 100, 7+4096)  -> fw_classic  dist + pred
* c3   BASELINE config 3: GenParams(8192, 1.0, 100, 7+8192)  -> rkleene(base_threshold=64) dist + via
* c16k the bench graph:   GenParams(16384, 0.1, 100, 7+16384) -> rkleene dist (the distances are the
       unique shortest-path lengths, so any exact solver must reproduce them; rkleene is the faster
       reference solver here) + via

Each digest is sha256 over the C-order bytes of the reference's int64 array (INF_RAW = 2**61 for
unreachable, -1 = None in index matrices). The matrices themselves (up to 2 GiB) are not kept.
Output: tests/golden/large.json, merged with any entries already there.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent / "large.json"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(which: list[str]) -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import apsp

    cases = {
        "c2": (4096, 1.0, "fw_classic"),
        "c3": (8192, 1.0, "rkleene"),
        "c16k": (16384, 0.1, "rkleene"),
    }
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    # JIT warm-up (scaling_trend.py:27-30)
    hw = apsp.cost_matrix_from_graph(apsp.generate(apsp.GenParams(64, 0.5, 100, 1)))
    apsp.fw_classic(hw)
    apsp.rkleene(hw)
    for key in which:
        n, rho, alg = cases[key]
        p = apsp.GenParams(n, rho, 100, 7 + n)
        t0 = time.perf_counter()
        g = apsp.generate(p)
        h = apsp.cost_matrix_from_graph(g)
        del g
        t1 = time.perf_counter()
        from apsp.solvers import SOLVERS
        s = SOLVERS[alg](h, workers=os.cpu_count())
        t2 = time.perf_counter()
        d = s.distances.raw
        fin = d[d < apsp.INF_RAW] if hasattr(apsp, "INF_RAW") else d[d < 2**61]
        entry = {
            "n": n, "rho": rho, "alpha": 100, "seed": 7 + n, "algorithm": alg,
            "input_sha256": sha(h.raw),
            "dist_sha256": sha(d),
            "max_finite": int(fin.max()) if fin.size else 0,
            "n_unreachable": int((d >= 2**61).sum()),
            "gen_s": round(t1 - t0, 1), "solve_s": round(t2 - t1, 1),
            "cores": os.cpu_count(),
        }
        if s.pred is not None:
            entry["pred_sha256"] = sha(s.pred.raw)
        if s.via is not None:
            entry["via_sha256"] = sha(s.via.raw)
            entry["base_threshold"] = 64
        res[key] = entry
        OUT.write_text(json.dumps(res, indent=1, sort_keys=True) + "\n")
        print(key, entry, flush=True)
        del s, h, d


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3", "c16k"])
