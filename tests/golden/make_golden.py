"""Generate the golden fixtures of tests/golden/ by running the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports apsp 0.1.0 read-only from /root/reference/pkg/src and records, for seeded inputs,
the reference's own outputs:

* c1_fw.npz        BASELINE config 1: GenParams(256, 0.1, 100, 7+256) -> fw_classic dist + pred
* rk_*.npz         rkleene dist + via at (n, rho, base_threshold) from SURVEY.md 8(c)
* sq.npz           fw_squaring dist + via + iterations
* minplus.npz      minplus_product (with offsets) / minplus_accumulate cases
* suite.npz        40 graphs of the reference's suite recipe (conftest.py:32-50, master seed
                   20260825): fw_classic dist+pred, rkleene(t=16) via, fw_squaring via+iterations
* gen.json         sha256 of cost_matrix_from_graph(generate(p)).raw for generator params
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import apsp
    from apsp.core import INF_RAW, CostMatrix, Graph
    from apsp.minplus import minplus_accumulate, minplus_product

    # 1. BASELINE config 1
    p = apsp.GenParams(256, 0.1, 100, 7 + 256)
    h = apsp.cost_matrix_from_graph(apsp.generate(p))
    s = apsp.fw_classic(h)
    np.savez_compressed(OUT / "c1_fw.npz", h=h.raw, dist=s.distances.raw, pred=s.pred.raw)

    # 2. rkleene via (bit-exact via cases)
    for n, rho, thr, seed in [(300, 0.1, 64, 11), (200, 0.05, 16, 12), (130, 1.0, 8, 13), (150, 0.1, 1, 14)]:
        g = apsp.generate(apsp.GenParams(n, rho, 100, seed))
        hm = apsp.cost_matrix_from_graph(g)
        r = apsp.rkleene(hm, base_threshold=thr)
        np.savez_compressed(OUT / f"rk_n{n}_t{thr}.npz", h=hm.raw, dist=r.distances.raw, via=r.via.raw,
                            thr=np.int64(thr))

    # 3. fw_squaring
    cases = {}
    for idx, (n, rho, seed) in enumerate([(5, 0.0, 0), (64, 0.2, 21), (97, 0.05, 22)]):
        if n == 5:
            hm = apsp.cost_matrix_from_graph(Graph(5, [(i, i + 1, 1) for i in range(4)]))
        else:
            hm = apsp.cost_matrix_from_graph(apsp.generate(apsp.GenParams(n, rho, 100, seed)))
        r = apsp.fw_squaring(hm)
        cases[f"h{idx}"] = hm.raw
        cases[f"dist{idx}"] = r.distances.raw
        cases[f"via{idx}"] = r.via.raw
        cases[f"it{idx}"] = np.int64(r.iterations)
    np.savez_compressed(OUT / "sq.npz", **cases)

    # 4. minplus product / accumulate (test_minplus.py patterns, incl. offsets and ties)
    rng = np.random.default_rng(20261018)
    mp = {}
    k = 0
    for n1, n2, n3, offs in [(12, 12, 12, (0, 0, 0)), (5, 5, 7, (0, 0, 5)), (7, 5, 5, (5, 0, 0)),
                             (33, 17, 40, (3, 9, 11)), (64, 64, 64, (0, 0, 0)), (1, 1, 1, (0, 0, 0))]:
        x = rng.integers(0, 51, size=(n1, n2)).astype(np.int64)
        x[rng.random((n1, n2)) < 0.25] = INF_RAW
        y = rng.integers(0, 51, size=(n2, n3)).astype(np.int64)
        y[rng.random((n2, n3)) < 0.25] = INF_RAW
        r = minplus_product(CostMatrix(x), CostMatrix(y), offsets=offs)
        mp[f"p{k}_x"], mp[f"p{k}_y"], mp[f"p{k}_off"] = x, y, np.asarray(offs, np.int64)
        mp[f"p{k}_dist"], mp[f"p{k}_via"] = r.distances.raw, r.via.raw
        z = rng.integers(0, 120, size=(n1, n3)).astype(np.int64)
        z[rng.random((n1, n3)) < 0.3] = INF_RAW
        vin = rng.integers(-1, 9, size=(n1, n3)).astype(np.int64)
        a = minplus_accumulate(CostMatrix(z), CostMatrix(x), CostMatrix(y), via=apsp.ViaMatrix(vin),
                               inner_offset=offs[1])
        mp[f"a{k}_z"], mp[f"a{k}_vin"] = z, vin
        mp[f"a{k}_dist"], mp[f"a{k}_via"] = a.distances.raw, a.via.raw
        k += 1
    np.savez_compressed(OUT / "minplus.npz", count=np.int64(k), **mp)

    # 5. suite recipe (conftest.py:32-50), first 40 generator graphs with n <= 96
    srng = np.random.default_rng(20260825)
    rhos = (0.05, 0.25, 0.5, 1.0)
    suite = {}
    kept = 0
    for i in range(292):
        n = int(srng.integers(1, 129))
        rho = rhos[i % 4]
        seed = int(srng.integers(0, 2**63))
        if n > 96 or kept >= 40:
            continue
        hm = apsp.cost_matrix_from_graph(apsp.generate(apsp.GenParams(n, rho, 100, seed)))
        fc = apsp.fw_classic(hm)
        rk = apsp.rkleene(hm, base_threshold=16)
        sq = apsp.fw_squaring(hm)
        suite[f"h{kept}"] = hm.raw
        suite[f"dist{kept}"] = fc.distances.raw
        suite[f"pred{kept}"] = fc.pred.raw
        suite[f"rkvia{kept}"] = rk.via.raw
        suite[f"sqvia{kept}"] = sq.via.raw
        suite[f"sqit{kept}"] = np.int64(sq.iterations)
        kept += 1
    np.savez_compressed(OUT / "suite.npz", count=np.int64(kept), **suite)

    # 6. generator hashes
    gen = []
    for v, rho, alpha, seed in [(256, 0.1, 100, 263), (1000, 0.5, 100, 5), (1023, 1.0, 100, 11), (513, 0.7, 3, 9),
                                (301, 0.9, 1_000_000_007, 77), (4096, 0.1, 100, 4103)]:
        g = apsp.generate(apsp.GenParams(v, rho, alpha, seed))
        raw = apsp.cost_matrix_from_graph(g).raw
        gen.append({"v": v, "rho": rho, "alpha": alpha, "seed": seed, "n_edges": g.n_edges,
                    "sha256": hashlib.sha256(np.ascontiguousarray(raw).tobytes()).hexdigest()})
    (OUT / "gen.json").write_text(json.dumps(gen, indent=1) + "\n")
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
