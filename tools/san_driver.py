#!/usr/bin/env python3
"""Small solves for compute-sanitizer (tools/sanitize.sh): every kernel family on a case the
sanitizer finishes in seconds, each checked against the oracle so the run is a real one.

usage: tools/san_driver.py CASE   (CASE in: fw_u8 fw_u16 fw_w32 fw_f32 rk_floor rk_aligned fused_u8 fused_w32
                                   minplus squaring classic)"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2310_03983_b200 as ap  # noqa: E402
from conftest import INF_RAW, random_graph_raw  # noqa: E402
from oracle import oracle as orc  # noqa: E402


def check(cond, what):
    if not cond:
        raise SystemExit(f"FAILED: {what}")
    print("ok", what, flush=True)


def main(case: str):
    if case.startswith("fw_"):
        tier = case[3:]
        wmax = {"u8": 9, "u16": 60, "w32": 5000, "f32": 9}[tier]
        raw = random_graph_raw(512, 0.05, wmax, 3)
        want, _ = orc.fw_classic(raw)
        if tier == "f32":   # continuous weights: the blocked f32 closure + deferred-argmin kernel
            h = ap.continuous_costs(ap.GenParams(512, 0.1, 100, 9))
            r = ap.solve(torch.from_numpy(h).cuda(), block=128)
            check(r.info["tier"] == "f32", "f32 tier")
            ok, why = ap.check_pred_paths(torch.from_numpy(h).cuda(), r.distances, r.index, 1e-5)
            check(ok, f"fw f32 pred paths ({why})")
            return
        s = ap.fw_classic(ap.CostMatrix(raw), tier=tier, block=128)
        check(np.array_equal(s.distances.raw, want), f"fw {tier} distances")
    elif case == "rk_floor":
        raw = random_graph_raw(301, 0.05, 9, 4)
        want, wv = orc.rkleene(raw, 64)
        r = ap.rkleene(ap.CostMatrix(raw))
        check(np.array_equal(r.distances.raw, want) and np.array_equal(r.via.raw, wv), "rkleene floor via")
        raw64 = random_graph_raw(301, 0.05, 1 << 40, 5)
        want, wv = orc.rkleene(raw64, 64)
        r = ap.rkleene(ap.CostMatrix(raw64))
        check(np.array_equal(r.distances.raw, want) and np.array_equal(r.via.raw, wv), "rkleene floor i64 odd n")
    elif case == "rk_aligned":
        raw = random_graph_raw(640, 0.05, 9, 6)
        want, _ = orc.rkleene(raw, 64)
        r = ap.rkleene(ap.CostMatrix(raw), split="aligned", track="pred", base_threshold=256)
        check(np.array_equal(r.distances.raw, want), "rkleene aligned")
    elif case.startswith("fused_"):
        from paper_2310_03983_b200.distributed import fw_blocked_emulated
        from paper_2310_03983_b200.distributed_rk import rkleene_emulated

        alpha = 100 if case == "fused_u8" else 50000
        h = torch.from_numpy(ap.dense_costs(ap.GenParams(600, 0.05, alpha, 7), np.int32)).cuda()
        single = ap.solve(h, "fw_blocked", block=128)
        d, p, info = fw_blocked_emulated(h, 2, block=128, fused=True)
        check(torch.equal(d, single.distances) and torch.equal(p, single.index), f"fused FW push ({info['tier']})")
        d2, p2, info2 = rkleene_emulated(h, 2, base_threshold=256, fused=True)
        check(torch.equal(d2, single.distances) and info2["replicas_equal"], f"fused R-Kleene ({info2['tier']})")
    elif case == "minplus":
        g = np.load(ROOT / "tests" / "golden" / "minplus.npz")
        for k in range(int(g["count"])):
            r = ap.minplus_product(ap.CostMatrix(g[f"p{k}_x"]), ap.CostMatrix(g[f"p{k}_y"]),
                                   offsets=tuple(int(o) for o in g[f"p{k}_off"]))
            check(np.array_equal(r.via.raw, g[f"p{k}_via"]), f"minplus golden {k}")
    elif case == "squaring":
        raw = random_graph_raw(200, 0.03, 9, 8)
        want, wv, it = orc.fw_squaring(raw)
        r = ap.fw_squaring(ap.CostMatrix(raw))
        check(np.array_equal(r.via.raw, wv) and r.iterations == it, "fw_squaring")
    elif case == "classic":
        raw = random_graph_raw(256, 0.05, 9, 9, zero_frac=0.02)
        want, wp = orc.fw_classic(raw)
        s = ap.fw_classic(ap.CostMatrix(raw), method="classic")
        check(np.array_equal(s.pred.raw, wp), "classic order pred")
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main(sys.argv[1])
