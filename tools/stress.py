#!/usr/bin/env python3
"""Randomised cross-checks of the product paths (run on a GPU box; not part of the test suite):
  * small n: every solver entry against the CPU oracle (distances bit-exact, pred certificate);
  * continuous fp32 (small n): FW and R-Kleene within 1e-5 of the float64 oracle, paths re-summed;
  * multi-rank schedules emulated on one GPU (fused peer stores): bitwise equal to one GPU;
  * large n (> 2048, streamed readback, narrowed transfers): host-buffer API == device API.
With APSP_B200_LIB=paper_2310_03983_b200/libapsp_b200_jitter.so (make -C ... jitter) every
synchronisation point of the rings and closures sleeps pseudo-randomly: the race stress run.
usage: tools/stress.py [seconds] [seed] [-v]"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2310_03983_b200 as ap  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2310_03983_b200.core import INF32, INF_RAW  # noqa: E402


def rand_raw(rng, n):
    dens = float(rng.choice([0.002, 0.01, 0.05, 0.3, 1.0]))
    wmax = int(rng.choice([1, 5, 100, 254, 300, 5000, 10 ** 6]))
    raw = rng.integers(1, wmax + 1, size=(n, n)).astype(np.int64)
    if rng.random() < 0.2:
        raw[rng.random((n, n)) < 0.1] = 0
    raw[rng.random((n, n)) >= dens] = INF_RAW
    np.fill_diagonal(raw, 0)
    return raw, dens, wmax


def extra_case(rng, verbose) -> int:
    """Continuous fp32 (FW + R-Kleene vs float64) or an emulated multi-rank schedule."""
    from paper_2310_03983_b200.distributed import fw_blocked_emulated
    from paper_2310_03983_b200.distributed_rk import rkleene_emulated

    if rng.random() < 0.5:
        n = int(rng.integers(1, 700))
        h = ap.continuous_costs(ap.GenParams(n, float(rng.choice([0.01, 0.1, 1.0])), 100, int(rng.integers(1 << 30))))
        tag = f"f32 n={n}"
        want = orc.fw_f64(h.astype(np.float64))
        hd = torch.from_numpy(h).cuda()
        try:
            for r in (ap.solve(hd), ap.solve(hd, "rkleene", track="pred", base_threshold=128)):
                d = r.distances.double().cpu().numpy()
                fin = np.isfinite(want)
                assert np.array_equal(np.isfinite(d), fin), "f32 reachability"
                assert (np.abs(d[fin] - want[fin]) <= 1e-5 * np.maximum(want[fin], 1e-30)).all(), "f32 tolerance"
                ok, why = ap.check_pred_paths(hd, r.distances, r.index, 1e-5)
                assert ok, f"f32 paths: {why}"
        except AssertionError as e:
            print(f"FAIL {tag}: {e}", flush=True)
            return 1
    else:
        n = int(rng.integers(300, 1300))
        world = int(rng.integers(2, 5))
        alpha = int(rng.choice([100, 400, 50000]))
        h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, float(rng.choice([0.02, 0.1])), alpha,
                                                         int(rng.integers(1 << 30))), np.int32)).cuda()
        tag = f"emulated n={n} world={world} alpha={alpha}"
        try:
            single = ap.solve(h, "fw_blocked", block=128)
            d, p, _ = fw_blocked_emulated(h, world, block=128, fused=True)
            assert torch.equal(d, single.distances) and torch.equal(p, single.index), "fused FW"
            rk1 = ap.solve(h, "rkleene", track="pred", base_threshold=256)
            d2, p2, info = rkleene_emulated(h, world, base_threshold=256, fused=True)
            assert torch.equal(d2, rk1.distances) and info["replicas_equal"], "fused R-Kleene"
        except AssertionError as e:
            print(f"FAIL {tag}: {e}", flush=True)
            return 1
    if verbose:
        print("ok", tag, flush=True)
    return 0


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-v" else int(time.time())
    print("seed", seed, "library", ap._native.lib_path(), flush=True)
    rng = np.random.default_rng(seed)
    t0 = time.time()
    cases = fails = 0
    while time.time() - t0 < budget:
        kind = rng.random()
        if kind < 0.12:
            cases += 1
            fails += extra_case(rng, "-v" in sys.argv)
            continue
        small = rng.random() < 0.7
        n = int(rng.integers(1, 700)) if small else int(rng.choice([2176, 2304, 2560, 3072, 3200, 4096]))
        raw, dens, wmax = rand_raw(rng, n)
        h = ap.CostMatrix(raw.copy(), _validated=True)
        tag = f"n={n} dens={dens} wmax={wmax} zeros={int((raw == 0).sum()) - n}"
        if "-v" in sys.argv:
            print("case", tag, flush=True)
        try:
            if small:
                want_d, want_p = orc.fw_classic(raw)
                s = ap.fw_classic(h)
                assert np.array_equal(s.distances.raw, want_d), "fw dist"
                ok, why = ap.check_pred_tree(raw, s.distances.raw, s.pred.raw, INF_RAW)
                assert ok, f"fw pred: {why}"
                c = ap.fw_classic(h, method="classic")
                assert np.array_equal(c.pred.raw, want_p), "classic pred"
                r = ap.rkleene(h)
                assert np.array_equal(r.distances.raw, want_d), "rk dist"
                rp = ap.rkleene(h, track="pred", split="aligned", base_threshold=128)
                ok, why = ap.check_pred_tree(raw, rp.distances.raw, rp.pred.raw, INF_RAW)
                assert ok and np.array_equal(rp.distances.raw, want_d), f"rk pred: {why}"
                bt = int(rng.choice([1, 8, 64]))
                od, ov = orc.rkleene(raw, base_threshold=bt)
                rv = ap.rkleene(h, base_threshold=bt)
                assert np.array_equal(rv.via.raw, ov) and np.array_equal(rv.distances.raw, od), "rk via"
                if n <= 300:
                    sd, sv, si = orc.fw_squaring(raw)
                    sq = ap.fw_squaring(h)
                    assert np.array_equal(sq.distances.raw, sd) and np.array_equal(sq.via.raw, sv), "squaring"
                    assert sq.iterations == si, "squaring iterations"
                # rectangular products on sub-blocks, with offsets, then an accumulate into the result
                n1, n2, n3 = (int(rng.integers(1, n + 1)) for _ in range(3))
                x, y = raw[:n1, :n2], raw[n - n2:, n - n3:]
                offs = tuple(int(o) for o in rng.integers(0, 1000, size=3))
                pd_, pv_ = orc.product(x, y, offs)
                pr = ap.minplus_product(ap.CostMatrix(x.copy()), ap.CostMatrix(y.copy()), offsets=offs)
                assert np.array_equal(pr.distances.raw, pd_) and np.array_equal(pr.via.raw, pv_), "product"
                z = raw[n - n1:, :n3]
                io = int(rng.integers(0, 1000))
                ad, av = orc.accumulate(z, x, y, pv_, io)
                ac = ap.minplus_accumulate(ap.CostMatrix(z.copy()), ap.CostMatrix(x.copy()), ap.CostMatrix(y.copy()),
                                           pr.via, inner_offset=io)
                assert np.array_equal(ac.distances.raw, ad) and np.array_equal(ac.via.raw, av), "accumulate"
            else:
                h32 = np.where(raw == INF_RAW, INF32, np.minimum(raw, 2 ** 20)).astype(np.int32)
                dev = ap.solve(torch.from_numpy(h32.copy()).cuda())
                host = ap.solve(h32)
                assert np.array_equal(host.distances, dev.distances.cpu().numpy()), "host32 dist"
                assert np.array_equal(host.index, dev.index.cpu().numpy()), "host32 pred"
                # an independent schedule (R-Kleene) and the pred certificate on the device
                hd = torch.from_numpy(h32.copy()).cuda()
                rk = ap.solve(hd, "rkleene", track="pred", base_threshold=1024)
                assert torch.equal(rk.distances, dev.distances), "fw == rkleene"
                ok, why = ap.check_pred_tree(hd, dev.distances, dev.index, INF32)
                assert ok, f"large pred: {why}"
                r64 = ap.fw_classic(ap.CostMatrix(np.where(raw == INF_RAW, INF_RAW, np.minimum(raw, 2 ** 20))))
                d64 = np.where(host.distances == INF32, INF_RAW, host.distances.astype(np.int64))
                assert np.array_equal(r64.distances.raw, d64), "int64 api dist"
        except ap.ApspError as e:   # range errors are legitimate for some draws
            if "range" not in str(e).lower():
                fails += 1
                print(f"FAIL {tag}: {type(e).__name__}: {e}", flush=True)
        except AssertionError as e:
            fails += 1
            print(f"FAIL {tag}: {e}", flush=True)
        cases += 1
    print(f"stress: {cases} cases, {fails} failures in {time.time() - t0:.0f}s", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
