"""GPU parity at BASELINE's stated sizes (SURVEY.md 8(d) "Check" column).

* C2  fw_classic n=4096 rho=1.0, C3 rkleene n=8192 rho=1.0 and the bench graph n=16384 rho=0.1:
  the GPU results hash to the digests of the REFERENCE's own int64 outputs, recorded in
  tests/golden/large.json by tests/golden/make_golden_large.py (which runs /root/reference in
  the build container).  Distances are bitwise on every path (int64 API, int32, integral fp32);
  ``method="classic"`` pred and the floor-split R-Kleene via are bitwise too.
* C2 continuous variant: fp32 weights U[1, 100) on the C2 mask, within rtol 1e-5 of the float64
  FW (oracle.fw_f64, bit-identical to networkx floyd_warshall_numpy: tests/test_oracle.py), and
  every predecessor path re-summed in float64 within the same tolerance.
* C5 grid n in {1024, 2048} x rho in {0.002 .. 1.0}: FW and R-Kleene, int32 and fp32, bitwise
  against the oracle (pinned to the reference by tests/test_oracle.py).
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, INF_RAW
from oracle import oracle as orc

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200.core import INF32

pytestmark = pytest.mark.gpu

LARGE = json.loads((GOLDEN / "large.json").read_text())
RTOL = 1e-5   # north star: float32 graphs within 1e-5 relative on distances


def as_ref_int64(a) -> np.ndarray:
    """int32 (INF32) / float32 (+inf, integral) / int64 -> the reference's int64 INF_RAW form."""
    if not isinstance(a, np.ndarray):
        a = a.cpu().numpy()
    if a.dtype == np.int64:
        return a
    inf = (a == INF32) if a.dtype == np.int32 else ~np.isfinite(a)
    out = np.where(inf, 0, a).astype(np.int64)
    out[inf] = INF_RAW
    return out


def as_int32(t):
    """Device fp32 (+inf) / int32 tensor -> int32 with INF32 (for the integer pred certificate)."""
    import torch

    if t.dtype == torch.int32:
        return t
    fin = torch.isfinite(t)
    return torch.where(fin, t, torch.zeros_like(t)).to(torch.int32).masked_fill(~fin, INF32)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(as_ref_int64(a)).tobytes()).hexdigest()


def gen(key: str, dtype):
    e = LARGE[key]
    return ap.dense_costs(ap.GenParams(e["n"], e["rho"], e["alpha"], e["seed"]), dtype)


def test_c2_fw_classic_reference_digests(cuda):
    import torch

    ref = LARGE["c2"]
    raw = gen("c2", np.int64)
    assert digest(raw) == ref["input_sha256"], "generator differs from the reference's generate()"
    s = ap.fw_classic(ap.CostMatrix(raw))                         # blocked (default)
    assert digest(s.distances.raw) == ref["dist_sha256"]
    ok, why = ap.check_pred_tree(raw, s.distances.raw, s.pred.raw, INF_RAW)
    assert ok, why
    c = ap.fw_classic(ap.CostMatrix(raw), method="classic")       # classic k order: pred bitwise
    assert digest(c.distances.raw) == ref["dist_sha256"]
    assert digest(c.pred.raw) == ref["pred_sha256"]
    r32 = ap.solve(gen("c2", np.int32))                           # int32 through apsp_solve_host
    assert digest(r32.distances) == ref["dist_sha256"]
    h32 = torch.from_numpy(gen("c2", np.float32)).cuda()          # fp32 (BASELINE C2 dtype), device API
    f = ap.solve(h32)
    assert digest(f.distances) == ref["dist_sha256"]
    fw32 = ap.solve(h32, tier="w32")                              # exact 32-bit tier, no narrow store
    assert digest(fw32.distances) == ref["dist_sha256"]


def test_c2_continuous_fp32_within_tolerance_of_float64(cuda):
    import torch

    e = LARGE["c2"]
    h = ap.continuous_costs(ap.GenParams(e["n"], e["rho"], e["alpha"], e["seed"]))
    want = orc.fw_f64(h.astype(np.float64))
    hd = torch.from_numpy(h).cuda()
    wd = torch.from_numpy(want).cuda()
    for r in (ap.solve(hd), ap.solve(hd, "rkleene", track="pred", base_threshold=512)):
        assert r.info["tier"] == "f32"
        d = r.distances.double()
        assert torch.equal(torch.isfinite(d), torch.isfinite(wd))
        fin = torch.isfinite(wd)
        rel = ((d[fin] - wd[fin]).abs() / wd[fin].clamp(min=1e-30)).max().item()
        assert rel <= RTOL, rel
        ok, why = ap.check_pred_paths(hd, r.distances, r.index, RTOL)
        assert ok, why


def test_c3_rkleene_reference_digests(cuda):
    import torch

    ref = LARGE["c3"]
    raw = gen("c3", np.int64)
    assert digest(raw) == ref["input_sha256"]
    r = ap.rkleene(ap.CostMatrix(raw))        # the reference's defaults: floor split, threshold 64, via
    assert digest(r.distances.raw) == ref["dist_sha256"]
    assert digest(r.via.raw) == ref["via_sha256"]
    h32 = torch.from_numpy(gen("c3", np.float32)).cuda()
    f = ap.solve(h32, "rkleene", track="pred", base_threshold=2048)   # aligned perf schedule, fp32
    assert digest(f.distances) == ref["dist_sha256"]
    ok, why = ap.check_pred_tree(as_int32(h32), as_int32(f.distances), f.index, INF32)
    assert ok, why


def test_bench_graph_reference_digest(cuda):
    import torch

    ref = LARGE["c16k"]
    h = gen("c16k", np.int32)
    s = ap.solve(h)                           # the bench's C ABI call: apsp_solve_host, host buffers
    assert digest(s.distances) == ref["dist_sha256"]
    hd = torch.from_numpy(h).cuda()
    ok, why = ap.check_pred_tree(hd, torch.from_numpy(s.distances).cuda(), torch.from_numpy(s.index).cuda(), INF32)
    assert ok, why


@pytest.mark.parametrize("n", [1024, 2048])
@pytest.mark.parametrize("rho", [0.002, 0.01, 0.1, 0.5, 1.0])
def test_c5_grid_fw_and_rkleene_vs_oracle(cuda, n, rho):
    import torch

    raw = ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int64)
    want, _ = orc.rkleene(raw, 64)
    h32 = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 7 + n), np.int32)).cuda()
    hf = h32.float().masked_fill(h32 == INF32, float("inf"))
    for h in (h32, hf):
        for alg in ("fw_blocked", "rkleene"):
            r = ap.solve(h, alg, track="pred")
            assert np.array_equal(as_ref_int64(r.distances), want), (alg, h.dtype)
            ok, why = ap.check_pred_tree(h32, as_int32(r.distances), r.index, INF32)
            assert ok, (alg, h.dtype, why)
