"""Property tests on the GPU solvers, after the reference's hypothesis suite
(test_solvers.py:139-192, test_minplus.py:184-214): every solver equals the oracle on random
graphs, results are idempotent, satisfy the triangle inequality, reconstruct valid paths, and
are deterministic across repeated calls."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from conftest import INF_RAW
from oracle import oracle as orc

import paper_2310_03983_b200 as ap

pytestmark = pytest.mark.gpu
SETTINGS = settings(deadline=None, max_examples=25, suppress_health_check=[HealthCheck.function_scoped_fixture])


@st.composite
def cost_matrices(draw, max_n=160, max_w=60):
    n = draw(st.integers(1, max_n))
    seed = draw(st.integers(0, 2**31))
    dens = draw(st.sampled_from([0.0, 0.02, 0.1, 0.5, 1.0]))
    zeros = draw(st.sampled_from([0.0, 0.0, 0.2]))
    rng = np.random.default_rng(seed)
    raw = rng.integers(1, max_w + 1, size=(n, n)).astype(np.int64)
    if zeros:
        raw[rng.random((n, n)) < zeros] = 0
    raw[rng.random((n, n)) >= dens] = INF_RAW
    np.fill_diagonal(raw, 0)
    return raw


@given(cost_matrices())
@SETTINGS
def test_all_solvers_match_oracle(cuda, raw):
    want, want_pred = orc.fw_classic(raw)
    h = ap.CostMatrix(raw)
    for name, solver in ap.SOLVERS.items():
        s = solver(h)
        assert np.array_equal(s.distances.raw, want), name
    s = ap.fw_classic(h)
    ok, why = ap.check_pred_tree(raw, s.distances.raw, s.pred.raw, INF_RAW)
    assert ok, why
    c = ap.fw_classic(h, method="classic")
    assert np.array_equal(c.pred.raw, want_pred)
    r = ap.rkleene(h, split="aligned", track="pred", base_threshold=128)
    assert np.array_equal(r.distances.raw, want)
    ok, why = ap.check_pred_tree(raw, r.distances.raw, r.pred.raw, INF_RAW)
    assert ok, why


@given(cost_matrices(max_n=96), st.sampled_from([1, 2, 16, 64]))
@SETTINGS
def test_rkleene_via_matches_oracle_and_invariant(cuda, raw, thr):
    want_d, want_via = orc.rkleene(raw, thr)
    r = ap.rkleene(ap.CostMatrix(raw), base_threshold=thr)
    assert np.array_equal(r.distances.raw, want_d)
    assert np.array_equal(r.via.raw, want_via)


@given(cost_matrices(max_n=120))
@SETTINGS
def test_idempotence_and_triangle_inequality(cuda, raw):
    s = ap.fw_classic(ap.CostMatrix(raw))
    d = s.distances
    again = ap.fw_classic(d)
    assert ap.matrices_equal(again.distances, d)
    dd = d.raw
    fin = dd != INF_RAW
    # saturated sums exceed INF_RAW but never undercut a finite cell (test_solvers.py:175-182)
    for k in range(dd.shape[0]):
        assert (dd <= dd[:, k, None] + dd[None, k, :]).all()
    assert (dd[fin] >= 0).all()


@given(cost_matrices(max_n=64), cost_matrices(max_n=64))
@SETTINGS
def test_minplus_product_matches_oracle(cuda, x, y):
    n = min(x.shape[0], y.shape[0])
    x, y = x[:n, :n], y[:n, :n]
    want = orc.product(x, y)
    r = ap.minplus_product(ap.CostMatrix(x), ap.CostMatrix(y))
    assert np.array_equal(r.distances.raw, want[0]) and np.array_equal(r.via.raw, want[1])


def test_determinism_repeated_calls(cuda):
    raw = ap.dense_costs(ap.GenParams(1500, 0.05, 100, 9), np.int64)
    a = ap.fw_classic(ap.CostMatrix(raw))
    for _ in range(3):
        b = ap.fw_classic(ap.CostMatrix(raw))
        assert np.array_equal(a.distances.raw, b.distances.raw) and np.array_equal(a.pred.raw, b.pred.raw)
