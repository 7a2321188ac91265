"""Path reconstruction (paths.py; reference semantics paths.py:34-105) on CPU, with the pred /
via matrices produced by the oracle (no GPU needed)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import INF_RAW, random_graph_raw
from oracle import oracle as orc

import paper_2310_03983_b200 as ap

CHAIN = ap.Graph(3, [(0, 1, 3), (1, 2, 4)])


def classic(g: ap.Graph):
    d, p = orc.fw_classic(ap.cost_matrix_from_graph(g).raw)
    return ap.CostMatrix(d), ap.PredMatrix(p)


def squaring(g: ap.Graph):
    d, v, _ = orc.fw_squaring(ap.cost_matrix_from_graph(g).raw)
    return ap.CostMatrix(d), ap.ViaMatrix(v)


def graph_of(raw: np.ndarray) -> ap.Graph:
    n = raw.shape[0]
    u, v = np.nonzero((raw != INF_RAW) & ~np.eye(n, dtype=bool))
    return ap.Graph(n, [(int(a), int(b), int(raw[a, b])) for a, b in zip(u, v)])


def edge_sum(g: ap.Graph, path: ap.Path) -> int:
    w = {(u, v): c for u, v, c in g.edges}
    return sum(w[(a, b)] for a, b in zip(path.vertices, path.vertices[1:]))


def test_pred_known_answers():
    d, p = classic(CHAIN)
    assert ap.path_from_pred(p, d, 2, 2) == ap.Path((2,), 0)
    got = ap.path_from_pred(p, d, 0, 2)
    assert got.vertices == (0, 1, 2) and got.total_cost == 7 == edge_sum(CHAIN, got)
    d0, p0 = classic(ap.Graph(2, []))
    assert ap.path_from_pred(p0, d0, 0, 1) is None
    with pytest.raises(IndexError):
        ap.path_from_pred(p, d, 0, 3)
    with pytest.raises(IndexError):
        ap.path_from_pred(p, d, -1, 0)
    with pytest.raises(ap.DimensionError):
        ap.path_from_pred(ap.PredMatrix(np.full((2, 2), -1)), d, 0, 1)


def test_pred_corruption():
    d, p = classic(CHAIN)
    hole = p.raw.copy()
    hole[0, 2] = -1                      # finite distance, no predecessor
    with pytest.raises(ap.CorruptPredError):
        ap.path_from_pred(ap.PredMatrix(hole), d, 0, 2)
    loop = p.raw.copy()
    loop[0, 2] = 2                       # the walk never leaves the target
    with pytest.raises(ap.CorruptPredError):
        ap.path_from_pred(ap.PredMatrix(loop), d, 0, 2)


def test_via_known_answers_and_corruption():
    g1 = ap.Graph(2, [(0, 1, 3)])
    d1, v1 = squaring(g1)
    assert ap.path_from_via(v1, d1, g1, 0, 1) == ap.Path((0, 1), 3)
    d, v = squaring(CHAIN)
    assert v[0, 2] == 1
    got = ap.path_from_via(v, d, CHAIN, 0, 2)
    assert got.vertices == (0, 1, 2) and got.total_cost == 7
    assert ap.path_from_via(v, d, CHAIN, 1, 1) == ap.Path((1,), 0)
    g0 = ap.Graph(2, [])
    d0, v0 = squaring(g0)
    assert ap.path_from_via(v0, d0, g0, 0, 1) is None
    no_edge = v.raw.copy()
    no_edge[0, 2] = -1                   # claims the missing edge (0, 2)
    with pytest.raises(ap.CorruptViaError):
        ap.path_from_via(ap.ViaMatrix(no_edge), d, CHAIN, 0, 2)
    self_split = v.raw.copy()
    self_split[0, 2] = 2                 # (0,2) splits into (0,2) forever
    with pytest.raises(ap.CorruptViaError):
        ap.path_from_via(ap.ViaMatrix(self_split), d, CHAIN, 0, 2)


@pytest.mark.parametrize("seed", range(6))
def test_pred_and_via_paths_sum_to_distances(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 40))
    raw = random_graph_raw(n, float(rng.choice([0.05, 0.2, 0.6])), 9, seed)
    g = graph_of(raw)
    d, p = orc.fw_classic(raw)
    rd, via = orc.rkleene(raw, 4)
    D, P, V = ap.CostMatrix(d), ap.PredMatrix(p), ap.ViaMatrix(via)
    RD = ap.CostMatrix(rd)
    for s in range(n):
        for t in range(n):
            a = ap.path_from_pred(P, D, s, t)
            b = ap.path_from_via(V, RD, g, s, t)
            if d[s, t] == INF_RAW:
                assert a is None and b is None
                continue
            for path in (a, b):
                assert path.vertices[0] == s and path.vertices[-1] == t
                assert edge_sum(g, path) == d[s, t] == path.total_cost
                assert len(path.vertices) <= n
