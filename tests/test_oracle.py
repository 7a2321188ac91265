"""Pin the CPU oracle (oracle/apsp_oracle.c) to the reference's own outputs.

tests/golden/*.npz were produced by tests/golden/make_golden.py running the reference
(apsp 0.1.0) itself; these tests prove the restatement is bit-exact before any GPU result
is judged against it.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, INF_RAW, golden
from oracle import oracle as orc


def test_three_cycle_known_answer():
    # test_solvers.py:32-33 THREE_CYCLE
    h = np.array([[0, 1, INF_RAW], [INF_RAW, 0, 2], [4, INF_RAW, 0]])
    d, pred = orc.fw_classic(h)
    assert d.tolist() == [[0, 1, 3], [6, 0, 2], [4, 5, 0]]
    d2, via = orc.rkleene(h, 1)
    assert d2.tolist() == d.tolist()


def test_chain_with_shortcut_pred():
    # test_solvers.py:62-66: d[0][2] = 7 through vertex 1
    h = np.array([[0, 3, 10], [INF_RAW, 0, 4], [INF_RAW, INF_RAW, 0]])
    d, pred = orc.fw_classic(h)
    assert d[0, 2] == 7 and pred[0, 2] == 1 and pred[0, 1] == 0 and pred[0, 0] == -1


def test_c1_fw_classic_bitwise():
    g = golden("c1_fw.npz")
    d, pred = orc.fw_classic(g["h"])
    assert np.array_equal(d, g["dist"])
    assert np.array_equal(pred, g["pred"])


@pytest.mark.parametrize("name", ["rk_n300_t64.npz", "rk_n200_t16.npz", "rk_n130_t8.npz", "rk_n150_t1.npz"])
def test_rkleene_via_bitwise(name):
    g = golden(name)
    d, via = orc.rkleene(g["h"], int(g["thr"]))
    assert np.array_equal(d, g["dist"])
    assert np.array_equal(via, g["via"])


def test_squaring_bitwise():
    g = golden("sq.npz")
    for i in range(3):
        d, via, it = orc.fw_squaring(g[f"h{i}"])
        assert np.array_equal(d, g[f"dist{i}"])
        assert np.array_equal(via, g[f"via{i}"])
        assert it == int(g[f"it{i}"])


def test_minplus_bitwise():
    g = golden("minplus.npz")
    for k in range(int(g["count"])):
        d, v = orc.product(g[f"p{k}_x"], g[f"p{k}_y"], tuple(g[f"p{k}_off"]))
        assert np.array_equal(d, g[f"p{k}_dist"]), k
        assert np.array_equal(v, g[f"p{k}_via"]), k
        d, v = orc.accumulate(g[f"a{k}_z"], g[f"p{k}_x"], g[f"p{k}_y"], g[f"a{k}_vin"], int(g[f"p{k}_off"][1]))
        assert np.array_equal(d, g[f"a{k}_dist"]), k
        assert np.array_equal(v, g[f"a{k}_via"]), k


def test_suite_bitwise():
    g = golden("suite.npz")
    for i in range(int(g["count"])):
        h = g[f"h{i}"]
        d, pred = orc.fw_classic(h)
        assert np.array_equal(d, g[f"dist{i}"]) and np.array_equal(pred, g[f"pred{i}"])
        d, via = orc.rkleene(h, 16)
        assert np.array_equal(d, g[f"dist{i}"]) and np.array_equal(via, g[f"rkvia{i}"])
        d, via, it = orc.fw_squaring(h)
        assert np.array_equal(via, g[f"sqvia{i}"]) and it == int(g[f"sqit{i}"])


def test_overflow_status():
    # test_minplus.py:243-250: MAX_FINITE_COST - 1 chain overflows
    big = (1 << 60) - 2
    m = np.array([[0, big, INF_RAW], [INF_RAW, 0, big], [INF_RAW, INF_RAW, 0]])
    with pytest.raises(orc.OracleRangeError):
        orc.product(m, m)
    with pytest.raises(orc.OracleRangeError):
        orc.fw_classic(m)


def test_generator_matches_reference_hashes():
    from paper_2310_03983_b200 import GenParams, cost_matrix_from_graph, dense_costs, generate

    for rec in json.loads((GOLDEN / "gen.json").read_text()):
        p = GenParams(rec["v"], rec["rho"], rec["alpha"], rec["seed"])
        raw = dense_costs(p, np.int64, chunk_rows=96)
        assert hashlib.sha256(np.ascontiguousarray(raw).tobytes()).hexdigest() == rec["sha256"], rec
        if rec["v"] <= 1024:
            g = generate(p)
            assert g.n_edges == rec["n_edges"]
            assert np.array_equal(cost_matrix_from_graph(g).raw, raw)


def test_dense_costs_dtypes():
    from paper_2310_03983_b200 import GenParams, dense_costs
    from paper_2310_03983_b200.core import INF32

    p = GenParams(300, 0.2, 100, 5)
    a = dense_costs(p, np.int64)
    b = dense_costs(p, np.int32)
    c = dense_costs(p, np.float32)
    fin = a != INF_RAW
    assert np.array_equal(b[fin], a[fin]) and (b[~fin] == INF32).all()
    assert np.array_equal(c[fin], a[fin].astype(np.float32)) and np.isinf(c[~fin]).all()


@pytest.mark.parametrize("n,density,seed", [(1, 1.0, 0), (57, 0.3, 1), (300, 0.05, 2), (256, 0.6, 3)])
def test_f64_fw_matches_networkx(n, density, seed):
    """oracle.fw_f64 (the C2 continuous-weight reference) is bit-identical to networkx
    floyd_warshall_numpy on the same float64 weights (SURVEY.md 8(d) C2 variant)."""
    nx = pytest.importorskip("networkx")
    rng = np.random.default_rng(seed)
    w = rng.uniform(1.0, 100.0, size=(n, n)).astype(np.float32).astype(np.float64)
    present = (rng.random((n, n)) < density) & ~np.eye(n, dtype=bool)
    g = nx.DiGraph()
    g.add_nodes_from(range(n))
    g.add_weighted_edges_from((int(i), int(j), float(w[i, j])) for i, j in zip(*np.nonzero(present)))
    want = nx.floyd_warshall_numpy(g, nodelist=range(n))
    h = np.where(present, w, np.inf)
    np.fill_diagonal(h, 0.0)
    got = orc.fw_f64(h)
    assert np.array_equal(got, want)
