"""Wire formats (reference textio.py; tests mirror reference tests/test_textio.py): exact layout,
INF literal, bit-identical round trips, malformed inputs, and a large-matrix round trip that the
reference's per-cell Python loop could not do quickly.  CPU only (host code of the library)."""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import INF_RAW

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200.textio import (
    format_graph,
    format_matrix,
    parse_graph,
    parse_matrix,
    read_graph,
    read_matrix,
    write_graph,
    write_matrix,
)


def test_graph_exact_layout_and_round_trips(tmp_path):
    g = ap.Graph(3, [(0, 1, 5), (2, 0, 7)])
    assert format_graph(g) == "3 2\n0 1 5\n2 0 7\n"
    assert format_graph(ap.Graph(2, [])) == "2 0\n"
    g = ap.Graph(4, [(0, 3, 9), (3, 1, 2), (1, 0, 1)])
    assert parse_graph(format_graph(g)) == g
    p1, p2 = tmp_path / "a.txt", tmp_path / "b.txt"
    write_graph(g, p1)
    write_graph(read_graph(p1), p2)
    assert p1.read_bytes() == p2.read_bytes()


@pytest.mark.parametrize("text", ["", "2\n", "2 1\n", "2 1\n0 1\n", "2 1\n0 1 5\n0 1 5\n", "2 1\n0 1 x\n", "x 0\n",
                                  "2 1\n0 1 5.5\n", "2 1\n0 0 3\n", "2 1\n0 1 0\n"])
def test_malformed_graph_text(text):
    with pytest.raises(ap.MalformedGraphError):
        parse_graph(text)


def test_matrix_exact_layout_and_inf():
    assert format_matrix(ap.CostMatrix.from_rows([[0, 3], [7, 0]])) == "2\n0 3\n7 0\n"
    assert format_matrix(ap.minplus_identity(2)) == "2\n0 INF\nINF 0\n"
    assert parse_matrix("2\n0 INF\nINF 0\n").raw.tolist() == [[0, INF_RAW], [INF_RAW, 0]]
    assert parse_matrix("2\n0 INF\nINF 0").raw.tolist() == [[0, INF_RAW], [INF_RAW, 0]]
    assert parse_matrix("1\n+7\n").raw.tolist() == [[7]]


@pytest.mark.parametrize("text", ["", "2\n0 1\n", "2\n0 1\n0 1\n0 1\n", "2\n0\n0 1\n", "2\n0 -1\nINF 0\n", "x\n",
                                  "2\n0 inf\nINF 0\n", "2\n0  1\n1 0\n", "0\n"])
def test_malformed_matrix_text(text):
    with pytest.raises((ap.DimensionError, ValueError)):
        parse_matrix(text)


@given(st.integers(1, 10), st.integers(0, 2**32), st.data())
@settings(deadline=None, max_examples=40)
def test_matrix_text_round_trip_is_identity(n, seed, data):
    rng = np.random.default_rng(seed)
    raw = rng.integers(0, 10**data.draw(st.integers(1, 17)), size=(n, n)).astype(np.int64)
    raw[rng.random((n, n)) < 0.3] = INF_RAW
    m = ap.CostMatrix(raw)
    text = format_matrix(m)
    assert format_matrix(parse_matrix(text)) == text
    assert np.array_equal(parse_matrix(text).raw, raw)


def test_matrix_file_round_trip_large(tmp_path):
    raw = ap.dense_costs(ap.GenParams(1500, 0.3, 100, 5), np.int64)
    m = ap.CostMatrix(raw)
    p1, p2 = tmp_path / "a.txt", tmp_path / "b.txt"
    write_matrix(m, p1)
    write_matrix(read_matrix(p1), p2)
    assert p1.read_bytes() == p2.read_bytes()
    assert np.array_equal(read_matrix(p1).raw, raw)
    # byte-exact with the reference formatter's layout on a slice
    small = ap.CostMatrix(raw[:40, :40].copy())
    want = "40\n" + "\n".join(" ".join("INF" if v == INF_RAW else str(v) for v in r) for r in raw[:40, :40]) + "\n"
    assert format_matrix(small) == want


def test_negative_matrix_rejected():
    with pytest.raises(ValueError):
        format_matrix(ap.CostMatrix.from_rows([[0, -1], [1, 0]]))
