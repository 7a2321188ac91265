"""The reference's benchmark CSV contract (records.py) against the reference's own output
(tests/golden/bench_records.csv, written by tests/golden/make_golden_records.py)."""

from __future__ import annotations

import pytest

from conftest import GOLDEN

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200 import records as rec

CFG = rec.BenchConfig(count=8, min_nodes=4, max_nodes=60, seed=3, repetitions=1)
GOLD = (GOLDEN / "bench_records.csv").read_text()


def golden_rows():
    lines = GOLD.splitlines()
    assert lines[0].startswith("# ") and lines[1] == rec.CSV_HEADER
    return [ln.split(",") for ln in lines[2:]]


def without_time(row):
    return row[:5] + row[6:]


def test_preamble_header_and_population_match_reference():
    assert GOLD.splitlines()[0] == "# " + rec.config_preamble(CFG)
    pop = {gid: (v, seed) for gid, v, rho, seed in rec.draw_population(CFG)}
    for r in golden_rows():
        gid, n, seed = int(r[0]), int(r[1]), int(r[8])
        assert pop[gid] == (n, seed)
        g = ap.generate(ap.GenParams(n, rec.draw_population(CFG)[gid][2], CFG.alpha, seed))
        assert g.n_edges == int(r[2]) and f"{ap.density(g):.6f}" == r[3]


def test_emit_csv_reproduces_reference_text():
    rows = golden_rows()
    records = [rec.BenchRecord(int(r[0]), int(r[1]), int(r[2]), float(r[3]), r[4], float(r[5]), int(r[6]), int(r[7]),
                               int(r[8])) for r in rows]
    skipped = rec.BenchRecord(99, 5, 0, 0.0, "rkleene", 0.0, 0, 0, 1, skipped=True)
    assert rec.emit_csv(records + [skipped], preamble=rec.config_preamble(CFG)) == GOLD


def test_config_validation():
    for bad in ({"count": -1}, {"min_nodes": 0}, {"min_nodes": 9, "max_nodes": 8}, {"rho": 1.5}, {"alpha": 0},
                {"repetitions": 0}, {"algorithms": ()}, {"algorithms": ("dijkstra",)}):
        with pytest.raises(ap.ParameterError):
            rec.BenchConfig(**bad)


@pytest.mark.gpu
def test_gpu_population_rows_match_reference(cuda):
    """run_population on the GPU solvers: every column except the wall time equals the
    reference run (iterations and relaxation counts included), and every record verified."""
    records = rec.run_population(CFG)
    assert all(r.verified for r in records)
    got = [without_time(ln.split(",")) for ln in rec.emit_csv(records).splitlines()[1:]]
    assert got == [without_time(r) for r in golden_rows()]
