"""Benchmark records in the reference's CSV contract (reference bench.py:33, 88-106, 189-207).

A result file written here reads like one from the reference's ``apsp bench``: the same
``# config`` preamble, the same header and field order, the same number formats, one row per
(graph, algorithm), ascending by edge count.  ``run_population`` draws the reference's graph
population (same Philox draws per graph, bench.py:109-118), times every enabled solver on the
GPU (the solve call only, minimum over repetitions) and checks every algorithm's distances
against the first one's -- so a GPU run and a reference run of the same ``BenchConfig`` list the
same graphs with comparable times.  No plots (out of scope).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .core import CapacityError, ParameterError, cost_matrix_from_graph, matrices_equal
from .graphgen import GenParams, density, generate

CSV_HEADER = "graph_id,n_nodes,n_edges,density,algorithm,wall_time_ms,iterations,relaxation_count,seed"
ALGORITHMS = ("fw_classic", "fw_squaring", "rkleene")


@dataclass(frozen=True)
class BenchConfig:
    """Population and solver knobs; the reference's defaults and validation (bench.py:48-78)."""

    count: int = 100
    min_nodes: int = 4
    max_nodes: int = 512
    rho: float | None = None
    alpha: int = 100
    seed: int = 0
    algorithms: tuple[str, ...] = ALGORITHMS
    repetitions: int = 3
    base_threshold: int = 64
    tile_size: int = 64
    workers: int | None = None

    def __post_init__(self):
        checks = [
            (self.count >= 0, f"count must be >= 0, got {self.count}"),
            (1 <= self.min_nodes <= self.max_nodes, f"bad node range [{self.min_nodes},{self.max_nodes}]"),
            (self.rho is None or 0.0 <= self.rho <= 1.0, f"rho must lie in [0,1], got {self.rho}"),
            (self.alpha >= 1, f"alpha must be >= 1, got {self.alpha}"),
            (self.repetitions >= 1, f"repetitions must be >= 1, got {self.repetitions}"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ParameterError(msg)
        if not self.algorithms:
            raise ParameterError("at least one algorithm is required")
        unknown = [a for a in self.algorithms if a not in ALGORITHMS]
        if unknown:
            raise ParameterError(f"unknown algorithms: {unknown}; known: {list(ALGORITHMS)}")


@dataclass(frozen=True)
class BenchRecord:
    """One (graph, algorithm) measurement (the reference's record fields)."""

    graph_id: int
    n_nodes: int
    n_edges: int
    density: float
    algorithm: str
    wall_time_ms: float
    iterations: int
    relaxation_count: int
    seed: int
    verified: bool = True
    skipped: bool = False
    info: dict = field(default=None, compare=False)

    def csv_row(self) -> str:
        return (f"{self.graph_id},{self.n_nodes},{self.n_edges},{self.density:.6f},{self.algorithm},"
                f"{self.wall_time_ms:.3f},{self.iterations},{self.relaxation_count},{self.seed}")


def draw_population(cfg: BenchConfig) -> list[tuple[int, int, float, int]]:
    """(graph_id, v, rho, graph_seed) per graph: the reference's draws, in order, from one Philox
    stream keyed by the master seed (v, then rho if not fixed, then the graph seed)."""
    rng = np.random.Generator(np.random.Philox(cfg.seed))
    out = []
    for gid in range(cfg.count):
        v = int(rng.integers(cfg.min_nodes, cfg.max_nodes, endpoint=True))
        rho = float(rng.random()) if cfg.rho is None else cfg.rho
        out.append((gid, v, rho, int(rng.integers(0, 2 ** 63))))
    return out


def run_population(cfg: BenchConfig, progress=None) -> list[BenchRecord]:
    """Solve every graph of the population with every enabled algorithm on the GPU."""
    from .solvers import SOLVERS

    records: list[BenchRecord] = []
    for gid, v, rho, gseed in draw_population(cfg):
        g = generate(GenParams(v, rho, cfg.alpha, gseed))
        h = cost_matrix_from_graph(g)
        dens = density(g)
        first = None
        for alg in cfg.algorithms:
            kw = {"tile_size": cfg.tile_size, "workers": cfg.workers}
            if alg == "rkleene":
                kw["base_threshold"] = cfg.base_threshold
            try:
                best, sol = float("inf"), None
                for _ in range(cfg.repetitions):
                    t0 = time.perf_counter()
                    sol = SOLVERS[alg](h, **kw)
                    best = min(best, (time.perf_counter() - t0) * 1e3)
            except CapacityError:
                records.append(BenchRecord(gid, v, g.n_edges, dens, alg, 0.0, 0, 0, gseed, skipped=True))
                continue
            ok = True if first is None else matrices_equal(first, sol.distances)
            first = sol.distances if first is None else first
            records.append(BenchRecord(gid, v, g.n_edges, dens, alg, best, sol.iterations, sol.relaxation_count,
                                       gseed, verified=ok, info=sol.info))
        if progress is not None:
            progress(gid, cfg.count, len(records))
    records.sort(key=lambda r: (r.n_edges, r.graph_id))
    return records


def emit_csv(records, preamble: str | None = None) -> str:
    """CSV text: optional ``# ``-prefixed preamble lines, the header, one row per non-skipped
    record, LF line endings."""
    lines = [f"# {ln}" for ln in preamble.splitlines()] if preamble else []
    lines.append(CSV_HEADER)
    lines += [r.csv_row() for r in records if not r.skipped]
    return "\n".join(lines) + "\n"


def config_preamble(cfg: BenchConfig) -> str:
    """The one-line config echo the reference CLI writes above the rows (cli.py:116-121)."""
    rho = "per-graph" if cfg.rho is None else cfg.rho
    workers = "auto" if cfg.workers is None else cfg.workers
    return (f"count={cfg.count} nodes=[{cfg.min_nodes},{cfg.max_nodes}] rho={rho} alpha={cfg.alpha} "
            f"seed={cfg.seed} algos={','.join(cfg.algorithms)} reps={cfg.repetitions} workers={workers}")


__all__ = ["ALGORITHMS", "BenchConfig", "BenchRecord", "CSV_HEADER", "config_preamble", "draw_population",
           "emit_csv", "run_population"]
