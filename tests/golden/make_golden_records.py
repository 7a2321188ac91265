"""Record the REFERENCE's benchmark CSV for a small population (build container only):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_records.py

Writes tests/golden/bench_records.csv: apsp.bench.run_benchmark + emit_csv with the CLI's config
echo as preamble (cli.py:113-122), for BenchConfig(count=8, min_nodes=4, max_nodes=60, seed=3,
repetitions=1). Every column but wall_time_ms is a pure function of the config
(reference bench.py:8-11), so tests compare those columns exactly.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "bench_records.csv"


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, "/root/reference/pkg/src")
    from apsp.bench import BenchConfig, emit_csv, run_benchmark

    cfg = BenchConfig(count=8, min_nodes=4, max_nodes=60, seed=3, repetitions=1)
    records = run_benchmark(cfg)
    echo = (f"count={cfg.count} nodes=[{cfg.min_nodes},{cfg.max_nodes}] "
            f"rho={'per-graph' if cfg.rho is None else cfg.rho} alpha={cfg.alpha} "
            f"seed={cfg.seed} algos={','.join(cfg.algorithms)} reps={cfg.repetitions} "
            f"workers={'auto' if cfg.workers is None else cfg.workers}")
    OUT.write_text(emit_csv(records, preamble=echo))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
