"""Public min-plus product / accumulate on the B200 (reference: minplus.py).

``minplus_product`` and ``minplus_accumulate`` keep the reference contract: smallest-k argmin
on ties, strict improvement, via in global vertex numbers through the offsets, the
self-witness clear of the product (minplus.py:99-111) and ``CostRangeError`` when a finite
result leaves the range.  The kernels are the same tile kernels that run R-Kleene.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import CostMatrix, DimensionError, ParameterError, ViaMatrix

DEFAULT_TILE_SIZE = 64


@dataclass(frozen=True)
class MinPlusResult:
    """Product distances, the argmin via matrix and the exact candidate count."""

    distances: CostMatrix
    via: ViaMatrix
    relaxation_count: int


def default_workers() -> int:
    """APSP_WORKERS, else the CPU count (minplus.py:55-66).  Kept for API parity."""
    env = os.environ.get("APSP_WORKERS")
    if env is not None:
        try:
            w = int(env)
        except ValueError as exc:
            raise ParameterError(f"APSP_WORKERS must be an integer, got {env!r}") from exc
        if w < 1:
            raise ParameterError(f"APSP_WORKERS must be >= 1, got {w}")
        return w
    return os.cpu_count() or 1


def _resolve_workers(workers: int | None) -> int:
    if workers is None:
        return default_workers()
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    return workers


def _run(accumulate: int, x: CostMatrix, y: CostMatrix, z: CostMatrix | None, via: ViaMatrix | None,
         offsets: tuple[int, int, int], tier) -> MinPlusResult:
    import torch

    from .solvers import _tier_arg

    lib = nat.load()
    n1, n2 = x.shape
    n3 = y.shape[1]
    dev = torch.device("cuda", torch.cuda.current_device())
    xt = torch.from_numpy(np.array(x.raw, dtype=np.int64)).to(dev)
    yt = torch.from_numpy(np.array(y.raw, dtype=np.int64)).to(dev)
    if z is not None:
        zt = torch.from_numpy(np.array(z.raw, dtype=np.int64)).to(dev)
        vt = torch.from_numpy(np.array(via.raw, dtype=np.int64)).to(dev, torch.int32)
    else:
        zt = torch.empty((n1, n3), dtype=torch.int64, device=dev)
        vt = torch.empty((n1, n3), dtype=torch.int32, device=dev)
    info = nat.ApspInfo()
    s = torch.cuda.current_stream(dev)
    st = lib.apsp_minplus(nat.DTYPE_I64, accumulate, n1, n2, n3, xt.data_ptr(), n2, yt.data_ptr(), n3,
                          zt.data_ptr(), n3, vt.data_ptr(), n3, offsets[0], offsets[1], offsets[2], _tier_arg(tier),
                          ctypes.c_void_p(s.cuda_stream), ctypes.byref(info))
    nat.check(st)
    return MinPlusResult(
        distances=CostMatrix(zt.cpu().numpy(), _validated=True),
        via=ViaMatrix(vt.cpu().numpy().astype(np.int64)),
        relaxation_count=n1 * n2 * n3,
    )


def minplus_product(x: CostMatrix, y: CostMatrix, *, tile_size: int = DEFAULT_TILE_SIZE,
                    workers: int | None = None, offsets: tuple[int, int, int] = (0, 0, 0),
                    tier=None) -> MinPlusResult:
    """distances[i][j] = min_k x[i][k] + y[k][j] (minplus.py:166-203)."""
    if x.n_cols != y.n_rows:
        raise DimensionError(f"inner dimensions disagree: {x.shape} x {y.shape}")
    if tile_size < 1:
        raise ParameterError(f"tile_size must be >= 1, got {tile_size}")
    _resolve_workers(workers)
    return _run(0, x, y, None, None, tuple(int(o) for o in offsets), tier)


def minplus_accumulate(z: CostMatrix, x: CostMatrix, y: CostMatrix, via: ViaMatrix | None = None, *,
                       tile_size: int = DEFAULT_TILE_SIZE, workers: int | None = None, inner_offset: int = 0,
                       tier=None) -> MinPlusResult:
    """distances = min(z, x (x) y); via changes only on strict improvement (minplus.py:206-252)."""
    if x.n_cols != y.n_rows:
        raise DimensionError(f"inner dimensions disagree: {x.shape} x {y.shape}")
    if z.shape != (x.n_rows, y.n_cols):
        raise DimensionError(f"accumulator shape {z.shape} != product shape {(x.n_rows, y.n_cols)}")
    if via is None:
        via = ViaMatrix.all_none(z.n_rows, z.n_cols)
    elif via.shape != z.shape:
        raise DimensionError(f"via shape {via.shape} != accumulator shape {z.shape}")
    if tile_size < 1:
        raise ParameterError(f"tile_size must be >= 1, got {tile_size}")
    _resolve_workers(workers)
    return _run(1, x, y, z, via, (0, int(inner_offset), 0), tier)


def results_equal(a: MinPlusResult, b: MinPlusResult) -> bool:
    """Bitwise comparison of two kernel results, counters included."""
    return (a.relaxation_count == b.relaxation_count and a.distances.shape == b.distances.shape
            and bool(np.array_equal(a.distances.raw, b.distances.raw))
            and bool(np.array_equal(a.via.raw, b.via.raw)))
