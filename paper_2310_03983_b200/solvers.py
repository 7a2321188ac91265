"""APSP solvers behind the reference's Python API (reference: solvers.py).

Every entry point takes the reference's ``CostMatrix`` (int64, INF_RAW) and returns the
reference's ``ApspSolution``; the work runs on the B200 through libapsp_b200.so:

* ``fw_classic``  -- blocked three-phase Floyd-Warshall (default, ``method="blocked"``) or the
  classic k-order kernel (``method="classic"``, bit-exact pred with the reference).
  Reference: solvers.py:118-155.
* ``rkleene``     -- recursive closure (solvers.py:207-296).  ``split="floor"`` with the given
  ``base_threshold`` reproduces the reference's via matrix bit-for-bit; ``split="aligned"``
  is the performance schedule (128-aligned splits, blocked-FW leaves).  ``track="pred"``
  returns predecessors instead of via.
* ``fw_squaring`` -- repeated min-plus squaring until unchanged (solvers.py:167-204).

``tile_size`` and ``workers`` are accepted and validated exactly like the reference
(they select CPU band sizes and thread counts there; the GPU grid replaces both).
Dense int32 / fp32 arrays (numpy or CUDA torch tensors) go through ``solve``.
"""

from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import (
    INF32,
    INF_RAW,
    ApspError,
    CostMatrix,
    DimensionError,
    ParameterError,
    PredMatrix,
    ViaMatrix,
)
from .minplus import DEFAULT_TILE_SIZE, _resolve_workers

DEFAULT_BASE_THRESHOLD = 64
DEFAULT_BLOCK = 0   # 0: the library picks by n (fw_sched.cu default_block: 128 ... 2048)


@dataclass(frozen=True)
class ApspSolution:
    """Closed distances plus reconstruction data (reference: solvers.py:49-64).

    Exactly one of via / pred is set.  ``info`` carries the engine's own telemetry (value
    tier, kernel launches, device time) and is excluded from equality.
    """

    distances: CostMatrix
    via: ViaMatrix | None
    pred: PredMatrix | None
    iterations: int
    relaxation_count: int
    algorithm: str
    info: dict | None = field(default=None, compare=False)


def _tier_arg(tier) -> int:
    if tier is None or tier == "auto":
        return nat.TIER_AUTO
    names = {v: k for k, v in nat.TIER_NAMES.items()}
    if isinstance(tier, str):
        if tier not in names:
            raise ParameterError(f"unknown tier {tier!r}; expected one of {sorted(names)}")
        return names[tier]
    return int(tier)


def _check_common(tile_size: int, workers) -> None:
    if tile_size < 1:
        raise ParameterError(f"tile_size must be >= 1, got {tile_size}")
    _resolve_workers(workers)


def _host_solve(alg: int, h: CostMatrix, *, idx_mode: int = nat.IDX_PRED, block: int = DEFAULT_BLOCK,
                base_threshold: int = 0, aligned: int = 0, tier=None, device: int = 0):
    lib = nat.load()
    n = h.n
    src = np.ascontiguousarray(h.raw, dtype=np.int64)
    dist = np.empty((n, n), dtype=np.int64)
    idx = np.empty((n, n), dtype=np.int64)
    info = nat.ApspInfo()
    st = lib.apsp_solve_host(alg, nat.DTYPE_I64, n, src.ctypes.data, dist.ctypes.data, idx.ctypes.data,
                             nat.DTYPE_I64, idx_mode, block, base_threshold, aligned, _tier_arg(tier), device,
                             ctypes.byref(info))
    nat.check(st)
    return dist, idx, info


def fw_classic(h: CostMatrix, *, tile_size: int = DEFAULT_TILE_SIZE, workers: int | None = None,
               method: str = "blocked", block: int = DEFAULT_BLOCK, tier=None, device: int = 0) -> ApspSolution:
    """Floyd-Warshall with predecessors.

    ``method="blocked"``: three-phase blocked FW (distances bit-exact with the reference,
    pred a valid shortest-path tree).  ``method="classic"``: k-order kernel, pred bit-exact
    with reference ``fw_classic`` (solvers.py:77-95).
    """
    _check_common(tile_size, workers)
    n = h.n
    if method == "blocked":
        alg = nat.ALG_FW_BLOCKED
    elif method == "classic":
        alg = nat.ALG_FW_CLASSIC
    else:
        raise ParameterError(f"method must be 'blocked' or 'classic', got {method!r}")
    dist, pred, info = _host_solve(alg, h, block=block, tier=tier, device=device)
    return ApspSolution(
        distances=CostMatrix(dist, _validated=True),
        via=None,
        pred=PredMatrix(pred, _validated=True),
        iterations=0,
        relaxation_count=n * n * n,
        algorithm="fw_classic",
        info=info.as_dict() | {"method": method},
    )


def fw_blocked(h: CostMatrix, **kw) -> ApspSolution:
    """Alias of ``fw_classic(h, method="blocked")``."""
    return fw_classic(h, method="blocked", **kw)


def rkleene(h: CostMatrix, *, base_threshold: int = DEFAULT_BASE_THRESHOLD, tile_size: int = DEFAULT_TILE_SIZE,
            workers: int | None = None, track: str = "via", split: str = "floor", tier=None,
            device: int = 0) -> ApspSolution:
    """Recursive blocked closure (solvers.py:207-296)."""
    n = h.n
    if base_threshold < 1:
        raise ParameterError(f"base_threshold must be >= 1, got {base_threshold}")
    _check_common(tile_size, workers)
    if track not in ("via", "pred"):
        raise ParameterError(f"track must be 'via' or 'pred', got {track!r}")
    if split not in ("floor", "aligned"):
        raise ParameterError(f"split must be 'floor' or 'aligned', got {split!r}")
    mode = nat.IDX_VIA if track == "via" else nat.IDX_PRED
    dist, idx, info = _host_solve(nat.ALG_RKLEENE, h, idx_mode=mode, base_threshold=base_threshold,
                                  aligned=int(split == "aligned"), tier=tier, device=device)
    return ApspSolution(
        distances=CostMatrix(dist, _validated=True),
        via=ViaMatrix(idx, _validated=True) if track == "via" else None,
        pred=PredMatrix(idx, _validated=True) if track == "pred" else None,
        iterations=0,
        relaxation_count=n * n * n,
        algorithm="rkleene",
        info=info.as_dict() | {"split": split, "track": track},
    )


def fw_squaring(h: CostMatrix, *, tile_size: int = DEFAULT_TILE_SIZE, workers: int | None = None, tier=None,
                device: int = 0) -> ApspSolution:
    """Repeated min-plus squaring until the matrix stops changing (solvers.py:167-204)."""
    _check_common(tile_size, workers)
    n = h.n
    dist, via, info = _host_solve(nat.ALG_FW_SQUARING, h, idx_mode=nat.IDX_VIA, tier=tier, device=device)
    return ApspSolution(
        distances=CostMatrix(dist, _validated=True),
        via=ViaMatrix(via, _validated=True),
        pred=None,
        iterations=info.iterations,
        relaxation_count=info.iterations * n * n * n,
        algorithm="fw_squaring",
        info=info.as_dict(),
    )


def detect_negative_cycle(distances: CostMatrix) -> bool:
    """True iff a diagonal cell of a closed distance matrix is negative (solvers.py:299-305)."""
    return bool((np.diagonal(distances.raw) < 0).any())


SOLVERS = {
    "fw_classic": fw_classic,
    "fw_squaring": fw_squaring,
    "rkleene": rkleene,
}


# ---- dense int32 / fp32 entry point -------------------------------------------------------

@dataclass(frozen=True)
class DenseSolution:
    """Result of ``solve`` on a dense int32 / fp32 matrix (numpy or torch, like the input)."""

    distances: object
    index: object          # pred (fw_*, rkleene track="pred") or via (rkleene "via", fw_squaring)
    index_kind: str
    info: dict


_ALGS = {"fw_blocked": nat.ALG_FW_BLOCKED, "fw_classic": nat.ALG_FW_CLASSIC, "rkleene": nat.ALG_RKLEENE,
         "fw_squaring": nat.ALG_FW_SQUARING}


def _dtype_code(dt) -> int:
    s = str(dt)
    if s.endswith("int32"):
        return nat.DTYPE_I32
    if s.endswith("float32"):
        return nat.DTYPE_F32
    if s.endswith("int64"):
        return nat.DTYPE_I64
    raise ParameterError(f"unsupported dtype {dt}; expected int32 (INF={INF32}), float32 (+inf) or int64 "
                         f"(INF={INF_RAW})")


def solve(h, algorithm: str = "fw_blocked", *, track: str = "pred", base_threshold: int = 512,
          split: str = "aligned", block: int = DEFAULT_BLOCK, tier=None, stream=None, workspace=None) -> DenseSolution:
    """APSP on a dense int32 / fp32 / int64 matrix.

    numpy input: host-level call (copy in, solve, copy out) -> numpy outputs.
    CUDA torch tensor: device-level call on a copy, on ``stream`` (default: torch's current
    stream) -> torch outputs, ready in ``stream`` order; ``stream`` first waits for the current
    stream (which produced ``h``).  ``workspace`` may be a preallocated uint8 CUDA tensor.
    """
    if algorithm not in _ALGS:
        raise ParameterError(f"unknown algorithm {algorithm!r}; expected one of {sorted(_ALGS)}")
    if track not in ("via", "pred"):
        raise ParameterError(f"track must be 'via' or 'pred', got {track!r}")
    if split not in ("floor", "aligned"):
        raise ParameterError(f"split must be 'floor' or 'aligned', got {split!r}")
    if base_threshold < 1:
        raise ParameterError(f"base_threshold must be >= 1, got {base_threshold}")
    alg = _ALGS[algorithm]
    mode = nat.IDX_VIA if (algorithm == "fw_squaring" or (algorithm == "rkleene" and track == "via")) \
        else nat.IDX_PRED
    kind = "via" if mode == nat.IDX_VIA else "pred"
    aligned = int(split == "aligned")
    lib = nat.load()
    info = nat.ApspInfo()
    if isinstance(h, np.ndarray):
        if h.ndim != 2 or h.shape[0] != h.shape[1] or h.size == 0:
            raise DimensionError(f"expected a non-empty square matrix, got shape {h.shape}")
        dt = _dtype_code(h.dtype)
        n = h.shape[0]
        src = np.ascontiguousarray(h)
        dist = np.empty_like(src)
        idx = np.empty((n, n), dtype=np.int32)
        st = lib.apsp_solve_host(alg, dt, n, src.ctypes.data, dist.ctypes.data, idx.ctypes.data, nat.DTYPE_I32,
                                 mode, block, base_threshold, aligned, _tier_arg(tier), 0, ctypes.byref(info))
        nat.check(st)
        return DenseSolution(dist, idx, kind, info.as_dict())
    import torch

    if not isinstance(h, torch.Tensor) or not h.is_cuda:
        raise ParameterError("solve expects a numpy array or a CUDA torch tensor")
    if h.dim() != 2 or h.shape[0] != h.shape[1] or h.numel() == 0:
        raise DimensionError(f"expected a non-empty square matrix, got shape {tuple(h.shape)}")
    dt = _dtype_code(h.dtype)
    n = h.shape[0]
    cur = torch.cuda.current_stream(h.device)
    s = stream if stream is not None else cur
    sp = ctypes.c_void_p(s.cuda_stream)
    ws_need = lib.apsp_workspace_bytes(alg, dt, n, block)
    # The library runs on `s`; whatever produced `h` (and a caller's `workspace`) was queued on
    # the current stream, so `s` waits for it, and the copies/allocations below are made on `s`.
    side = s != cur
    if side:
        s.wait_stream(cur)
    # (the stream / device context managers cost ~10 us per call at small n: entered only when
    # they change something)
    with torch.cuda.stream(s) if side else contextlib.nullcontext():
        dist = h.contiguous().clone()
        idx = torch.empty((n, n), dtype=torch.int32, device=h.device)
        if workspace is None and ws_need:
            workspace = torch.empty(ws_need, dtype=torch.uint8, device=h.device)
    if side:
        # the outputs are handed back to a caller on `cur` (who syncs with `s` before reading,
        # as with any side-stream result): their blocks must not be recycled while `cur` uses them
        for t in (dist, idx):
            t.record_stream(cur)
    wp = workspace.data_ptr() if workspace is not None else None
    wb = workspace.numel() if workspace is not None else 0
    with torch.cuda.device(h.device) if h.device.index != torch.cuda.current_device() else contextlib.nullcontext():
        if alg == nat.ALG_FW_BLOCKED:
            st = lib.apsp_fw_blocked(dt, n, dist.data_ptr(), n, idx.data_ptr(), n, block, _tier_arg(tier), wp, wb,
                                     sp, ctypes.byref(info))
        elif alg == nat.ALG_FW_CLASSIC:
            st = lib.apsp_fw_classic(dt, n, dist.data_ptr(), n, idx.data_ptr(), n, sp, ctypes.byref(info))
        elif alg == nat.ALG_RKLEENE:
            st = lib.apsp_rkleene(dt, n, dist.data_ptr(), n, idx.data_ptr(), n, mode, base_threshold, aligned,
                                  _tier_arg(tier), wp, wb, sp, ctypes.byref(info))
        else:
            st = lib.apsp_fw_squaring(dt, n, dist.data_ptr(), n, idx.data_ptr(), n, _tier_arg(tier), wp, wb, sp,
                                      ctypes.byref(info))
    nat.check(st)
    return DenseSolution(dist, idx, kind, info.as_dict())


__all__ = ["ApspSolution", "DenseSolution", "SOLVERS", "detect_negative_cycle", "fw_blocked", "fw_classic",
           "fw_squaring", "rkleene", "solve", "ApspError"]
