"""numpy front end of apsp_oracle.c (TEST INFRASTRUCTURE ONLY; see the package docstring).

Each function mirrors one reference entry point (file:line in apsp_oracle.c) on int64
arrays with INF_RAW = 2**61, returning plain numpy arrays.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

INF_RAW = 1 << 61
HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


class OracleRangeError(Exception):
    """The oracle's kernel status 1 (the reference raises CostRangeError)."""


def build() -> Path:
    """Compile liboracle.so with gcc (idempotent)."""
    src = HERE / "apsp_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        i64, p, i = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        lib.oracle_fw_classic.argtypes = [i64, p, p, i64, i]
        lib.oracle_fw_via_block.argtypes = [i64, p, p, i64, i64]
        lib.oracle_fw_steps.argtypes = [i64, p, p, i64, i64, i]
        lib.oracle_product.argtypes = [i64, i64, i64, p, i64, p, i64, p, p, i64, i64, i64, i64]
        lib.oracle_accumulate.argtypes = [i64, i64, i64, p, i64, p, i64, p, i64, p, i64, p, p, i64, i64]
        lib.oracle_rkleene.argtypes = [i64, p, p, i64, i]
        lib.oracle_fw_squaring.argtypes = [i64, p, p, p, i]
        lib.oracle_fw_f64.argtypes = [i64, p, i]
        lib.oracle_fw_f64.restype = None
        _lib = lib
    return _lib


def _c64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64)).copy()


def _check(st: int) -> None:
    if st == 1:
        raise OracleRangeError("shortest-path cost left the representable finite range")
    if st:
        raise RuntimeError(f"oracle status {st}")


def threads() -> int:
    return int(os.environ.get("APSP_ORACLE_THREADS", os.cpu_count() or 1))


def fw_classic(h, k_end: int = -1, nthreads: int | None = None):
    """(dist, pred) of reference fw_classic (solvers.py:118-155); k_end bounds the steps."""
    d = _c64(h)
    n = d.shape[0]
    pred = np.empty_like(d)
    _check(_load().oracle_fw_classic(n, d.ctypes.data, pred.ctypes.data, k_end, nthreads or threads()))
    return d, pred


def fw_steps(d: np.ndarray, pred: np.ndarray, k0: int, k1: int, nthreads: int | None = None) -> None:
    """In place: steps [k0, k1) of fw_classic on an initialised (d, pred) state."""
    assert d.dtype == np.int64 and pred.dtype == np.int64 and d.flags.c_contiguous and pred.flags.c_contiguous
    _check(_load().oracle_fw_steps(d.shape[0], d.ctypes.data, pred.ctypes.data, k0, k1, nthreads or threads()))


def rkleene(h, base_threshold: int = 64, nthreads: int | None = None):
    """(dist, via) of reference rkleene (solvers.py:207-296)."""
    d = _c64(h)
    n = d.shape[0]
    via = np.empty_like(d)
    _check(_load().oracle_rkleene(n, d.ctypes.data, via.ctypes.data, base_threshold, nthreads or threads()))
    return d, via


def fw_squaring(h, nthreads: int | None = None):
    """(dist, via, iterations) of reference fw_squaring (solvers.py:167-204)."""
    d = _c64(h)
    n = d.shape[0]
    via = np.empty_like(d)
    it = ctypes.c_int64(0)
    _check(_load().oracle_fw_squaring(n, d.ctypes.data, via.ctypes.data, ctypes.byref(it), nthreads or threads()))
    return d, via, int(it.value)


def fw_f64(h, nthreads: int | None = None) -> np.ndarray:
    """float64 FW distances (+inf unreachable), bit-identical to networkx floyd_warshall_numpy
    on the same float64 matrix (the C2 continuous-weight check)."""
    d = np.ascontiguousarray(np.asarray(h, dtype=np.float64)).copy()
    _load().oracle_fw_f64(d.shape[0], d.ctypes.data, nthreads or threads())
    return d


def product(x, y, offsets=(0, 0, 0)):
    """(dist, via) of reference minplus_product (minplus.py:166-203)."""
    x, y = _c64(x), _c64(y)
    n1, n2 = x.shape
    n3 = y.shape[1]
    d = np.empty((n1, n3), np.int64)
    v = np.empty((n1, n3), np.int64)
    _check(_load().oracle_product(n1, n2, n3, x.ctypes.data, n2, y.ctypes.data, n3, d.ctypes.data, v.ctypes.data,
                                  n3, *offsets))
    return d, v


def accumulate(z, x, y, via=None, inner_offset: int = 0):
    """(dist, via) of reference minplus_accumulate (minplus.py:206-252)."""
    x, y, z = _c64(x), _c64(y), _c64(z)
    n1, n2 = x.shape
    n3 = y.shape[1]
    vin = _c64(np.full((n1, n3), -1) if via is None else via)
    d = np.empty((n1, n3), np.int64)
    v = np.empty((n1, n3), np.int64)
    _check(_load().oracle_accumulate(n1, n2, n3, x.ctypes.data, n2, y.ctypes.data, n3, z.ctypes.data, n3,
                                     vin.ctypes.data, n3, d.ctypes.data, v.ctypes.data, n3, inner_offset))
    return d, v


__all__ = ["INF_RAW", "OracleRangeError", "accumulate", "build", "fw_classic", "fw_f64", "fw_squaring", "fw_steps",
           "product",
           "rkleene", "threads"]
