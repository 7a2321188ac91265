"""ctypes binding of libapsp_b200.so (the C ABI declared in include/apsp_b200.h).

The shared library is the product: there is no CPU fallback.  If it is missing, or no CUDA
device is visible, every solver raises ``NativeUnavailableError`` instead of computing.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .core import (
    ApspError,
    CostRangeError,
    DimensionError,
    MalformedGraphError,
    NegativeWeightError,
    ParameterError,
)

LIB_NAME = "libapsp_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

# apsp_status
OK, ERANGE, EINVAL, ECUDA, ENCCL, ENEGATIVE, EDIAGONAL, EDIMENSION, ECONVERGE = range(9)
# apsp_dtype
DTYPE_I32, DTYPE_F32, DTYPE_I64 = 0, 1, 2
# apsp_tier
TIER_AUTO, TIER_U8, TIER_W32, TIER_I32, TIER_F32, TIER_I64, TIER_U16 = -1, 0, 1, 2, 3, 4, 5
TIER_NAMES = {TIER_U8: "u8", TIER_U16: "u16", TIER_W32: "w32", TIER_I32: "i32", TIER_F32: "f32", TIER_I64: "i64"}
# apsp_idx_mode
IDX_PRED, IDX_VIA = 0, 1
# apsp_algorithm
ALG_FW_BLOCKED, ALG_FW_CLASSIC, ALG_RKLEENE, ALG_FW_SQUARING = 0, 1, 2, 3

EXPORTED_SYMBOLS = (
    "apsp_last_error",
    "apsp_abi_version",
    "apsp_set_profiling",
    "apsp_launch_count",
    "apsp_profile_read",
    "apsp_workspace_bytes",
    "apsp_fw_blocked",
    "apsp_fw_classic",
    "apsp_rkleene",
    "apsp_fw_squaring",
    "apsp_minplus",
    "apsp_solve_host",
    "apsp_scan",
    "apsp_shard_scratch_bytes",
    "apsp_shard_prepare",
    "apsp_shard_pivot",
    "apsp_shard_pivot_fused",
    "apsp_shard_update",
    "apsp_shard_finish",
    "apsp_side_stream",
    "apsp_rk_shard_scratch_bytes",
    "apsp_rk_shard_leaf",
    "apsp_rk_shard_product",
    "apsp_rk_shard_product_fused",
    "apsp_format_matrix_i64",
    "apsp_parse_matrix_i64",
)


class NativeUnavailableError(ApspError):
    """The CUDA extension is not built or no GPU is visible (no fallback exists)."""


class ApspInfo(ctypes.Structure):
    _fields_ = [
        ("tier", ctypes.c_int32),
        ("tiers_tried", ctypes.c_int32),
        ("iterations", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("max_finite", ctypes.c_int64),
        ("relaxations", ctypes.c_int64),
        ("device_ms", ctypes.c_double),
        ("flags", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("kernel_ms", ctypes.c_double),
        ("block", ctypes.c_int32),
        ("d2h_bytes_per_cell", ctypes.c_int32),
        ("h2d_bytes_per_cell", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {
            "tier": TIER_NAMES.get(self.tier, str(self.tier)),
            "tiers_tried": [TIER_NAMES[t] for t in TIER_NAMES if self.tiers_tried & (1 << t)],
            "iterations": self.iterations,
            "launches": self.launches,
            "max_finite": self.max_finite,
            "relaxations": self.relaxations,
            "device_ms": self.device_ms,
            "classic_for_zero_edges": bool(self.flags & 1),
            "kernel_launches": self.kernel_launches,
            "kernel_ms": self.kernel_ms,
            "block": self.block,
            "d2h_bytes_per_cell": self.d2h_bytes_per_cell,
            "h2d_bytes_per_cell": self.h2d_bytes_per_cell,
        }


class ScanResult(ctypes.Structure):
    _fields_ = [
        ("negative", ctypes.c_int32),
        ("diag_nonzero", ctypes.c_int32),
        ("non_integral", ctypes.c_int32),
        ("any_finite", ctypes.c_int32),
        ("max_finite", ctypes.c_int64),
        ("max_finite_f", ctypes.c_float),
        ("zero_offdiag", ctypes.c_int32),
        ("finite_offdiag", ctypes.c_uint64),
    ]


_i32, _i64, _vp, _sz = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
_info_p = ctypes.POINTER(ApspInfo)
_scan_p = ctypes.POINTER(ScanResult)

_SIGNATURES = {
    "apsp_last_error": (ctypes.c_char_p, []),
    "apsp_abi_version": (_i32, []),
    "apsp_set_profiling": (None, [_i32]),
    "apsp_launch_count": (ctypes.c_longlong, []),
    "apsp_profile_read": (_i32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32)]),
    "apsp_workspace_bytes": (_sz, [_i32, _i32, _i64, _i32]),
    "apsp_fw_blocked": (_i32, [_i32, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _vp, _sz, _vp, _info_p]),
    "apsp_fw_classic": (_i32, [_i32, _i64, _vp, _i64, _vp, _i64, _vp, _info_p]),
    "apsp_rkleene": (_i32, [_i32, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _sz, _vp, _info_p]),
    "apsp_fw_squaring": (_i32, [_i32, _i64, _vp, _i64, _vp, _i64, _i32, _vp, _sz, _vp, _info_p]),
    "apsp_minplus": (_i32, [_i32, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                            _i64, _i64, _i64, _i32, _vp, _info_p]),
    "apsp_solve_host": (_i32, [_i32, _i32, _i64, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32,
                               _info_p]),
    "apsp_scan": (_i32, [_i32, _vp, _i64, _i64, _i64, _i64, _scan_p, _vp]),
    "apsp_shard_scratch_bytes": (_sz, [_i32, _i64, _i64, _i32]),
    "apsp_shard_prepare": (_i32, [_i32, _i32, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp]),
    "apsp_shard_pivot": (_i32, [_i32, _i64, _i32, _vp, _i64, _vp, _i64, _i64, _i64, _vp, _sz, _vp]),
    "apsp_shard_pivot_fused": (_i32, [_i32, _i64, _i32, _vp, _i64, _vp, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _sz,
                                      _vp]),
    "apsp_shard_update": (_i32, [_i32, _i64, _i32, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64,
                                 _i64, _i64, _vp, _sz, _vp]),
    "apsp_side_stream": (_vp, []),
    "apsp_rk_shard_scratch_bytes": (_sz, [_i64, _i32]),
    "apsp_rk_shard_leaf": (_i32, [_i32, _vp, _i64, _vp, _i64, _i64, _i64, _i32, _vp, _sz, _vp]),
    "apsp_rk_shard_product": (_i32, [_i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64,
                                     _i64, _i64, _i64, _i32, _vp, _sz, _vp]),
    "apsp_rk_shard_product_fused": (_i32, [_i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64,
                                           _i64, _i64, _i64, _i64, _i32, _i32, _vp, _vp, _vp, _sz, _vp]),
    "apsp_format_matrix_i64": (_i64, [_vp, _i64, _vp, _i64]),
    "apsp_parse_matrix_i64": (_i64, [_vp, _i64, _i64, _vp, ctypes.POINTER(ctypes.c_int64)]),
    "apsp_shard_finish": (_i32, [_i32, _i32, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                                 ctypes.POINTER(ctypes.c_int64), _vp]),
}

_lib = None


def lib_path() -> Path:
    return Path(os.environ.get("APSP_B200_LIB", str(LIB_PATH)))


def load(require_gpu: bool = True):
    """Load the extension (once).  ``require_gpu`` additionally checks for a CUDA device."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not path.exists():
            raise NativeUnavailableError(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2310_03983_b200/csrc`")
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.apsp_abi_version() != 2:
            raise NativeUnavailableError("libapsp_b200.so ABI version mismatch")
        _lib = lib
    if require_gpu:
        _require_device()
    return _lib


_device_ok = None


def _require_device() -> None:
    global _device_ok
    if _device_ok is None:
        try:
            import torch

            _device_ok = bool(torch.cuda.is_available())
        except Exception:  # pragma: no cover - torch is part of the image
            _device_ok = False
    if not _device_ok:
        raise NativeUnavailableError("no CUDA device visible: the B200 engine has no CPU fallback")


def last_error() -> str:
    return (_lib.apsp_last_error() or b"").decode("utf-8", "replace") if _lib else ""


def check(status: int) -> None:
    """Map an apsp_status to the reference's exception classes (core.py:23-56)."""
    if status == OK:
        return
    msg = last_error()
    exc = {
        ERANGE: CostRangeError,
        EINVAL: ParameterError,
        ENEGATIVE: NegativeWeightError,
        EDIAGONAL: MalformedGraphError,
        EDIMENSION: DimensionError,
    }.get(status, ApspError)
    raise exc(msg or f"apsp status {status}")
