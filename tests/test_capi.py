"""The C ABI library: it loads without a GPU and exports every symbol include/apsp_b200.h
declares; status codes map onto the reference's exception classes; without a device the
package refuses to compute (no CPU fallback)."""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200 import _native as nat


def declared_symbols():
    text = (ROOT / "include" / "apsp_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:[a-z_0-9]+\*?\s+)+\*?(apsp_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(nat.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_all_symbols():
    lib = nat.load(require_gpu=False)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.apsp_abi_version() == 2


def test_workspace_query_is_host_only():
    lib = nat.load(require_gpu=False)
    n = 16384
    ws = lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, 128)
    assert ws >= n * n * 8
    assert lib.apsp_workspace_bytes(nat.ALG_FW_CLASSIC, nat.DTYPE_I32, n, 128) == 0


def test_status_mapping():
    nat.load(require_gpu=False)
    for code, exc in [(nat.ERANGE, ap.CostRangeError), (nat.EINVAL, ap.ParameterError),
                      (nat.ENEGATIVE, ap.NegativeWeightError), (nat.EDIAGONAL, ap.MalformedGraphError),
                      (nat.EDIMENSION, ap.DimensionError), (nat.ECUDA, ap.ApspError)]:
        with pytest.raises(exc):
            nat.check(code)
    nat.check(nat.OK)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ap.minplus_identity(4)
    for solver in ap.SOLVERS.values():
        with pytest.raises(nat.NativeUnavailableError):
            solver(h)
    with pytest.raises(nat.NativeUnavailableError):
        ap.solve(np.zeros((4, 4), np.int32))


def test_host_level_call_reports_missing_device_as_error():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = nat.load(require_gpu=False)
    h = np.zeros((4, 4), np.int64)
    out = np.empty_like(h)
    idx = np.empty_like(h)
    info = nat.ApspInfo()
    st = lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I64, 4, h.ctypes.data, out.ctypes.data, idx.ctypes.data,
                             nat.DTYPE_I64, 0, 128, 64, 0, -1, 0, ctypes.byref(info))
    assert st == nat.ECUDA
    assert "CUDA" in nat.last_error()
