"""Out-of-bounds write checks through the device-level C ABI (stand-in for compute-sanitizer
memcheck, which the GPU pool does not allow): every caller buffer is embedded in a larger
allocation -- rows of canaries above and below, ld > n so every row carries canary columns, and
canaries past the end of the workspace. After each solve the result must equal the oracle and
every canary must be intact (ragged n, odd n, every tier and schedule)."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from conftest import INF_RAW, random_graph_raw
from oracle import oracle as orc

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200 import _native as nat
from paper_2310_03983_b200.core import INF32

pytestmark = pytest.mark.gpu

CANARY = 0x5A5A5A5A
GUARD = 3          # canary rows above and below
PADC = 20          # canary columns right of every row (ld = n + PADC)


class Guarded:
    """An n x n view with canaries around it (int32 or float32 cells, or int64)."""

    def __init__(self, n, dtype, fill=None):
        self.n, self.ld = n, n + PADC
        self.buf = torch.full((n + 2 * GUARD, self.ld), 0, dtype=dtype, device="cuda")
        self.buf.view(torch.int32 if dtype != torch.int64 else torch.int64).fill_(CANARY)
        self.view = self.buf[GUARD:GUARD + n, :n]
        if fill is not None:
            self.view.copy_(fill)

    def ptr(self):
        return self.view.data_ptr()

    def intact(self) -> bool:
        raw = self.buf.view(torch.int32 if self.buf.dtype != torch.int64 else torch.int64)
        mask = torch.ones_like(raw, dtype=torch.bool)
        mask[GUARD:GUARD + self.n, :self.n] = False
        return bool((raw[mask] == CANARY).all().item())


def guarded_ws(nbytes):
    ws = torch.full((nbytes + 8192,), 0x5A, dtype=torch.uint8, device="cuda")
    return ws, lambda: bool((ws[nbytes:] == 0x5A).all().item())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to32(raw):
    h = raw.astype(np.int64)
    h[raw == INF_RAW] = INF32
    return torch.from_numpy(h.astype(np.int32)).cuda()


def back64(t):
    a = t.cpu().numpy().astype(np.int64)
    a[a == INF32] = INF_RAW
    return a


@pytest.mark.parametrize("n,wmax,tier,block", [(300, 9, "u8", 128), (257, 400, "auto", 128), (333, 50000, "w32", 256),
                                               (129, 9, "u8", 256), (700, 9, "auto", 0), (1100, 9, "auto", 128),
                                               # persistent 64-wide u16 / w32 tasks, the device-signalled
                                               # chain with half-row cross launches (n > 2560)
                                               (640, 300, "u16", 0), (520, 50000, "w32", 0), (2600, 9, "u8", 0)])
def test_fw_blocked_guarded(cuda, n, wmax, tier, block):
    lib = nat.load()
    raw = random_graph_raw(n, 0.05, wmax, n + wmax)
    want, _ = orc.fw_classic(raw)
    d = Guarded(n, torch.int32, to32(raw))
    p = Guarded(n, torch.int32)
    need = lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, block)
    ws, ws_ok = guarded_ws(need)
    info = nat.ApspInfo()
    tcode = nat.TIER_AUTO if tier == "auto" else {v: k for k, v in nat.TIER_NAMES.items()}[tier]
    nat.check(lib.apsp_fw_blocked(nat.DTYPE_I32, n, d.ptr(), d.ld, p.ptr(), p.ld, block, tcode, ws.data_ptr(), need,
                                  stream(), ctypes.byref(info)))
    torch.cuda.synchronize()
    assert np.array_equal(back64(d.view), want)
    assert d.intact() and p.intact() and ws_ok()
    ok, why = ap.check_pred_tree(raw, back64(d.view), p.view.cpu().numpy().astype(np.int64), INF_RAW)
    assert ok, why


@pytest.mark.parametrize("n", [200, 513])
def test_fw_f32_continuous_guarded(cuda, n):
    lib = nat.load()
    h = torch.from_numpy(ap.continuous_costs(ap.GenParams(n, 0.2, 100, n))).cuda()
    want = orc.fw_f64(h.double().cpu().numpy())
    d = Guarded(n, torch.float32, h)
    p = Guarded(n, torch.int32)
    need = lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, nat.DTYPE_F32, n, 0)
    ws, ws_ok = guarded_ws(need)
    info = nat.ApspInfo()
    nat.check(lib.apsp_fw_blocked(nat.DTYPE_F32, n, d.ptr(), d.ld, p.ptr(), p.ld, 0, nat.TIER_AUTO, ws.data_ptr(),
                                  need, stream(), ctypes.byref(info)))
    torch.cuda.synchronize()
    got = d.view.double().cpu().numpy()
    fin = np.isfinite(want)
    assert (np.abs(got[fin] - want[fin]) <= 1e-5 * want[fin].clip(min=1e-30)).all()
    assert d.intact() and p.intact() and ws_ok()


@pytest.mark.parametrize("n,thr,aligned,mode", [(301, 64, 0, nat.IDX_VIA), (255, 16, 0, nat.IDX_VIA),
                                                (640, 256, 1, nat.IDX_PRED), (389, 128, 1, nat.IDX_PRED)])
def test_rkleene_guarded(cuda, n, thr, aligned, mode):
    lib = nat.load()
    raw = random_graph_raw(n, 0.05, 9, n + thr)
    want, want_via = orc.rkleene(raw, thr)
    d = Guarded(n, torch.int32, to32(raw))
    p = Guarded(n, torch.int32)
    need = lib.apsp_workspace_bytes(nat.ALG_RKLEENE, nat.DTYPE_I32, n, 0)
    ws, ws_ok = guarded_ws(need)
    info = nat.ApspInfo()
    nat.check(lib.apsp_rkleene(nat.DTYPE_I32, n, d.ptr(), d.ld, p.ptr(), p.ld, mode, thr, aligned, nat.TIER_AUTO,
                               ws.data_ptr(), need, stream(), ctypes.byref(info)))
    torch.cuda.synchronize()
    assert np.array_equal(back64(d.view), want)
    if mode == nat.IDX_VIA:
        assert np.array_equal(p.view.cpu().numpy().astype(np.int64), want_via)
    assert d.intact() and p.intact() and ws_ok()


@pytest.mark.parametrize("n", [97, 256])
def test_classic_and_squaring_guarded(cuda, n):
    lib = nat.load()
    raw = random_graph_raw(n, 0.05, 9, 7 * n, zero_frac=0.01)
    want, want_pred = orc.fw_classic(raw)
    d = Guarded(n, torch.int32, to32(raw))
    p = Guarded(n, torch.int32)
    info = nat.ApspInfo()
    nat.check(lib.apsp_fw_classic(nat.DTYPE_I32, n, d.ptr(), d.ld, p.ptr(), p.ld, stream(), ctypes.byref(info)))
    torch.cuda.synchronize()
    assert np.array_equal(back64(d.view), want)
    assert np.array_equal(p.view.cpu().numpy().astype(np.int64), want_pred)
    assert d.intact() and p.intact()
    sd, sv, si = orc.fw_squaring(raw)
    d2 = Guarded(n, torch.int32, to32(raw))
    v2 = Guarded(n, torch.int32)
    need = lib.apsp_workspace_bytes(nat.ALG_FW_SQUARING, nat.DTYPE_I32, n, 0)
    ws, ws_ok = guarded_ws(need)
    nat.check(lib.apsp_fw_squaring(nat.DTYPE_I32, n, d2.ptr(), d2.ld, v2.ptr(), v2.ld, nat.TIER_AUTO, ws.data_ptr(),
                                   need, stream(), ctypes.byref(info)))
    torch.cuda.synchronize()
    assert np.array_equal(back64(d2.view), sd) and np.array_equal(v2.view.cpu().numpy().astype(np.int64), sv)
    assert d2.intact() and v2.intact() and ws_ok()
