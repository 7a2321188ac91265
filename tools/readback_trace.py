#!/usr/bin/env python3
"""Time the phases of apsp_solve_host at n (default 16384): device solve alone vs. the host
call, and the packed readback's host wait+widen time (APSP_READBACK_TRACE)."""

from __future__ import annotations

import ctypes
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402
from paper_2310_03983_b200 import _native as nat  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
    h = ap.dense_costs(ap.GenParams(n, 0.1, 100, 7 + n), np.int32)
    lib = nat.load()
    hin = torch.from_numpy(h).pin_memory()
    dout = torch.empty((n, n), dtype=torch.int32).pin_memory()
    pout = torch.empty((n, n), dtype=torch.int32).pin_memory()
    info = nat.ApspInfo()
    for label, env in (("packed", "1"), ("plain", "0")):
        os.environ["APSP_PACKED_READBACK"] = env
        ts = []
        for i in range(5):
            if i == 4:
                os.environ["APSP_READBACK_TRACE"] = "1"
            t = time.perf_counter()
            nat.check(lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, hin.data_ptr(), dout.data_ptr(),
                                          pout.data_ptr(), nat.DTYPE_I32, nat.IDX_PRED, 0, 0, 0, nat.TIER_AUTO, 0,
                                          ctypes.byref(info)))
            ts.append((time.perf_counter() - t) * 1e3)
            os.environ.pop("APSP_READBACK_TRACE", None)
        print(f"{label}: host call ms {' '.join(f'{x:.1f}' for x in ts)}; device solve {info.device_ms:.1f} ms; "
              f"d2h {info.d2h_bytes_per_cell} B/cell", flush=True)
    x = torch.empty(n * n, dtype=torch.int32, device="cuda")
    for nbytes, label in ((n * n * 4, "H2D 4B/cell"), (n * n * 3, "D2H 3B/cell"), (n * n * 8, "D2H 8B/cell")):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if label.startswith("H2D"):
            e0.record(); x.copy_(hin.view(-1), non_blocking=True); e1.record()
        else:
            src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
            e0.record(); dst.copy_(src, non_blocking=True); e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{label}: {nbytes / 2**20:.0f} MiB in {ms:.2f} ms = {nbytes / ms / 1e6:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
