#!/usr/bin/env python3
"""Where the fixed per-solve time goes at small n: CUDA-event time of ap.solve (Python API),
of the bare device ABI call on preallocated buffers, and the library's own device_ms.
usage: tools/overhead.py [n ...]"""
import ctypes
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402
from paper_2310_03983_b200 import _native as nat  # noqa: E402


def ev_time(fn, reps=20):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


lib = nat.load()
for n in [int(x) for x in (sys.argv[1:] or ["128", "256", "1024"])]:
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.int32)).cuda()
    dist = torch.empty_like(h)
    pred = torch.empty((n, n), dtype=torch.int32, device="cuda")
    wsb = lib.apsp_workspace_bytes(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, 0)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    info = nat.ApspInfo()
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def abi():
        dist.copy_(h)
        nat.check(lib.apsp_fw_blocked(nat.DTYPE_I32, n, dist.data_ptr(), n, pred.data_ptr(), n, 0, nat.TIER_AUTO,
                                      ws.data_ptr(), wsb, sp, ctypes.byref(info)))

    t_api = ev_time(lambda: ap.solve(h))
    t_abi = ev_time(abi)
    print(f"n={n}: ap.solve {t_api:.3f} ms | C ABI on preallocated buffers {t_abi:.3f} ms | "
          f"library device_ms {info.device_ms:.3f} | launches {info.launches}", flush=True)
