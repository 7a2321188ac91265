#!/usr/bin/env python3
"""Device time of the sharded R-Kleene schedule (emulated ranks on one B200) vs the one-GPU
aligned R-Kleene.  usage: tools/rk_shard_timing.py n thr world [world ...]"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_03983_b200 as ap  # noqa: E402
from paper_2310_03983_b200.distributed_rk import rkleene_emulated  # noqa: E402


def timed(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def main():
    n, thr = int(sys.argv[1]), int(sys.argv[2])
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 7 + n), np.float32)).cuda()
    ms, single = timed(lambda: ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=thr))
    print(f"one-GPU rkleene n={n} thr={thr}: {ms:.2f} ms tier={single.info['tier']}", flush=True)
    for w in map(int, sys.argv[3:]):
        ms, (d, p, info) = timed(lambda: rkleene_emulated(h, w, base_threshold=thr))
        same = torch.equal(d, single.distances) and torch.equal(p, single.index)
        print(f"emulated world={w}: {ms:.2f} ms (all ranks, sequential) bitwise_equal={same} "
              f"replicas_equal={info['replicas_equal']}", flush=True)


if __name__ == "__main__":
    main()
