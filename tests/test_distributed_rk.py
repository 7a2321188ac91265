"""World-size-2 tests of the multi-GPU R-Kleene schedule (replicated matrix, products split by
output row bands, band all-gather) over gloo on CPU.

The schedule is the product code in paper_2310_03983_b200.distributed_rk; the per-replica
arithmetic is the exact CPU stand-in in tests/rk_ops_cpu.py.  Two ranks must produce replicas
bit-identical to one rank, distances equal to the oracle, and predecessors that pass the
reconstruction certificate.
"""

from __future__ import annotations

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import INF_RAW, random_graph_raw


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, h, thr, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from rk_ops_cpu import CpuRkOps

        from paper_2310_03983_b200 import _native as nat
        from paper_2310_03983_b200.distributed import RankState, TorchComm
        from paper_2310_03983_b200.distributed_rk import run_rk_schedule

        n = h.shape[0]
        comm = TorchComm(torch.device("cpu"))
        rs = RankState(rank, 0, n)
        tier, gmax = run_rk_schedule([rs], world, n, thr, CpuRkOps(), comm, nat.DTYPE_I64,
                                     [torch.from_numpy(h.copy())], None, comm.allreduce_max)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), d=rs.state.D.numpy()[:n, :n], p=rs.state.P.numpy()[:n, :n],
                 tier=tier, gmax=gmax)
    finally:
        dist.destroy_process_group()


def _solve(h, world, thr):
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), h, thr, td), nprocs=world, join=True)
        return [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]


def _single(h, thr):
    from rk_ops_cpu import CpuRkOps

    from paper_2310_03983_b200 import _native as nat
    from paper_2310_03983_b200.distributed import EmulatedComm, RankState
    from paper_2310_03983_b200.distributed_rk import run_rk_schedule

    n = h.shape[0]
    rs = RankState(0, 0, n)
    run_rk_schedule([rs], 1, n, thr, CpuRkOps(), EmulatedComm(), nat.DTYPE_I64, [torch.from_numpy(h.copy())])
    return rs.state.D.numpy()[:n, :n], rs.state.P.numpy()[:n, :n]


@pytest.mark.parametrize("n,thr,density", [(300, 128, 0.03), (200, 100, 0.1), (390, 128, 0.01)])
def test_two_ranks_replicas_match_one_rank_and_oracle(n, thr, density):
    from oracle import oracle as orc

    import paper_2310_03983_b200 as ap

    h = random_graph_raw(n, density, 100, seed=n + thr)
    want_d, _ = orc.fw_classic(h)
    one_d, one_p = _single(h, thr)
    assert np.array_equal(one_d, want_d)
    parts = _solve(h, 2, thr)
    for p in parts:                                   # both replicas, bit-identical to one rank
        assert np.array_equal(p["d"], one_d)
        assert np.array_equal(p["p"], one_p)
    ok, why = ap.check_pred_tree(h, one_d, one_p.astype(np.int64), INF_RAW)
    assert ok, why


def test_row_bands_cover_and_align():
    from paper_2310_03983_b200.distributed_rk import rk_split, row_bands

    for m in (128, 256, 384, 1024, 16384, 4096 + 128):
        for world in (1, 2, 3, 4, 8):
            bands = row_bands(m, world)
            assert bands[0][0] == 0 and bands[-1][1] == m
            assert all(b[0] == a[1] for a, b in zip(bands, bands[1:]))
            assert all(lo % 128 == 0 and hi >= lo for lo, hi in bands)
        assert rk_split(m) % 128 == 0 and 0 < rk_split(m) < m or m == 128
