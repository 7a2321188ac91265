"""World-size-2 tests of the multi-GPU row-band schedule over gloo on CPU.

The schedule (ownership, panel broadcast, tier agreement, certificate) is the product code in
paper_2310_03983_b200.distributed; the per-shard arithmetic is the exact CPU stand-in in
tests/shard_ops_cpu.py.  Distances must equal the oracle bit-for-bit and the predecessors must
pass the reconstruction certificate -- for every split of the rows across the two ranks.
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


def _worker(rank, world, port, h, block, out_dir, tier=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_ops_cpu import CpuShardOps

        from paper_2310_03983_b200 import _native as nat
        from paper_2310_03983_b200.distributed import RankState, TorchComm, layout, run_schedule

        n = h.shape[0]
        comm = TorchComm(torch.device("cpu"))
        N, R = layout(n, world, block)
        row0 = rank * R
        rv = max(0, min(R, n - row0))
        hl = torch.from_numpy(h[row0:row0 + rv].copy())
        ops = CpuShardOps(block)
        rs = RankState(rank, row0, rv)
        try:
            tier, gmax = run_schedule([rs], world, n, block, ops, comm, nat.DTYPE_I64, [hl], tier,
                                      comm.allreduce_max)
        except Exception as exc:   # recorded for the parent (e.g. a refused forced tier)
            np.savez(os.path.join(out_dir, f"r{rank}.npz"), err=np.array(type(exc).__name__))
            return
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), d=rs.state.D.numpy()[:rv, :n], p=rs.state.P.numpy()[:rv, :n],
                 tier=tier, gmax=gmax, classic=bool(rs.info.get("classic_for_zero_edges")))
    finally:
        dist.destroy_process_group()


def _solve(h, world, block, tier=None, want_info=False):
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), h, block, td, tier), nprocs=world, join=True)
        parts = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
        if "err" in parts[0]:
            return str(parts[0]["err"])
        if want_info:
            return parts
        d = np.concatenate([p["d"] for p in parts])
        pr = np.concatenate([p["p"] for p in parts])
        return d, pr, int(parts[0]["tier"]), [int(p["gmax"]) for p in parts]


@pytest.mark.parametrize("n,block,density", [(200, 64, 0.05), (60, 64, 0.2), (256, 32, 0.02), (97, 16, 0.1),
                                             (130, 16, 0.03)])
def test_two_ranks_match_oracle(n, block, density):
    from oracle import oracle as orc

    import paper_2310_03983_b200 as ap

    h = random_graph_raw(n, density, 100, seed=n + block)
    want_d, _ = orc.fw_classic(h)
    d, pred, tier, gmaxes = _solve(h, 2, block)
    assert np.array_equal(d, want_d)
    ok, why = ap.check_pred_tree(h, d, pred.astype(np.int64), INF_RAW)
    assert ok, why
    assert len(set(gmaxes)) == 1            # every rank agreed on the certificate input


def test_layout_rows_are_block_multiples():
    from paper_2310_03983_b200.distributed import layout

    for n in (1, 60, 200, 16384, 32768, 20000):
        for world in (1, 2, 4, 8):
            for block in (128, 256):
                N, R = layout(n, world, block)
                assert N >= n and R * world == N and R % block == 0


def test_shard_block_rule():
    from paper_2310_03983_b200.distributed import layout, shard_block

    assert shard_block(16384, 1) == 1024          # single rank: the single-GPU rule
    assert shard_block(32768, 8) == 256           # owner pivot share capped at N/(16P)
    assert shard_block(4096, 2) == 128
    for n, w in [(20480, 2), (26112, 4), (32768, 8), (1000, 3)]:
        b = shard_block(n, w)
        N, R = layout(n, w, b)
        assert R % b == 0 and b % 128 == 0


def test_tier_selection_mirrors_library():
    from paper_2310_03983_b200 import _native as nat
    from paper_2310_03983_b200.distributed import pick_tiers

    dense = {"non_integral": 0, "max_finite": 100, "finite_offdiag": 16384 * 800}
    assert pick_tiers(nat.DTYPE_I32, dense, 16384) == [nat.TIER_U8, nat.TIER_U16, nat.TIER_W32, nat.TIER_I32]
    assert pick_tiers(nat.DTYPE_I32, dense | {"max_finite": 200}, 16384) == [nat.TIER_U16, nat.TIER_W32,
                                                                             nat.TIER_I32]
    sparse = dense | {"finite_offdiag": 16384 * 16}      # rho=0.002-like: skip u8, start at u16
    assert pick_tiers(nat.DTYPE_I32, sparse, 16384) == [nat.TIER_U16, nat.TIER_W32, nat.TIER_I32]
    tiny = dense | {"finite_offdiag": 2048 * 2}          # degree ~2: straight to w32
    assert pick_tiers(nat.DTYPE_I32, tiny, 2048) == [nat.TIER_W32, nat.TIER_I32]
    assert pick_tiers(nat.DTYPE_I64, dense | {"max_finite": 1 << 30}, 16384) == [nat.TIER_I64]
    assert pick_tiers(nat.DTYPE_F32, dense | {"non_integral": 1}, 16384) == [nat.TIER_F32]


def test_two_ranks_zero_cost_edges_take_the_classic_order():
    """Zero-cost edges (allowed by the reference's CostMatrix): the rows are gathered, solved in
    classic k order and scattered back -- distances and pred bit-exact with fw_classic."""
    from oracle import oracle as orc

    h = random_graph_raw(150, 0.05, 9, seed=21, zero_frac=0.03)
    want_d, want_p = orc.fw_classic(h)
    parts = _solve(h, 2, 32, want_info=True)
    d = np.concatenate([p["d"] for p in parts])
    pr = np.concatenate([p["p"] for p in parts])
    assert all(bool(p["classic"]) for p in parts)
    assert np.array_equal(d, want_d) and np.array_equal(pr.astype(np.int64), want_p)


def test_two_ranks_forced_tier_names():
    """A forced tier is given by name like on one GPU, and one that cannot hold the input is
    refused on every rank (ParameterError) instead of failing inside the schedule."""
    from oracle import oracle as orc

    h = random_graph_raw(90, 0.1, 100, seed=5)
    want_d, _ = orc.fw_classic(h)
    d, _, tier, _ = _solve(h, 2, 16, tier="w32")
    from paper_2310_03983_b200 import _native as nat

    assert tier == nat.TIER_W32 and np.array_equal(d, want_d)
    wide = random_graph_raw(90, 0.1, 1000, seed=6)
    assert _solve(wide, 2, 16, tier="u8") == "ParameterError"
