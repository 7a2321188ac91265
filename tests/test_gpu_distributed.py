"""GPU tests of the multi-GPU row-band schedule.

* fw_blocked_emulated runs all ranks' kernels in this process on one B200 (sequentially; no
  rank waits on another) and must be bit-identical -- distances AND predecessors -- to the
  single-GPU solver at the same pivot block.
* fw_blocked_sharded is exercised end to end over a 1-rank NCCL process group.
* rkleene_emulated / rkleene_sharded (replicated matrix, products split by output row bands)
  must equal the single-GPU aligned R-Kleene bit for bit, on every replica.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from conftest import INF_RAW, random_graph_raw
from oracle import oracle as orc

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200.core import INF32

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world,block", [(1000, 3, 128), (2048, 4, 256), (777, 2, 256), (300, 4, 128)])
def test_emulated_ranks_bitwise_equal_single_gpu(cuda, n, world, block):
    from paper_2310_03983_b200.distributed import fw_blocked_emulated

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.05, 100, n), np.int32)).cuda()
    single = ap.solve(h, "fw_blocked", block=block)
    d, p, info = fw_blocked_emulated(h, world, block=block)
    assert info["tier"] == single.info["tier"]
    assert torch.equal(d, single.distances)
    assert torch.equal(p, single.index)
    ok, why = ap.check_pred_tree(h, d, p, INF32)
    assert ok, why


def test_emulated_tier_fallback(cuda):
    from paper_2310_03983_b200.distributed import fw_blocked_emulated

    n = 600
    raw = np.full((n, n), INF32, np.int32)
    np.fill_diagonal(raw, 0)
    raw[np.arange(n - 1), np.arange(1, n)] = 2          # a long path: u8 certificate must fail
    h = torch.from_numpy(raw).cuda()
    d, p, info = fw_blocked_emulated(h, 3, block=128)
    assert info["tier"] == "w32"
    single = ap.solve(h, "fw_blocked", block=128)
    assert torch.equal(d, single.distances) and torch.equal(p, single.index)


def _nccl_worker(rank, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2310_03983_b200.distributed import TorchComm, fw_blocked_sharded

    from paper_2310_03983_b200.distributed_rk import rkleene_sharded

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(512, 0.1, 100, 3), np.int32)).cuda()
    comm = TorchComm(torch.device("cuda", 0))
    r = fw_blocked_sharded(h, 512, comm=comm, block=128)
    single = ap.solve(h, "fw_blocked", block=128)
    ok = bool(torch.equal(r.distances, single.distances) and torch.equal(r.pred, single.index))
    k = rkleene_sharded(h, 512, comm=comm, base_threshold=128)
    ks = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=128)
    ok = ok and bool(torch.equal(k.distances, ks.distances) and torch.equal(k.pred, ks.index))
    out.put(ok)
    dist.destroy_process_group()


def test_sharded_entry_over_nccl(cuda):
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    proc = ctx.Process(target=_nccl_worker, args=(0, port, q))
    proc.start()
    proc.join(timeout=300)
    assert proc.exitcode == 0
    assert q.get(timeout=5)


@pytest.mark.parametrize("n,world,thr,rho", [(1000, 2, 256, 0.05), (2048, 3, 512, 0.1), (700, 4, 128, 0.02),
                                             (1500, 2, 2048, 0.1)])
def test_rkleene_emulated_ranks_bitwise_equal_single_gpu(cuda, n, world, thr, rho):
    from paper_2310_03983_b200.distributed_rk import rkleene_emulated

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, n + 1), np.int32)).cuda()
    single = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=thr)
    d, p, info = rkleene_emulated(h, world, base_threshold=thr)
    assert info["replicas_equal"]
    assert info["tier"] == single.info["tier"]
    assert torch.equal(d, single.distances)
    assert torch.equal(p, single.index)
    ok, why = ap.check_pred_tree(h, d, p, INF32)
    assert ok, why


def test_rkleene_emulated_tier_fallback(cuda):
    from paper_2310_03983_b200.distributed_rk import rkleene_emulated

    n = 600
    raw = np.full((n, n), INF32, np.int32)
    np.fill_diagonal(raw, 0)
    raw[np.arange(n - 1), np.arange(1, n)] = 2          # a long path: u8 certificate must fail
    h = torch.from_numpy(raw).cuda()
    d, p, info = rkleene_emulated(h, 3, base_threshold=128)
    assert info["tier"] == "w32" and info["replicas_equal"]
    single = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=128)
    assert torch.equal(d, single.distances) and torch.equal(p, single.index)


@pytest.mark.parametrize("n,world,thr,rho", [(1000, 3, 256, 0.05), (2048, 4, 512, 0.1)])
def test_rkleene_fused_peer_stores_emulated(cuda, n, world, thr, rho):
    """Fused exchange: each rank's product epilogue writes its band into every replica."""
    from paper_2310_03983_b200.distributed_rk import rkleene_emulated

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, n + 2), np.int32)).cuda()
    single = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=thr)
    d, p, info = rkleene_emulated(h, world, base_threshold=thr, fused=True)
    assert info["fused"] and info["replicas_equal"]
    assert torch.equal(d, single.distances) and torch.equal(p, single.index)


def _ipc_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_03983_b200.distributed import TorchComm
        from paper_2310_03983_b200.distributed_rk import rkleene_sharded

        n = 900
        h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.05, 100, 77), np.int32)).cuda()
        r = rkleene_sharded(h, n, comm=TorchComm(torch.device("cuda", 0)), base_threshold=256, fused=True)
        torch.cuda.synchronize()
        if rank == 0:
            single = ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=256)
            out.put(bool(torch.equal(r.distances, single.distances) and torch.equal(r.pred, single.index)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_rkleene_fused_ipc_two_processes_one_gpu(cuda):
    """Two processes, one GPU: replicas mapped with CUDA IPC, bands pushed by the product
    kernel's peer stores, gloo all-reduce as the per-product barrier (host-side; no kernel waits
    on another)."""
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5)


@pytest.mark.parametrize("n,world,block", [(1000, 3, 128), (2048, 4, 256), (777, 2, 256)])
def test_fused_panel_push_emulated(cuda, n, world, block):
    """FW fused panel push: the owner's pivot kernel stores the whole panel into every other
    rank's receive slot; receivers read only their own slots."""
    from paper_2310_03983_b200.distributed import fw_blocked_emulated

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.05, 100, n + 5), np.int32)).cuda()
    single = ap.solve(h, "fw_blocked", block=block)
    d, p, info = fw_blocked_emulated(h, world, block=block, fused=True)
    assert info["tier"] == single.info["tier"]
    assert torch.equal(d, single.distances) and torch.equal(p, single.index)


@pytest.mark.parametrize("world,block", [(3, 128), (2, 256)])
def test_fused_panel_push_w32_emulated(cuda, world, block):
    """The fused push on the w32 tier (weights past the u16 range): minplus_w32nt_kernel's
    whole-panel peer stores, bitwise equal to one GPU."""
    from paper_2310_03983_b200.distributed import fw_blocked_emulated

    n = 900
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.05, 50000, 17), np.int32)).cuda()
    single = ap.solve(h, "fw_blocked", block=block)
    assert single.info["tier"] == "w32"
    d, p, info = fw_blocked_emulated(h, world, block=block, fused=True)
    assert info["tier"] == "w32"
    assert torch.equal(d, single.distances) and torch.equal(p, single.index)


def test_sharded_zero_cost_edges_classic_order(cuda):
    """Zero-cost edges on the sharded path: gathered, solved in classic k order on one GPU,
    scattered back -- bit-exact with reference fw_classic (the oracle)."""
    from paper_2310_03983_b200.distributed import fw_blocked_emulated

    raw = random_graph_raw(500, 0.03, 9, 77, zero_frac=0.02)
    want_d, want_p = orc.fw_classic(raw)
    h32 = raw.astype(np.int64)
    h32[raw == INF_RAW] = INF32
    h = torch.from_numpy(h32.astype(np.int32)).cuda()
    d, p, info = fw_blocked_emulated(h, 3, block=128)
    assert info.get("classic_for_zero_edges")
    dd = d.cpu().numpy().astype(np.int64)
    dd[dd == INF32] = INF_RAW
    assert np.array_equal(dd, want_d) and np.array_equal(p.cpu().numpy().astype(np.int64), want_p)


def _fw_ipc_worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_03983_b200.distributed import TorchComm, fw_blocked_sharded, layout

        n, block = 1100, 128
        h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.05, 100, 91), np.int32)).cuda()
        N, R = layout(n, world, block)
        row0 = rank * R
        rv = max(0, min(R, n - row0))
        r = fw_blocked_sharded(h[row0:row0 + rv].contiguous(), n, comm=TorchComm(torch.device("cuda", 0)),
                               block=block, fused=True)
        torch.cuda.synchronize()
        single = ap.solve(h, "fw_blocked", block=block)
        ok = bool(torch.equal(r.distances, single.distances[row0:row0 + rv]) and
                  torch.equal(r.pred, single.index[row0:row0 + rv]))
        out.put((rank, ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_fused_panel_push_ipc_two_processes_one_gpu(cuda):
    """Two processes, one GPU: receive slots mapped with CUDA IPC, panels pushed by the pivot
    kernel's peer stores, gloo all-reduces as the slot / readiness barriers (host-side)."""
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_fw_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res[0] and res[1]
