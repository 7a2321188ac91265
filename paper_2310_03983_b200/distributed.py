"""Multi-GPU blocked Floyd-Warshall: one process per GPU, 1D row bands, NCCL panel broadcast.

SURVEY.md 8(e): FW shards naturally with one exchange step per pivot block.  Rank r owns rows
[r*R, (r+1)*R) of the padded N x N matrix (R = N / world, a multiple of the pivot block b, so a
pivot block never straddles ranks).  Per pivot block [k0, k0+b), owned by rank o:

  1. o      apsp_shard_pivot: close the b x b diagonal block (classic order), then
            row panel <- Dg (x) row panel                      (both on o's rows only)
  2. all    the b x N row panel -- values and predecessors, ~b*N*(1+4) bytes per round --
            reaches every rank: fused (u8/u16): the owner's pivot kernel stores it into each
            peer's receive slot over NVLink (CUDA IPC), with 4-byte all-reduces as barriers;
            otherwise an NCCL broadcast
  3. all    apsp_shard_update: column panel <- colpanel (x) Dg (Dg = columns k0.. of the
            received panel), then phase 3 on the local rows with the received panel as B

A row-band layout needs one broadcast per round (the column panel is local to every rank);
on NVSwitch every GPU has full bandwidth to every peer, so the 2D grid of the survey buys no
bandwidth, only smaller messages.  The arithmetic is the single-GPU schedule exactly, so the
distances are bit-identical to one GPU and the predecessors identical at the same b.

The schedule is written once over abstract per-rank ``ops`` and a ``bcast`` hook:
* ``CudaShardOps`` + ``TorchComm`` (NCCL, torchrun)      -- the product path;
* ``CudaShardOps`` + in-process emulation of all ranks on one GPU (tests);
* CPU ops in tests/ + ``TorchComm`` over gloo            -- the world_size-2 CPU tests.
"""

from __future__ import annotations

import ctypes
import json
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .core import (
    INF32,
    INF_RAW,
    ApspError,
    CostRangeError,
    MalformedGraphError,
    NegativeWeightError,
    ParameterError,
)

U8_LIMIT, U16_LIMIT, W32_LIMIT = 254, 510, (1 << 24) - 2
TIER_LIMIT = {nat.TIER_U8: U8_LIMIT, nat.TIER_U16: U16_LIMIT, nat.TIER_W32: W32_LIMIT, nat.TIER_I32: INF32 - 1,
              nat.TIER_I64: (1 << 60) - 1}


def round_up(v: int, m: int) -> int:
    return (v + m - 1) // m * m


def shard_block(n: int, world: int) -> int:
    """Pivot block for the sharded solve.

    Starts from the single-GPU size rule (fw_sched.cu default_block).  The owner of a pivot block
    does its b^2*N pivot work alone while every rank does (N/P)*N*b of phase 3, so the owner's
    extra share is b*P/N: b is capped at N/(16 P) (~6%).  Then lowered until a rank's row band
    holds whole blocks without extra padding."""
    b = 128 if n <= 6144 else 256 if n <= 12288 else 1024 if n <= 24576 else 2048
    while b > 128 and b > n / (16 * world):
        b //= 2
    while b > 128 and layout(n, world, b)[0] > 1.01 * layout(n, world, 128)[0]:
        b //= 2
    return b


def layout(n: int, world: int, block: int) -> tuple[int, int]:
    """(N, R): padded order and rows per rank (R a multiple of block)."""
    N = round_up(max(n, 1), block * world)
    return N, N // world


def pick_tiers(dtype_code: int, scan: dict, n: int = 0) -> list[int]:
    """Narrowest exact tier first (mirror of engine.cu pick_tiers, including the sparse-graph
    distance estimate 0.5 * w_max * ln(n) / ln(average degree) that skips hopeless tiers)."""
    import math

    integral = dtype_code != nat.DTYPE_F32 or not scan["non_integral"]
    w = scan["max_finite"]
    nv = max(n, 2)
    deg = max(scan.get("finite_offdiag", nv * nv) / nv, 1.5)
    m_est = (0.8 if deg < 8 else 0.5) * w * math.log(nv) / math.log(deg)
    t = []
    if integral and w <= U8_LIMIT and m_est + w <= U8_LIMIT:
        t.append(nat.TIER_U8)
    if integral and w <= U16_LIMIT and m_est + w <= U16_LIMIT:
        t.append(nat.TIER_U16)
    if integral and w <= W32_LIMIT:
        t.append(nat.TIER_W32)
    t.append({nat.DTYPE_F32: nat.TIER_F32, nat.DTYPE_I32: nat.TIER_I32}.get(dtype_code, nat.TIER_I64))
    return t


def resolve_tier(tier, dtype_code: int, scan: dict):
    """A caller's forced tier (None / "auto", a name such as "u8", or a tier code) -> its code,
    or None for the automatic choice. A forced tier must hold the input exactly (as the
    single-GPU engine's pick_tiers: narrow integer tiers need integral costs within range);
    the certificate still decides whether the result fits."""
    if tier is None or tier == "auto" or tier == nat.TIER_AUTO:
        return None
    from .solvers import _tier_arg

    code = _tier_arg(tier)
    if code not in nat.TIER_NAMES:
        raise ParameterError(f"unknown tier {tier!r}")
    integral = dtype_code != nat.DTYPE_F32 or not scan["non_integral"]
    w = scan["max_finite"]
    fits = {nat.TIER_U8: integral and w <= U8_LIMIT, nat.TIER_U16: integral and w <= U16_LIMIT,
            nat.TIER_W32: integral and w <= W32_LIMIT,
            nat.TIER_I32: dtype_code != nat.DTYPE_F32 and w <= INF32 - 1,
            nat.TIER_F32: dtype_code == nat.DTYPE_F32, nat.TIER_I64: dtype_code == nat.DTYPE_I64}[code]
    if not fits:
        raise ParameterError(f"tier {nat.TIER_NAMES[code]!r} cannot hold this input exactly")
    return code


def merge_scans(scans: list[dict]) -> dict:
    out = {k: 0 for k in ("negative", "diag_nonzero", "non_integral", "zero_offdiag")}
    out["max_finite"] = -1
    for s in scans:
        for k in out:
            out[k] = max(out[k], int(s[k]))
    out["finite_offdiag"] = sum(int(s.get("finite_offdiag", 0)) for s in scans)
    return out


def check_scan(scan: dict) -> None:
    if scan["negative"]:
        raise NegativeWeightError("solver input contains a negative finite cost")
    if scan["diag_nonzero"]:
        raise MalformedGraphError("solver input must have a zero diagonal")


# ---- the schedule --------------------------------------------------------------------------

@dataclass
class RankState:
    rank: int
    row0: int
    rows_valid: int
    state: object = None
    info: dict = field(default_factory=dict)


def run_schedule(ranks: list[RankState], world: int, n: int, block: int, ops, comm, dtype_code: int,
                 h_locals: list, tier_req: int | None = None, allreduce_max=None):
    """Solve with the given local ranks; returns (tier, global max finite)."""
    N, R = layout(n, world, block)
    scan = merged_scan(ranks, ops, h_locals, n, allreduce_max)
    forced = resolve_tier(tier_req, dtype_code, scan)
    if scan["zero_offdiag"]:
        return classic_fallback(ranks, world, n, ops, comm, dtype_code, h_locals, R, N, allreduce_max)
    tiers = [forced] if forced is not None else pick_tiers(dtype_code, scan, n)
    for tier in tiers:
        for rk, h in zip(ranks, h_locals):
            rk.state = ops.alloc(tier, R, N)
            ops.prepare(rk.state, h, n, rk.row0, dtype_code)
        run_rounds(ranks, N, R, block, ops, comm)
        local_max = max(ops.max_finite(rk.state, rk.rows_valid, n) for rk in ranks)
        gmax = allreduce_max(local_max) if allreduce_max else local_max
        if tier == nat.TIER_F32:
            return tier, gmax
        if gmax < 0 or gmax + scan["max_finite"] <= TIER_LIMIT[tier]:
            return tier, gmax
    if dtype_code == nat.DTYPE_I32:
        raise CostRangeError("shortest-path cost left the representable int32 range")
    raise CostRangeError("no value tier could represent the result")


EXACT_TIER = {nat.DTYPE_I32: nat.TIER_I32, nat.DTYPE_F32: nat.TIER_F32, nat.DTYPE_I64: nat.TIER_I64}


def classic_fallback(ranks, world, n, ops, comm, dtype_code, h_locals, R, N, allreduce_max):
    """Zero-cost edges (allowed by the reference's CostMatrix, core.py:161-230): many cells
    relaxing at once could make equal-distance vertices point at each other, so -- as on one
    GPU -- the predecessors come from the classic k order (bit-exact with reference fw_classic).
    The rows are gathered on rank 0, solved there by the classic kernel, and scattered back into
    every rank's state in the exact tier; returns (tier, global max finite) like run_schedule."""
    full = comm.gather_rows(ranks, h_locals, n, R)          # rank 0: the n x n input, else None
    res = ops.classic(full, n, dtype_code) if full is not None else None
    rows = comm.scatter_rows(ranks, res, n, R)               # per local rank: (dist rows, pred rows)
    tier = EXACT_TIER[dtype_code]
    for rk, (d, p) in zip(ranks, rows):
        rk.state = ops.alloc(tier, R, N)
        ops.prepare(rk.state, d, n, rk.row0, dtype_code)
        ops.set_pred_rows(rk.state, p)
    local_max = max(ops.max_finite(rk.state, rk.rows_valid, n) for rk in ranks)
    gmax = allreduce_max(local_max) if allreduce_max else local_max
    for rk in ranks:
        rk.info = {"classic_for_zero_edges": True}
    return tier, gmax


def run_rounds(ranks: list[RankState], N: int, R: int, b: int, ops, comm) -> None:
    """The pivot rounds with one-block lookahead.

    Round K (pivot rows owned by o, local rows [lr, lr+b)):
      * wait for panel K
      * owner o' of block K+1: finish round K on its rows [lr', lr'+b) first, then run the
        K+1 pivot on the high-priority side stream and start broadcasting panel K+1
        (asynchronously, into the other receive slot)
      * everyone: round K on all remaining local rows, concurrent with pivot / broadcast K+1
    """
    nblocks = N // b

    def owner(k0):
        o = k0 // R
        return o, k0 - o * R

    # fused panel push (u8/u16, CudaShardOps(fused=True)): the owner's pivot kernel stores the
    # whole panel into every peer's receive slot; the comm only adds tiny barriers
    fused = bool(getattr(ops, "fused_for", lambda st: False)(ranks[0].state))
    if fused:
        fused = bool(comm.connect_slots(ranks, ops))
    o, lr = owner(0)
    panels = None
    for rk in ranks:
        if rk.rank == o:
            panels = ops.pivot(rk.state, lr, 0, side=False, slot=0)
    handle = comm.bcast_start(ranks, o, panels, 0, ops, fused=fused)
    for K in range(nblocks):
        k0 = K * b
        o, lr = owner(k0)
        cur = comm.bcast_wait(handle, ranks, ops)
        nxt = K + 1 < nblocks
        o1, lr1 = owner(k0 + b) if nxt else (-1, -1)
        if nxt:
            if fused:   # every rank is done with slot (K+1) % 2 (read by round K-1) before the push
                comm.slot_barrier(ranks, ops)
            nxt_panels = None
            for rk, (pv, pp) in zip(ranks, cur):
                if rk.rank == o1:
                    ops.update(rk.state, pv, pp, k0, lr1, lr1 + b, -1, -1)
                    nxt_panels = ops.pivot(rk.state, lr1, k0 + b, side=True, slot=(K + 1) % 2)
            handle = comm.bcast_start(ranks, o1, nxt_panels, (K + 1) % 2, ops, fused=fused)
        for rk, (pv, pp) in zip(ranks, cur):
            lo, hi = (lr, lr + b) if rk.rank == o else (-1, -1)
            if rk.rank == o1:              # its K+1 pivot rows are done already (adjacent bands merge)
                lo, hi = (lr1, lr1 + b) if lo < 0 else (min(lo, lr1), max(hi, lr1 + b))
            ops.update(rk.state, pv, pp, k0, 0, R, lo, hi)


def allreduce_sum(allreduce_max, v: int) -> int:
    """Sum over ranks through the comm's all-reduce (TorchComm exposes allreduce_sum)."""
    owner = getattr(allreduce_max, "__self__", None)
    return owner.allreduce_sum(v) if owner is not None and hasattr(owner, "allreduce_sum") else v


def merged_scan(ranks, ops, h_locals, n, allreduce_max):
    scans = [ops.scan(h, rk.row0, rk.rows_valid, n) for rk, h in zip(ranks, h_locals)]
    scan = merge_scans(scans)
    if allreduce_max is not None:
        edges = scan.pop("finite_offdiag")
        scan = {k: allreduce_max(v) for k, v in scan.items()}
        scan["finite_offdiag"] = allreduce_sum(allreduce_max, edges)
    check_scan(scan)
    for rk in ranks:
        rk.scan = scan
    return scan


# ---- CUDA shard ops --------------------------------------------------------------------------

_TORCH_STORE = {nat.TIER_U8: "uint8", nat.TIER_U16: "uint16", nat.TIER_W32: "int32", nat.TIER_I32: "int32", nat.TIER_F32: "float32",
                nat.TIER_I64: "int64"}


@dataclass
class CudaShard:
    tier: int
    R: int
    N: int
    D: object
    P: object
    scratch: object
    stream: object
    pv: object = None      # two receive slots for the broadcast panel (values, pred)
    pp: object = None
    peer_pv: list = field(default_factory=list)   # fused push: peers' receive slots [peer][slot]
    peer_pp: list = field(default_factory=list)
    peer_keep: list = field(default_factory=list)  # IPC mappings kept alive


class CudaShardOps:
    """Per-rank device state and the C-ABI shard calls, on torch's current stream."""

    def __init__(self, device, block: int, fused: bool = False):
        import torch

        self.torch = torch
        self.device = torch.device(device)
        self.block = block
        self.lib = nat.load()
        self.side = torch.cuda.Stream(self.device, priority=-100)   # lookahead pivots
        self.fused = fused

    def fused_for(self, st) -> bool:
        """Fused panel push (the pivot kernel's own peer stores) for the bulk-staged tiers."""
        return self.fused and st.tier in (nat.TIER_U8, nat.TIER_U16, nat.TIER_W32)

    def set_peer_slots(self, st: CudaShard, peer_pv: list, peer_pp: list, keep=()) -> None:
        if len(peer_pv) > 7:
            raise ParameterError("the fused panel push supports at most 8 ranks")
        st.peer_pv, st.peer_pp, st.peer_keep = list(peer_pv), list(peer_pp), list(keep)

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def scan(self, h, row0: int, rows_valid: int, n: int) -> dict:
        r = nat.ScanResult()
        if rows_valid > 0:
            nat.check(self.lib.apsp_scan(_dtype_of(h), h.data_ptr(), n, rows_valid, n, row0, ctypes.byref(r),
                                         self._stream()))
        mx = int(r.max_finite) if r.any_finite else -1
        return {"negative": r.negative, "diag_nonzero": r.diag_nonzero, "non_integral": r.non_integral,
                "zero_offdiag": r.zero_offdiag, "max_finite": mx, "finite_offdiag": int(r.finite_offdiag)}

    def alloc(self, tier: int, R: int, N: int) -> CudaShard:
        t = self.torch
        dt = getattr(t, _TORCH_STORE[tier])
        sb = self.lib.apsp_shard_scratch_bytes(tier, N, R, self.block)
        return CudaShard(tier, R, N, t.empty((R, N), dtype=dt, device=self.device),
                         t.empty((R, N), dtype=t.int32, device=self.device),
                         t.empty(sb, dtype=t.uint8, device=self.device),
                         t.empty(sb, dtype=t.uint8, device=self.device),      # side-stream scratch
                         [t.empty((self.block, N), dtype=dt, device=self.device) for _ in range(2)],
                         [t.empty((self.block, N), dtype=t.int32, device=self.device) for _ in range(2)])

    def prepare(self, st: CudaShard, h, n: int, row0: int, dtype_code: int) -> None:
        hp = h.data_ptr() if h is not None and h.numel() else None
        nat.check(self.lib.apsp_shard_prepare(dtype_code, st.tier, n, st.N, row0, st.R, hp, n, st.D.data_ptr(),
                                              st.N, st.P.data_ptr(), st.N, self._stream()))

    def pivot(self, st: CudaShard, lrow: int, k0: int, side: bool, slot: int | None = None):
        """Pivot of block k0 (its rows are local rows [lrow, lrow+b)); side=True runs it on the
        high-priority side stream after the work already queued on the current stream.  Fused:
        the pivot kernel also stores the whole panel into every peer's receive slot ``slot``."""
        t = self.torch
        if side:
            self.side.wait_stream(t.cuda.current_stream(self.device))
            stream, scratch = self.side, st.stream
        else:
            stream, scratch = t.cuda.current_stream(self.device), st.scratch
        if self.fused_for(st) and st.peer_pv and slot is not None:
            es = st.D.element_size()
            base_v = st.D.data_ptr() + lrow * st.N * es
            base_p = st.P.data_ptr() + lrow * st.N * 4
            npr = len(st.peer_pv)
            dv = (ctypes.c_int64 * npr)(*[pv[slot].data_ptr() - base_v for pv in st.peer_pv])
            dp = (ctypes.c_int64 * npr)(*[pp[slot].data_ptr() - base_p for pp in st.peer_pp])
            nat.check(self.lib.apsp_shard_pivot_fused(st.tier, st.N, self.block, st.D.data_ptr(), st.N,
                                                      st.P.data_ptr(), st.N, lrow, k0, npr, dv, dp,
                                                      scratch.data_ptr(), scratch.numel(),
                                                      ctypes.c_void_p(stream.cuda_stream)))
            return st.D[lrow:lrow + self.block], st.P[lrow:lrow + self.block], (stream if side else None)
        nat.check(self.lib.apsp_shard_pivot(st.tier, st.N, self.block, st.D.data_ptr(), st.N, st.P.data_ptr(), st.N,
                                            lrow, k0, scratch.data_ptr(), scratch.numel(),
                                            ctypes.c_void_p(stream.cuda_stream)))
        return st.D[lrow:lrow + self.block], st.P[lrow:lrow + self.block], (stream if side else None)

    def recv_buffers(self, st: CudaShard, slot: int):
        return st.pv[slot], st.pp[slot]

    def join_side(self) -> None:
        self.torch.cuda.current_stream(self.device).wait_stream(self.side)

    def update(self, st: CudaShard, pv, pp, k0: int, row_lo: int, row_hi: int, skip_lo: int, skip_hi: int) -> None:
        nat.check(self.lib.apsp_shard_update(st.tier, st.N, self.block, row_lo, row_hi, st.D.data_ptr(), st.N,
                                             st.P.data_ptr(), st.N, pv.data_ptr(), st.N, pp.data_ptr(), st.N, k0,
                                             skip_lo, skip_hi, st.scratch.data_ptr(), st.scratch.numel(),
                                             self._stream()))

    def classic(self, h, n: int, dtype_code: int):
        """Classic-order FW of the whole (gathered) matrix on this GPU (apsp_fw_classic)."""
        t = self.torch
        d = h.contiguous().clone()
        p = t.empty((n, n), dtype=t.int32, device=self.device)
        info = nat.ApspInfo()
        nat.check(self.lib.apsp_fw_classic(dtype_code, n, d.data_ptr(), n, p.data_ptr(), n, self._stream(),
                                           ctypes.byref(info)))
        return d, p

    def set_pred_rows(self, st: CudaShard, p) -> None:
        if p is not None and p.numel():
            st.P[:p.shape[0], :p.shape[1]].copy_(p)

    def max_finite(self, st: CudaShard, rows_valid: int, n: int) -> int:
        mx = ctypes.c_int64(-1)
        nat.check(self.lib.apsp_shard_finish(st.tier, nat.DTYPE_I32, rows_valid, n, st.D.data_ptr(), st.N,
                                             None, st.N, None, n, None, n, ctypes.byref(mx), self._stream()))
        return int(mx.value)

    def finish(self, st: CudaShard, rows_valid: int, n: int, dtype_code: int, dist, pred) -> None:
        mx = ctypes.c_int64(-1)
        nat.check(self.lib.apsp_shard_finish(st.tier, dtype_code, rows_valid, n, st.D.data_ptr(), st.N,
                                             st.P.data_ptr(), st.N, dist.data_ptr(), n, pred.data_ptr(), n,
                                             ctypes.byref(mx), self._stream()))


def _dtype_of(t) -> int:
    s = str(t.dtype)
    return {"torch.int32": nat.DTYPE_I32, "torch.float32": nat.DTYPE_F32, "torch.int64": nat.DTYPE_I64}[s]


# ---- communicators ---------------------------------------------------------------------------

class TorchComm:
    """torch.distributed (NCCL on GPUs, gloo on CPU): this process is one rank."""

    def __init__(self, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.device(device) if device is not None else torch.device("cpu")

    def allreduce_max(self, v: int) -> int:
        t = self.torch.tensor([int(v)], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def allreduce_sum(self, v: int) -> int:
        t = self.torch.tensor([int(v)], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return int(t.item())

    def gather_rows(self, ranks, h_locals, n: int, R: int):
        """Every rank's input rows -> the n x n matrix on rank 0 (None elsewhere)."""
        (rk,), (h,) = ranks, h_locals
        t = self.torch
        dtype = h.dtype if h is not None else t.int32
        pad = t.zeros((R, n), dtype=dtype, device=self.device)
        if rk.rows_valid:
            pad[:rk.rows_valid].copy_(h)
        parts = [t.empty_like(pad) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(pad, parts, dst=0, group=self.group)
        return t.cat(parts)[:n].contiguous() if self.rank == 0 else None

    def scatter_rows(self, ranks, res, n: int, R: int):
        """Rank 0's (dist, pred) n x n result -> every rank's rows [(dist rows, pred rows)]."""
        (rk,) = ranks
        t = self.torch
        meta = [res[0].dtype if res is not None else None]
        self.dist.broadcast_object_list(meta, src=0, group=self.group)
        dd = t.empty((R, n), dtype=meta[0], device=self.device)
        pp = t.empty((R, n), dtype=t.int32, device=self.device)
        if self.rank == 0:
            d, p = res
            D = t.zeros((R * self.world, n), dtype=d.dtype, device=self.device)
            P = t.full((R * self.world, n), -1, dtype=t.int32, device=self.device)
            D[:n].copy_(d)
            P[:n].copy_(p)
            dl, pl = list(D.chunk(self.world)), list(P.chunk(self.world))
        else:
            dl = pl = None
        self.dist.scatter(dd, dl, src=0, group=self.group)
        self.dist.scatter(pp, pl, src=0, group=self.group)
        return [(dd[:rk.rows_valid], pp[:rk.rows_valid])]

    def _flag(self, stream=None):
        """A 4-byte all-reduce issued on `stream` (default: current): the collective's
        completion orders every rank's queued work before whatever waits on the handle."""
        t = self.torch.zeros(1, dtype=self.torch.int32, device=self.device)
        ctx = self.torch.cuda.stream(stream) if stream is not None else _null_ctx()
        with ctx:
            return self.dist.all_reduce(t, group=self.group, async_op=True)

    def peers_reachable(self) -> bool:
        """True on every rank iff every rank's GPU can store into every other rank's GPU
        (cudaDeviceCanAccessPeer for each ordered pair; the IPC mappings then enable peer access
        themselves). All ranks get the same answer, so they agree on fused vs NCCL exchange."""
        if self.world == 1:
            return True
        if self.device.type != "cuda":
            return False
        devs = [None] * self.world
        self.dist.all_gather_object(devs, self.device.index, group=self.group)
        mine = self.device.index
        ok = all(d == mine or self.torch.cuda.can_device_access_peer(mine, d) for d in devs)
        return self.allreduce_min(int(ok)) == 1

    def allreduce_min(self, v: int) -> int:
        t = self.torch.tensor([int(v)], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def connect_slots(self, ranks, ops) -> bool:
        """Fused panel push: map every peer's two receive slots (values, pred) into this process
        with CUDA IPC handles exchanged over the process group. Returns False (every rank) when
        some pair of GPUs has no peer access: the rounds then use the NCCL broadcast."""
        (rk,) = ranks
        st = rk.state
        if self.world == 1:
            ops.set_peer_slots(st, [], [])
            return True
        if not self.peers_reachable():
            ops.set_peer_slots(st, [], [])
            return False
        from torch.multiprocessing.reductions import reduce_tensor

        mine = [reduce_tensor(x) for x in (st.pv[0], st.pv[1], st.pp[0], st.pp[1])]
        every = [None] * self.world
        self.dist.all_gather_object(every, mine, group=self.group)
        peer_pv, peer_pp, keep = [], [], []
        for r, handles in enumerate(every):
            if r == rk.rank:
                continue
            v0, v1, p0, p1 = (f(*a) for f, a in handles)
            peer_pv.append([v0, v1])
            peer_pp.append([p0, p1])
            keep += [v0, v1, p0, p1]
        ops.set_peer_slots(st, peer_pv, peer_pp, keep=keep)
        self._flag().wait()
        return True

    def slot_barrier(self, ranks, ops):
        if self.world > 1:
            self._flag().wait()

    def bcast_start(self, ranks, owner: int, owner_panels, slot: int, ops, fused: bool = False):
        """Asynchronous broadcast of panel (values, pred) from owner into receive slot `slot`.
        On the owner the collective is issued on the stream that produced the panel.  Fused:
        the owner's pivot kernel already stored the panel into every receive slot; a 4-byte
        all-reduce after it (on the pivot's stream) is the readiness signal."""
        (rk,) = ranks
        if self.world == 1:                  # nothing to send (NCCL would still copy 5*b*N bytes)
            pv, pp, _ = owner_panels
            return [], [(pv, pp)], True
        if fused:
            if rk.rank == owner:
                pv, pp, stream = owner_panels
            else:
                (pv, pp), stream = ops.recv_buffers(rk.state, slot), None
            return [self._flag(stream)], [(pv, pp)], rk.rank == owner
        if rk.rank == owner:
            pv, pp, stream = owner_panels
        else:
            (pv, pp), stream = ops.recv_buffers(rk.state, slot), None
        ctx = self.torch.cuda.stream(stream) if stream is not None else _null_ctx()
        wire = pv.view(self.torch.int16) if pv.dtype == self.torch.uint16 else pv   # NCCL has no uint16
        with ctx:
            works = [self.dist.broadcast(wire, src=owner, group=self.group, async_op=True),
                     self.dist.broadcast(pp, src=owner, group=self.group, async_op=True)]
        return works, [(pv, pp)], rk.rank == owner

    def bcast_wait(self, handle, ranks, ops):
        works, panels, is_owner = handle
        for w in works:
            w.wait()
        if is_owner and hasattr(ops, "join_side"):
            ops.join_side()
        return panels


class _null_ctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class EmulatedComm:
    """All ranks in this process on one device: every rank reads the owner's panel directly
    (fused: each rank reads its own receive slot, filled by the owner's pivot kernel)."""

    def connect_slots(self, ranks, ops) -> bool:
        for rk in ranks:
            others = [o.state for o in ranks if o is not rk]
            ops.set_peer_slots(rk.state, [o.pv for o in others], [o.pp for o in others])
        return True

    def slot_barrier(self, ranks, ops):
        return None   # one process, stream order: the side-stream pivot follows all queued updates

    def gather_rows(self, ranks, h_locals, n: int, R: int):
        import torch

        return torch.cat([h for rk, h in zip(ranks, h_locals) if rk.rows_valid])[:n].contiguous()

    def scatter_rows(self, ranks, res, n: int, R: int):
        d, p = res
        return [(d[rk.row0:rk.row0 + rk.rows_valid], p[rk.row0:rk.row0 + rk.rows_valid]) for rk in ranks]

    def bcast_start(self, ranks, owner: int, owner_panels, slot: int, ops, fused: bool = False):
        pv, pp, _ = owner_panels
        if fused:
            return [(pv, pp) if rk.rank == owner else ops.recv_buffers(rk.state, slot) for rk in ranks]
        return [(pv, pp) for _ in ranks]

    def bcast_wait(self, handle, ranks, ops):
        if hasattr(ops, "join_side"):
            ops.join_side()
        return handle


# ---- public entry points ---------------------------------------------------------------------

@dataclass
class ShardedResult:
    distances: object        # local rows [row0, row0 + rows_valid) x n (device tensor)
    pred: object
    row0: int
    rows_valid: int
    info: dict = field(default_factory=dict)


def fw_blocked_sharded(h_local, n: int, *, comm: TorchComm, block: int = 256, tier=None, ops=None,
                       fused: bool = True):
    """SPMD entry: this rank's rows of the input (torch CUDA tensor, rows x n) -> its rows of
    dist / pred.  Must be called by every rank of ``comm`` with the same n and block."""
    import torch

    world, rank = comm.world, comm.rank
    N, R = layout(n, world, block)
    row0 = rank * R
    rows_valid = max(0, min(R, n - row0))
    if h_local is not None and tuple(h_local.shape) != (rows_valid, n):
        raise ParameterError(f"rank {rank} expects {rows_valid} x {n} input rows, got {tuple(h_local.shape)}")
    ops = ops or CudaShardOps(h_local.device, block, fused=fused)
    rs = RankState(rank, row0, rows_valid)
    dtype_code = _dtype_of(h_local)
    t0 = time.perf_counter()
    tier, gmax = run_schedule([rs], world, n, block, ops, comm, dtype_code, [h_local],
                              None if tier is None else tier, comm.allreduce_max)
    dist = torch.empty((rows_valid, n), dtype=h_local.dtype, device=h_local.device)
    pred = torch.empty((rows_valid, n), dtype=torch.int32, device=h_local.device)
    if rows_valid:
        ops.finish(rs.state, rows_valid, n, dtype_code, dist, pred)
    return ShardedResult(dist, pred, row0, rows_valid,
                         {"tier": nat.TIER_NAMES[tier], "max_finite": gmax, "world": world, "N": N, "R": R,
                          "block": block, "host_s": time.perf_counter() - t0} | rs.info)


def fw_blocked_emulated(h, world: int, *, block: int = 256, tier=None, fused: bool = False):
    """All ``world`` ranks of the row-band schedule in this process on h's device (sequential;
    no rank waits on another).  Returns full (dist, pred) tensors.  Used to test the sharded
    path on one GPU."""
    import torch

    n = h.shape[0]
    N, R = layout(n, world, block)
    ops = CudaShardOps(h.device, block, fused=fused)
    ranks, hs = [], []
    for r in range(world):
        row0 = r * R
        rv = max(0, min(R, n - row0))
        ranks.append(RankState(r, row0, rv))
        hs.append(h[row0:row0 + rv].contiguous() if rv else h[:0])
    tier_code, gmax = run_schedule(ranks, world, n, block, ops, EmulatedComm(), _dtype_of(h), hs,
                                   None if tier is None else tier, None)
    dist = torch.empty_like(h)
    pred = torch.empty((n, n), dtype=torch.int32, device=h.device)
    for rk in ranks:
        if rk.rows_valid:
            ops.finish(rk.state, rk.rows_valid, n, _dtype_of(h), dist[rk.row0:rk.row0 + rk.rows_valid],
                       pred[rk.row0:rk.row0 + rk.rows_valid])
    return dist, pred, {"tier": nat.TIER_NAMES[tier_code], "max_finite": gmax} | ranks[0].info


# ---- multi-GPU bench leg (torchrun) ----------------------------------------------------------

def bench_main(args, metric, unit, config, make_input, weak_n, ClockSampler, cpu_baseline=None, tier_peak=None,
               tier_op=None):
    """bench.py --gpus N under torchrun: weak-scaled n (or n=32768 with --strong), row bands,
    max-over-ranks device time; per-rank phase-3 roofline and rank 0's bounded CPU baseline."""
    import os

    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Keep stdout to the one JSON line: the process's fd 1 points at stderr for the whole run
    # (NCCL prints its version banner with printf at communicator init), and the JSON line goes
    # to the saved original stdout.
    import sys

    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = TorchComm(dev)
    world, rank = comm.world, comm.rank
    n = args.n or weak_n(world)
    block = args.block or shard_block(n, world)
    N, R = layout(n, world, block)
    row0 = rank * R
    rv = max(0, min(R, n - row0))
    from .graphgen import GenParams, dense_costs

    rk = getattr(args, "alg", "fw") == "rkleene"
    fused = os.environ.get("APSP_FUSED_PUSH", "1") != "0"
    if rk:   # replicated matrix: every rank generates (and holds) the whole input
        row0, rv = 0, n
    t = time.perf_counter()
    h_np = dense_costs(GenParams(n, args.rho, 100, 7 + n), np.int32, rows=(row0, row0 + rv))
    if rank == 0:
        print(f"[bench] rank0 generated rows {row0}..{row0 + rv} of n={n} in {time.perf_counter() - t:.1f}s",
              file=__import__("sys").stderr, flush=True)
    h = torch.from_numpy(h_np).to(dev)
    if rk:
        from .distributed_rk import CudaRkOps, rkleene_sharded

        ops = CudaRkOps(dev, fused=fused)

        def step():
            return rkleene_sharded(h, n, comm=comm, base_threshold=2048, ops=ops)
    else:
        ops = CudaShardOps(dev, block, fused=fused)

        def step():
            return fw_blocked_sharded(h, n, comm=comm, block=block, ops=ops)
    lib = ops.lib

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = lib.apsp_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(args.steps):
            res = step()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    launches = comm.allreduce_sum(lib.apsp_launch_count() - launches0)   # all ranks' kernels
    # per-rank roofline of the dominant kernel (FW phase 3 on the local rows): one extra, untimed
    # solve with every phase-3 launch bracketed by CUDA events on its stream
    roofline = None
    if not rk:
        lib.apsp_set_profiling(1)
        step()
        torch.cuda.synchronize()
        lib.apsp_set_profiling(0)
        kms, kl = ctypes.c_double(0), ctypes.c_int32(0)
        nat.check(lib.apsp_profile_read(ctypes.byref(kms), ctypes.byref(kl)))
        upd = R * (N - block) ** 2          # sum over rounds of (local rows - owned pivot rows) x (N - b) x b
        rate = upd / (kms.value / 1e3) if kms.value > 0 else 0.0
        every = [None] * world
        dist.all_gather_object(every, (rank, rate, kms.value, int(kl.value)), group=None)
        tier = res.info["tier"]
        peak = (tier_peak or {}).get(tier)
        rates = [r[1] for r in sorted(every)]
        roofline = {"bound": "alu", "kernel": f"minplus phase 3 ({tier} tier) on each rank's rows",
                    "op": (tier_op or {}).get(tier), "unit": "T updates/s",
                    "achieved": min(rates) / 1e12, "peak": peak / 1e12 if peak else None,
                    "frac": (min(rates) / peak) if peak else None,
                    "per_rank": [{"rank": r, "achieved": x / 1e12, "kernel_ms": ms, "launches": nl,
                                  "frac": (x / peak) if peak else None} for r, x, ms, nl in sorted(every)],
                    "updates_per_rank": upd, "traffic": None,
                    "measurement": "CUDA events around every phase-3 launch on its stream (apsp_profile_read), "
                                   "one extra solve; achieved = the slowest rank"}
    cpu = None
    if cpu_baseline is not None and not getattr(args, "no_cpu", False):
        if rank == 0:   # the other ranks wait at the barrier below
            from .graphgen import GenParams as _GP, dense_costs as _dc

            cpu = cpu_baseline(_dc(_GP(n, args.rho, 100, 7 + n), np.int32))
        dist.barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    total_ms = float(ms.item())
    value = n ** 3 * args.steps / (total_ms / 1e3)
    # e2e: pinned host rows in, device solve, host rows out, all ranks
    e2e = None
    if not args.no_e2e:
        hin = torch.from_numpy(h_np).pin_memory()
        dout = torch.empty_like(hin).pin_memory()
        pout = torch.empty(hin.shape, dtype=torch.int32).pin_memory()
        dist.barrier()
        t = time.perf_counter()
        for _ in range(args.steps):
            hd = hin.to(dev, non_blocking=True)
            if rk:
                r = rkleene_sharded(hd, n, comm=comm, base_threshold=2048, ops=ops)
            else:
                r = fw_blocked_sharded(hd, n, comm=comm, block=block, ops=ops)
            if not rk or rank == 0:   # R-Kleene: every replica holds the result; rank 0 reads it
                dout.copy_(r.distances, non_blocking=True)
                pout.copy_(r.pred, non_blocking=True)
            torch.cuda.synchronize()
        dist.barrier()
        dt = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": n ** 3 * args.steps / float(dt.item()), "unit": unit,
               "h2d_bytes_per_step": n * n * 4 * (world if rk else 1), "d2h_bytes_per_step": 2 * n * n * 4,
               "api": ("paper_2310_03983_b200.distributed_rk.rkleene_sharded from pinned host matrices" if rk else
                       "paper_2310_03983_b200.distributed.fw_blocked_sharded from pinned host rows")}
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if getattr(args, "strong", False) else "weak", "vs_baseline": None,
                "dtype": f"tier {res.info['tier']}; int32 in/out",
                "data": "synthetic (reference generator, bit-identical to apsp.generate)",
                "config": config(n, args.rho, world) | (
                    {"workload": f"aligned R-Kleene APSP (replicated matrix, row-band products), distances+"
                                 f"predecessors, n={n}, generator graph GenParams(n, rho={args.rho}, alpha=100, "
                                 f"seed=7+n), int32 in/out", "alg": "rkleene", "base_threshold": 2048,
                     "fused_exchange": fused} if rk else
                    {"block": block, "rows_per_rank": R, "fused_exchange": fused}),
                "clocks": clk.summary(), "gpu_launches": launches, "e2e": e2e, "cpu_baseline": cpu,
                "roofline": roofline, "tier": res.info["tier"]}
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    dist.barrier()
    dist.destroy_process_group()
