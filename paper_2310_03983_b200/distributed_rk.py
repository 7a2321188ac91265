"""Multi-GPU R-Kleene: replicated matrix, every block product split by output row bands.

SURVEY.md 8(e): "R-Kleene shards each of the 6 block products by output row bands, with operand
broadcast.  The recursion leaves and the closure chain stay serialized."  Here every rank holds
the whole padded N x N store matrix and predecessor matrix (N = 128-multiple; one u8 matrix at
n = 32768 is 1 GiB, pred 4 GiB -- small against 180 GB of HBM), so operands never move:

  close(lo, hi)                              (solvers.py:239-286, 128-aligned split)
    leaf           every rank, redundantly  (apsp_rk_shard_leaf; latency-bound, on the chain)
    each product   rank r computes its band of output rows (apsp_rk_shard_product), then the
                   bands are all-gathered (values + pred, NCCL over NVLink/NVSwitch)

A product's output rows are independent (C[i][j] depends on A row i, B column j and C[i][j]),
so each band equals the same rows of the one-GPU product and every replica stays bit-identical
to the single-GPU aligned R-Kleene (``solve(h, "rkleene", track="pred", split="aligned")``).

Work per rank is (products / P) + leaves; exchange per product is its output block once
(m * n * (store bytes + 4)), e.g. 16384^2 * 5 B = 1.3 GiB for a top-level product at n = 32768
against ~18 ms of 8-GPU compute.

Fused exchange (``fused=True``, bulk-staged tiers u8/u16/w32): instead of all-gathering the bands
after a product, the product kernel's epilogue stores every improved segment into every peer's
replica as well (peer memory mapped with CUDA IPC, NVLink/NVSwitch stores), so the exchange
overlaps the remaining tiles and the host only adds a 4-byte all-reduce as the per-product
barrier.  Emulated ranks on one GPU exercise the same kernel path with in-process replicas.

The schedule is written once over per-rank ``ops`` and a comm with ``gather_bands``:
* ``CudaRkOps`` + ``TorchComm``            -- the product path (torchrun, one process per GPU);
* ``CudaRkOps`` + ``EmulatedComm``         -- all ranks in one process on one GPU (tests);
* CPU ops in tests/ + ``TorchComm`` (gloo)  -- the world_size-2 CPU tests.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

from . import _native as nat
from .core import CostRangeError, ParameterError
from .distributed import (
    TIER_LIMIT,
    EmulatedComm,
    RankState,
    ShardedResult,
    TorchComm,
    _dtype_of,
    _TORCH_STORE,
    merged_scan,
    pick_tiers,
    resolve_tier,
    round_up,
)

TILE = 128


def rk_split(m: int) -> int:
    """Size of the first half of an m-block (rkleene.cu RK::split, aligned): ceil(tiles / 2) tiles."""
    return ((m // TILE + 1) // 2) * TILE


def row_bands(m: int, world: int) -> list[tuple[int, int]]:
    """Tile-aligned split of m output rows over the ranks: [(lo, hi)] per rank."""
    tiles = m // TILE
    per = -(-tiles // world)
    return [(min(m, r * per * TILE), min(m, (r + 1) * per * TILE)) for r in range(world)]


def run_rkleene(ranks: list[RankState], world: int, N: int, thr: int, ops, comm) -> None:
    """The recursion of rkleene.cu RK::close on every local rank's replica.

    Operand specs: ("D", i, j) the matrix, ("S", 0, 0) the value snapshot, ("P", i, j) the pred
    matrix, ("SP", 0, 0) the pred snapshot (the aliasing rules of solvers.py:250-286)."""

    fused = bool(getattr(ops, "fused_for", lambda st: False)(ranks[0].state))

    def product(A, B, r0, c0, m, n, k, PB, inner_off):
        bands = row_bands(m, world)
        for rk in ranks:
            lo, hi = bands[rk.rank]
            if hi > lo:
                ops.product(rk.state, A, B, r0, c0, lo, hi, n, k, PB, inner_off)
        if fused:
            comm.product_barrier(ranks, ops)      # bands already stored into every replica
        else:
            comm.gather_bands(ranks, ops, r0, c0, n, bands)

    def snap(i, j, rows, cols, idx):
        for rk in ranks:
            ops.snap(rk.state, i, j, rows, cols, idx)
        if fused:   # the snapshot's source is the next product's output: no peer may store into
            comm.product_barrier(ranks, ops)      # it before every rank has taken its copy

    def close(lo, hi):
        m = hi - lo
        if m <= thr or m <= TILE:
            for rk in ranks:
                ops.leaf(rk.state, lo, m)
            return
        mid = lo + rk_split(m)
        a, d = mid - lo, hi - mid
        close(lo, mid)
        snap(lo, mid, a, d, True)                                               # B <- A (x) B
        product(("D", lo, lo), ("S", 0, 0), lo, mid, a, d, a, ("SP", 0, 0), lo)
        snap(mid, lo, d, a, False)                                              # C <- C (x) A
        product(("S", 0, 0), ("D", lo, lo), mid, lo, d, a, a, ("P", lo, lo), lo)
        product(("D", mid, lo), ("D", lo, mid), mid, mid, d, d, a, ("P", lo, mid), lo)   # D <- min(D, C B)
        close(mid, hi)
        snap(lo, mid, a, d, False)                                              # B <- B (x) D
        product(("S", 0, 0), ("D", mid, mid), lo, mid, a, d, d, ("P", mid, mid), mid)
        snap(mid, lo, d, a, True)                                               # C <- D (x) C
        product(("D", mid, mid), ("S", 0, 0), mid, lo, d, a, d, ("SP", 0, 0), mid)
        product(("D", lo, mid), ("D", mid, lo), lo, lo, a, a, d, ("P", mid, lo), mid)    # A <- min(A, B C)

    close(0, N)


def run_rk_schedule(ranks, world, n, thr, ops, comm, dtype_code, h_fulls, tier_req=None, allreduce_max=None):
    """Tier loop around run_rkleene (every rank holds the full input); returns (tier, max finite)."""
    N = round_up(max(n, 1), TILE)
    for rk in ranks:
        rk.row0, rk.rows_valid = 0, n
    scan = merged_scan(ranks[:1], ops, h_fulls[:1], n, None)   # every rank holds the same input
    forced = resolve_tier(tier_req, dtype_code, scan)
    tiers = [forced] if forced is not None else pick_tiers(dtype_code, scan, n)
    for tier in tiers:
        for rk, h in zip(ranks, h_fulls):
            rk.state = ops.alloc(tier, N, thr)
            ops.prepare(rk.state, h, n, dtype_code)
        if getattr(ops, "fused_for", lambda st: False)(ranks[0].state):
            if comm.connect_replicas(ranks, ops):
                comm.product_barrier(ranks, ops)  # every replica prepared before any peer store
            else:
                ops.fused = False                 # no peer access between some GPUs: all-gather
        run_rkleene(ranks, world, N, thr, ops, comm)
        gmax = ops.max_finite(ranks[0].state, n)
        if allreduce_max is not None:
            gmax = allreduce_max(gmax)
        if tier == nat.TIER_F32 or gmax < 0 or gmax + scan["max_finite"] <= TIER_LIMIT[tier]:
            return tier, gmax
    if dtype_code == nat.DTYPE_I32:
        raise CostRangeError("shortest-path cost left the representable int32 range")
    raise CostRangeError("no value tier could represent the result")


# ---- CUDA ops ---------------------------------------------------------------------------------

@dataclass
class CudaRk:
    tier: int
    N: int
    thr: int
    es: int
    D: object
    P: object
    S: object
    SP: object
    scratch: object
    peer_dc: object = None      # ctypes int64 arrays: byte deltas to the peer replicas (fused)
    peer_di: object = None
    npeers: int = 0
    peer_views: list = field(default_factory=list)   # keeps IPC mappings alive


class CudaRkOps:
    """One replica per rank and the C-ABI R-Kleene shard calls, on torch's current stream."""

    def __init__(self, device, fused: bool = False):
        import torch

        self.torch = torch
        self.device = torch.device(device)
        self.lib = nat.load()
        self.fused = fused

    def fused_for(self, st) -> bool:
        """Fused peer stores are available for the bulk-staged tiers."""
        return self.fused and st.tier in (nat.TIER_U8, nat.TIER_U16, nat.TIER_W32)

    def set_peers(self, st: CudaRk, peer_D: list, peer_P: list, keep=()) -> None:
        """Peer replicas (tensors aliasing peer memory, same layout): byte deltas for the epilogue."""
        n = len(peer_D)
        if n > 7:
            raise ParameterError("fused exchange supports at most 8 ranks")
        st.npeers = n
        st.peer_dc = (ctypes.c_int64 * max(n, 1))(*[d.data_ptr() - st.D.data_ptr() for d in peer_D])
        st.peer_di = (ctypes.c_int64 * max(n, 1))(*[p.data_ptr() - st.P.data_ptr() for p in peer_P])
        st.peer_views = list(keep)

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    def scan(self, h, row0, rows_valid, n):
        from .distributed import CudaShardOps

        return CudaShardOps.scan(self, h, row0, rows_valid, n)

    def alloc(self, tier: int, N: int, thr: int) -> CudaRk:
        t = self.torch
        dt = getattr(t, _TORCH_STORE[tier])
        h = rk_split(N) if N > TILE else N
        sb = self.lib.apsp_rk_shard_scratch_bytes(N, thr)
        D = t.empty((N, N), dtype=dt, device=self.device)
        return CudaRk(tier, N, thr, D.element_size(), D, t.empty((N, N), dtype=t.int32, device=self.device),
                      t.empty((h, h), dtype=dt, device=self.device), t.empty((h, h), dtype=t.int32, device=self.device),
                      t.empty(sb, dtype=t.uint8, device=self.device))

    def prepare(self, st: CudaRk, h, n: int, dtype_code: int) -> None:
        nat.check(self.lib.apsp_shard_prepare(dtype_code, st.tier, n, st.N, 0, st.N, h.data_ptr(), n,
                                              st.D.data_ptr(), st.N, st.P.data_ptr(), st.N, self._stream()))

    def snap(self, st: CudaRk, i: int, j: int, rows: int, cols: int, idx: bool) -> None:
        st.S[:rows, :cols].copy_(st.D[i:i + rows, j:j + cols])
        if idx:
            st.SP[:rows, :cols].copy_(st.P[i:i + rows, j:j + cols])

    def _ptr(self, st: CudaRk, spec, row_off: int = 0):
        name, i, j = spec
        if name == "D":
            return st.D.data_ptr() + ((i + row_off) * st.N + j) * st.es, st.N
        if name == "S":
            ld = st.S.shape[1]
            return st.S.data_ptr() + ((i + row_off) * ld + j) * st.es, ld
        if name == "P":
            return st.P.data_ptr() + ((i + row_off) * st.N + j) * 4, st.N
        ld = st.SP.shape[1]
        return st.SP.data_ptr() + ((i + row_off) * ld + j) * 4, ld

    def product(self, st: CudaRk, A, B, r0, c0, lo, hi, n, k, PB, inner_off) -> None:
        a, lda = self._ptr(st, A, lo)
        b, ldb = self._ptr(st, B)
        pb, ldpb = self._ptr(st, PB)
        c = st.D.data_ptr() + ((r0 + lo) * st.N + c0) * st.es
        p = st.P.data_ptr() + ((r0 + lo) * st.N + c0) * 4
        if self.fused_for(st) and st.peer_dc is not None:
            nat.check(self.lib.apsp_rk_shard_product_fused(
                st.tier, a, lda, b, ldb, c, st.N, p, st.N, pb, ldpb, hi - lo, n, k, inner_off, st.N, st.thr,
                st.npeers, st.peer_dc, st.peer_di, st.scratch.data_ptr(), st.scratch.numel(), self._stream()))
            return
        nat.check(self.lib.apsp_rk_shard_product(st.tier, a, lda, b, ldb, c, st.N, p, st.N, pb, ldpb, hi - lo, n, k,
                                                 inner_off, st.N, st.thr, st.scratch.data_ptr(), st.scratch.numel(),
                                                 self._stream()))

    def leaf(self, st: CudaRk, lo: int, m: int) -> None:
        nat.check(self.lib.apsp_rk_shard_leaf(st.tier, st.D.data_ptr(), st.N, st.P.data_ptr(), st.N, lo, m, st.thr,
                                              st.scratch.data_ptr(), st.scratch.numel(), self._stream()))

    def band(self, st: CudaRk, r0: int, c0: int, rows: int, n: int):
        """Views of output rows [r0, r0 + rows) x [c0, c0 + n): (values, pred)."""
        return st.D[r0:r0 + rows, c0:c0 + n], st.P[r0:r0 + rows, c0:c0 + n]

    def max_finite(self, st: CudaRk, n: int) -> int:
        mx = ctypes.c_int64(-1)
        nat.check(self.lib.apsp_shard_finish(st.tier, nat.DTYPE_I32, n, n, st.D.data_ptr(), st.N, None, st.N, None, n,
                                             None, n, ctypes.byref(mx), self._stream()))
        return int(mx.value)

    def finish(self, st: CudaRk, n: int, dtype_code: int, dist, pred) -> None:
        mx = ctypes.c_int64(-1)
        nat.check(self.lib.apsp_shard_finish(st.tier, dtype_code, n, n, st.D.data_ptr(), st.N, st.P.data_ptr(), st.N,
                                             dist.data_ptr(), n, pred.data_ptr(), n, ctypes.byref(mx),
                                             self._stream()))


# ---- band exchange ----------------------------------------------------------------------------

def _torch_gather_bands(self: TorchComm, ranks, ops, r0, c0, n, bands):
    """All-gather of the product's output bands (values, then pred) from every rank."""
    if self.world == 1:
        return
    torch, dist = self.torch, self.dist
    (rk,) = ranks
    rows = max(hi - lo for lo, hi in bands)
    if rows == 0:
        return
    lo, hi = bands[rk.rank]
    mine = ops.band(rk.state, r0 + lo, c0, hi - lo, n)
    for q in range(2):
        src = mine[q]
        send = torch.empty((rows, n), dtype=src.dtype, device=src.device)
        if hi > lo:
            send[:hi - lo].copy_(src)
        recv = torch.empty((self.world * rows, n), dtype=src.dtype, device=src.device)
        wire_s, wire_r = send, recv
        if src.dtype == torch.uint16:                       # NCCL has no uint16
            wire_s, wire_r = send.view(torch.int16), recv.view(torch.int16)
        if hasattr(dist, "all_gather_into_tensor") and src.device.type == "cuda":
            dist.all_gather_into_tensor(wire_r, wire_s, group=self.group)
        else:
            dist.all_gather(list(wire_r.chunk(self.world)), wire_s, group=self.group)
        for r, (l2, h2) in enumerate(bands):
            if r != rk.rank and h2 > l2:
                ops.band(rk.state, r0 + l2, c0, h2 - l2, n)[q].copy_(recv[r * rows:r * rows + h2 - l2])


def _emulated_gather_bands(self: EmulatedComm, ranks, ops, r0, c0, n, bands):
    """All ranks in this process: copy each owner's band into every other replica."""
    for rk in ranks:
        lo, hi = bands[rk.rank]
        if hi <= lo:
            continue
        src = ops.band(rk.state, r0 + lo, c0, hi - lo, n)
        for other in ranks:
            if other is not rk:
                dst = ops.band(other.state, r0 + lo, c0, hi - lo, n)
                dst[0].copy_(src[0])
                dst[1].copy_(src[1])


def _torch_connect_replicas(self: TorchComm, ranks, ops):
    """Map every peer's replica into this process (CUDA IPC handles exchanged over the process
    group) and hand the byte deltas to the ops; world 1 has no peers."""
    (rk,) = ranks
    st = rk.state
    if self.world == 1:
        ops.set_peers(st, [], [])
        return True
    if not self.peers_reachable():
        return False
    from torch.multiprocessing.reductions import reduce_tensor

    mine = (reduce_tensor(st.D), reduce_tensor(st.P))
    every = [None] * self.world
    self.dist.all_gather_object(every, mine, group=self.group)
    peer_D, peer_P = [], []
    for r, ((fd, ad), (fp, ap_)) in enumerate(every):
        if r != rk.rank:
            peer_D.append(fd(*ad))
            peer_P.append(fp(*ap_))
    ops.set_peers(st, peer_D, peer_P, keep=peer_D + peer_P)
    return True


def _torch_product_barrier(self: TorchComm, ranks, ops):
    """Every rank's fused product has landed in every replica: a 4-byte all-reduce on the
    compute stream orders the next product after all peers' stores."""
    if self.world == 1:
        return
    t = self.torch.zeros(1, dtype=self.torch.int32, device=self.device)
    self.dist.all_reduce(t, group=self.group)


def _emulated_connect_replicas(self: EmulatedComm, ranks, ops):
    for rk in ranks:
        others = [o.state for o in ranks if o is not rk]
        ops.set_peers(rk.state, [o.D for o in others], [o.P for o in others])
    return True


def _emulated_product_barrier(self: EmulatedComm, ranks, ops):
    return None   # one stream, one process: stream order is the barrier


TorchComm.gather_bands = _torch_gather_bands
EmulatedComm.gather_bands = _emulated_gather_bands
TorchComm.connect_replicas = _torch_connect_replicas
EmulatedComm.connect_replicas = _emulated_connect_replicas
TorchComm.product_barrier = _torch_product_barrier
EmulatedComm.product_barrier = _emulated_product_barrier


# ---- public entry points ------------------------------------------------------------------------

def rkleene_sharded(h, n: int, *, comm: TorchComm, base_threshold: int = 1024, tier=None, ops=None,
                    fused: bool = True):
    """SPMD entry: every rank passes the full input (torch CUDA tensor, n x n, int32 or fp32)
    and receives the full (dist, pred) -- bit-identical to the one-GPU aligned R-Kleene."""
    import torch

    if tuple(h.shape) != (n, n):
        raise ParameterError(f"rank {comm.rank} expects the full {n} x {n} input, got {tuple(h.shape)}")
    if base_threshold < 1:
        raise ParameterError(f"base_threshold must be >= 1, got {base_threshold}")
    ops = ops or CudaRkOps(h.device, fused=fused)
    rs = RankState(comm.rank, 0, n)
    dtype_code = _dtype_of(h)
    t0 = time.perf_counter()
    tier, gmax = run_rk_schedule([rs], comm.world, n, base_threshold, ops, comm, dtype_code, [h],
                                 tier, comm.allreduce_max)
    dist = torch.empty((n, n), dtype=h.dtype, device=h.device)
    pred = torch.empty((n, n), dtype=torch.int32, device=h.device)
    ops.finish(rs.state, n, dtype_code, dist, pred)
    return ShardedResult(dist, pred, 0, n, {"tier": nat.TIER_NAMES[tier], "max_finite": gmax, "world": comm.world,
                                            "N": rs.state.N, "base_threshold": base_threshold,
                                            "host_s": time.perf_counter() - t0})


def rkleene_emulated(h, world: int, *, base_threshold: int = 1024, tier=None, fused: bool = False):
    """All ``world`` ranks in this process on h's device (one replica each; sequential, no rank
    waits on another).  Returns (dist, pred, info) of rank 0's replica."""
    import torch

    n = h.shape[0]
    ops = CudaRkOps(h.device, fused=fused)
    ranks = [RankState(r, 0, n) for r in range(world)]
    tier_code, gmax = run_rk_schedule(ranks, world, n, base_threshold, ops, EmulatedComm(), _dtype_of(h),
                                      [h] * world, tier, None)
    dist = torch.empty_like(h)
    pred = torch.empty((n, n), dtype=torch.int32, device=h.device)
    ops.finish(ranks[0].state, n, _dtype_of(h), dist, pred)
    replicas_equal = all(torch.equal(ranks[0].state.D, rk.state.D) and torch.equal(ranks[0].state.P, rk.state.P)
                         for rk in ranks[1:])
    return dist, pred, {"tier": nat.TIER_NAMES[tier_code], "max_finite": gmax, "replicas_equal": replicas_equal,
                        "fused": ops.fused_for(ranks[0].state)}
