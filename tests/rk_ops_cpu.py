"""CPU stand-in for CudaRkOps (TEST INFRASTRUCTURE): the replicated R-Kleene shard ops in exact
int64 numpy, so the multi-rank schedule of paper_2310_03983_b200.distributed_rk runs over gloo
with world_size 2 on a machine without GPUs."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
from shard_ops_cpu import INF_RAW, CpuShardOps


@dataclass
class CpuRk:
    tier: int
    N: int
    D: torch.Tensor
    P: torch.Tensor
    S: torch.Tensor
    SP: torch.Tensor


class CpuRkOps:
    scan = CpuShardOps.scan

    def alloc(self, tier, N, thr):
        h = ((N // 128 + 1) // 2) * 128 if N > 128 else N
        return CpuRk(tier, N, torch.full((N, N), INF_RAW, dtype=torch.int64), torch.full((N, N), -1, dtype=torch.int32),
                     torch.empty((h, h), dtype=torch.int64), torch.empty((h, h), dtype=torch.int32))

    def prepare(self, st, h, n, dtype_code):
        D, P = st.D.numpy(), st.P.numpy()
        D[:n, :n] = h.numpy()
        fin = D[:n, :n] != INF_RAW
        P[:n, :n] = np.where(fin, np.arange(n)[:, None], -1)
        for i in range(st.N):
            D[i, i] = 0
            P[i, i] = -1

    def snap(self, st, i, j, rows, cols, idx):
        st.S[:rows, :cols].copy_(st.D[i:i + rows, j:j + cols])
        if idx:
            st.SP[:rows, :cols].copy_(st.P[i:i + rows, j:j + cols])

    def _arr(self, st, spec, rows, cols, row_off=0):
        name, i, j = spec
        t = {"D": st.D, "S": st.S, "P": st.P, "SP": st.SP}[name]
        return t.numpy()[i + row_off:i + row_off + rows, j:j + cols]

    def product(self, st, A, B, r0, c0, lo, hi, n, k, PB, inner_off):
        a = self._arr(st, A, hi - lo, k, lo).copy()
        b = self._arr(st, B, k, n).copy()
        pb = self._arr(st, PB, k, n).copy()
        C = st.D.numpy()[r0 + lo:r0 + hi, c0:c0 + n]
        PC = st.P.numpy()[r0 + lo:r0 + hi, c0:c0 + n]
        CpuShardOps._product(C, PC, a, b, pb)

    def leaf(self, st, lo, m):
        G = st.D.numpy()[lo:lo + m, lo:lo + m]
        PG = st.P.numpy()[lo:lo + m, lo:lo + m]
        for k in range(m):                                   # classic closure (FW rule)
            c = G[:, k:k + 1] + G[k:k + 1, :]
            imp = c < G
            G[imp] = c[imp]
            PG[imp] = np.broadcast_to(PG[k:k + 1, :], G.shape)[imp]

    def band(self, st, r0, c0, rows, n):
        return st.D[r0:r0 + rows, c0:c0 + n], st.P[r0:r0 + rows, c0:c0 + n]

    def max_finite(self, st, n):
        a = st.D.numpy()[:n, :n]
        fin = a != INF_RAW
        return int(a[fin].max()) if fin.any() else -1
