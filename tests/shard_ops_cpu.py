"""CPU stand-in for CudaShardOps (TEST INFRASTRUCTURE): the same pivot / update semantics in
exact int64 numpy, so the multi-rank schedule of paper_2310_03983_b200.distributed can be run
over gloo with world_size 2 on a machine without GPUs."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

INF_RAW = 1 << 61


@dataclass
class CpuShard:
    tier: int
    R: int
    N: int
    D: torch.Tensor
    P: torch.Tensor
    pv: list
    pp: list


class CpuShardOps:
    def __init__(self, block: int):
        self.block = block

    def scan(self, h, row0, rows_valid, n):
        a = h.numpy() if rows_valid else np.zeros((0, n), np.int64)
        fin = a != INF_RAW
        diag = np.zeros_like(fin)
        for i in range(rows_valid):
            diag[i, row0 + i] = True
        return {"negative": int((a[fin] < 0).any()), "diag_nonzero": int((a[diag] != 0).any()),
                "non_integral": 0, "zero_offdiag": int(((a == 0) & fin & ~diag).any()),
                "max_finite": int(a[fin].max()) if fin.any() else -1, "finite_offdiag": int((fin & ~diag).sum())}

    def alloc(self, tier, R, N):
        b = self.block
        return CpuShard(tier, R, N, torch.full((R, N), INF_RAW, dtype=torch.int64),
                        torch.full((R, N), -1, dtype=torch.int32),
                        [torch.empty((b, N), dtype=torch.int64) for _ in range(2)],
                        [torch.empty((b, N), dtype=torch.int32) for _ in range(2)])

    def prepare(self, st, h, n, row0, dtype_code):
        D, P = st.D.numpy(), st.P.numpy()
        rv = h.shape[0] if h is not None else 0
        if rv:
            D[:rv, :n] = h.numpy()
            fin = D[:rv, :n] != INF_RAW
            P[:rv, :n] = np.where(fin, (row0 + np.arange(rv))[:, None], -1)
        for il in range(st.R):
            i = row0 + il
            if i < st.N:
                D[il, i] = 0
                P[il, i] = -1

    @staticmethod
    def _product(C, PC, A, B, PB, skip_rows=None, skip_cols=None):
        """C <- min(C, A (x) B) with smallest-k strict-improvement argmin; PC <- PB[k*][j]."""
        cand = A[:, :, None] + B[None, :, :]
        best = cand.min(axis=1)
        arg = cand.argmin(axis=1)
        imp = best < C
        if skip_rows is not None:
            imp[skip_rows[0]:skip_rows[1], :] = False
        if skip_cols is not None:
            imp[:, skip_cols[0]:skip_cols[1]] = False
        cols = np.broadcast_to(np.arange(C.shape[1]), C.shape)
        newp = PB[arg, cols]
        C[imp] = best[imp]
        PC[imp] = newp[imp]

    def pivot(self, st, lrow, k0, side=False, slot=None):
        b = self.block
        D, P = st.D.numpy(), st.P.numpy()
        G = D[lrow:lrow + b, k0:k0 + b]
        PG = P[lrow:lrow + b, k0:k0 + b]
        for k in range(b):                                   # classic closure (FW rule)
            c = G[:, k:k + 1] + G[k:k + 1, :]
            imp = c < G
            G[imp] = c[imp]
            PG[imp] = np.broadcast_to(PG[k:k + 1, :], G.shape)[imp]
        T = D[lrow:lrow + b]
        snap = P[lrow:lrow + b].copy()
        self._product(T, P[lrow:lrow + b], G.copy(), T.copy(), snap, skip_cols=(k0, k0 + b))
        return st.D[lrow:lrow + b], st.P[lrow:lrow + b], None

    def recv_buffers(self, st, slot):
        return st.pv[slot], st.pp[slot]

    def update(self, st, pv, pp, k0, row_lo, row_hi, skip_lo, skip_hi):
        b = self.block
        D, P = st.D.numpy()[row_lo:row_hi], st.P.numpy()[row_lo:row_hi]
        pvn, ppn = pv.numpy(), pp.numpy()
        skip = (skip_lo - row_lo, skip_hi - row_lo) if skip_lo >= 0 else None
        self._product(D[:, k0:k0 + b], P[:, k0:k0 + b], D[:, k0:k0 + b].copy(), pvn[:, k0:k0 + b],
                      ppn[:, k0:k0 + b], skip_rows=skip)
        self._product(D, P, D[:, k0:k0 + b].copy(), pvn, ppn, skip_rows=skip, skip_cols=(k0, k0 + b))

    def max_finite(self, st, rows_valid, n):
        a = st.D.numpy()[:rows_valid, :n]
        fin = a != INF_RAW
        return int(a[fin].max()) if fin.any() else -1

    def classic(self, h, n, dtype_code):
        """Zero-cost-edge fallback: classic-order FW of the gathered matrix (the oracle)."""
        from oracle import oracle as orc

        d, p = orc.fw_classic(h.numpy().astype(np.int64))
        return torch.from_numpy(d), torch.from_numpy(p.astype(np.int32))

    def set_pred_rows(self, st, p):
        if p is not None and p.numel():
            st.P[:p.shape[0], :p.shape[1]].copy_(p)
