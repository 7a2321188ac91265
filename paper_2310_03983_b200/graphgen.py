"""Seeded random digraph generator G = f(v, rho, alpha, seed) (reference: graphgen.py).

``generate`` keeps the reference contract bit-for-bit: a numpy ``Generator(Philox(seed))``
consumed as three row-major v x v blocks -- probability uniforms, presence uniforms, weights
(graphgen.py:60-71) -- with edge (i, j) present iff ``presence < clip(rho * prob, 0, 1)``.

``dense_costs`` is the B200-side producer: it builds the dense cost matrix directly (int64,
int32 or fp32) in row chunks without a Python edge list.  Each block is drawn from its own
Philox stream advanced to the block's counter offset, and the weight block re-implements
numpy's buffered 32-bit Lemire draw (bounded_integers: buffered_bounded_lemire_uint32) so
the chunked result equals ``cost_matrix_from_graph(generate(p))`` exactly, rejections included.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import INF32, INF_RAW, Graph, ParameterError


@dataclass(frozen=True)
class GenParams:
    """Generator parameters; rho already normalised to [0, 1] (graphgen.py:26-43)."""

    v: int
    rho: float
    alpha: int
    seed: int

    def __post_init__(self):
        if not isinstance(self.v, int) or self.v < 1:
            raise ParameterError(f"v must be an integer >= 1, got {self.v!r}")
        if not 0.0 <= self.rho <= 1.0:
            raise ParameterError(f"rho must lie in [0,1] after normalization, got {self.rho!r}")
        if not isinstance(self.alpha, int) or self.alpha < 1:
            raise ParameterError(f"alpha must be an integer >= 1, got {self.alpha!r}")
        if not isinstance(self.seed, int) or not 0 <= self.seed < 2**64:
            raise ParameterError(f"seed must be a 64-bit unsigned integer, got {self.seed!r}")


def normalize_rho(value: float) -> float:
    """[0,1] passes through, (1,100] is read as percent, anything else is rejected."""
    v = float(value)
    if not 0.0 <= v <= 100.0:
        raise ParameterError(f"rho must lie in [0,1] or (1,100] percent, got {value!r}")
    return v if v <= 1.0 else v / 100.0


def generate(params: GenParams) -> Graph:
    """Edge-list graph; identical draws and edge order to the reference generator."""
    mask, weights = _monolithic_draws(params)
    rows, cols = np.nonzero(mask)
    w = weights[rows, cols]
    return Graph(params.v, zip(rows.tolist(), cols.tolist(), w.tolist()))


def density(g: Graph) -> float:
    """Directed density m / (n (n - 1))."""
    g.validate()
    return 0.0 if g.n < 2 else g.n_edges / (g.n * (g.n - 1))


def _monolithic_draws(p: GenParams):
    rng = np.random.Generator(np.random.Philox(p.seed))
    prob = rng.random((p.v, p.v))
    pres = rng.random((p.v, p.v))
    weights = rng.integers(1, p.alpha, size=(p.v, p.v), endpoint=True)
    mask = pres < np.clip(p.rho * prob, 0.0, 1.0)
    np.fill_diagonal(mask, False)
    return mask, weights


def _stream_at(seed: int, n_uint64: int) -> np.random.Philox:
    """Philox positioned after n_uint64 outputs (4 outputs per counter step)."""
    bg = np.random.Philox(seed)
    bg.advance(n_uint64 // 4)
    rest = n_uint64 % 4
    if rest:
        bg.random_raw(rest)
    return bg


class _LemireStream:
    """numpy's buffered bounded Lemire draw of integers in [0, rng], rng < 2**32 - 1.

    One uint64 feeds two uint32 draws (low half first); a draw whose low product word falls
    below (2**32 - 1 - rng) % (rng + 1) is rejected and redrawn.  The buffer lives for the
    whole block, exactly like the single ``integers`` call of the reference.
    """

    def __init__(self, bg: np.random.Philox, rng: int):
        self.bg = bg
        self.excl = np.uint64(rng + 1)
        self.threshold = (0xFFFFFFFF - rng) % (rng + 1)
        self.pending = np.empty(0, dtype=np.uint32)

    def take(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.int64)
        filled = 0
        while filled < count:
            need = count - filled
            if self.pending.size < need:
                raw = self.bg.random_raw((need - self.pending.size + 1) // 2 + 16)
                halves = np.empty(raw.size * 2, dtype=np.uint32)
                halves[0::2] = (raw & np.uint64(0xFFFFFFFF)).astype(np.uint32)
                halves[1::2] = (raw >> np.uint64(32)).astype(np.uint32)
                self.pending = np.concatenate([self.pending, halves])
            m = self.pending.astype(np.uint64) * self.excl
            leftover = m & np.uint64(0xFFFFFFFF)
            ok = leftover >= np.uint64(self.threshold)
            idx = np.flatnonzero(ok)
            use = idx[:need]
            out[filled:filled + use.size] = (m[use] >> np.uint64(32)).astype(np.int64)
            filled += use.size
            consumed = int(use[-1]) + 1 if use.size else self.pending.size
            self.pending = self.pending[consumed:]
        return out


def dense_costs(params: GenParams, dtype=np.int64, chunk_rows: int = 512,
                rows: tuple[int, int] | None = None) -> np.ndarray:
    """Dense cost matrix of ``generate(params)`` (zero diagonal, Infinity elsewhere).

    dtype int64 -> INF_RAW, int32 -> INF32, float32 -> +inf.  Equal to
    ``cost_matrix_from_graph(generate(params)).raw`` after sentinel mapping.  ``rows=(r0, r1)``
    returns only those rows (a rank's row band): the uniform streams jump straight to row r0;
    the weight stream is replayed up to r0 to count Lemire rejections exactly.
    """
    v, seed = params.v, params.seed
    r_lo, r_hi = (0, v) if rows is None else (max(0, rows[0]), min(v, rows[1]))
    dtype = np.dtype(dtype)
    if dtype == np.int64:
        inf = INF_RAW
    elif dtype == np.int32:
        inf = INF32
        if params.alpha >= INF32:
            raise ParameterError("alpha does not fit the int32 domain")
    elif dtype == np.float32:
        inf = np.inf
    else:
        raise ParameterError(f"unsupported dtype {dtype}")
    out = np.empty((max(0, r_hi - r_lo), v), dtype=dtype)
    if r_hi <= r_lo:
        return out
    g_prob = np.random.Generator(_stream_at(seed, r_lo * v))
    g_pres = np.random.Generator(_stream_at(seed, v * v + r_lo * v))
    rng = params.alpha - 1
    lemire = None
    if 0 < rng < 0xFFFFFFFF:
        lemire = _LemireStream(_stream_at(seed, 2 * v * v), rng)
        done = 0
        while done < r_lo * v:                     # replay (rejections shift the stream)
            step = min(r_lo * v - done, chunk_rows * v)
            lemire.take(step)
            done += step
    elif rng != 0:
        mask, weights = _monolithic_draws(params)   # 64-bit weight path: rare, do it whole
        full = np.where(mask, weights, inf).astype(dtype)
        np.fill_diagonal(full, 0)
        return full[r_lo:r_hi].copy()
    for r0 in range(r_lo, r_hi, chunk_rows):
        r1 = min(r_hi, r0 + chunk_rows)
        prob = g_prob.random((r1 - r0, v))
        pres = g_pres.random((r1 - r0, v))
        w = (lemire.take((r1 - r0) * v).reshape(r1 - r0, v) + 1) if lemire else np.ones((r1 - r0, v), np.int64)
        mask = pres < np.clip(params.rho * prob, 0.0, 1.0)
        block = out[r0 - r_lo:r1 - r_lo]
        block[...] = inf
        block[mask] = w[mask].astype(dtype)
        idx = np.arange(r0, r1)
        block[idx - r0, idx] = 0
    return out


def continuous_costs(params: GenParams) -> np.ndarray:
    """BASELINE config 2's continuous variant: the edge mask of
    ``generate(params)`` with float32 weights drawn U[1, 100) from ``default_rng(params.seed)``
    in row-major edge order; zero diagonal, +inf for non-edges."""
    h = dense_costs(params, np.float32)
    fin = np.isfinite(h)
    np.fill_diagonal(fin, False)
    rng = np.random.default_rng(params.seed)
    h[fin] = rng.uniform(1.0, 100.0, size=int(fin.sum())).astype(np.float32)
    return h
