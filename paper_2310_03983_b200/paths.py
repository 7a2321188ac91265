"""Shortest-path reconstruction from pred / via matrices (reference: paths.py), plus the
whole-matrix predecessor certificate used to validate blocked-FW and R-Kleene pred.

``path_from_pred`` / ``path_from_via`` keep the reference semantics (paths.py:34-105): None for
unreachable targets, ``CorruptPredError`` / ``CorruptViaError`` on inconsistency.

``check_pred_tree`` validates every (i, j) at once, the way SURVEY.md 8(c) defines pred
parity for non-classic orders: for each reachable pair, p = pred[i][j] is a vertex with an
input edge (p, j) and d[i][p] + w(p, j) == d[i][j]; walking pred from any j reaches i within
n - 1 hops (pointer doubling).  That is equivalent to reconstructing every path and
re-summing its length.  It runs on numpy or on CUDA torch tensors (test infrastructure).
"""

from __future__ import annotations

from .core import (
    CorruptPredError,
    CorruptViaError,
    CostMatrix,
    DimensionError,
    Graph,
    Path,
    PredMatrix,
    ViaMatrix,
)


def _check_pair(n: int, s: int, t: int) -> None:
    if not (0 <= s < n and 0 <= t < n):
        raise IndexError(f"vertex pair ({s},{t}) out of range for n={n}")


def path_from_pred(pred: PredMatrix, distances: CostMatrix, source: int, target: int) -> Path | None:
    """Vertex sequence source -> target read off row ``source`` of ``pred`` (reference
    semantics, paths.py:34-63): None if unreachable, CorruptPredError if the walk hits a None
    predecessor or has not reached the source after n hops."""
    n = distances.n
    if pred.shape != distances.shape:
        raise DimensionError(f"pred shape {pred.shape} != distances shape {distances.shape}")
    _check_pair(n, source, target)
    if source == target:
        return Path((source,), 0)
    if distances[source, target].is_infinite:
        return None
    parent = pred.raw[source].tolist()          # one row of the int64 matrix, -1 = None
    hops = [target]
    for _ in range(n):
        if hops[-1] == source:
            break
        up = parent[hops[-1]]
        if up < 0:
            raise CorruptPredError(f"pred[{source}][{hops[-1]}] is None but distance to {target} is finite")
        hops.append(up)
    else:
        if hops[-1] != source:
            raise CorruptPredError(f"backtracking from {target} exceeded {n} steps")
    return Path(hops[::-1], distances[source, target].value)


class _EdgeIndex:
    """Weight lookup over a graph's edge list: sorted u*n+v keys, binary search."""

    def __init__(self, graph: Graph):
        import numpy as np

        e = np.asarray(graph.edges, dtype=np.int64).reshape(-1, 3)
        key = e[:, 0] * graph.n + e[:, 1]
        order = np.argsort(key, kind="stable")
        self.n, self.key, self.w = graph.n, key[order], e[order, 2]

    def weight(self, u: int, v: int):
        import numpy as np

        q = u * self.n + v
        at = int(np.searchsorted(self.key, q))
        return int(self.w[at]) if at < len(self.key) and self.key[at] == q else None


def path_from_via(via: ViaMatrix, distances: CostMatrix, graph: Graph, source: int, target: int) -> Path | None:
    """Expand source -> target through via midpoints down to graph edges (reference semantics,
    paths.py:66-105): a None via cell must be a direct edge, and no segment may split more than
    n times deep (CorruptViaError).  The cost is the sum of the actual edge weights.

    The path is refined in place: ``seq`` holds the vertices found so far and ``depth[x]`` the
    split depth of the segment seq[x] -> seq[x+1]; the cursor advances only past direct edges.
    """
    n = distances.n
    if via.shape != distances.shape:
        raise DimensionError(f"via shape {via.shape} != distances shape {distances.shape}")
    _check_pair(n, source, target)
    if source == target:
        return Path((source,), 0)
    if distances[source, target].is_infinite:
        return None
    mid = via.raw
    edges = _EdgeIndex(graph)
    seq, depth = [source, target], [0]
    total, x = 0, 0
    while x < len(seq) - 1:
        i, j, d = seq[x], seq[x + 1], depth[x]
        if d > n:
            raise CorruptViaError(f"via expansion of ({source},{target}) nested deeper than n={n}")
        k = int(mid[i, j])
        if k < 0:
            w = edges.weight(i, j)
            if w is None:
                raise CorruptViaError(f"via[{i}][{j}] is None but the graph has no direct edge ({i},{j})")
            total += w
            x += 1
        else:
            seq.insert(x + 1, k)
            depth[x:x + 1] = [d + 1, d + 1]
    return Path(seq, total)


def check_pred_tree(h, dist, pred, inf) -> tuple[bool, str]:
    """Certificate that ``pred`` encodes shortest paths of ``dist`` over input ``h``.

    ``h``, ``dist``, ``pred`` are same-shape numpy arrays or torch tensors; ``inf`` is the
    Infinity sentinel of h/dist.  Returns (ok, reason).
    """
    try:
        import torch
    except Exception:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(dist, torch.Tensor):
        xp_where, xp_arange = torch.where, lambda n: torch.arange(n, device=dist.device)

        def take_rows(mat, cols):
            return torch.gather(mat, 1, cols)

        def anyf(x):
            return bool(x.any().item())
        to64 = (lambda t: t.to(torch.int64))
    else:
        import numpy as np

        xp_where, xp_arange = np.where, np.arange

        def take_rows(mat, cols):
            return np.take_along_axis(mat, cols, axis=1)

        def anyf(x):
            return bool(x.any())
        to64 = (lambda t: t.astype(np.int64))
    n = dist.shape[0]
    ar = xp_arange(n)
    fin = dist != inf
    offdiag = ar[:, None] != ar[None, :]
    need = fin & offdiag
    p = to64(pred)
    if anyf(need & ((p < 0) | (p >= n))):
        return False, "reachable pair without a valid predecessor"
    if anyf(~need & (p != -1)):
        return False, "predecessor set on a diagonal or unreachable pair"
    ps = xp_where(need, p, ar[:, None] + 0 * p)   # safe index where not needed
    d_ip = take_rows(to64(dist), ps)                                   # d[i][p]
    w_pj = to64(h)[ps, ar[None, :] + 0 * ps]                           # h[p][j]
    if anyf(need & (w_pj == inf)):
        return False, "predecessor hop is not an input edge"
    if anyf(need & (d_ip == inf)):
        return False, "predecessor unreachable from the source"
    if anyf(need & (d_ip + w_pj != to64(dist))):
        return False, "d[i][p] + w(p,j) != d[i][j]"
    # termination: pointer doubling of the parent map j -> pred[i][j] (root i -> i)
    anc = xp_where(need, p, ar[:, None] + 0 * p)
    steps = 1
    while steps < n:
        anc = take_rows(anc, anc)
        steps *= 2
    if anyf(need & (anc != ar[:, None])):
        return False, "pred walk does not reach the source (cycle)"
    return True, "ok"


def check_pred_paths(h, dist, pred, rtol: float = 1e-5) -> tuple[bool, str]:
    """Floating-point predecessor certificate: reconstruct every path of ``pred`` and re-sum it.

    For fp32 (continuous-weight) results, where d[i][p] + w(p, j) need not round to d[i][j]
    exactly: for every reachable pair the pred walk from j must reach i along input edges, and
    the float64 sum of its edge weights must equal d[i][j] within ``rtol`` (relative).  The
    walks are summed for all pairs at once by pointer doubling (the sum from a vertex's 2^t-th
    ancestor to it doubles with the hop count; the root i carries 0).  Unreachable = +inf.
    numpy arrays or CUDA torch tensors; returns (ok, reason).
    """
    try:
        import torch
    except Exception:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(dist, torch.Tensor):
        dev = dist.device
        f64 = (lambda t: t.to(torch.float64))
        i64 = (lambda t: t.to(torch.int64))
        where, isfin, absf = torch.where, torch.isfinite, torch.abs
        ar = torch.arange(dist.shape[0], device=dev)

        def take_rows(mat, cols):
            return torch.gather(mat, 1, cols)

        def anyf(x):
            return bool(x.any().item())
    else:
        import numpy as np

        f64 = (lambda t: np.asarray(t, dtype=np.float64))
        i64 = (lambda t: np.asarray(t, dtype=np.int64))
        where, isfin, absf = np.where, np.isfinite, np.abs
        ar = np.arange(dist.shape[0])

        def take_rows(mat, cols):
            return np.take_along_axis(mat, cols, axis=1)

        def anyf(x):
            return bool(x.any())
    n = dist.shape[0]
    d = f64(dist)
    need = isfin(d) & (ar[:, None] != ar[None, :])
    p = i64(pred)
    if anyf(need & ((p < 0) | (p >= n))):
        return False, "reachable pair without a valid predecessor"
    if anyf(~need & (p != -1)):
        return False, "predecessor set on a diagonal or unreachable pair"
    anc = where(need, p, ar[:, None] + 0 * p)
    w = f64(h)[anc, ar[None, :] + 0 * anc]                              # h[pred[i][j]][j]
    if anyf(need & ~isfin(w)):
        return False, "predecessor hop is not an input edge"
    acc = where(need, w, 0 * w)
    steps = 1
    while steps < n:
        acc = acc + take_rows(acc, anc)
        anc = take_rows(anc, anc)
        steps *= 2
    if anyf(need & (anc != ar[:, None])):
        return False, "pred walk does not reach the source (cycle)"
    err = where(need, absf(acc - d), 0 * d)
    bad = err > rtol * where(need, absf(d), 0 * d)
    if anyf(bad):
        return False, f"re-summed path length differs from d[i][j] beyond rtol={rtol}"
    return True, "ok"
