"""Shortest-path reconstruction from pred / via matrices (reference: paths.py), plus the
whole-matrix predecessor certificate used to validate blocked-FW and R-Kleene pred.

``path_from_pred`` / ``path_from_via`` follow the reference semantics exactly (paths.py:34-105):
None for unreachable targets, ``CorruptPredError`` / ``CorruptViaError`` on inconsistency.

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
    """Backtrack target <- pred[source][target] until the source (paths.py:34-63)."""
    n = distances.n
    if pred.shape != distances.shape:
        raise DimensionError(f"pred shape {pred.shape} != distances shape {distances.shape}")
    _check_pair(n, source, target)
    if source == target:
        return Path((source,), 0)
    if distances[source, target].is_infinite:
        return None
    walk = [target]
    cur = target
    while cur != source:
        if len(walk) > n:
            raise CorruptPredError(f"backtracking from {target} exceeded {n} steps")
        prev = pred[source, cur]
        if prev is None:
            raise CorruptPredError(f"pred[{source}][{cur}] is None but distance to {target} is finite")
        walk.append(prev)
        cur = prev
    walk.reverse()
    return Path(walk, distances[source, target].value)


def path_from_via(via: ViaMatrix, distances: CostMatrix, graph: Graph, source: int, target: int) -> Path | None:
    """Expand (source, target) through via midpoints down to direct edges (paths.py:66-105)."""
    n = distances.n
    if via.shape != distances.shape:
        raise DimensionError(f"via shape {via.shape} != distances shape {distances.shape}")
    _check_pair(n, source, target)
    if source == target:
        return Path((source,), 0)
    if distances[source, target].is_infinite:
        return None
    weight = {(u, v): w for u, v, w in graph.edges}
    out = [source]
    total = 0
    todo = [(source, target, 0)]
    while todo:
        i, j, depth = todo.pop()
        if depth > n:
            raise CorruptViaError(f"via expansion of ({source},{target}) nested deeper than n={n}")
        k = via[i, j]
        if k is None:
            w = weight.get((i, j))
            if w is None:
                raise CorruptViaError(f"via[{i}][{j}] is None but the graph has no direct edge ({i},{j})")
            out.append(j)
            total += w
        else:
            todo.append((k, j, depth + 1))
            todo.append((i, k, depth + 1))
    return Path(out, total)


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
