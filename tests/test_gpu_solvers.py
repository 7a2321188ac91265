"""GPU parity of the solvers against the reference (golden fixtures) and the CPU oracle.

Parity bar:
* distances: bit-exact for integer inputs;
* fw_classic(method="classic") pred and rkleene(split="floor") via: bit-exact;
* blocked-FW pred and R-Kleene pred: validated by the whole-matrix reconstruction
  certificate (paths.check_pred_tree);
* continuous fp32: within 1e-5 relative of a float64 Floyd-Warshall.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import INF_RAW, golden, random_graph_raw
from oracle import oracle as orc

import paper_2310_03983_b200 as ap
from paper_2310_03983_b200.core import INF32

pytestmark = pytest.mark.gpu


def pred_ok(h, dist, pred, inf=INF_RAW):
    ok, why = ap.check_pred_tree(h, dist, pred, inf)
    assert ok, why


# ---- Floyd-Warshall ------------------------------------------------------------------------

def test_c1_blocked_and_classic(cuda):
    g = golden("c1_fw.npz")
    h = ap.CostMatrix(g["h"])
    s = ap.fw_classic(h)                        # blocked (default)
    assert np.array_equal(s.distances.raw, g["dist"])
    pred_ok(g["h"], s.distances.raw, s.pred.raw)
    assert s.info["tier"] == "u8"
    c = ap.fw_classic(h, method="classic")      # classic order: pred bit-exact
    assert np.array_equal(c.distances.raw, g["dist"])
    assert np.array_equal(c.pred.raw, g["pred"])


@pytest.mark.parametrize("tier", ["u8", "u16", "w32", "i64"])
def test_c1_every_tier(cuda, tier):
    g = golden("c1_fw.npz")
    s = ap.fw_classic(ap.CostMatrix(g["h"]), tier=tier)
    assert s.info["tier"] == tier
    assert np.array_equal(s.distances.raw, g["dist"])
    pred_ok(g["h"], s.distances.raw, s.pred.raw)


def test_suite_graphs(cuda):
    g = golden("suite.npz")
    for i in range(int(g["count"])):
        h = ap.CostMatrix(g[f"h{i}"])
        s = ap.fw_classic(h)
        assert np.array_equal(s.distances.raw, g[f"dist{i}"]), i
        pred_ok(g[f"h{i}"], s.distances.raw, s.pred.raw)
        c = ap.fw_classic(h, method="classic")
        assert np.array_equal(c.pred.raw, g[f"pred{i}"]), i
        r = ap.rkleene(h, base_threshold=16)
        assert np.array_equal(r.distances.raw, g[f"dist{i}"]), i
        assert np.array_equal(r.via.raw, g[f"rkvia{i}"]), i
        q = ap.fw_squaring(h)
        assert np.array_equal(q.distances.raw, g[f"dist{i}"]), i
        assert np.array_equal(q.via.raw, g[f"sqvia{i}"]), i
        assert q.iterations == int(g[f"sqit{i}"]), i


def test_known_answers(cuda):
    three = ap.cost_matrix_from_graph(ap.Graph(3, [(0, 1, 1), (1, 2, 2), (2, 0, 4)]))
    for solver in ap.SOLVERS.values():
        assert solver(three).distances.raw.tolist() == [[0, 1, 3], [6, 0, 2], [4, 5, 0]]
    chain = ap.cost_matrix_from_graph(ap.Graph(3, [(0, 1, 3), (1, 2, 4), (0, 2, 10)]))
    s = ap.fw_classic(chain)
    assert s.distances[0, 2].value == 7 and s.pred[0, 2] == 1
    one = ap.cost_matrix_from_graph(ap.Graph(3, [(0, 1, 3)]))
    s = ap.fw_classic(one)
    assert s.pred[0, 1] == 0 and s.pred[0, 2] is None and s.pred[0, 0] is None
    edgeless = ap.cost_matrix_from_graph(ap.Graph(3, []))
    s = ap.fw_classic(edgeless)
    assert ap.matrices_equal(s.distances, ap.minplus_identity(3)) and (s.pred.raw == -1).all()
    for n in (1, 2, 7, 33):
        assert ap.fw_classic(ap.minplus_identity(n)).relaxation_count == n ** 3
    path5 = ap.cost_matrix_from_graph(ap.Graph(5, [(i, i + 1, 1) for i in range(4)]))
    assert ap.fw_squaring(path5).iterations == 3


@pytest.mark.parametrize("n,density,wmax,seed", [(1, 1.0, 5, 1), (2, 1.0, 5, 2), (127, 0.1, 100, 3),
                                                  (129, 0.05, 100, 4), (300, 0.02, 100, 5), (385, 1.0, 9, 6),
                                                  (640, 0.01, 200, 7)])
def test_fw_ragged_sizes_vs_oracle(cuda, n, density, wmax, seed):
    raw = random_graph_raw(n, density, wmax, seed)
    want_d, want_p = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    c = ap.fw_classic(ap.CostMatrix(raw), method="classic")
    assert np.array_equal(c.distances.raw, want_d) and np.array_equal(c.pred.raw, want_p)


@pytest.mark.parametrize("n,density", [(50, 0.1), (100, 0.05), (128, 0.03), (128, 1.0), (77, 0.2)])
def test_single_block_closure_is_classic_order(cuda, n, density):
    # n <= 128: the blocked solve is one phase-1 closure, whose deferred-pred u8 kernel must
    # reproduce the classic k order bit-for-bit (dist and pred), like reference fw_classic
    raw = random_graph_raw(n, density, 9, seed=1000 + n)
    want_d, want_p = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert s.info["tier"] == "u8"
    assert np.array_equal(s.distances.raw, want_d)
    assert np.array_equal(s.pred.raw, want_p)


def test_zero_weight_edges(cuda):
    raw = random_graph_raw(257, 0.05, 20, 9, zero_frac=0.3)
    want_d, _ = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    # zero-cost edges: predecessors come from the classic k order (a tree by construction)
    assert s.info["classic_for_zero_edges"]
    r = ap.rkleene(ap.CostMatrix(raw), track="pred", split="aligned", base_threshold=128)
    assert np.array_equal(r.distances.raw, want_d)
    pred_ok(raw, r.distances.raw, r.pred.raw)
    v = ap.rkleene(ap.CostMatrix(raw))
    assert np.array_equal(v.distances.raw, want_d)


def ring_with_chords(n, step, seed):
    """Unit ring i -> i+1 plus weight-2 chords i -> i+step: max distance ~ 2n/step (known range)."""
    rng = np.random.default_rng(seed)
    raw = np.full((n, n), INF_RAW, np.int64)
    idx = np.arange(n)
    raw[idx, (idx + 1) % n] = 1
    keep = rng.random(n) < 0.9
    raw[idx[keep], (idx[keep] + step) % n] = 2
    np.fill_diagonal(raw, 0)
    return raw


@pytest.mark.parametrize("n,step,b", [(384, 3, 128), (1000, 7, 256), (2048, 13, 256)])
def test_u16_tier_fw_and_rkleene(cuda, n, step, b):
    # max distance in (254, 508]: u8 cannot certify, u16 can; forced and auto both exact
    raw = ring_with_chords(n, step, seed=n)
    want_d, _ = orc.rkleene(raw, 64)
    m = want_d[want_d != INF_RAW].max()
    assert 254 < m + 2 <= 510
    for tier in ("u16", None):
        s = ap.fw_classic(ap.CostMatrix(raw), tier=tier, block=b)
        assert s.info["tier"] == "u16"
        assert np.array_equal(s.distances.raw, want_d)
        pred_ok(raw, s.distances.raw, s.pred.raw)
    r = ap.rkleene(ap.CostMatrix(raw), split="aligned", track="pred", base_threshold=256, tier="u16")
    assert r.info["tier"] == "u16"
    assert np.array_equal(r.distances.raw, want_d)
    pred_ok(raw, r.distances.raw, r.pred.raw)


def test_tier_fallback_and_wide_costs(cuda):
    # long paths: u8 and u16 certificates must fail and fall back to w32, results exact
    n = 300
    raw = np.full((n, n), INF_RAW, np.int64)
    np.fill_diagonal(raw, 0)
    for i in range(n - 1):
        raw[i, i + 1] = 3
    s = ap.fw_classic(ap.CostMatrix(raw))
    # (u8 itself may be skipped when an earlier call of this shape needed u16: fw_sched.cu skip-ahead)
    assert s.info["tier"] == "w32" and "u16" in s.info["tiers_tried"]
    want_d, _ = orc.fw_classic(raw)
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    # costs beyond 2^24: straight to the exact int64 tier
    big = random_graph_raw(200, 0.1, 1 << 40, 11)
    s = ap.fw_classic(ap.CostMatrix(big))
    assert s.info["tier"] == "i64"
    want_d, _ = orc.fw_classic(big)
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(big, s.distances.raw, s.pred.raw)


def test_errors(cuda):
    for solver in ap.SOLVERS.values():
        with pytest.raises(ap.NegativeWeightError):
            solver(ap.CostMatrix.from_rows([[0, -2], [1, 0]]))
        with pytest.raises(ap.MalformedGraphError):
            solver(ap.CostMatrix.from_rows([[0, 1], [1, 3]]))
        with pytest.raises(ap.ParameterError):
            solver(ap.minplus_identity(2), tile_size=0)
        h = ap.cost_matrix_from_graph(ap.Graph(3, [(0, 1, 1), (1, 2, 2), (2, 0, 4)]))
        before = h.raw.copy()
        solver(h)
        assert np.array_equal(h.raw, before)
    with pytest.raises(ap.ParameterError):
        ap.rkleene(ap.minplus_identity(2), base_threshold=0)
    big = (1 << 60) - 2
    m = ap.CostMatrix.from_rows([[0, big, ap.INF], [ap.INF, 0, big], [ap.INF, ap.INF, 0]])
    with pytest.raises(ap.CostRangeError):
        ap.fw_classic(m)
    with pytest.raises(ap.CostRangeError):
        ap.fw_classic(m, method="classic")


def test_int32_and_fp32_dense_entry(cuda):
    import torch

    p = ap.GenParams(700, 0.1, 100, 707)
    h64 = ap.dense_costs(p, np.int64)
    want_d, _ = orc.fw_classic(h64)
    h32 = ap.dense_costs(p, np.int32)
    r = ap.solve(h32)
    assert r.distances.dtype == np.int32
    fin = want_d != INF_RAW
    assert np.array_equal(r.distances[fin], want_d[fin]) and (r.distances[~fin] == INF32).all()
    pred_ok(h32, r.distances, r.index, INF32)
    hf = ap.dense_costs(p, np.float32)
    rt = ap.solve(torch.from_numpy(hf).cuda())
    df = rt.distances.cpu().numpy()
    assert np.array_equal(df[fin], want_d[fin].astype(np.float32)) and np.isinf(df[~fin]).all()
    assert rt.info["tier"] == "u8"


def test_fp32_continuous_tolerance(cuda):
    import torch

    rng = np.random.default_rng(3)
    n = 400
    w = rng.uniform(1.0, 100.0, size=(n, n)).astype(np.float32)
    w[rng.random((n, n)) > 0.05] = np.inf
    np.fill_diagonal(w, 0.0)
    ref = w.astype(np.float64)
    for k in range(n):
        np.minimum(ref, ref[:, k:k + 1] + ref[k:k + 1, :], out=ref)
    for alg in ("fw_blocked", "fw_classic", "rkleene"):
        r = ap.solve(torch.from_numpy(w).cuda(), alg)
        assert r.info["tier"] == "f32"
        d = r.distances.cpu().numpy().astype(np.float64)
        fin = np.isfinite(ref)
        assert (np.isfinite(d) == fin).all()
        assert np.allclose(d[fin], ref[fin], rtol=1e-5, atol=0), alg


def test_fp32_continuous_bulk_kernel(cuda):
    # block 256 / long R-Kleene products: the bulk-staged fp32 kernel (k >= 256); tolerance vs
    # float64, and blocked FW == R-Kleene within the same tolerance; predecessors certified
    import torch

    rng = np.random.default_rng(5)
    n = 1000
    w = rng.uniform(1.0, 100.0, size=(n, n)).astype(np.float32)
    w[rng.random((n, n)) > 0.02] = np.inf
    np.fill_diagonal(w, 0.0)
    ref = w.astype(np.float64)
    for k in range(n):
        np.minimum(ref, ref[:, k:k + 1] + ref[k:k + 1, :], out=ref)
    fin = np.isfinite(ref)
    h = torch.from_numpy(w).cuda()
    for r in (ap.solve(h, "fw_blocked", block=256),
              ap.solve(h, "rkleene", track="pred", split="aligned", base_threshold=256)):
        assert r.info["tier"] == "f32"
        d = r.distances.cpu().numpy().astype(np.float64)
        assert (np.isfinite(d) == fin).all()
        assert np.allclose(d[fin], ref[fin], rtol=1e-5, atol=0)
        p = r.index.cpu().numpy()
        # every finite off-diagonal cell's pred is a real last hop: d[i][p] + w[p][j] == d[i][j]
        ii, jj = np.nonzero(fin & ~np.eye(n, dtype=bool))
        pp = p[ii, jj].astype(np.int64)
        assert (pp >= 0).all()
        assert np.allclose(d[ii, pp] + w[pp, jj].astype(np.float64), d[ii, jj], rtol=1e-5)


# ---- R-Kleene -------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["rk_n300_t64.npz", "rk_n200_t16.npz", "rk_n130_t8.npz", "rk_n150_t1.npz"])
def test_rkleene_via_bitwise(cuda, name):
    g = golden(name)
    r = ap.rkleene(ap.CostMatrix(g["h"]), base_threshold=int(g["thr"]))
    assert np.array_equal(r.distances.raw, g["dist"])
    assert np.array_equal(r.via.raw, g["via"])


@pytest.mark.parametrize("split", ["floor", "aligned"])
def test_rkleene_pred_and_aligned(cuda, split):
    raw = random_graph_raw(777, 0.03, 100, 21)
    want_d, _ = orc.fw_classic(raw)
    r = ap.rkleene(ap.CostMatrix(raw), base_threshold=256, track="pred", split=split)
    assert np.array_equal(r.distances.raw, want_d)
    pred_ok(raw, r.distances.raw, r.pred.raw)
    v = ap.rkleene(ap.CostMatrix(raw), base_threshold=256, split=split)
    assert np.array_equal(v.distances.raw, want_d)
    d, via = want_d, v.via.raw
    rows, cols = np.nonzero(via >= 0)
    mids = via[rows, cols]
    assert (d[rows, mids] + d[mids, cols] == d[rows, cols]).all()
    assert (mids != rows).all() and (mids != cols).all()


# ---- min-plus products ----------------------------------------------------------------------

def test_minplus_golden(cuda):
    g = golden("minplus.npz")
    for k in range(int(g["count"])):
        x, y = ap.CostMatrix(g[f"p{k}_x"]), ap.CostMatrix(g[f"p{k}_y"])
        r = ap.minplus_product(x, y, offsets=tuple(int(o) for o in g[f"p{k}_off"]))
        assert np.array_equal(r.distances.raw, g[f"p{k}_dist"]), k
        assert np.array_equal(r.via.raw, g[f"p{k}_via"]), k
        a = ap.minplus_accumulate(ap.CostMatrix(g[f"a{k}_z"]), x, y, ap.ViaMatrix(g[f"a{k}_vin"]),
                                  inner_offset=int(g[f"p{k}_off"][1]))
        assert np.array_equal(a.distances.raw, g[f"a{k}_dist"]), k
        assert np.array_equal(a.via.raw, g[f"a{k}_via"]), k


def test_minplus_tiers_and_errors(cuda):
    rng = np.random.default_rng(5)
    x = rng.integers(0, 1 << 33, size=(70, 90)).astype(np.int64)
    y = rng.integers(0, 1 << 33, size=(90, 50)).astype(np.int64)
    x[rng.random(x.shape) < 0.2] = INF_RAW
    want = orc.product(x, y)
    r = ap.minplus_product(ap.CostMatrix(x), ap.CostMatrix(y))
    assert np.array_equal(r.distances.raw, want[0]) and np.array_equal(r.via.raw, want[1])
    with pytest.raises(ap.DimensionError):
        ap.minplus_product(ap.CostMatrix(np.zeros((2, 3), np.int64)), ap.CostMatrix(np.zeros((2, 3), np.int64)))
    big = (1 << 60) - 2
    m = ap.CostMatrix.from_rows([[0, big, ap.INF], [ap.INF, 0, big], [ap.INF, ap.INF, 0]])
    with pytest.raises(ap.CostRangeError):
        ap.minplus_product(m, m)
    with pytest.raises(ap.NegativeWeightError):
        ap.minplus_product(ap.CostMatrix.from_rows([[0, -1], [1, 0]]), ap.minplus_identity(2))
    # a forced tier that cannot hold the partial sums is refused, never silently narrowed
    w = ap.CostMatrix.from_rows([[0, 300], [ap.INF, 0]])
    with pytest.raises(ap.ParameterError):
        ap.minplus_product(w, w, tier="u8")
    r8 = ap.minplus_product(ap.CostMatrix.from_rows([[0, 100], [ap.INF, 0]]), ap.minplus_identity(2), tier="u8")
    assert r8.distances.raw.tolist() == [[0, 100], [INF_RAW, 0]]


# ---- larger sizes: size-independent properties ---------------------------------------------

def test_c2_shape_fw_equals_rkleene_and_oracle(cuda):
    p = ap.GenParams(2048, 1.0, 100, 7 + 2048)
    raw = ap.dense_costs(p, np.int64)
    want_d, _ = orc.rkleene(raw, 64)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    r = ap.rkleene(ap.CostMatrix(raw), base_threshold=512, split="aligned", track="pred")
    assert np.array_equal(r.distances.raw, want_d)
    pred_ok(raw, r.distances.raw, r.pred.raw)


def test_large_fw_device_properties(cuda):
    import torch

    p = ap.GenParams(8192, 0.1, 100, 7 + 8192)
    h = torch.from_numpy(ap.dense_costs(p, np.int32)).cuda()
    a = ap.solve(h, "fw_blocked")
    b = ap.solve(h, "rkleene", track="pred", base_threshold=1024)
    assert torch.equal(a.distances, b.distances)
    w = ap.solve(h, "fw_blocked", tier="w32")
    assert torch.equal(a.distances, w.distances)
    ok, why = ap.check_pred_tree(h, a.distances, a.index, INF32)
    assert ok, why
    ok, why = ap.check_pred_tree(h, b.distances, b.index, INF32)
    assert ok, why
    # Bellman fixpoint on a row sample: with the pred certificate above (every distance is the
    # length of a real path) this proves the sampled rows exact, independent of any CPU run.
    H = h.to(torch.int64)
    H = torch.where(h == INF32, torch.tensor(INF_RAW, device=h.device), H)
    D = a.distances.to(torch.int64)
    D = torch.where(a.distances == INF32, torch.tensor(INF_RAW, device=h.device), D)
    for r in range(0, 8192, 1021):
        best = H[r].clone()
        for k0 in range(0, 8192, 1024):
            cand = (D[r, k0:k0 + 1024, None] + H[k0:k0 + 1024, :]).amin(dim=0)
            best = torch.minimum(best, cand)
        best = torch.where(best >= INF_RAW, torch.tensor(INF_RAW, device=h.device), best)
        assert torch.equal(best, D[r]), r


@pytest.mark.parametrize("block", [0, 128, 256])
def test_w32_bulk_tier_wide_weights(cuda, block):
    # weights up to 50000: only w32 / i64 certify; the w32 tier runs the bulk-staged kernel
    # (7-bit tags, 3-chunk decode windows) in phases 2/3 and in the R-Kleene products
    raw = random_graph_raw(777, 0.05, 50000, 5)
    want_d, _ = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw), block=block)
    assert s.info["tier"] == "w32"
    assert np.array_equal(s.distances.raw, want_d)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    r = ap.rkleene(ap.CostMatrix(raw), split="aligned", track="pred", base_threshold=256)
    assert r.info["tier"] == "w32"
    assert np.array_equal(r.distances.raw, want_d)
    pred_ok(raw, r.distances.raw, r.pred.raw)


def test_graph_replay_with_changing_inputs(cuda):
    """Repeated solves of one shape on the same buffers replay a CUDA graph (N <= 2048): every
    call must still read the current input (different graphs, reused buffers)."""
    import torch

    n = 1500
    dist = torch.empty((n, n), dtype=torch.int32, device="cuda")
    pred = torch.empty((n, n), dtype=torch.int32, device="cuda")
    lib = ap._native.load()
    ws_n = lib.apsp_workspace_bytes(ap._native.ALG_FW_BLOCKED, ap._native.DTYPE_I32, n, 0)
    ws = torch.empty(ws_n, dtype=torch.uint8, device="cuda")
    import ctypes

    stream = torch.cuda.current_stream()
    for it in range(6):                       # sightings 1 (plain), 2 (capture), 3+ (replay)
        seed = 100 + it
        h = ap.dense_costs(ap.GenParams(n, 0.02 if it % 2 else 0.1, 100, seed), np.int32)
        dist.copy_(torch.from_numpy(h))
        info = ap._native.ApspInfo()
        st = lib.apsp_fw_blocked(ap._native.DTYPE_I32, n, dist.data_ptr(), n, pred.data_ptr(), n, 0,
                                 ap._native.TIER_AUTO, ws.data_ptr(), ws.numel(), ctypes.c_void_p(stream.cuda_stream),
                                 ctypes.byref(info))
        ap._native.check(st)
        torch.cuda.synchronize()
        h64 = h.astype(np.int64)
        h64[h64 == INF32] = INF_RAW
        want, _ = orc.fw_classic(h64)
        got = dist.cpu().numpy().astype(np.int64)
        got[got == INF32] = INF_RAW
        assert np.array_equal(got, want), it
        ok, why = ap.check_pred_tree(h64, got, pred.cpu().numpy().astype(np.int64), INF_RAW)
        assert ok, (it, why)


def test_results_independent_of_tile_size_and_workers(cuda):
    """Reference determinism-under-parallelism criterion (test_solvers.py:195-210,
    test_acceptance.py:53-71): identical dist / pred / via for every tile_size and worker count
    (both are accepted and validated; neither changes the GPU grid)."""
    raw = random_graph_raw(300, 0.08, 50, 17)
    h = ap.CostMatrix(raw)
    base_f = ap.fw_classic(h)
    base_r = ap.rkleene(h, base_threshold=16)
    for tile_size in (1, 8, 16, 64, 1024):
        for workers in (1, 2, 3, 4, None):
            f = ap.fw_classic(h, tile_size=tile_size, workers=workers)
            assert np.array_equal(f.distances.raw, base_f.distances.raw)
            assert np.array_equal(f.pred.raw, base_f.pred.raw)
    for tile_size in (1, 64):
        r = ap.rkleene(h, base_threshold=16, tile_size=tile_size, workers=2)
        assert np.array_equal(r.via.raw, base_r.via.raw)


@pytest.mark.parametrize("alpha", [100, 3000, 10 ** 6])
def test_host_readback_narrowed_equals_device_result(cuda, alpha, monkeypatch):
    """apsp_solve_host narrows the int32 result for the PCIe readback (csrc/hostio.cu): 1 byte
    (u8 range), 2 bytes (u16 range) or none (wide) for dist, 2 bytes for pred. The host arrays
    must equal the device-resident result and the plain int32 readback, cell for cell. n=2050
    makes every row start 8 bytes off a 16-byte boundary (scalar heads in the widening loops)."""
    import ctypes

    import torch
    from paper_2310_03983_b200 import _native as nat

    n = 2050
    h32 = ap.dense_costs(ap.GenParams(n, 0.1, alpha, 11 + alpha), np.int32)
    dev = ap.solve(torch.from_numpy(h32).cuda())
    want_d, want_p = dev.distances.cpu().numpy(), dev.index.cpu().numpy()
    r = ap.solve(h32)
    m = r.info["max_finite"]
    width = 1 if m <= 254 else 2 if m <= 65534 else 4
    assert width == {100: 1, 3000: 2, 10 ** 6: 4}[alpha] or alpha == 3000
    assert np.array_equal(r.distances, want_d) and np.array_equal(r.index, want_p)
    lib = nat.load()
    info = nat.ApspInfo()
    d = np.empty((n, n), np.int32)
    p64 = np.empty((n, n), np.int64)
    st = lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, h32.ctypes.data, d.ctypes.data, p64.ctypes.data,
                             nat.DTYPE_I64, nat.IDX_PRED, 0, 0, 0, nat.TIER_AUTO, 0, ctypes.byref(info))
    nat.check(st)
    assert info.d2h_bytes_per_cell == width + 2
    assert np.array_equal(d, want_d) and np.array_equal(p64, want_p.astype(np.int64))
    monkeypatch.setenv("APSP_PACKED_READBACK", "0")
    st = lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, h32.ctypes.data, d.ctypes.data, p64.ctypes.data,
                             nat.DTYPE_I64, nat.IDX_PRED, 0, 0, 0, nat.TIER_AUTO, 0, ctypes.byref(info))
    nat.check(st)
    assert info.d2h_bytes_per_cell == 12
    assert np.array_equal(d, want_d) and np.array_equal(p64, want_p.astype(np.int64))


def test_host_upload_narrowed_and_fallbacks(cuda):
    """apsp_solve_host narrows the int32 costs for the upload (csrc/hostio.cu): the width comes
    from the first rows and every cell is checked while packing. A late cell that does not fit
    (a wide cost, a negative cost) aborts to the plain int32 upload, so results and errors are
    those of the caller's matrix."""
    import ctypes

    import torch
    from paper_2310_03983_b200 import _native as nat

    n = 2048
    lib = nat.load()

    def host(h):
        info = nat.ApspInfo()
        d = np.empty((n, n), np.int32)
        p = np.empty((n, n), np.int32)
        st = lib.apsp_solve_host(nat.ALG_FW_BLOCKED, nat.DTYPE_I32, n, h.ctypes.data, d.ctypes.data, p.ctypes.data,
                                 nat.DTYPE_I32, nat.IDX_PRED, 0, 0, 0, nat.TIER_AUTO, 0, ctypes.byref(info))
        return st, d, p, info

    for alpha, width in ((100, 1), (3000, 2), (10 ** 6, 4)):
        h = ap.dense_costs(ap.GenParams(n, 0.1, alpha, 5 + alpha), np.int32)
        st, d, p, info = host(h)
        nat.check(st)
        dev = ap.solve(torch.from_numpy(h).cuda())
        assert info.h2d_bytes_per_cell == width
        assert np.array_equal(d, dev.distances.cpu().numpy()) and np.array_equal(p, dev.index.cpu().numpy())
    h = ap.dense_costs(ap.GenParams(n, 0.1, 100, 9), np.int32)
    h[n - 1, 3] = 70000                                   # fits neither u8 nor u16: plain upload
    st, d, p, info = host(h)
    nat.check(st)
    assert info.h2d_bytes_per_cell == 4
    dev = ap.solve(torch.from_numpy(h).cuda())
    assert np.array_equal(d, dev.distances.cpu().numpy()) and np.array_equal(p, dev.index.cpu().numpy())
    h[n - 1, 3] = -5                                      # negative cost: the device scan's error
    st, _, _, _ = host(h)
    from paper_2310_03983_b200.core import NegativeWeightError
    with pytest.raises(NegativeWeightError):
        nat.check(st)


@pytest.mark.parametrize("algorithm,kw", [("rkleene", {"track": "via"}), ("rkleene", {"track": "pred"}),
                                          ("fw_squaring", {})])
def test_host_transfers_other_algorithms(cuda, algorithm, kw):
    """The narrowed host transfers carry R-Kleene via / pred and squaring via indices too: the
    host-buffer result equals the device-resident one cell for cell."""
    import torch

    n = 2048
    h32 = ap.dense_costs(ap.GenParams(n, 0.1, 100, 77), np.int32)
    dev = ap.solve(torch.from_numpy(h32).cuda(), algorithm, **kw)
    r = ap.solve(h32, algorithm, **kw)
    assert r.info["d2h_bytes_per_cell"] == 3 and r.info["h2d_bytes_per_cell"] == 1
    assert np.array_equal(r.distances, dev.distances.cpu().numpy())
    assert np.array_equal(r.index, dev.index.cpu().numpy())


@pytest.mark.parametrize("alpha", [100, 3000, 10 ** 6])
def test_int64_api_narrowed_transfers(cuda, alpha):
    """The reference-facing int64 API (CostMatrix in, int64 ApspSolution out) moves its data
    narrowed too: int64 costs -> u8/u16 up, dist u8/u16 (INF_RAW = all-ones) and pred u16 down.
    Results equal the device-resident int64 solve cell for cell; a late wide cell or a negative
    cost falls back to the plain int64 upload with the reference's error."""
    import torch
    from paper_2310_03983_b200.core import NegativeWeightError

    n = 2048
    h64 = ap.dense_costs(ap.GenParams(n, 0.1, alpha, 21 + alpha), np.int64)
    dev = ap.solve(torch.from_numpy(h64).cuda())   # before CostMatrix freezes h64
    s = ap.fw_classic(ap.CostMatrix(h64))
    d = np.asarray(s.distances.raw)
    assert np.array_equal(d, dev.distances.cpu().numpy())
    assert np.array_equal(np.asarray(s.pred.raw), dev.index.cpu().numpy().astype(np.int64))
    up = {100: 1, 3000: 2, 10 ** 6: 8}[alpha]
    m = s.info["max_finite"]
    down = (1 if m <= 254 else 2 if m <= 65534 else 8) + 2
    assert s.info["h2d_bytes_per_cell"] == up and s.info["d2h_bytes_per_cell"] == down
    if alpha == 100:
        h64 = h64.copy()   # CostMatrix froze the first one
        h64[n - 1, 5] = 70000
        dev2 = ap.solve(torch.from_numpy(h64).cuda())
        s2 = ap.fw_classic(ap.CostMatrix(h64))
        assert s2.info["h2d_bytes_per_cell"] == 8
        assert np.array_equal(np.asarray(s2.distances.raw), dev2.distances.cpu().numpy())
        h64 = h64.copy()
        h64[n - 1, 5] = -3
        with pytest.raises(NegativeWeightError):
            ap.fw_classic(ap.CostMatrix(h64))


@pytest.mark.parametrize("n", [512, 520, 301])
@pytest.mark.parametrize("wmax,zero", [(60, 0.0), (60, 0.2), (400, 0.0), (100000, 0.0)])
def test_classic_order_narrow_stores_bitwise(cuda, n, wmax, zero):
    """Classic k order (K1) on the narrowest certified store: u8 (small weights), u16 (sums past
    254) or the exact store, through the packed-pair streaming kernel (n a multiple of 16 / 8)
    or the scalar one (n = 301). Distances and pred bit-exact with reference fw_classic."""
    raw = random_graph_raw(n, 0.05, wmax, n + wmax, zero_frac=zero)
    want_d, want_p = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw), method="classic")
    assert np.array_equal(s.distances.raw, want_d)
    assert np.array_equal(s.pred.raw, want_p)
    if zero:   # the blocked solver falls back to the same classic order
        b = ap.fw_classic(ap.CostMatrix(raw))
        assert b.info["classic_for_zero_edges"]
        assert np.array_equal(b.distances.raw, want_d) and np.array_equal(b.pred.raw, want_p)


def test_streamed_last_round_readback(cuda):
    """apsp_solve_host streams the blocked FW's last round to the host band by band (N > 2048,
    no graph replay). The streamed rows stand only when the u8 attempt certifies: a ring with
    chords (true max distance ~2n/step > 254) makes the u8 attempt fail, the u16 run follows and
    the host arrays must still equal the device-resident result."""
    import torch

    n = 2304
    for raw, want_tier in ((ring_with_chords(n, 16, 5), "u16"),
                           (ap.dense_costs(ap.GenParams(n, 0.1, 100, 31), np.int64), "u8")):
        h32 = np.where(raw == INF_RAW, INF32, raw).astype(np.int32)
        dev = ap.solve(torch.from_numpy(h32.copy()).cuda())
        r = ap.solve(h32)
        # (the device call may take u16 straight away after the ring's u8 -> u16 fallback:
        # fw_sched.cu skip-ahead; u8 and u16 results are bitwise identical)
        assert r.info["tier"] == want_tier and dev.info["tier"] in (want_tier, "u16")
        if want_tier == "u16":
            assert "u8" in r.info["tiers_tried"]
        assert np.array_equal(r.distances, dev.distances.cpu().numpy())
        assert np.array_equal(r.index, dev.index.cpu().numpy())


@pytest.mark.parametrize("n", [643, 301])
def test_rkleene_floor_int64_tier_odd_n(cuda, n):
    """Floor-split R-Kleene on the exact int64 tier with odd n: the int64 store must start
    8-byte aligned in the workspace (regression: a 4-byte offset faulted with misaligned
    address). Found by tools/stress.py."""
    raw = random_graph_raw(n, 0.002, 10 ** 6, n)
    want_d, _ = orc.fw_classic(raw)
    r = ap.rkleene(ap.CostMatrix(raw), tier="i64")
    assert np.array_equal(r.distances.raw, want_d)
    assert r.info["tier"] == "i64"


@pytest.mark.parametrize("n,rho", [(128, 0.5), (300, 0.3), (1000, 0.1), (1537, 0.3), (2100, 0.1)])
def test_persistent_small_n_schedule(cuda, n, rho, monkeypatch):
    """The one-launch dataflow schedule of small-n u8 FW (fw_persist.cuh) against the oracle and
    the launch-based schedule (APSP_NO_PERSIST=1): equal distances, both pred trees valid."""
    import torch

    raw = ap.dense_costs(ap.GenParams(n, rho, 100, 3 * n), np.int64)
    want, _ = orc.rkleene(raw, 64)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert s.info["tier"] == "u8"
    assert np.array_equal(s.distances.raw, want)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, 3 * n), np.int32)).cuda()
    a = ap.solve(h)
    monkeypatch.setenv("APSP_NO_PERSIST", "1")
    b = ap.solve(h)
    assert torch.equal(a.distances, b.distances)
    ok, why = ap.check_pred_tree(h, b.distances, b.index, INF32)
    assert ok, why


def test_speculative_tier_follows_the_input(cuda):
    """Repeated calls of one shape start the tier that certified last time before the scan is
    read back (fw_sched.cu spec_lookup). Whatever the call history, each input must give exactly
    the result of its first call: inputs that need another tier, long paths whose narrow
    certificates fail, error inputs and zero-cost edges (classic order) included."""
    import torch

    n = 640

    def dev(raw):
        h = raw.copy()
        h[raw == INF_RAW] = INF32
        return torch.from_numpy(h.astype(np.int32)).cuda()

    narrow = ap.dense_costs(ap.GenParams(n, 0.1, 100, 5), np.int64)
    wide = random_graph_raw(n, 0.05, 50000, 9)
    path = np.full((n, n), INF_RAW, np.int64)
    np.fill_diagonal(path, 0)
    path[np.arange(n - 1), np.arange(1, n)] = 3
    mid = ring_with_chords(n, 4, 5)   # max distance ~ 2n/4 = 320: u8 fails its certificate, u16 holds
    cases = {"narrow": (narrow, "u8"), "wide": (wide, "w32"), "path": (path, "w32"), "mid": (mid, "u16")}
    first = {}
    # "mid" then "wide": a speculative u16 attempt on weights up to 50000 (saturated on store, then
    # discarded) must neither fault nor leak into the result
    for name in ["narrow", "narrow", "narrow", "wide", "narrow", "wide", "wide", "path", "path", "narrow", "path",
                 "mid", "mid", "wide", "mid", "narrow", "mid"]:
        raw, tier = cases[name]
        s = ap.solve(dev(raw))
        # after "mid" (u8 failed, u16 used) a u8 input may skip ahead to u16: same bits either way
        assert s.info["tier"] == tier or (tier, s.info["tier"]) == ("u8", "u16"), name
        d, p = s.distances.cpu().numpy(), s.index.cpu().numpy()
        if name not in first:
            want, _ = orc.fw_classic(raw)
            got = d.astype(np.int64)
            got[d == INF32] = INF_RAW
            assert np.array_equal(got, want), name
            pred_ok(raw, got, p.astype(np.int64))
            first[name] = (d, p)
        else:
            assert np.array_equal(d, first[name][0]) and np.array_equal(p, first[name][1]), name
    bad = dev(narrow)
    bad[1, 2] = -1
    with pytest.raises(ap.NegativeWeightError):
        ap.solve(bad)
    zero = narrow.copy()
    zero[3, 4] = 0
    s = ap.solve(dev(zero))
    want_d, want_p = orc.fw_classic(zero)
    got = s.distances.cpu().numpy().astype(np.int64)
    got[got == INF32] = INF_RAW
    assert np.array_equal(got, want_d) and np.array_equal(s.index.cpu().numpy().astype(np.int64), want_p)
    s = ap.solve(dev(narrow))
    assert np.array_equal(s.distances.cpu().numpy(), first["narrow"][0])
    # host-buffer calls (band sink; no speculation) after same-shape calls match the device path,
    # zero-cost edges (classic order) included
    for raw in (narrow, narrow, zero, narrow):
        h32 = dev(raw).cpu().numpy()
        host = ap.solve(h32)
        d = ap.solve(torch.from_numpy(h32).cuda())
        assert np.array_equal(host.distances, d.distances.cpu().numpy())
        assert np.array_equal(host.index, d.index.cpu().numpy())


@pytest.mark.parametrize("n,rho,seed,tier", [(320, 0.05, 1, "u16"), (1024, 0.01, 7 + 1024, None),
                                             (2048, 0.01, 7 + 2048, None)])
def test_persistent_small_n_u16(cuda, n, rho, seed, tier, monkeypatch):
    """The 64-wide persistent schedule on the u16 tier (two 32-k tag windows per task): equal
    to the oracle, valid pred tree, and equal distances to the launch-based schedule. The two
    larger graphs pick u16 themselves (the C5 configs), the small one is forced."""
    import torch

    raw = ap.dense_costs(ap.GenParams(n, rho, 100, seed), np.int64)
    want, _ = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw), tier=tier)
    assert s.info["tier"] == "u16"
    assert np.array_equal(s.distances.raw, want)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, seed), np.int32)).cuda()
    a = ap.solve(h, tier=tier)
    assert a.info["tier"] == "u16"
    monkeypatch.setenv("APSP_NO_PERSIST", "1")
    b = ap.solve(h, tier=tier)
    assert torch.equal(a.distances, b.distances)
    ok, why = ap.check_pred_tree(h, a.distances, a.index, INF32)
    assert ok, why


@pytest.mark.parametrize("n,rho,block", [(300, 0.1, 0), (700, 0.05, 128), (1500, 0.05, 0), (3200, 0.02, 0)])
def test_u8_u16_results_identical(cuda, n, rho, block):
    """u8 and u16 run the same kernels with the same tie rules: forced to either tier, one input
    gives bitwise equal distances AND predecessors (the speculative u8 -> u16 skip-ahead in
    fw_sched.cu relies on it)."""
    import torch

    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, rho, 100, n + 11), np.int32)).cuda()
    a = ap.solve(h, block=block, tier="u8")
    b = ap.solve(h, block=block, tier="u16")
    assert a.info["tier"] == "u8" and b.info["tier"] == "u16"
    assert torch.equal(a.distances, b.distances) and torch.equal(a.index, b.index)


def test_speculative_skip_ahead_u8_to_u16(cuda):
    """A shape whose scan picks u8 first but whose certificate needs u16: the first call tries
    both, repeated calls start u16 right away (skip-ahead) and return bitwise the same."""
    import torch

    n = 1024
    h = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.02, 100, 7 + n), np.int32)).cuda()
    first = ap.solve(h)
    assert first.info["tier"] == "u16"
    again = [ap.solve(h) for _ in range(3)]
    for r in again:
        assert r.info["tier"] == "u16"
        assert torch.equal(r.distances, first.distances) and torch.equal(r.index, first.index)
    assert "u8" not in again[-1].info["tiers_tried"]
    raw = first.distances.cpu().numpy().astype(np.int64)
    h64 = h.cpu().numpy().astype(np.int64)
    h64[h64 == INF32] = INF_RAW
    raw[raw == INF32] = INF_RAW
    want, _ = orc.fw_classic(h64)
    assert np.array_equal(raw, want)


@pytest.mark.parametrize("n,rho,wmax", [(300, 0.05, 50000), (1000, 0.01, 3000), (2048, 0.002, 100)])
def test_persistent_small_n_w32(cuda, n, rho, wmax, monkeypatch):
    """The 64-wide persistent schedule on the w32 tier (one unsigned 32-bit key per cell,
    VIADDMNMX.U32): equal to the oracle, valid pred tree, equal distances to the launch-based
    schedule."""
    import torch

    raw = random_graph_raw(n, rho, wmax, n + wmax) if wmax > 500 else ap.dense_costs(
        ap.GenParams(n, rho, wmax, 7 + n), np.int64)
    want, _ = orc.fw_classic(raw)
    s = ap.fw_classic(ap.CostMatrix(raw))
    assert s.info["tier"] == "w32"
    assert np.array_equal(s.distances.raw, want)
    pred_ok(raw, s.distances.raw, s.pred.raw)
    h32 = raw.copy()
    h32[raw == INF_RAW] = INF32
    h = torch.from_numpy(h32.astype(np.int32)).cuda()
    a = ap.solve(h)
    assert a.info["tier"] == "w32"
    monkeypatch.setenv("APSP_NO_PERSIST", "1")
    b = ap.solve(h)
    assert torch.equal(a.distances, b.distances)
    ok, why = ap.check_pred_tree(h, a.distances, a.index, INF32)
    assert ok, why


def test_skip_ahead_returns_to_u8(cuda):
    """After a shape needed u16, a same-shape input that fits u8 may run once on u16 (skip-ahead,
    same bits), but its certificate shows u8 would have held: the next call is u8 again."""
    import torch

    n = 1024
    need16 = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 0.02, 100, 7 + n), np.int32)).cuda()
    dense = torch.from_numpy(ap.dense_costs(ap.GenParams(n, 1.0, 100, 5), np.int32)).cuda()
    assert ap.solve(need16).info["tier"] == "u16"
    assert ap.solve(need16).info["tier"] == "u16"
    a = ap.solve(dense)
    b = ap.solve(dense)
    assert a.info["tier"] in ("u8", "u16") and b.info["tier"] == "u8"
    assert torch.equal(a.distances, b.distances) and torch.equal(a.index, b.index)
