// R-Kleene recursion, min-plus squaring and the public min-plus product / accumulate.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "engine.h"

namespace apsp {

// ---- R-Kleene ---------------------------------------------------------------------------
struct RK {
  int store;
  size_t es;
  char* D;
  int64_t ld;
  int32_t* P;     // idx matrix (pred or via), ld = ld
  int mode;
  int thr;
  bool aligned;
  char* sV;       // snapshot values (half x half)
  int32_t* sP;    // snapshot idx
  int64_t sld;
  Status* st;
  cudaStream_t s;
  char* prep = nullptr;     // narrow tiers, aligned split: bulk-copy operand layouts (half x half)
  char* leafws = nullptr;   // aligned leaves: fw_scratch_bytes(thr, 128, es)
  // aligned split: the two independent products of each half (B and C updates) run
  // concurrently on a second stream, with their own snapshot / layout buffers
  char* sV2 = nullptr;
  char* prep2 = nullptr;
  cudaStream_t s2 = nullptr;
  cudaEvent_t evFork = nullptr, evJoin = nullptr;
  int launches = 0;

  char* at(int64_t i, int64_t j) const { return D + (i * ld + j) * es; }
  int32_t* pat(int64_t i, int64_t j) const { return P + i * ld + j; }

  int mp(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t r0, int64_t c0, int64_t m, int64_t n,
         int64_t k, const int32_t* predB, int64_t ldpb, int64_t inner_off) {
    return mp_on(s, prep, A, lda, B, ldb, r0, c0, m, n, k, predB, ldpb, inner_off);
  }
  int mp_on(cudaStream_t st_, char* prep_, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t r0,
            int64_t c0, int64_t m, int64_t n, int64_t k, const int32_t* predB, int64_t ldpb, int64_t inner_off) {
    NvtxRange r("apsp.rkleene.product");
    MinplusArgs a = minplus_args();
    a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
    a.C = at(r0, c0); a.ldc = ld;
    a.idx = pat(r0, c0); a.ldi = ld;
    a.predB = predB; a.ldp = ldpb;
    a.m = m; a.n = n; a.k = k;
    a.inner_off = inner_off;
    a.mode = mode;
    a.status = st;
    launches++;
    const bool al16 = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                      (size_t(lda) * es) % 16 == 0 && (size_t(ldb) * es) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(at(r0, c0)) & 15) == 0 && (size_t(ld) * es) % 16 == 0;
    if (prep_ && al16 && bulk_store(store, k) && m % TILE_ALIGN == 0 && n % TILE_ALIGN == 0 && k % 32 == 0) {
      int rc = launch_prep_bulk(store, A, lda, B, ldb, m, n, k, prep_a(prep_), prep_b(prep_, m, k), st_);
      if (rc) return rc;
      a.Aprep = prep_a(prep_);
      a.Bprep = prep_b(prep_, m, k);
      launches += 2;
    }
    return timed_minplus(store, a, st_);
  }
  int snap_vals(int64_t r0, int64_t c0, int64_t rows, int64_t cols, char* dst = nullptr) {
    launches++;
    return launch_copy_block(store, at(r0, c0), ld, dst ? dst : sV, sld, rows, cols, s);
  }
  int snap_idx(int64_t r0, int64_t c0, int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return 0;
    launches++;
    APSP_CUDA_TRY(cudaMemcpy2DAsync(sP, size_t(sld) * 4, pat(r0, c0), size_t(ld) * 4, size_t(cols) * 4, size_t(rows),
                                    cudaMemcpyDeviceToDevice, s));
    return 0;
  }
  bool pairs() const { return aligned && s2 && sV2 && prep2 && evFork && evJoin; }
  int fork() {
    APSP_CUDA_TRY(cudaEventRecord(evFork, s));
    APSP_CUDA_TRY(cudaStreamWaitEvent(s2, evFork, 0));
    return 0;
  }
  int join() {
    APSP_CUDA_TRY(cudaEventRecord(evJoin, s2));
    APSP_CUDA_TRY(cudaStreamWaitEvent(s, evJoin, 0));
    return 0;
  }

  int64_t split(int64_t m) const {
    if (!aligned) return m / 2;
    const int64_t tiles = m / TILE_ALIGN;
    return ((tiles + 1) / 2) * TILE_ALIGN;
  }

  int leaf(int64_t lo, int64_t m) {
    if (aligned && m > 128) {
      // leaves run the lookahead schedule too (phases 1-2 of K+1 beside phase 3 of K)
      return fw_blocked_view(store, at(lo, lo), ld, pat(lo, lo), ld, m, DEFAULT_BLOCK, mode, lo, st, s, &launches,
                             sP, leafws, getenv("APSP_NO_LOOKAHEAD") ? nullptr : side_stream());
    }
    launches += int(m > 128 ? m : 1);
    return launch_block_close(store, D, ld, lo, m, P, ld, mode, lo, st, s);
  }

  // solvers.py:239-286, every block op as C <- min(C, X (x) Y) with strict-improvement argmin
  int close(int64_t lo, int64_t hi) {
    const int64_t m = hi - lo;
    if (m <= thr || (aligned && m <= TILE_ALIGN)) return leaf(lo, m);
    const int64_t mid = lo + split(m);
    const int64_t a = mid - lo, d = hi - mid;
    const bool pred = mode == IDX_PRED;
    int rc = close(lo, mid);
    if (pairs()) {
      // B <- A (x) B and C <- C (x) A read only A and their own snapshots: run them side by side
      if (!rc) rc = snap_vals(lo, mid, a, d);
      if (!rc && pred) rc = snap_idx(lo, mid, a, d);
      if (!rc) rc = snap_vals(mid, lo, d, a, sV2);
      if (!rc) rc = fork();
      if (!rc) rc = mp_on(s2, prep2, sV2, sld, at(lo, lo), ld, mid, lo, d, a, a, pat(lo, lo), ld, lo);
      if (!rc) rc = mp(at(lo, lo), ld, sV, sld, lo, mid, a, d, a, pred ? sP : nullptr, sld, lo);
      if (!rc) rc = join();
    } else {
      // B <- A (x) B   (B aliased: snapshot B values and, for pred, B's pred rows)
      if (!rc) rc = snap_vals(lo, mid, a, d);
      if (!rc && pred) rc = snap_idx(lo, mid, a, d);
      if (!rc) rc = mp(at(lo, lo), ld, sV, sld, lo, mid, a, d, a, pred ? sP : nullptr, sld, lo);
      // C <- C (x) A   (C aliased as the left operand)
      if (!rc) rc = snap_vals(mid, lo, d, a);
      if (!rc) rc = mp(sV, sld, at(lo, lo), ld, mid, lo, d, a, a, pat(lo, lo), ld, lo);
    }
    // D <- min(D, C (x) B)
    if (!rc) rc = mp(at(mid, lo), ld, at(lo, mid), ld, mid, mid, d, d, a, pat(lo, mid), ld, lo);
    if (!rc) rc = close(mid, hi);
    if (pairs()) {
      // B <- B (x) D and C <- D (x) C read only D and their own snapshots
      if (!rc) rc = snap_vals(lo, mid, a, d);
      if (!rc) rc = snap_vals(mid, lo, d, a, sV2);
      if (!rc && pred) rc = snap_idx(mid, lo, d, a);
      if (!rc) rc = fork();
      if (!rc) rc = mp_on(s2, prep2, sV, sld, at(mid, mid), ld, lo, mid, a, d, d, pat(mid, mid), ld, mid);
      if (!rc) rc = mp(at(mid, mid), ld, sV2, sld, mid, lo, d, a, d, pred ? sP : nullptr, sld, mid);
      if (!rc) rc = join();
    } else {
      // B <- B (x) D   (B aliased as the left operand)
      if (!rc) rc = snap_vals(lo, mid, a, d);
      if (!rc) rc = mp(sV, sld, at(mid, mid), ld, lo, mid, a, d, d, pat(mid, mid), ld, mid);
      // C <- D (x) C   (C aliased as the right operand)
      if (!rc) rc = snap_vals(mid, lo, d, a);
      if (!rc && pred) rc = snap_idx(mid, lo, d, a);
      if (!rc) rc = mp(at(mid, mid), ld, sV, sld, mid, lo, d, a, d, pred ? sP : nullptr, sld, mid);
    }
    // A <- min(A, B (x) C)
    if (!rc) rc = mp(at(lo, mid), ld, at(mid, lo), ld, lo, lo, a, a, d, pat(mid, lo), ld, mid);
    return rc;
  }
};

// Largest block side below the root: floor split -> ceil(N/2); aligned split -> the first
// half, ceil(tiles/2) tiles.
int64_t rk_half(int64_t N, int aligned) {
  return aligned ? ((N / TILE_ALIGN + 1) / 2) * TILE_ALIGN : N - N / 2;
}

size_t rk_extra_bytes(int64_t N, int aligned, int thr) {
  const int64_t h = rk_half(N, aligned);
  // floor split (the reference's): operand layouts for the products whose sides happen to be
  // 128-aligned (every product above the leaves when N is a power of two), which then run on
  // the bulk-staged kernels instead of the register-staged ones (n=8192: 44 -> see DESIGN.md)
  if (!aligned) return prep_bytes(h, h, h) + 512;
  const int64_t leaf = std::max<int64_t>(round_up(std::min<int64_t>(thr, N), TILE_ALIGN), TILE_ALIGN);
  // prep + prep2 (concurrent product pair), leaf FW scratch, second value snapshot (<= 8 B / cell)
  return 2 * (prep_bytes(h, h, h) + 512) + fw_scratch_bytes(leaf, TILE_ALIGN, 4) + 512 +
         size_t(h + 8) * (h + 8) * 8 + 512;
}

size_t rk_ws_bytes(int dtype, int64_t n, int aligned, int thr) {
  const int64_t N = aligned ? round_up(n, TILE_ALIGN) : n;
  const int64_t h = rk_half(N, aligned);
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  return header_bytes() + size_t(N) * N * (es + 4) + size_t(h + 8) * (h + 8) * (es + 4) + 1024 + 5 * 256 +
         rk_extra_bytes(N, aligned, thr);
}

int rkleene_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* idx, int64_t ldi, int idx_mode, int thr,
                 int aligned, int tier_req, void* ws, size_t ws_bytes, cudaStream_t s, apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  if (thr < 1) return set_error(APSP_EINVAL, "base_threshold must be >= 1, got %d", thr);
  const int64_t N = aligned ? round_up(n, TILE_ALIGN) : n;
  const int64_t h = rk_half(N, aligned);
  Scratch sc;
  int rc = sc.acquire(ws, ws_bytes, rk_ws_bytes(dtype, n, aligned, thr), s);
  if (rc) return rc;
  Header* hdr_dev = static_cast<Header*>(sc.base);
  // every region starts 256-byte aligned (odd N with the floor split would leave the int64
  // store 4 bytes off)
  auto align256 = [](char* q) {
    return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(q) + 255) & ~uintptr_t(255));
  };
  char* p = align256(static_cast<char*>(sc.base) + header_bytes());
  int32_t* P = reinterpret_cast<int32_t*>(p);
  p = align256(p + size_t(N) * N * 4);
  int32_t* sP = reinterpret_cast<int32_t*>(p);
  p = align256(p + size_t(h + 8) * (h + 8) * 4);
  char* D = p;
  p = align256(p + size_t(N) * N * (dtype == APSP_DTYPE_I64 ? 8 : 4));
  char* sV = p;
  p = align256(p + size_t(h + 8) * (h + 8) * (dtype == APSP_DTYPE_I64 ? 8 : 4) + 512);
  char* rkprep = (aligned || !getenv("APSP_RK_FLOOR_REGISTER")) ? p : nullptr;
  char* rkprep2 = aligned ? rkprep + ((prep_bytes(h, h, h) + 511) / 256) * 256 : nullptr;
  char* sV2 = aligned ? rkprep2 + ((prep_bytes(h, h, h) + 511) / 256) * 256 : nullptr;
  char* leafws = aligned ? sV2 + ((size_t(h + 8) * (h + 8) * 8 + 511) / 256) * 256 : nullptr;
  cudaStream_t s2 = (aligned && !getenv("APSP_NO_LOOKAHEAD")) ? side_stream() : nullptr;
  cudaEvent_t evs[2] = {nullptr, nullptr};
  if (s2) {
    cudaError_t e = cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      if (evs[0]) cudaEventDestroy(evs[0]);
      return set_cuda_error(e, "product-pair events", __FILE__, __LINE__);
    }
  }
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      if (e[0]) cudaEventDestroy(e[0]);
      if (e[1]) cudaEventDestroy(e[1]);
    }
  } ev_guard{evs};
  Header hdr{};
  Timer tm(s);
  rc = launch_scan(dtype, dist, ld, n, n, 0, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  const ScanResult scan = hdr.scan;
  rc = check_scan(scan);
  if (rc) return rc;
  if (scan.zero_offdiag && idx_mode == IDX_PRED && idx) {
    rc = fw_classic_impl(dtype, n, dist, ld, idx, ldi, s, info);
    if (!rc && info) info->flags |= FLAG_CLASSIC_FOR_ZERO_EDGES;
    return rc;
  }
  std::vector<int> tiers = pick_tiers(dtype, scan, tier_req, aligned != 0, n);
  if (tiers.empty()) return set_error(APSP_EINVAL, "tier %d cannot hold this input", tier_req);
  int used = -1, tried = 0, launches = 2;
  for (int tier : tiers) {
    const int store = tier_store(tier);
    if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
    if (store == STORE_I64 && dtype != APSP_DTYPE_I64) return set_error(APSP_EINVAL, "int64 tier needs int64 input");
    tried |= 1 << tier;
    APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status, 0, sizeof(Status), s));
    rc = launch_to_store(dtype, dist, ld, n, store, D, N, N, idx_mode == IDX_PRED ? P : nullptr, N, 1, s);
    if (!rc && idx_mode == IDX_VIA) rc = launch_fill_idx(P, N, N, N, -1, s);
    RK rk{store, store_elem_size(store), D, N, P, idx_mode, thr, aligned != 0, sV, sP, h, &hdr_dev->status, s};
    rk.prep = rkprep;
    rk.leafws = leafws;
    rk.prep2 = rkprep2;
    rk.sV2 = sV2;
    rk.s2 = s2;
    rk.evFork = evs[0];
    rk.evJoin = evs[1];
    if (!rc) rc = rk.close(0, N);
    bool ok = false;
    if (!rc) rc = certify(tier, store, D, N, n, n, scan, hdr_dev, hdr, s, ok);
    if (rc) return rc;
    launches += rk.launches + 3;
    if (ok) {
      used = tier;
      break;
    }
  }
  if (used < 0) {
    if (dtype == APSP_DTYPE_I32) return set_error(APSP_ERANGE, "shortest-path cost left the representable int32 range");
    return set_error(APSP_ERANGE, "no value tier could represent the result");
  }
  rc = launch_from_store(tier_store(used), D, N, n, n, dtype, dist, ld, s);
  if (!rc && idx) rc = launch_copy_idx(P, N, n, n, APSP_DTYPE_I32, idx, ldi, s);
  if (rc) return rc;
  const double ms = tm.stop();
  if (info) {
    info->tier = used;
    info->tiers_tried = tried;
    info->iterations = 0;
    info->launches = launches + 2;
    info->max_finite = hdr.cert.max_finite;
    info->relaxations = n * n * n;
    info->device_ms = ms;
    info->flags = 0;
    g_prof.collect(info);
  }
  return 0;
}

// ---- fw_squaring ----------------------------------------------------------------------------
size_t sq_ws_bytes(int dtype, int64_t n) {
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  return header_bytes() + 2 * size_t(n) * n * (es + 4) + 1024;
}

int squaring_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* via, int64_t ldv, int tier_req, void* ws,
                  size_t ws_bytes, cudaStream_t s, apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  Scratch sc;
  int rc = sc.acquire(ws, ws_bytes, sq_ws_bytes(dtype, n), s);
  if (rc) return rc;
  Header* hdr_dev = static_cast<Header*>(sc.base);
  char* p = static_cast<char*>(sc.base) + header_bytes();
  int32_t* P0 = reinterpret_cast<int32_t*>(p);
  int32_t* P1 = P0 + n * n;
  char* D0 = reinterpret_cast<char*>(P1 + n * n);
  const size_t esmax = dtype == APSP_DTYPE_I64 ? 8 : 4;
  char* D1 = D0 + size_t(n) * n * esmax;
  Header hdr{};
  Timer tm(s);
  rc = launch_scan(dtype, dist, ld, n, n, 0, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  const ScanResult scan = hdr.scan;
  rc = check_scan(scan);
  if (rc) return rc;
  std::vector<int> tiers = pick_tiers(dtype, scan, tier_req, false, n);
  if (tiers.empty()) return set_error(APSP_EINVAL, "tier %d cannot hold this input", tier_req);
  int used = -1, tried = 0, iters = 0, launches = 2;
  char* cur = D0;
  int32_t* curP = P0;
  for (int tier : tiers) {
    const int store = tier_store(tier);
    if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
    if (store == STORE_I64 && dtype != APSP_DTYPE_I64) return set_error(APSP_EINVAL, "int64 tier needs int64 input");
    tried |= 1 << tier;
    const size_t es = store_elem_size(store);
    cur = D0;
    curP = P0;
    char* nxt = D1;
    int32_t* nxtP = P1;
    APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status, 0, sizeof(Status), s));
    rc = launch_to_store(dtype, dist, ld, n, store, cur, n, n, nullptr, n, 0, s);
    if (!rc) rc = launch_fill_idx(curP, n, n, n, -1, s);
    if (rc) return rc;
    iters = 0;
    bool overflow = false;
    while (true) {
      APSP_CUDA_TRY(cudaMemcpyAsync(nxt, cur, size_t(n) * n * es, cudaMemcpyDeviceToDevice, s));
      APSP_CUDA_TRY(cudaMemcpyAsync(nxtP, curP, size_t(n) * n * 4, cudaMemcpyDeviceToDevice, s));
      APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status.changed, 0, sizeof(int32_t), s));
      MinplusArgs a = minplus_args();
      a.A = cur; a.lda = n; a.B = cur; a.ldb = n; a.C = nxt; a.ldc = n; a.idx = nxtP; a.ldi = n;
      a.predB = nullptr; a.ldp = n; a.m = n; a.n = n; a.k = n; a.inner_off = 0; a.mode = IDX_VIA;
        a.status = &hdr_dev->status;
      a.track_changed = 1;
      rc = timed_minplus(store, a, s);
      if (!rc) rc = read_header(hdr_dev, hdr, s);
      if (rc) return rc;
      launches += 4;
      iters++;
      std::swap(cur, nxt);
      std::swap(curP, nxtP);
      overflow |= hdr.status.overflow != 0;
      if (!hdr.status.changed) break;
      if (iters > n + 1) return set_error(APSP_ECONVERGE, "squaring failed to converge within %lld rounds", (long long)(n + 1));
    }
    bool ok = false;
    rc = certify(tier, store, cur, n, n, n, scan, hdr_dev, hdr, s, ok);
    if (rc) return rc;
    if (ok) {
      used = tier;
      break;
    }
  }
  if (used < 0) {
    if (dtype == APSP_DTYPE_I32) return set_error(APSP_ERANGE, "shortest-path cost left the representable int32 range");
    return set_error(APSP_ERANGE, "no value tier could represent the result");
  }
  rc = launch_from_store(tier_store(used), cur, n, n, n, dtype, dist, ld, s);
  if (!rc && via) rc = launch_copy_idx(curP, n, n, n, APSP_DTYPE_I32, via, ldv, s);
  if (rc) return rc;
  const double ms = tm.stop();
  if (info) {
    info->tier = used;
    info->tiers_tried = tried;
    info->iterations = iters;
    info->launches = launches + 2;
    info->max_finite = hdr.cert.max_finite;
    info->relaxations = int64_t(iters) * n * n * n;
    info->device_ms = ms;
    info->flags = 0;
    g_prof.collect(info);
  }
  return 0;
}

// ---- public min-plus product / accumulate ----------------------------------------------------
int minplus_impl(int dtype, int accumulate, int64_t n1, int64_t n2, int64_t n3, const void* x, int64_t ldx,
                 const void* y, int64_t ldy, void* z, int64_t ldz, int32_t* via, int64_t ldv, int64_t row_off,
                 int64_t inner_off, int64_t col_off, int tier_req, cudaStream_t s, apsp_info* info) {
  if (n1 < 1 || n2 < 1 || n3 < 1) return set_error(APSP_EDIMENSION, "min-plus operands must be non-empty");
  const size_t esmax = dtype == APSP_DTYPE_I64 ? 8 : 4;
  const size_t need = header_bytes() + (size_t(n1) * n2 + size_t(n2) * n3 + size_t(n1) * n3) * esmax + 1024;
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, need, s);
  if (rc) return rc;
  Header* hdr_dev = static_cast<Header*>(sc.base);
  char* Xs = static_cast<char*>(sc.base) + header_bytes();
  char* Ys = Xs + size_t(n1) * n2 * esmax;
  char* Zs = Ys + size_t(n2) * n3 * esmax;
  Header hdr{};
  Timer tm(s);
  // operand ranges: the tier must hold every partial sum x + y (and z)
  ScanResult sx{}, sy{}, sz{};
  rc = launch_scan(dtype, x, ldx, n1, n2, -1, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  sx = hdr.scan;
  rc = launch_scan(dtype, y, ldy, n2, n3, -1, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  sy = hdr.scan;
  if (accumulate) {
    rc = launch_scan(dtype, z, ldz, n1, n3, -1, &hdr_dev->scan, s);
    if (!rc) rc = read_header(hdr_dev, hdr, s);
    if (rc) return rc;
    sz = hdr.scan;
  }
  if (sx.negative) return set_error(APSP_ENEGATIVE, "left operand contains a negative finite cost");
  if (sy.negative) return set_error(APSP_ENEGATIVE, "right operand contains a negative finite cost");
  if (sz.negative) return set_error(APSP_ENEGATIVE, "accumulator contains a negative finite cost");
  const bool integral = dtype != APSP_DTYPE_F32 || !(sx.non_integral || sy.non_integral || sz.non_integral);
  const int64_t sum = std::max<int64_t>(sx.max_finite + sy.max_finite, sz.max_finite);
  int tier = tier_req;
  if (tier >= 0) {
    // A forced tier must hold every partial sum exactly: the product has no certificate pass,
    // so a narrower store would silently wrap a cost (e.g. 300 -> 44 in u8).
    const bool int_tier = tier == APSP_TIER_U8 || tier == APSP_TIER_U16 || tier == APSP_TIER_W32 ||
                          tier == APSP_TIER_I32;
    bool fits = tier == APSP_TIER_F32 ? dtype == APSP_DTYPE_F32
              : tier == APSP_TIER_I64 ? dtype == APSP_DTYPE_I64
              : tier == APSP_TIER_I32 ? dtype != APSP_DTYPE_F32 && sum <= tier_limit(tier)
              : int_tier && integral && sum <= tier_limit(tier);
    if (!fits)
      return set_error(APSP_EINVAL, "forced tier %d cannot hold the operands exactly (max partial sum %lld)", tier,
                       (long long)sum);
  }
  if (tier < 0) {
    if (integral && sum <= U8_INF - 1) tier = APSP_TIER_U8;
    else if (integral && sum <= W32_INF - 1) tier = APSP_TIER_W32;
    else if (dtype == APSP_DTYPE_F32) tier = APSP_TIER_F32;
    else if (dtype == APSP_DTYPE_I32) tier = APSP_TIER_I32;
    else tier = APSP_TIER_I64;
  }
  const int store = tier_store(tier);
  if (store < 0 || store == STORE_U16) return set_error(APSP_EINVAL, "tier %d not available for products", tier);
  rc = launch_to_store_rect(dtype, x, ldx, n1, n2, store, Xs, n2, s);
  if (!rc) rc = launch_to_store_rect(dtype, y, ldy, n2, n3, store, Ys, n3, s);
  if (rc) return rc;
  if (accumulate) {
    rc = launch_to_store_rect(dtype, z, ldz, n1, n3, store, Zs, n3, s);
  } else {
    // product: C starts at Infinity, via at None (_product_band fills dist/via per row, minplus.py:84-88)
    rc = launch_to_store_rect(dtype, nullptr, 0, n1, n3, store, Zs, n3, s);
    if (!rc && via) rc = launch_fill_idx(via, ldv, n1, n3, -1, s);
  }
  if (rc) return rc;
  APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status, 0, sizeof(Status), s));
  MinplusArgs a = minplus_args();
  a.A = Xs; a.lda = n2; a.B = Ys; a.ldb = n3; a.C = Zs; a.ldc = n3; a.idx = via; a.ldi = ldv;
  a.predB = nullptr; a.ldp = 0; a.m = n1; a.n = n3; a.k = n2; a.inner_off = inner_off; a.mode = IDX_VIA;
  a.status = &hdr_dev->status;
  rc = timed_minplus(store, a, s);
  if (!rc && !accumulate && via)
    rc = launch_witness_clear(store, Xs, n2, Ys, n3, Zs, n3, via, ldv, n1, n2, n3, row_off, inner_off, col_off, s);
  if (!rc) rc = launch_max_finite(store, Zs, n3, n1, n3, &hdr_dev->cert, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  if (tier == APSP_TIER_I64 && hdr.cert.max_finite > MAX_FINITE_COST)
    return set_error(APSP_ERANGE, "product cost left the representable finite range");
  rc = launch_from_store(store, Zs, n3, n1, n3, dtype, z, ldz, s);
  if (rc) return rc;
  const double ms = tm.stop();
  if (info) {
    info->tier = tier;
    info->tiers_tried = 1 << tier;
    info->iterations = 0;
    info->launches = 8;
    info->max_finite = hdr.cert.max_finite;
    info->relaxations = n1 * n2 * n3;
    info->device_ms = ms;
    info->flags = 0;
    g_prof.collect(info);
  }
  return 0;
}


}  // namespace apsp
