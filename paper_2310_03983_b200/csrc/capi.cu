// C ABI and native orchestration: blocked FW rounds, R-Kleene recursion, squaring loop,
// min-plus products, value-tier selection and certification, host-level entry.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <vector>
#include "../../include/apsp_b200.h"
#include "launch.h"
#include <nvtx3/nvToolsExt.h>

namespace apsp {
const char* last_error();
long long launch_count();
}

using namespace apsp;

namespace {

constexpr int DEFAULT_BLOCK = 128;
constexpr int TILE_ALIGN = 128;

// Opt-in event timing of the min-plus tile launches (apsp_set_profiling).
struct Profiler {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  size_t used = 0;
  void reset() { used = 0; }
  void begin(cudaStream_t s) {
    if (!on) return;
    if (used == ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      ev.emplace_back(a, b);
    }
    cudaEventRecord(ev[used].first, s);
  }
  void end(cudaStream_t s) {
    if (!on) return;
    cudaEventRecord(ev[used].second, s);
    used++;
  }
  // after the stream is synchronised
  void collect(apsp_info* info) {
    if (!info) return;
    double ms = 0;
    for (size_t i = 0; i < used; i++) {
      float t = 0;
      cudaEventElapsedTime(&t, ev[i].first, ev[i].second);
      ms += t;
    }
    info->kernel_launches = int32_t(used);
    info->kernel_ms = ms;
  }
};
thread_local Profiler g_prof;

int timed_minplus(int store, const MinplusArgs& a, cudaStream_t s) {
  g_prof.begin(s);
  const int rc = launch_minplus(store, a, s);
  g_prof.end(s);
  return rc;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

int tier_store(int tier) {
  switch (tier) {
    case APSP_TIER_U8: return STORE_U8;
    case APSP_TIER_U16: return STORE_U16;
    case APSP_TIER_W32: return STORE_W32;
    case APSP_TIER_I32: return STORE_I32;
    case APSP_TIER_F32: return STORE_F32;
    case APSP_TIER_I64: return STORE_I64;
  }
  return -1;
}

// Largest finite value a tier can hold.  A result is certified exact when
// max_finite + w_max <= limit: every cell with true distance <= limit is computed exactly
// (all partial sums of its shortest path are <= it), and a reachable cell beyond the limit
// would force a cell within (limit - w_max, limit] along its shortest path.
int64_t tier_limit(int tier) {
  switch (tier) {
    case APSP_TIER_U8: return U8_INF - 1;
    case APSP_TIER_U16: return U16_INF - 1;
    case APSP_TIER_W32: return W32_INF - 1;
    case APSP_TIER_I32: return INF32 - 1;
    case APSP_TIER_I64: return MAX_FINITE_COST;
  }
  return INT64_MAX;
}

// Keep freed stream-ordered allocations in the device pool across calls (the default
// release threshold of 0 returns them to the driver at every synchronisation).
// The library's scratch comes from the device's default stream-ordered pool; keep freed blocks
// reserved (release threshold = max) so repeated solves do not remap GBs of workspace.
void keep_pool() {
  static std::atomic<bool> done[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || done[dev].load()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[dev].store(true);
}

struct Scratch {
  void* base = nullptr;
  bool owned = false;
  cudaStream_t s = nullptr;
  ~Scratch() {
    if (owned && base) cudaFreeAsync(base, s);
  }
  int acquire(void* ws, size_t ws_bytes, size_t need, cudaStream_t st) {
    s = st;
    if (ws) {
      if (ws_bytes < need) return set_error(APSP_EINVAL, "workspace too small: %zu < %zu bytes", ws_bytes, need);
      base = ws;
      return 0;
    }
    keep_pool();
    APSP_CUDA_TRY(cudaMallocAsync(&base, need, st));
    owned = true;
    return 0;
  }
};

struct Header {   // first 256 bytes of every workspace
  Status status;
  ScanResult scan;
  ScanResult cert;
};

int read_header(Header* dev, Header& host, cudaStream_t s) {
  APSP_CUDA_TRY(cudaMemcpyAsync(&host, dev, sizeof(Header), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

int check_scan(const ScanResult& sc) {
  if (sc.negative) return set_error(APSP_ENEGATIVE, "solver input contains a negative finite cost");
  if (sc.diag_nonzero) return set_error(APSP_EDIAGONAL, "solver input must have a zero diagonal");
  return 0;
}

// Bulk-staged (pre-laid-out panel) products for this tier and inner length k.  The exact fp32
// kernel (1 CTA / SM, compare-select) only pays off on long products: k >= 256 (measured
// n=8192 FW 119 vs 126 ms; at k = 128 the 64 x 64 register-staged kernel is faster).
int64_t kF32MinK = getenv("APSP_F32_MINK") ? atoll(getenv("APSP_F32_MINK")) : 128;
bool bulk_store(int store, int64_t k) {
  static const bool f32 = !getenv("APSP_F32_BULK") || atoi(getenv("APSP_F32_BULK")) != 0;
  return store == STORE_U8 || store == STORE_U16 || store == STORE_W32 || (store == STORE_F32 && f32 && k >= kF32MinK);
}

// Candidate tiers, narrowest first.  allow_u16: the caller runs only aligned products (the
// u16 tier exists only as bulk-staged tiles).
std::vector<int> pick_tiers(int dtype, const ScanResult& sc, int forced, bool allow_u16, int64_t n_vert) {
  const bool integral = dtype != APSP_DTYPE_F32 || !sc.non_integral;
  const int64_t w = sc.max_finite;
  if (forced >= 0) {
    // a forced tier must be able to hold the input (the certificate covers the result)
    bool fits = forced == APSP_TIER_U8 ? integral && w <= U8_INF - 1
              : forced == APSP_TIER_U16 ? allow_u16 && integral && w <= U16_INF - 1
              : forced == APSP_TIER_W32 ? integral && w <= W32_INF - 1
              : forced == APSP_TIER_I32 ? (dtype != APSP_DTYPE_F32 && w <= INF32 - 1)
              : forced == APSP_TIER_F32 ? dtype == APSP_DTYPE_F32
              : forced == APSP_TIER_I64 ? dtype == APSP_DTYPE_I64 : false;
    if (!fits) return {};
    return {forced};
  }
  // Skip narrow tiers whose certificate would almost surely fail: on random-like graphs the
  // largest distance grows like w_max * ln(n) / ln(average degree), with a larger constant on
  // very sparse graphs (degree < 8: the diameter's long tails; fitted on the generator sweep,
  // profiles/r01_configs_sparse.json).  The estimate only picks the starting tier; the
  // certificate still decides exactness.
  const double n = n_vert > 0 ? double(n_vert) : 1.0;
  const double deg = std::max(double(sc.finite_offdiag) / n, 1.5);
  const double m_est = (deg < 8.0 ? 0.8 : 0.5) * double(w) * std::log(std::max(n, 2.0)) / std::log(deg);
  std::vector<int> t;
  if (integral && w <= U8_INF - 1 && m_est + w <= U8_INF - 1) t.push_back(APSP_TIER_U8);
  if (allow_u16 && integral && w <= U16_INF - 1 && m_est + w <= U16_INF - 1) t.push_back(APSP_TIER_U16);
  if (integral && w <= W32_INF - 1) t.push_back(APSP_TIER_W32);
  if (dtype == APSP_DTYPE_F32) t.push_back(APSP_TIER_F32);
  else if (dtype == APSP_DTYPE_I32) t.push_back(APSP_TIER_I32);
  else t.push_back(APSP_TIER_I64);
  return t;
}

size_t header_bytes() { return 256; }

// ---- blocked FW on an m x m view (m multiple of b) -------------------------------------
//
// Round K (pivot block [k0, k0+b)):
//   phase 1  close the diagonal block in classic k order (block_close; b > 128: blocked FW
//            on the b x b sub-view)
//   phase 2  row panel <- Dg (x) row panel, column panel <- column panel (x) Dg: one min-plus
//            product each against the CLOSED diagonal block (equal distances to the classic
//            in-block k loop); pred of the row panel is read from a snapshot because the
//            product rewrites those rows
//   phase 3  every other tile: C <- min(C, colpanel (x) rowpanel), pred <- pred[k*][j]
// Lookahead: phase 3 of round K is split into (3a) the tiles of pivot cross K+1 and (3b) the
// rest; phases 1-2 of round K+1 run on a high-priority side stream concurrently with 3b.
// 3b never touches cross K+1 and phases 1-2 of K+1 never touch cross K, so the overlap is
// race-free; round K+1's 3a waits for both.
struct FwCtx {
  int store = 0;
  size_t es = 1;
  char* D = nullptr;
  int64_t ld = 0;
  int32_t* P = nullptr;
  int64_t ldp = 0;
  int64_t m = 0;
  int b = 128;
  int mode = IDX_PRED;
  int64_t via_off = 0;
  Status* st = nullptr;
  cudaStream_t side = nullptr;   // nullptr: no lookahead
  int32_t* predsnap = nullptr;   // b x m
  char* rowsnap = nullptr;       // b x m values (b > 128 only)
  char* colsnap = nullptr;       // m x b values (b > 128 only)
  char* prep[2] = {nullptr, nullptr};  // narrow tiers: bulk-copy layouts of the panels, by round parity
  char* p2prep = nullptr;        // narrow tiers: bulk-copy layouts of the phase-2 operands
  char* sub = nullptr;           // scratch of the phase-1 sub-run when b > 128
  int launches = 0;
};

size_t fw_scratch_bytes(int64_t m, int b, size_t es) {
  size_t v = size_t(b) * m * 4 + 256;                      // pred row-panel snapshot
  if (b > TILE_ALIGN) v += 2 * size_t(b) * m * es + 256;   // value snapshots (non-narrow tiers)
  v += 2 * (prep_bytes(m, m, b) + 256);                 // phase-3 panel layouts (double buffered)
  v += prep_bytes(m, b, b) + 256;                       // phase-2 layouts (max of row/col product)
  if (b > TILE_ALIGN) v += fw_scratch_bytes(b, TILE_ALIGN, es) + 256;   // phase-1 sub-run
  return v;
}

// carve the scratch of fw_scratch_bytes
void fw_carve(FwCtx& c, char* scratch, int64_t N) {
  char* p = scratch;
  c.predsnap = reinterpret_cast<int32_t*>(p);
  p += size_t(c.b) * N * 4 + 256;
  if (c.b > TILE_ALIGN) {
    c.rowsnap = p;
    c.colsnap = p + size_t(c.b) * N * c.es + 128;
    p += 2 * size_t(c.b) * N * c.es + 256;
  }
  for (int q = 0; q < 2; q++) {
    c.prep[q] = p;
    p += prep_bytes(N, N, c.b) + 256;
  }
  c.p2prep = p;
  p += prep_bytes(N, c.b, c.b) + 256;
  if (c.b > TILE_ALIGN) c.sub = p;
}

uint32_t* prep_a(char* slot) { return reinterpret_cast<uint32_t*>(slot); }
uint16_t* prep_b(char* slot, int64_t m, int64_t k) {
  return reinterpret_cast<uint16_t*>(slot + ((size_t(m) * k * 4 + 255) / 256) * 256);
}

int fw_run(FwCtx& c, cudaStream_t s);

// ---- CUDA-graph replay of a solve's device schedule ----------------------------------------
// Between the input scan and the certificate a solve is a fixed chain of launches (FW rounds
// with their lookahead fork/join, or the R-Kleene recursion).  Repeated solves of one shape on
// the same buffers (iterative workloads, benchmarks) replay it as one CUDA graph: the second
// solve with a given key captures the chain, later ones launch the instantiated graph, which
// removes the per-launch gaps that dominate small n.  APSP_NO_GRAPHS=1 disables it; profiling
// (per-launch events) always runs the plain chain.
struct GraphKey {
  int dev, kind, store, mode;
  int64_t N, b;
  const void *D, *P, *scratch, *extra;
  cudaStream_t s;
  bool operator==(const GraphKey& o) const {
    return dev == o.dev && kind == o.kind && store == o.store && mode == o.mode && N == o.N && b == o.b &&
           D == o.D && P == o.P && scratch == o.scratch && extra == o.extra && s == o.s;
  }
};
struct GraphEntry {
  GraphKey key{};
  bool valid = false;
  cudaGraphExec_t exec = nullptr;   // null: seen once, not captured yet
  long long launches = 0;
};
constexpr int GRAPH_SLOTS = 8;
std::mutex g_graph_mu;
GraphEntry g_graphs[GRAPH_SLOTS];
int g_graph_next = 0;

bool graphs_enabled() {
  static const bool on = !getenv("APSP_NO_GRAPHS");
  return on;
}

// Private per-device stream the graphs are captured on and launched from (the caller's stream
// may be the legacy default stream, which cannot be captured).  It is ordered after everything
// already queued on the caller's stream, and the caller's stream after the graph.
cudaStream_t graph_stream() {
  static cudaStream_t streams[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) return nullptr;
  return streams[dev];
}

int stream_after(cudaStream_t later, cudaStream_t earlier) {
  cudaEvent_t e;
  APSP_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaError_t r = cudaEventRecord(e, earlier);
  if (r == cudaSuccess) r = cudaStreamWaitEvent(later, e, 0);
  cudaEventDestroy(e);
  if (r != cudaSuccess) return set_cuda_error(r, "stream ordering", __FILE__, __LINE__);
  return 0;
}

// Runs body(s) directly, or captures / replays it as a graph per the cache.  Launch counts of
// a replay are credited from the capture.
template <typename F>
int run_graphed(const GraphKey& key, cudaStream_t s, F&& body) {
  cudaStream_t gs = graphs_enabled() && !g_prof.on ? graph_stream() : nullptr;
  if (!gs) return body(s);
  GraphEntry* hit = nullptr;
  cudaGraphExec_t exec = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_graph_mu);
    for (auto& e : g_graphs)
      if (e.valid && e.key == key) hit = &e;
    if (hit && hit->exec) {
      exec = hit->exec;
      const long long n = hit->launches;
      int rc = stream_after(gs, s);
      if (!rc && cudaGraphLaunch(exec, gs) != cudaSuccess) rc = set_error(APSP_ECUDA, "graph launch");
      if (!rc) rc = stream_after(s, gs);
      if (!rc) count_launches(n);
      return rc;
    }
    if (!hit) {   // first sighting: remember the key, run plainly
      GraphEntry& e = g_graphs[g_graph_next];
      g_graph_next = (g_graph_next + 1) % GRAPH_SLOTS;
      if (e.exec) cudaGraphExecDestroy(e.exec);
      e = GraphEntry{};
      e.key = key;
      e.valid = true;
    }
  }
  if (!hit) return body(s);
  // second sighting: capture on the private stream, instantiate, launch
  int rc = stream_after(gs, s);
  if (rc) return rc;
  const long long before = launch_count();
  APSP_CUDA_TRY(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
  rc = body(gs);
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(gs, &g);
  if (rc || ec != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    if (rc) return rc;
    return set_cuda_error(ec, "graph capture", __FILE__, __LINE__);
  }
  const cudaError_t ei = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (ei != cudaSuccess) return set_cuda_error(ei, "graph instantiate", __FILE__, __LINE__);
  if (cudaGraphLaunch(exec, gs) != cudaSuccess) {
    cudaGraphExecDestroy(exec);
    return set_error(APSP_ECUDA, "graph launch");
  }
  rc = stream_after(s, gs);
  std::lock_guard<std::mutex> lock(g_graph_mu);
  for (auto& e : g_graphs)
    if (e.valid && e.key == key && !e.exec) {
      e.exec = exec;
      e.launches = launch_count() - before;
      return rc;
    }
  cudaGraphExecDestroy(exec);   // slot recycled meanwhile (released once the launch completes)
  return rc;
}

// NVTX ranges name the phases for nsys/ncu (`ncu --nvtx --nvtx-include "apsp.fw.phase3/"`).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

int fw_phase1(FwCtx& c, int64_t k0, cudaStream_t s) {
  NvtxRange r("apsp.fw.phase1");
  c.launches++;
  if (c.b <= TILE_ALIGN)
    return launch_block_close(c.store, c.D, c.ld, k0, c.b, c.P, c.ldp, c.mode, c.via_off + k0, c.st, s);
  FwCtx sub = c;
  sub.D = c.D + (k0 * c.ld + k0) * c.es;
  sub.P = c.P ? c.P + k0 * c.ldp + k0 : nullptr;
  sub.m = c.b;
  sub.b = TILE_ALIGN;
  sub.via_off = c.via_off + k0;
  sub.side = nullptr;
  sub.rowsnap = sub.colsnap = nullptr;
  sub.prep[0] = sub.prep[1] = sub.p2prep = sub.sub = nullptr;
  if (c.sub) fw_carve(sub, c.sub, c.b);
  sub.launches = 0;
  const int rc = fw_run(sub, s);
  c.launches += sub.launches;
  return rc;
}

int fw_phase2(FwCtx& c, int64_t k0, cudaStream_t s) {
  NvtxRange r("apsp.fw.phase2");
  const int64_t b = c.b, m = c.m;
  char* Dg = c.D + (k0 * c.ld + k0) * c.es;
  char* rowp = c.D + k0 * c.ld * c.es;
  char* colp = c.D + k0 * c.es;
  const bool nt = bulk_store(c.store, c.b) && c.p2prep;   // bulk-staged tiles (prep = snapshot)
  const bool snap = !nt && b > TILE_ALIGN;
  if (c.P && c.mode == IDX_PRED) {
    APSP_CUDA_TRY(cudaMemcpy2DAsync(c.predsnap, size_t(m) * 4, c.P + k0 * c.ldp, size_t(c.ldp) * 4, size_t(m) * 4,
                                    size_t(b), cudaMemcpyDeviceToDevice, s));
  }
  int rc = 0;
  if (nt && c.prep[0]) {
    // Both panels in ONE cross-list launch: the tiles of the pivot row band compute
    // Dg (x) row panel and those of the pivot column band column panel (x) Dg, because the
    // A / B layouts are the full column / row panels (their pivot rows / columns are Dg).  The
    // diagonal tiles compute Dg (x) Dg, which never strictly improves a closed block.  The
    // layouts live in this round's phase-3 slot (free: its last reader, phase 3 two rounds
    // back, is ordered before us) and are rebuilt from the updated panels right after.
    char* slot = c.prep[(k0 / b) & 1];
    rc = launch_prep_bulk(c.store, colp, c.ld, rowp, c.ld, m, m, b, prep_a(slot), prep_b(slot, m, b), s);
    if (rc) return rc;
    MinplusArgs x = minplus_args();
    x.A = colp; x.lda = c.ld;
    x.B = rowp; x.ldb = c.ld;
    x.C = c.D; x.ldc = c.ld;
    x.idx = c.P; x.ldi = c.ldp;
    x.predB = c.predsnap; x.ldp = m;
    x.m = m; x.n = m; x.k = b;
    x.inner_off = c.via_off + k0;
    x.mode = c.mode;
    x.only_lo = k0; x.only_hi = k0 + b;
    x.status = c.st;
    x.Aprep = prep_a(slot);
    x.Bprep = prep_b(slot, m, b);
    c.launches += 5;
    rc = launch_minplus(c.store, x, s);
    if (rc) return rc;
    return launch_prep_bulk(c.store, colp, c.ld, rowp, c.ld, m, m, b, prep_a(slot), prep_b(slot, m, b), s);
  }
  if (snap) {
    rc = launch_copy_block(c.store, rowp, c.ld, c.rowsnap, m, b, m, s);
    if (!rc) rc = launch_copy_block(c.store, colp, c.ld, c.colsnap, b, m, b, s);
    if (rc) return rc;
  }
  MinplusArgs a = minplus_args();
  a.A = Dg; a.lda = c.ld;
  a.B = snap ? c.rowsnap : rowp; a.ldb = snap ? m : c.ld;
  a.C = rowp; a.ldc = c.ld;
  a.idx = c.P ? c.P + k0 * c.ldp : nullptr; a.ldi = c.ldp;
  a.predB = c.predsnap; a.ldp = m;
  a.m = b; a.n = m; a.k = b;
  a.inner_off = c.via_off + k0;
  a.mode = c.mode;
  a.skip_col_lo = k0; a.skip_col_hi = k0 + b;
  a.status = c.st;
  if (nt) {
    rc = launch_prep_bulk(c.store, Dg, c.ld, rowp, c.ld, b, m, b, prep_a(c.p2prep), prep_b(c.p2prep, b, b), s);
    if (rc) return rc;
    a.Aprep = prep_a(c.p2prep);
    a.Bprep = prep_b(c.p2prep, b, b);
    c.launches += 2;
  }
  rc = launch_minplus(c.store, a, s);
  if (rc) return rc;
  MinplusArgs q = minplus_args();
  q.A = snap ? c.colsnap : colp; q.lda = snap ? b : c.ld;
  q.B = Dg; q.ldb = c.ld;
  q.C = colp; q.ldc = c.ld;
  q.idx = c.P ? c.P + k0 : nullptr; q.ldi = c.ldp;
  q.predB = c.P ? c.P + k0 * c.ldp + k0 : nullptr; q.ldp = c.ldp;
  q.m = m; q.n = b; q.k = b;
  q.inner_off = c.via_off + k0;
  q.mode = c.mode;
  q.skip_row_lo = k0; q.skip_row_hi = k0 + b;
  q.status = c.st;
  if (nt) {
    rc = launch_prep_bulk(c.store, colp, c.ld, Dg, c.ld, m, b, b, prep_a(c.p2prep), prep_b(c.p2prep, m, b), s);
    if (rc) return rc;
    q.Aprep = prep_a(c.p2prep);
    q.Bprep = prep_b(c.p2prep, m, b);
    c.launches += 2;
  }
  c.launches += 2;
  rc = launch_minplus(c.store, q, s);
  if (rc || !c.prep[0] || !bulk_store(c.store, c.b)) return rc;
  char* slot = c.prep[(k0 / b) & 1];
  c.launches += 2;
  return launch_prep_bulk(c.store, colp, c.ld, rowp, c.ld, m, m, b, prep_a(slot), prep_b(slot, m, b), s);
}

// phase 3 of pivot block k0; only_next >= 0 restricts to cross only_next, skip_next >= 0
// additionally skips cross skip_next.
int fw_phase3(FwCtx& c, int64_t k0, int64_t only_next, int64_t skip_next, cudaStream_t s) {
  NvtxRange r(only_next >= 0 ? "apsp.fw.phase3a" : skip_next >= 0 ? "apsp.fw.phase3b" : "apsp.fw.phase3");
  MinplusArgs a = minplus_args();
  a.A = c.D + k0 * c.es; a.lda = c.ld;
  a.B = c.D + k0 * c.ld * c.es; a.ldb = c.ld;
  a.C = c.D; a.ldc = c.ld;
  a.idx = c.P; a.ldi = c.ldp;
  a.predB = c.P ? c.P + k0 * c.ldp : nullptr; a.ldp = c.ldp;
  a.m = c.m; a.n = c.m; a.k = c.b;
  a.inner_off = c.via_off + k0;
  a.mode = c.mode;
  a.skip_row_lo = k0; a.skip_row_hi = k0 + c.b;
  a.skip_col_lo = k0; a.skip_col_hi = k0 + c.b;
  if (only_next >= 0) { a.only_lo = only_next; a.only_hi = only_next + c.b; }
  if (skip_next >= 0) {   // 3b: disjoint from the 3a launch queued just before it
    a.skip2_lo = skip_next; a.skip2_hi = skip_next + c.b;
    a.pdl = getenv("APSP_NO_PDL") ? 0 : 1;
  }
  a.status = c.st;
  if (c.prep[0] && bulk_store(c.store, c.b)) {
    char* slot = c.prep[(k0 / c.b) & 1];
    a.Aprep = prep_a(slot);
    a.Bprep = prep_b(slot, c.m, c.b);
  }
  c.launches++;
  return timed_minplus(c.store, a, s);
}

int fw_run(FwCtx& c, cudaStream_t s) {
  const int64_t b = c.b;
  int rc = fw_phase1(c, 0, s);
  if (!rc) rc = fw_phase2(c, 0, s);
  if (rc) return rc;
  cudaEvent_t evA = nullptr, evB = nullptr;
  if (c.side) {
    cudaError_t e = cudaEventCreateWithFlags(&evA, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&evB, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      if (evA) cudaEventDestroy(evA);
      return set_cuda_error(e, "lookahead events", __FILE__, __LINE__);
    }
  }
  for (int64_t k0 = 0; !rc && k0 < c.m; k0 += b) {
    const int64_t k1 = k0 + b;
    if (k1 >= c.m) {
      rc = fw_phase3(c, k0, -1, -1, s);
    } else if (c.side) {
      rc = fw_phase3(c, k0, k1, -1, s);                       // 3a: next pivot cross
      if (!rc && cudaEventRecord(evA, s) != cudaSuccess) rc = set_error(APSP_ECUDA, "event record");
      if (!rc && cudaStreamWaitEvent(c.side, evA, 0) != cudaSuccess) rc = set_error(APSP_ECUDA, "stream wait");
      if (!rc) rc = fw_phase1(c, k1, c.side);
      if (!rc) rc = fw_phase2(c, k1, c.side);
      if (!rc && cudaEventRecord(evB, c.side) != cudaSuccess) rc = set_error(APSP_ECUDA, "event record");
      if (!rc) rc = fw_phase3(c, k0, -1, k1, s);               // 3b: the rest
      if (!rc && cudaStreamWaitEvent(s, evB, 0) != cudaSuccess) rc = set_error(APSP_ECUDA, "stream wait");
    } else {
      rc = fw_phase3(c, k0, -1, -1, s);
      if (!rc) rc = fw_phase1(c, k1, s);
      if (!rc) rc = fw_phase2(c, k1, s);
    }
  }
  if (evA) cudaEventDestroy(evA);
  if (evB) cudaEventDestroy(evB);
  return rc;
}

// High-priority side stream of the current device (created once per device, thread-safe).
cudaStream_t side_stream() {
  static cudaStream_t streams[64] = {};
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!streams[dev]) {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&streams[dev], cudaStreamNonBlocking, hi) != cudaSuccess) return nullptr;
  }
  return streams[dev];
}

// convenience for callers with a plain view (R-Kleene leaves): lookahead when `side` is given;
// scratch laid out by fw_carve (fw_scratch_bytes(m, b, es) bytes) or, if null, only a pred
// snapshot
int fw_blocked_view(int store, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t m, int b, int mode,
                    int64_t via_off, Status* st, cudaStream_t s, int* launches, int32_t* predsnap,
                    char* scratch = nullptr, cudaStream_t side = nullptr) {
  FwCtx c;
  c.store = store; c.es = store_elem_size(store);
  c.D = static_cast<char*>(D); c.ld = ld; c.P = P; c.ldp = ldp;
  c.m = m; c.b = b; c.mode = mode; c.via_off = via_off; c.st = st;
  c.side = side;
  if (scratch) fw_carve(c, scratch, m);
  else c.predsnap = predsnap;
  const int rc = fw_run(c, s);
  *launches += c.launches;
  return rc;
}

int certify(int tier, int store, const void* D, int64_t ld, int64_t rows, int64_t cols, const ScanResult& sc,
            Header* hdr_dev, Header& hdr, cudaStream_t s, bool& ok) {
  int rc = launch_max_finite(store, D, ld, rows, cols, &hdr_dev->cert, s);
  if (rc) return rc;
  rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  ok = true;
  if (hdr.status.overflow) {
    if (tier == APSP_TIER_I64) return set_error(APSP_ERANGE, "shortest-path cost left the representable finite range");
    ok = false;
  }
  if (tier == APSP_TIER_F32) return 0;
  const int64_t M = hdr.cert.max_finite;
  if (M >= 0 && M + sc.max_finite > tier_limit(tier)) {
    if (tier == APSP_TIER_I64) {
      if (M > MAX_FINITE_COST) return set_error(APSP_ERANGE, "shortest-path cost left the representable finite range");
    } else {
      ok = false;
    }
  }
  return 0;
}

struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    g_prof.reset();
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  double stop() {
    float ms = 0;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

int fw_classic_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, cudaStream_t s,
                    apsp_info* info);

// Zero-cost edges let equal-distance vertices point at each other when many cells are
// relaxed at once (blocked phase 3, R-Kleene products); only the classic k order keeps the
// predecessor graph a tree then.  Such inputs are solved by the classic kernel, which is
// bit-exact with the reference for both dist and pred.
constexpr int32_t FLAG_CLASSIC_FOR_ZERO_EDGES = 1;

// Pivot block by size (measured on B200, profiles/r01_summary.md): small n is bound by the
// phase-1 chain (b = 128), large n by per-tile overheads that a longer k amortises
// (n=16384: b=1024 145 ms vs 256 161 ms; n=32768: b=2048).  Padding waste is kept below ~1%.
int default_block(int64_t n) {
  int b = n <= 6144 ? 128 : n <= 12288 ? 256 : n <= 24576 ? 1024 : 2048;
  while (b > 128 && double(round_up(n, b)) > 1.01 * double(round_up(n, 128))) b /= 2;
  return b;
}

size_t fw_ws_bytes(int dtype, int64_t n, int block) {
  const int64_t N = round_up(std::max<int64_t>(n, 1), block);
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  return header_bytes() + size_t(N) * N * (es + 4) + 256 + fw_scratch_bytes(N, block, es);
}

int fw_blocked_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, int b, int tier_req,
                    void* ws, size_t ws_bytes, cudaStream_t s, apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  if (b <= 0) b = default_block(n);
  if (b % 128 || b < 128 || b > 4096) return set_error(APSP_EINVAL, "blocked FW block must be a multiple of 128 in [128, 4096] (got %d)", b);
  const int64_t N = round_up(n, b);
  Scratch sc;
  int rc = sc.acquire(ws, ws_bytes, fw_ws_bytes(dtype, n, b), s);
  if (rc) return rc;
  Header* hdr_dev = static_cast<Header*>(sc.base);
  int32_t* P = reinterpret_cast<int32_t*>(static_cast<char*>(sc.base) + header_bytes());
  char* D = reinterpret_cast<char*>(P) + size_t(N) * N * 4;
  char* scratch = D + size_t(N) * N * (dtype == APSP_DTYPE_I64 ? 8 : 4) + 256;
  Header hdr{};
  Timer tm(s);
  rc = launch_scan(dtype, dist, ld, n, n, 0, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  const ScanResult scan = hdr.scan;
  rc = check_scan(scan);
  if (rc) return rc;
  if (scan.zero_offdiag && pred) {
    rc = fw_classic_impl(dtype, n, dist, ld, pred, ldp, s, info);
    if (!rc && info) info->flags |= FLAG_CLASSIC_FOR_ZERO_EDGES;
    return rc;
  }
  std::vector<int> tiers = pick_tiers(dtype, scan, tier_req, true, n);
  if (tiers.empty()) return set_error(APSP_EINVAL, "tier %d cannot hold this input", tier_req);
  // no padding: solve straight into the caller's pred matrix (saves an N^2 int32 copy)
  int32_t* Pw = P;
  int64_t ldpw = N;
  if (pred && N == n && ldp >= n && ldp % 4 == 0 && (reinterpret_cast<uintptr_t>(pred) & 15) == 0) {
    Pw = pred;
    ldpw = ldp;
  }
  int launches = 2, used = -1, tried = 0;
  for (int tier : tiers) {
    const int store = tier_store(tier);
    if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
    if (store == STORE_I64 && dtype != APSP_DTYPE_I64) return set_error(APSP_EINVAL, "int64 tier needs int64 input");
    tried |= 1 << tier;
    APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status, 0, sizeof(Status), s));
    rc = launch_to_store(dtype, dist, ld, n, store, D, N, N, Pw, ldpw, 1, s);
    if (!rc) {
      FwCtx c;
      c.store = store; c.es = store_elem_size(store);
      c.D = D; c.ld = N; c.P = Pw; c.ldp = ldpw; c.m = N; c.b = b; c.mode = IDX_PRED; c.via_off = 0;
      c.st = &hdr_dev->status;
      c.side = getenv("APSP_NO_LOOKAHEAD") ? nullptr : side_stream();
      fw_carve(c, scratch, N);
      if (getenv("APSP_NO_BULK")) c.prep[0] = c.prep[1] = nullptr;
      // graph replay only where launch gaps dominate (N <= 2048): a graph drops the lookahead
      // stream's priority, which costs more than the gaps at larger N (n=8192 21.6 -> 25 ms)
      if (N <= 2048) {
        int dev = 0;
        cudaGetDevice(&dev);
        const GraphKey key{dev, 1, store, c.mode, N, b, D, Pw, scratch, c.side, s};
        rc = run_graphed(key, s, [&](cudaStream_t st) { return fw_run(c, st); });
      } else {
        rc = fw_run(c, s);
      }
      launches += c.launches;
    }
    bool ok = false;
    if (!rc) rc = certify(tier, store, D, N, n, n, scan, hdr_dev, hdr, s, ok);
    if (rc) return rc;
    launches += 2;
    if (ok) {
      used = tier;
      break;
    }
  }
  if (used < 0) {
    if (dtype == APSP_DTYPE_I32)
      return set_error(APSP_ERANGE, "shortest-path cost left the representable int32 range");
    return set_error(APSP_ERANGE, "no value tier could represent the result");
  }
  rc = launch_from_store(tier_store(used), D, N, n, n, dtype, dist, ld, s);
  if (!rc && pred && Pw != pred) {
    rc = launch_copy_idx(P, N, n, n, APSP_DTYPE_I32, pred, ldp, s);
    launches++;
  }
  if (rc) return rc;
  launches++;
  const double ms = tm.stop();
  if (info) {
    info->block = b;
    info->tier = used;
    info->tiers_tried = tried;
    info->iterations = 0;
    info->launches = launches;
    info->max_finite = hdr.cert.max_finite;
    info->relaxations = n * n * n;
    info->device_ms = ms;
    info->flags = 0;
    g_prof.collect(info);
  }
  return 0;
}

int api_store(int dtype) {
  return dtype == APSP_DTYPE_I32 ? STORE_I32 : dtype == APSP_DTYPE_F32 ? STORE_F32 : STORE_I64;
}

int fw_classic_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, cudaStream_t s,
                    apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, header_bytes(), s);
  if (rc) return rc;
  Header* hdr_dev = static_cast<Header*>(sc.base);
  Header hdr{};
  Timer tm(s);
  rc = launch_scan(dtype, dist, ld, n, n, 0, &hdr_dev->scan, s);
  if (!rc) rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  const ScanResult scan = hdr.scan;
  rc = check_scan(scan);
  if (rc) return rc;
  const int store = api_store(dtype);
  APSP_CUDA_TRY(cudaMemsetAsync(&hdr_dev->status, 0, sizeof(Status), s));
  // pred init in place (to_store with identical in/out is elementwise)
  rc = launch_to_store(dtype, dist, ld, n, store, dist, ld, n, pred, ldp, 1, s);
  for (int64_t k = 0; !rc && k < n; k++) rc = launch_fw_step(store, dist, ld, n, k, pred, ldp, IDX_PRED, 0, &hdr_dev->status, s);
  if (rc) return rc;
  const int tier = dtype == APSP_DTYPE_I32 ? APSP_TIER_I32 : dtype == APSP_DTYPE_F32 ? APSP_TIER_F32 : APSP_TIER_I64;
  bool ok = false;
  rc = certify(tier, store, dist, ld, n, n, scan, hdr_dev, hdr, s, ok);
  if (rc) return rc;
  if (!ok) return set_error(APSP_ERANGE, "shortest-path cost left the representable int32 range");
  const double ms = tm.stop();
  if (info) {
    info->tier = tier;
    info->tiers_tried = 1 << tier;
    info->iterations = 0;
    info->launches = int32_t(n + 3);
    info->max_finite = hdr.cert.max_finite;
    info->relaxations = n * n * n;
    info->device_ms = ms;
    info->flags = 0;
    g_prof.collect(info);
  }
  return 0;
}

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
    if (prep_ && bulk_store(store, k) && m % TILE_ALIGN == 0 && n % TILE_ALIGN == 0 && k % 32 == 0) {
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
  if (!aligned) return 0;
  const int64_t h = rk_half(N, aligned);
  const int64_t leaf = std::max<int64_t>(round_up(std::min<int64_t>(thr, N), TILE_ALIGN), TILE_ALIGN);
  // prep + prep2 (concurrent product pair), leaf FW scratch, second value snapshot (<= 8 B / cell)
  return 2 * (prep_bytes(h, h, h) + 512) + fw_scratch_bytes(leaf, TILE_ALIGN, 4) + 512 +
         size_t(h + 8) * (h + 8) * 8 + 512;
}

size_t rk_ws_bytes(int dtype, int64_t n, int aligned, int thr = 1 << 30) {
  const int64_t N = aligned ? round_up(n, TILE_ALIGN) : n;
  const int64_t h = rk_half(N, aligned);
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  return header_bytes() + size_t(N) * N * (es + 4) + size_t(h + 8) * (h + 8) * (es + 4) + 1024 +
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
  char* p = static_cast<char*>(sc.base) + header_bytes();
  int32_t* P = reinterpret_cast<int32_t*>(p);
  p += size_t(N) * N * 4;
  int32_t* sP = reinterpret_cast<int32_t*>(p);
  p += size_t(h + 8) * (h + 8) * 4;
  char* D = p;
  p += size_t(N) * N * (dtype == APSP_DTYPE_I64 ? 8 : 4);
  char* sV = p;
  p += size_t(h + 8) * (h + 8) * (dtype == APSP_DTYPE_I64 ? 8 : 4) + 512;
  char* rkprep = aligned ? p : nullptr;
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
    // product: C starts at Infinity, via at None (minplus.py:398-400)
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

}  // namespace


// ---- row-band shards of a blocked FW (multi-GPU building blocks) ---------------------------
//
// Rank r owns rows [row0, row0 + R) of the padded N x N matrix (R a multiple of b).  Per
// pivot block [k0, k0 + b) with owner o (local pivot rows [lrow, lrow + b) on o):
//   owner:     shard_pivot  = phase 1 on the diagonal block + row panel <- Dg (x) row panel
//   broadcast  row panel values (b x N) and pred (b x N) from o        (NCCL, caller)
//   everyone:  shard_update = column panel <- colpanel (x) Dg; phase 3 on the local rows
// The arithmetic is exactly the single-GPU schedule, so results are bit-identical to one GPU
// at the same b.
namespace {

size_t shard_scratch_bytes(int64_t N, int64_t R, int b, size_t es) {
  size_t v = size_t(b) * N * 4 + 256;                                         // pred row-panel snapshot
  if (b > TILE_ALIGN) v += size_t(b) * N * es + size_t(R) * b * es + 512;     // value snapshots
  v += std::max(prep_bytes(b, N, b), prep_bytes(std::max<int64_t>(R, b), N, b)) + 256;   // panel layouts
  if (b > TILE_ALIGN) v += fw_scratch_bytes(b, TILE_ALIGN, es) + 256;        // phase-1 sub-run
  return v;
}

struct ShardScratch {
  int32_t* predsnap;
  char* rowsnap;
  char* colsnap;
  char* prep;
  char* sub;
};

ShardScratch shard_carve(void* scratch, int64_t N, int64_t R, int b, size_t es) {
  ShardScratch c{};
  char* p = static_cast<char*>(scratch);
  c.predsnap = reinterpret_cast<int32_t*>(p);
  p += size_t(b) * N * 4 + 256;
  if (b > TILE_ALIGN) {
    c.rowsnap = p;
    c.colsnap = p + size_t(b) * N * es + 256;
    p += size_t(b) * N * es + size_t(R) * b * es + 512;
  }
  c.prep = p;
  p += std::max(prep_bytes(b, N, b), prep_bytes(std::max<int64_t>(R, b), N, b)) + 256;
  if (b > TILE_ALIGN) c.sub = p;
  return c;
}

int shard_pivot_impl(int tier, int64_t N, int b, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, cudaStream_t s, int npeers = 0,
                     const int64_t* peer_dv = nullptr, const int64_t* peer_dp = nullptr) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  const size_t es = store_elem_size(store);
  if (scratch_bytes < shard_scratch_bytes(N, b, b, es)) return set_error(APSP_EINVAL, "shard scratch too small");
  const ShardScratch sc = shard_carve(scratch, N, b, b, es);
  char* D = static_cast<char*>(Dv);
  FwCtx c;
  c.store = store; c.es = es;
  c.D = D + (lrow * ld + k0) * es; c.ld = ld;
  c.P = P ? P + lrow * ldp + k0 : nullptr; c.ldp = ldp;
  c.m = b; c.b = b; c.mode = IDX_PRED; c.via_off = k0;
  c.predsnap = sc.predsnap;
  c.sub = sc.sub;
  int rc = fw_phase1(c, 0, s);                           // diagonal block, classic order
  if (rc) return rc;
  char* rowp = D + lrow * ld * es;
  const bool nt = bulk_store(store, b);
  const bool snap = !nt && b > TILE_ALIGN;
  if (P) APSP_CUDA_TRY(cudaMemcpy2DAsync(sc.predsnap, size_t(N) * 4, P + lrow * ldp, size_t(ldp) * 4, size_t(N) * 4,
                                         size_t(b), cudaMemcpyDeviceToDevice, s));
  if (snap && (rc = launch_copy_block(store, rowp, ld, sc.rowsnap, N, b, N, s))) return rc;
  MinplusArgs a = minplus_args();
  a.A = c.D; a.lda = ld;
  a.B = snap ? sc.rowsnap : rowp; a.ldb = snap ? N : ld;
  a.C = rowp; a.ldc = ld;
  a.idx = P ? P + lrow * ldp : nullptr; a.ldi = ldp;
  a.predB = sc.predsnap; a.ldp = N;
  a.m = b; a.n = N; a.k = b; a.inner_off = k0; a.mode = IDX_PRED;
  if (npeers > 0) {
    // fused panel push: the product also covers the diagonal tiles (Dg (x) Dg never improves a
    // closed block) and stores every cell of the b x N panel, values and pred, into each
    // peer's receive slot (address + peer_dv / peer_dp bytes, IPC-mapped over NVLink)
    if (!nt || !(store == STORE_U8 || store == STORE_U16))
      return set_error(APSP_EINVAL, "the fused panel push needs the u8 / u16 tier");
    if (npeers > MAX_PEERS) return set_error(APSP_EINVAL, "npeers %d outside [0, %d]", npeers, MAX_PEERS);
    a.npeers = npeers;
    a.push_all = 1;
    for (int r = 0; r < npeers; r++) {
      a.peer_dC[r] = peer_dv[r];
      a.peer_dI[r] = peer_dp[r];
    }
  } else {
    a.skip_col_lo = k0; a.skip_col_hi = k0 + b;
  }
  if (nt) {
    if ((rc = launch_prep_bulk(store, c.D, ld, rowp, ld, b, N, b, prep_a(sc.prep), prep_b(sc.prep, b, b), s)))
      return rc;
    a.Aprep = prep_a(sc.prep);
    a.Bprep = prep_b(sc.prep, b, b);
  }
  return launch_minplus(store, a, s);
}

int shard_update_impl(int tier, int64_t N, int b, int64_t row_lo, int64_t row_hi, void* Dv, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  const int64_t R = row_hi - row_lo;
  if (R <= 0) return 0;
  const size_t es = store_elem_size(store);
  if (scratch_bytes < shard_scratch_bytes(N, R, b, es)) return set_error(APSP_EINVAL, "shard scratch too small");
  const ShardScratch sc = shard_carve(scratch, N, R, b, es);
  char* D = static_cast<char*>(Dv) + row_lo * ld * es;      // the processed row range
  int32_t* Pr = P ? P + row_lo * ldp : nullptr;
  const char* pv = static_cast<const char*>(panel);
  const bool nt = bulk_store(store, b);
  const bool snap = !nt && b > TILE_ALIGN;
  const bool skip = skip_lo >= 0 && skip_hi > skip_lo;
  int rc = 0;
  if (snap && (rc = launch_copy_block(store, D + k0 * es, ld, sc.colsnap, b, R, b, s))) return rc;
  // column panel of the rows against the (received) closed diagonal block
  MinplusArgs q = minplus_args();
  q.A = snap ? sc.colsnap : D + k0 * es; q.lda = snap ? b : ld;
  q.B = pv + k0 * es; q.ldb = ldpv;
  q.C = D + k0 * es; q.ldc = ld;
  q.idx = Pr ? Pr + k0 : nullptr; q.ldi = ldp;
  q.predB = ppanel ? ppanel + k0 : nullptr; q.ldp = ldpp;
  q.m = R; q.n = b; q.k = b; q.inner_off = k0; q.mode = IDX_PRED;
  if (skip) { q.skip_row_lo = skip_lo - row_lo; q.skip_row_hi = skip_hi - row_lo; }
  if (nt) {
    if ((rc = launch_prep_bulk(store, D + k0 * es, ld, pv + k0 * es, ldpv, R, b, b, prep_a(sc.prep),
                                 prep_b(sc.prep, R, b), s)))
      return rc;
    q.Aprep = prep_a(sc.prep);
    q.Bprep = prep_b(sc.prep, R, b);
  }
  if ((rc = launch_minplus(store, q, s))) return rc;
  // phase 3 of the rows
  MinplusArgs a = minplus_args();
  a.A = D + k0 * es; a.lda = ld;
  a.B = pv; a.ldb = ldpv;
  a.C = D; a.ldc = ld;
  a.idx = Pr; a.ldi = ldp;
  a.predB = ppanel; a.ldp = ldpp;
  a.m = R; a.n = N; a.k = b; a.inner_off = k0; a.mode = IDX_PRED;
  if (skip) { a.skip_row_lo = skip_lo - row_lo; a.skip_row_hi = skip_hi - row_lo; }
  a.skip_col_lo = k0; a.skip_col_hi = k0 + b;
  if (nt) {
    if ((rc = launch_prep_bulk(store, D + k0 * es, ld, pv, ldpv, R, N, b, prep_a(sc.prep), prep_b(sc.prep, R, b),
                                 s)))
      return rc;
    a.Aprep = prep_a(sc.prep);
    a.Bprep = prep_b(sc.prep, R, b);
  }
  return timed_minplus(store, a, s);
}

// ---- sharded R-Kleene: replicated matrix, every block product split by output row bands ----
// Every rank holds the whole N x N store matrix (N a multiple of 128, aligned split).  The host
// schedule (distributed.py run_rkleene) mirrors RK::close; each of the six block products is
// computed by every rank on its band of output rows (rk_shard_product) and the bands are then
// all-gathered; the diagonal leaves are closed redundantly on every rank (rk_shard_leaf), so all
// replicas stay bit-identical to the single-GPU aligned R-Kleene.
size_t rk_shard_scratch_bytes(int64_t N, int thr) {
  const int64_t h = rk_half(N, 1);
  const int64_t leaf = std::max<int64_t>(round_up(std::min<int64_t>(thr, N), TILE_ALIGN), TILE_ALIGN);
  return 256 + prep_bytes(h, h, h) + 512 + fw_scratch_bytes(leaf, TILE_ALIGN, 4) + 512;
}

int rk_shard_leaf_impl(int tier, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  if (lo % TILE_ALIGN || m % TILE_ALIGN || m <= 0) return set_error(APSP_EINVAL, "leaf blocks must be 128-aligned");
  const int64_t N = ld;
  if (scratch_bytes < rk_shard_scratch_bytes(N, thr)) return set_error(APSP_EINVAL, "rk shard scratch too small");
  Status* st = static_cast<Status*>(scratch);
  char* leafws = static_cast<char*>(scratch) + 256 + ((prep_bytes(rk_half(N, 1), rk_half(N, 1), rk_half(N, 1)) + 511) / 256) * 256;
  char* D = static_cast<char*>(Dv);
  const size_t es = store_elem_size(store);
  int launches = 0;
  if (m > TILE_ALIGN)
    return fw_blocked_view(store, D + (lo * ld + lo) * es, ld, P + lo * ldp + lo, ldp, m, DEFAULT_BLOCK, IDX_PRED, lo,
                           st, s, &launches, nullptr, leafws, getenv("APSP_NO_LOOKAHEAD") ? nullptr : side_stream());
  return launch_block_close(store, D, ld, lo, m, P, ldp, IDX_PRED, lo, st, s);
}

int rk_shard_product_impl(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* predB, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          cudaStream_t s, int npeers = 0, const int64_t* peer_dc = nullptr,
                          const int64_t* peer_di = nullptr) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  if (m <= 0 || n <= 0 || k <= 0) return 0;
  if (scratch_bytes < rk_shard_scratch_bytes(N, thr)) return set_error(APSP_EINVAL, "rk shard scratch too small");
  char* prep = static_cast<char*>(scratch) + 256;
  MinplusArgs a = minplus_args();
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.C = C; a.ldc = ldc;
  a.idx = idx; a.ldi = ldi;
  a.predB = predB; a.ldp = ldpb;
  a.m = m; a.n = n; a.k = k;
  a.inner_off = inner_off;
  a.mode = IDX_PRED;
  a.status = static_cast<Status*>(scratch);
  if (npeers < 0 || npeers > MAX_PEERS) return set_error(APSP_EINVAL, "npeers %d outside [0, %d]", npeers, MAX_PEERS);
  a.npeers = npeers;
  for (int r = 0; r < npeers; r++) {
    a.peer_dC[r] = peer_dc[r];
    a.peer_dI[r] = peer_di[r];
  }
  if (bulk_store(store, k) && m % TILE_ALIGN == 0 && n % TILE_ALIGN == 0 && k % 32 == 0) {   // as RK::mp
    int rc = launch_prep_bulk(store, A, lda, B, ldb, m, n, k, prep_a(prep), prep_b(prep, m, k), s);
    if (rc) return rc;
    a.Aprep = prep_a(prep);
    a.Bprep = prep_b(prep, m, k);
  }
  return timed_minplus(store, a, s);
}

}  // namespace

// =============================================================================================
extern "C" {

const char* apsp_last_error(void) { return apsp::last_error(); }
void apsp_set_profiling(int on) { g_prof.on = on != 0; }
long long apsp_launch_count(void) { return apsp::launch_count(); }

int apsp_scan(int dtype, const void* h, int64_t ld, int64_t rows, int64_t cols, int64_t diag_off,
              apsp_scan_result* out, void* stream) {
  static_assert(sizeof(apsp_scan_result) == sizeof(ScanResult), "scan result layout");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, sizeof(ScanResult), s);
  if (rc) return rc;
  rc = launch_scan(dtype, h, ld, rows, cols, diag_off, static_cast<ScanResult*>(sc.base), s);
  if (rc) return rc;
  APSP_CUDA_TRY(cudaMemcpyAsync(out, sc.base, sizeof(ScanResult), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

size_t apsp_shard_scratch_bytes(int tier, int64_t N, int64_t rows, int block) {
  const int store = tier_store(tier);
  return shard_scratch_bytes(N, rows, block, store < 0 ? 8 : store_elem_size(store));
}

int apsp_shard_prepare(int dtype, int tier, int64_t n, int64_t N, int64_t row0, int64_t rows, const void* h,
                       int64_t ldh, void* D, int64_t ld, int32_t* P, int64_t ldp, void* stream) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  return launch_to_store_rows(dtype, h, ldh, n, store, D, ld, N, P, ldp, 1, row0, rows, (cudaStream_t)stream);
}

int apsp_shard_pivot(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, void* stream) {
  return shard_pivot_impl(tier, N, block, D, ld, P, ldp, lrow, k0, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_shard_update(int tier, int64_t N, int block, int64_t row_lo, int64_t row_hi, void* D, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, void* stream) {
  return shard_update_impl(tier, N, block, row_lo, row_hi, D, ld, P, ldp, panel, ldpv, ppanel, ldpp, k0, skip_lo,
                           skip_hi, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_shard_pivot_fused(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                           int64_t k0, int npeers, const int64_t* peer_dv, const int64_t* peer_dp, void* scratch,
                           size_t scratch_bytes, void* stream) {
  return shard_pivot_impl(tier, N, block, D, ld, P, ldp, lrow, k0, scratch, scratch_bytes, (cudaStream_t)stream,
                          npeers, peer_dv, peer_dp);
}

void* apsp_side_stream(void) { return side_stream(); }

int apsp_shard_finish(int tier, int dtype, int64_t rows, int64_t n, const void* D, int64_t ld, const int32_t* P,
                      int64_t ldp, void* dist, int64_t ldd, int32_t* pred, int64_t ldpo, int64_t* max_finite,
                      void* stream) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, sizeof(ScanResult), s);
  if (rc) return rc;
  ScanResult* r = static_cast<ScanResult*>(sc.base);
  if (rows > 0) {
    rc = launch_max_finite(store, D, ld, rows, n, r, s);
    if (!rc && dist) rc = launch_from_store(store, D, ld, rows, n, dtype, dist, ldd, s);
    if (!rc && pred && P) rc = launch_copy_idx(P, ldp, rows, n, APSP_DTYPE_I32, pred, ldpo, s);
    if (rc) return rc;
  } else {
    APSP_CUDA_TRY(cudaMemsetAsync(r, 0, sizeof(ScanResult), s));
  }
  ScanResult h{};
  APSP_CUDA_TRY(cudaMemcpyAsync(&h, r, sizeof(ScanResult), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  if (max_finite) *max_finite = rows > 0 && h.max_finite >= 0 ? h.max_finite : -1;
  return 0;
}

size_t apsp_rk_shard_scratch_bytes(int64_t N, int thr) { return rk_shard_scratch_bytes(N, thr); }

int apsp_rk_shard_product_fused(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                                int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                                int64_t k, int64_t inner_off, int64_t N, int thr, int npeers, const int64_t* peer_dc,
                                const int64_t* peer_di, void* scratch, size_t scratch_bytes, void* stream) {
  return rk_shard_product_impl(tier, A, lda, B, ldb, C, ldc, idx, ldi, pred_b, ldpb, m, n, k, inner_off, N, thr,
                               scratch, scratch_bytes, (cudaStream_t)stream, npeers, peer_dc, peer_di);
}

int apsp_rk_shard_leaf(int tier, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, void* stream) {
  return rk_shard_leaf_impl(tier, D, ld, P, ldp, lo, m, thr, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_rk_shard_product(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          void* stream) {
  return rk_shard_product_impl(tier, A, lda, B, ldb, C, ldc, idx, ldi, pred_b, ldpb, m, n, k, inner_off, N, thr,
                               scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_abi_version(void) { return APSP_ABI_VERSION; }

size_t apsp_workspace_bytes(int algorithm, int dtype, int64_t n, int block) {
  switch (algorithm) {
    case APSP_ALG_FW_BLOCKED: return fw_ws_bytes(dtype, n, block > 0 ? block : default_block(n));
    case APSP_ALG_RKLEENE: return std::max(rk_ws_bytes(dtype, n, 1, 1 << 30), rk_ws_bytes(dtype, n, 0));
    case APSP_ALG_FW_SQUARING: return sq_ws_bytes(dtype, n);
    case APSP_ALG_FW_CLASSIC: return 0;
  }
  return 0;
}

int apsp_fw_blocked(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, int block, int tier,
                    void* ws, size_t ws_bytes, void* stream, apsp_info* info) {
  return fw_blocked_impl(dtype, n, dist, ld, pred, ldp, block, tier, ws, ws_bytes, (cudaStream_t)stream, info);
}

int apsp_fw_classic(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, void* stream,
                    apsp_info* info) {
  return fw_classic_impl(dtype, n, dist, ld, pred, ldp, (cudaStream_t)stream, info);
}

int apsp_rkleene(int dtype, int64_t n, void* dist, int64_t ld, int32_t* idx, int64_t ldi, int idx_mode,
                 int base_threshold, int aligned, int tier, void* ws, size_t ws_bytes, void* stream, apsp_info* info) {
  return rkleene_impl(dtype, n, dist, ld, idx, ldi, idx_mode, base_threshold, aligned, tier, ws, ws_bytes,
                      (cudaStream_t)stream, info);
}

int apsp_fw_squaring(int dtype, int64_t n, void* dist, int64_t ld, int32_t* via, int64_t ldv, int tier, void* ws,
                     size_t ws_bytes, void* stream, apsp_info* info) {
  return squaring_impl(dtype, n, dist, ld, via, ldv, tier, ws, ws_bytes, (cudaStream_t)stream, info);
}

int apsp_minplus(int dtype, int accumulate, int64_t n1, int64_t n2, int64_t n3, const void* x, int64_t ldx,
                 const void* y, int64_t ldy, void* z, int64_t ldz, int32_t* via, int64_t ldv, int64_t row_off,
                 int64_t inner_off, int64_t col_off, int tier, void* stream, apsp_info* info) {
  return minplus_impl(dtype, accumulate, n1, n2, n3, x, ldx, y, ldy, z, ldz, via, ldv, row_off, inner_off, col_off,
                      tier, (cudaStream_t)stream, info);
}

int apsp_solve_host(int algorithm, int dtype, int64_t n, const void* h, void* dist_out, void* idx_out, int idx_dtype,
                    int idx_mode, int block, int base_threshold, int aligned, int tier, int device, apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  if (idx_dtype != APSP_DTYPE_I32 && idx_dtype != APSP_DTYPE_I64)
    return set_error(APSP_EINVAL, "index dtype must be int32 or int64");
  APSP_CUDA_TRY(cudaSetDevice(device));
  keep_pool();
  cudaStream_t s;
  APSP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  const size_t bytes = size_t(n) * n * es;
  void* d = nullptr;
  int32_t* p = nullptr;
  void* pw = nullptr;
  int rc = 0;
  auto fail = [&](int code) {
    if (d) cudaFreeAsync(d, s);
    if (p) cudaFreeAsync(p, s);
    if (pw) cudaFreeAsync(pw, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  cudaError_t e = cudaMallocAsync(&d, bytes, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&p, size_t(n) * n * 4, s);
  if (e == cudaSuccess && idx_dtype == APSP_DTYPE_I64 && idx_out) e = cudaMallocAsync(&pw, size_t(n) * n * 8, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(set_cuda_error(e, "host staging", __FILE__, __LINE__));
  switch (algorithm) {
    case APSP_ALG_FW_BLOCKED: rc = fw_blocked_impl(dtype, n, d, n, p, n, block, tier, nullptr, 0, s, info); break;
    case APSP_ALG_FW_CLASSIC: rc = fw_classic_impl(dtype, n, d, n, p, n, s, info); break;
    case APSP_ALG_RKLEENE:
      rc = rkleene_impl(dtype, n, d, n, p, n, idx_mode, base_threshold, aligned, tier, nullptr, 0, s, info);
      break;
    case APSP_ALG_FW_SQUARING: rc = squaring_impl(dtype, n, d, n, p, n, tier, nullptr, 0, s, info); break;
    default: rc = set_error(APSP_EINVAL, "unknown algorithm %d", algorithm);
  }
  if (rc) return fail(rc);
  e = cudaMemcpyAsync(dist_out, d, bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && idx_out) {
    if (idx_dtype == APSP_DTYPE_I64) {
      rc = launch_copy_idx(p, n, n, n, APSP_DTYPE_I64, pw, n, s);
      if (rc) return fail(rc);
      e = cudaMemcpyAsync(idx_out, pw, size_t(n) * n * 8, cudaMemcpyDeviceToHost, s);
    } else {
      e = cudaMemcpyAsync(idx_out, p, size_t(n) * n * 4, cudaMemcpyDeviceToHost, s);
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(set_cuda_error(e, "host readback", __FILE__, __LINE__));
  return fail(0);
}

}  // extern "C"
