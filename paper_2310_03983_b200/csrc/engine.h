// Internal interfaces of the host-side orchestration (engine.cu: tiers, workspaces,
// certificate, streams; fw_sched.cu: blocked FW rounds; rkleene.cu: R-Kleene, squaring and
// public products; shard.cu: multi-GPU building blocks).  Not part of the C ABI.
#pragma once
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <memory>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "../../include/apsp_b200.h"
#include "launch.h"

namespace apsp {
const char* last_error();
long long launch_count();

void keep_pool();

constexpr int DEFAULT_BLOCK = 128;
constexpr int TILE_ALIGN = 128;

// Zero-cost edges let equal-distance vertices point at each other when many cells are
// relaxed at once (blocked phase 3, R-Kleene products); only the classic k order keeps the
// predecessor graph a tree then.  Such inputs are solved by the classic kernel, which is
// bit-exact with the reference for both dist and pred.
constexpr int32_t FLAG_CLASSIC_FOR_ZERO_EDGES = 1;

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
extern thread_local Profiler g_prof;

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

// NVTX ranges name the phases for nsys/ncu (`ncu --nvtx --nvtx-include "apsp.fw.phase3/"`).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

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
  char* prep[3] = {nullptr, nullptr, nullptr};  // bulk tiers: layouts of the panels, by round mod 3
  int32_t* predsnap3[3] = {nullptr, nullptr, nullptr};  // pivot-row pred after phase 2, by round mod 3
  bool deep = false;             // two-deep lookahead (the next cross on the side stream)
  char* p2prep = nullptr;        // narrow tiers: bulk-copy layouts of the phase-2 operands
  char* sub = nullptr;           // scratch of the phase-1 sub-run when b > 128
  int* spin = nullptr;           // device-signalled chain: exit counts and the diagonal flag
  int* tflags = nullptr;         // per-tile round flags of the device-signalled chain
  int launches = 0;
  struct BandSink* sink = nullptr;   // last round in row bands, each handed to the sink
};

// Consumer of the final rows of a blocked FW solve: with a sink, the last round's phase 3 runs
// in row bands and band() is called right after each band's launch on s (rows [r0, r1) of the
// padded matrix are final once that launch completes; c.store says which value tier produced
// them -- an attempt that later fails its certificate is followed by another run).
struct BandSink {
  virtual ~BandSink() = default;
  virtual int band(int64_t r0, int64_t r1, const FwCtx& c, cudaStream_t s) = 0;
};

// Device time of one call (apsp_info.device_ms). The event pair is created once per host thread
// and device. stop() synchronises on the end event; mark() + elapsed() let a call that
// synchronises anyway (the certificate readback) take the end point there, without one more
// host round trip at the end of a stream-ordered call.
struct Timer {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  bool marked = false;
  static int& depth() {   // nested calls (e.g. the zero-cost-edge fallback) get their own pair
    thread_local int d = 0;
    return d;
  }
  explicit Timer(cudaStream_t st) : s(st) {
    g_prof.reset();
    int dev = 0;
    cudaGetDevice(&dev);
    thread_local cudaEvent_t ev[64][4][2] = {};
    if (dev < 0 || dev >= 64) dev = 0;
    const int lvl = std::min(depth()++, 3);
    if (!ev[dev][lvl][0]) {
      cudaEventCreate(&ev[dev][lvl][0]);
      cudaEventCreate(&ev[dev][lvl][1]);
    }
    a = ev[dev][lvl][0];
    b = ev[dev][lvl][1];
    cudaEventRecord(a, s);
  }
  ~Timer() { depth()--; }
  void mark() {
    cudaEventRecord(b, s);
    marked = true;
  }
  double elapsed() {   // after a synchronisation that covers the mark
    float ms = 0;
    if (!marked) return stop();
    if (cudaEventQuery(b) != cudaSuccess) cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
  double stop() {
    float ms = 0;
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
};

inline uint32_t* prep_a(char* slot) { return reinterpret_cast<uint32_t*>(slot); }
inline uint16_t* prep_b(char* slot, int64_t m, int64_t k) {
  return reinterpret_cast<uint16_t*>(slot + ((size_t(m) * k * 4 + 255) / 256) * 256);
}

int timed_minplus(int store, const MinplusArgs& a, cudaStream_t s);

int64_t round_up(int64_t v, int64_t m);

int tier_store(int tier);

int64_t tier_limit(int tier);

int read_header(Header* dev, Header& host, cudaStream_t s);

int check_scan(const ScanResult& sc);

bool bulk_store(int store, int64_t k);

std::vector<int> pick_tiers(int dtype, const ScanResult& sc, int forced, bool allow_u16, int64_t n_vert);

int certify(int tier, int store, const void* D, int64_t ld, int64_t rows, int64_t cols, const ScanResult& sc,
            Header* hdr_dev, Header& hdr, cudaStream_t s, bool& ok);
int certify_check(int tier, const ScanResult& sc, const Header& hdr, bool& ok);

int api_store(int dtype);

cudaStream_t side_stream();

size_t header_bytes();

size_t fw_scratch_bytes(int64_t m, int b, size_t es);

void fw_carve(FwCtx& c, char* scratch, int64_t N);

int fw_phase1(FwCtx& c, int64_t k0, cudaStream_t s, const int* wait_count = nullptr, int wait_target = 0,
              uint32_t* nxA = nullptr, uint16_t* nxB = nullptr, int32_t* nxPred = nullptr, int64_t nxPredLd = 0);

int fw_run(FwCtx& c, cudaStream_t s);

int fw_blocked_view(int store, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t m, int b, int mode,
                    int64_t via_off, Status* st, cudaStream_t s, int* launches, int32_t* predsnap,
                    char* scratch = nullptr, cudaStream_t side = nullptr);

int default_block(int64_t n);

size_t fw_ws_bytes(int dtype, int64_t n, int block);

int fw_blocked_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, int b, int tier_req,
                    void* ws, size_t ws_bytes, cudaStream_t s, apsp_info* info, BandSink* sink = nullptr);

int fw_classic_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, cudaStream_t s,
                    apsp_info* info);

int64_t rk_half(int64_t N, int aligned);

size_t rk_ws_bytes(int dtype, int64_t n, int aligned, int thr = 1 << 30);

int rkleene_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* idx, int64_t ldi, int idx_mode, int thr,
                 int aligned, int tier_req, void* ws, size_t ws_bytes, cudaStream_t s, apsp_info* info);

size_t sq_ws_bytes(int dtype, int64_t n);

int squaring_impl(int dtype, int64_t n, void* dist, int64_t ld, int32_t* via, int64_t ldv, int tier_req, void* ws,
                  size_t ws_bytes, cudaStream_t s, apsp_info* info);

int minplus_impl(int dtype, int accumulate, int64_t n1, int64_t n2, int64_t n3, const void* x, int64_t ldx,
                 const void* y, int64_t ldy, void* z, int64_t ldz, int32_t* via, int64_t ldv, int64_t row_off,
                 int64_t inner_off, int64_t col_off, int tier_req, cudaStream_t s, apsp_info* info);

size_t shard_scratch_bytes(int64_t N, int64_t R, int b, size_t es);

int shard_pivot_impl(int tier, int64_t N, int b, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, cudaStream_t s, int npeers = 0,
                     const int64_t* peer_dv = nullptr, const int64_t* peer_dp = nullptr);

int shard_update_impl(int tier, int64_t N, int b, int64_t row_lo, int64_t row_hi, void* Dv, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, cudaStream_t s);

size_t rk_shard_scratch_bytes(int64_t N, int thr);

int rk_shard_leaf_impl(int tier, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, cudaStream_t s);

int rk_shard_product_impl(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* predB, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          cudaStream_t s, int npeers = 0, const int64_t* peer_dc = nullptr,
                          const int64_t* peer_di = nullptr);

// hostio.cu: narrowed device->host readback of an int32 result (apsp_solve_host).
int readback_packed(int64_t n, const void* d, int es, const int32_t* p, int64_t max_finite, void* dist_out,
                    void* idx_out, int idx_dtype, cudaStream_t s, bool& handled);
int32_t readback_width(int64_t n, int64_t max_finite, int es, bool idx);   // bytes per cell when handled
int upload_packed(int64_t n, const void* h, int es, void* d, cudaStream_t s, bool& handled, int& width);
// last-round streaming readback of apsp_solve_host's blocked FW (nullptr when it does not apply)
std::unique_ptr<BandSink> make_band_stream(int64_t n, int es, void* dist_out, void* idx_out, int idx_dtype,
                                           cudaStream_t s);
bool finish_band_stream(BandSink* b);   // true: dist/idx already hold the certified result

}  // namespace apsp
