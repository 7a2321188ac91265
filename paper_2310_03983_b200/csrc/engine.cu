// Engine services shared by the schedules: value tiers and their certificate, scratch,
// launch profiling, streams.
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


// The library's scratch comes from the device's default stream-ordered pool.  The default
// release threshold of 0 hands freed blocks back to the driver at every synchronisation; keep
// them reserved (threshold = max) so repeated solves do not remap GBs of workspace.
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


// The header comes back through a per-thread pinned buffer: a pageable copy is staged by the
// driver and costs several microseconds more on every solve (measured at n=256, where the host
// reads are a third of the call).
int read_header(Header* dev, Header& host, cudaStream_t s) {
  static thread_local Header* pinned = nullptr;
  static thread_local bool tried = false;
  if (!tried) {
    tried = true;
    if (cudaMallocHost(&pinned, sizeof(Header)) != cudaSuccess) {
      pinned = nullptr;
      cudaGetLastError();
    }
  }
  Header* dst = pinned ? pinned : &host;
  APSP_CUDA_TRY(cudaMemcpyAsync(dst, dev, sizeof(Header), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  if (pinned) host = *pinned;
  return 0;
}

int check_scan(const ScanResult& sc) {
  if (sc.negative) return set_error(APSP_ENEGATIVE, "solver input contains a negative finite cost");
  if (sc.diag_nonzero) return set_error(APSP_EDIAGONAL, "solver input must have a zero diagonal");
  return 0;
}

// Bulk-staged (pre-laid-out panel) products for this tier and inner length k.  The exact fp32
// tier uses them from k = 128 on (APSP_F32_MINK; the deferred-argmin kernel: n=4096 FW
// 17.8 -> 14.6 ms, n=8192 118 -> 75 ms); below that the 64 x 64 register-staged kernel.
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

// Off by default: grouping cuts phase-3b DRAM reads by 15 % at n=16384 with the same time, but
// costs 1.5 % at n=8192 (profiles/r02_raster_ab.txt); the kernel is ALU-bound either way.
int raster_group() {
  static const int g = getenv("APSP_RASTER_G") ? atoi(getenv("APSP_RASTER_G")) : 1;
  return g;
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


int certify(int tier, int store, const void* D, int64_t ld, int64_t rows, int64_t cols, const ScanResult& sc,
            Header* hdr_dev, Header& hdr, cudaStream_t s, bool& ok) {
  int rc = launch_max_finite(store, D, ld, rows, cols, &hdr_dev->cert, s);
  if (rc) return rc;
  rc = read_header(hdr_dev, hdr, s);
  if (rc) return rc;
  return certify_check(tier, sc, hdr, ok);
}

// the host half of certify, on a header already read back (status + cert of this attempt)
int certify_check(int tier, const ScanResult& sc, const Header& hdr, bool& ok) {
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

int api_store(int dtype) {
  return dtype == APSP_DTYPE_I32 ? STORE_I32 : dtype == APSP_DTYPE_F32 ? STORE_F32 : STORE_I64;
}

}  // namespace apsp
