// Host readback of apsp_solve_host (include/apsp_b200.h): the n x n int32 distances and
// predecessors leave the GPU narrowed, and host threads widen them into the caller's buffers.
//
// Over PCIe the readback of an int32 result is 8 bytes per cell (dist + pred). Most results need
// far fewer bits: a u8-tier result has max_finite <= 254, and predecessors are < n. One device
// pass packs dist to 1 or 2 bytes (INF32 -> all-ones) and pred to 2 bytes (p + 1, so -1 -> 0).
// The packed rows then come back in row chunks. Each chunk gets its own event, and a host worker
// pool widens chunk c while chunk c+1 is still on the wire. The pool writes with streaming stores,
// so the output lines are not read first
// (hostwiden.cpp, AVX-512 when the host has it). At n=16384 u8 this moves 768 MiB instead of 2 GiB.
//
// The pack kernel flags any value outside the promised width. A flagged result falls back to the
// plain int32 copies, so the output is always the exact device result.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <cstdio>
#include <mutex>
#include <thread>
#include <vector>
#include <sched.h>
#include "engine.h"

namespace apsp {

namespace {

constexpr int32_t kInf32 = INF32;   // the API's int32 "no path" (core.py INF32)

template <typename TD> __device__ __forceinline__ TD inf_of() { return sizeof(TD) == 4 ? TD(INF32) : TD(INF_RAW); }

// four consecutive cells as 64-bit lanes (int32 results sign-extend)
template <typename TD>
__device__ __forceinline__ void load4(const TD* d, int64_t g, int64_t (&x)[4]) {
  if constexpr (sizeof(TD) == 4) {
    const int4 v = reinterpret_cast<const int4*>(d)[g];
    x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
  } else {
    const longlong2 a = reinterpret_cast<const longlong2*>(d)[2 * g], b = reinterpret_cast<const longlong2*>(d)[2 * g + 1];
    x[0] = a.x; x[1] = a.y; x[2] = b.x; x[3] = b.y;
  }
}

template <int DW, bool PRED, typename TD>
__global__ void pack_result_kernel(const TD* __restrict__ d, const int32_t* __restrict__ p, int64_t cells,
                                   void* __restrict__ dpk, uint16_t* __restrict__ ppk, int32_t lim,
                                   int* __restrict__ bad) {
  const int64_t groups = cells >> 2;
  int flag = 0;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < groups; g += int64_t(gridDim.x) * blockDim.x) {
    if (DW) {
      int64_t x[4];
      load4(d, g, x);
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const bool inf = x[q] == int64_t(inf_of<TD>());
        flag |= !inf && (x[q] < 0 || x[q] > lim);
        o[q] = inf ? (DW == 1 ? 0xFFu : 0xFFFFu) : uint32_t(x[q]);
      }
      if (DW == 1) reinterpret_cast<uint32_t*>(dpk)[g] = o[0] | o[1] << 8 | o[2] << 16 | o[3] << 24;
      else reinterpret_cast<uint2*>(dpk)[g] = make_uint2(o[0] | o[1] << 16, o[2] | o[3] << 16);
    }
    if (PRED) {
      const int4 v = reinterpret_cast<const int4*>(p)[g];
      reinterpret_cast<uint2*>(ppk)[g] = make_uint2(uint32_t(v.x + 1) | uint32_t(v.y + 1) << 16,
                                                    uint32_t(v.z + 1) | uint32_t(v.w + 1) << 16);
    }
  }
  if (flag) atomicOr(bad, 1);
}

template <typename TD>
void launch_pack(int dw, bool pk, const void* d, const int32_t* p, int64_t cells, void* dev, uint16_t* ppk, int* bad,
                 cudaStream_t s) {
  const int grid = 148 * 8;
  const int32_t lim = dw == 1 ? 254 : 65534;
  const TD* dd = static_cast<const TD*>(d);
  if (dw == 1 && pk) pack_result_kernel<1, true, TD><<<grid, 256, 0, s>>>(dd, p, cells, dev, ppk, lim, bad);
  else if (dw == 1) pack_result_kernel<1, false, TD><<<grid, 256, 0, s>>>(dd, p, cells, dev, ppk, lim, bad);
  else if (dw == 2 && pk) pack_result_kernel<2, true, TD><<<grid, 256, 0, s>>>(dd, p, cells, dev, ppk, lim, bad);
  else if (dw == 2) pack_result_kernel<2, false, TD><<<grid, 256, 0, s>>>(dd, p, cells, dev, ppk, lim, bad);
  else pack_result_kernel<0, true, TD><<<grid, 256, 0, s>>>(dd, p, cells, dev, ppk, lim, bad);
}

// ---- pinned staging, grow-only, process-wide ------------------------------------------------

struct Pinned {
  std::mutex mu;
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaError_t reserve(size_t need) {   // caller holds mu
    if (bytes >= need) return cudaSuccess;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    bytes = 0;
    const cudaError_t e = cudaHostAlloc(&ptr, need, cudaHostAllocPortable);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
};
Pinned g_down, g_up;   // readback / upload staging

int host_workers() {
  if (const char* e = std::getenv("APSP_HOST_THREADS")) return std::max(1, std::atoi(e));
  cpu_set_t set;
  int n = 0;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
  if (n <= 0) n = int(std::thread::hardware_concurrency());
  return std::clamp(n, 1, 16);
}

// row chunks of a transfer: >= 16 of them, each at most 2048 rows
int64_t chunk_rows(int64_t n) { return std::min<int64_t>(2048, std::max<int64_t>(1, (n + 15) / 16)); }

template <int W, typename TD>
__global__ void widen_costs_kernel(const void* __restrict__ src, TD* __restrict__ d, int64_t cells) {
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < (cells >> 2);
       g += int64_t(gridDim.x) * blockDim.x) {
    uint32_t x[4];
    if (W == 1) {
      const uint32_t w = reinterpret_cast<const uint32_t*>(src)[g];
      for (int q = 0; q < 4; q++) x[q] = (w >> (8 * q)) & 0xFFu;
    } else {
      const uint2 w = reinterpret_cast<const uint2*>(src)[g];
      x[0] = w.x & 0xFFFFu; x[1] = w.x >> 16; x[2] = w.y & 0xFFFFu; x[3] = w.y >> 16;
    }
    constexpr uint32_t ALL = W == 1 ? 0xFFu : 0xFFFFu;
    TD o[4];
    for (int q = 0; q < 4; q++) o[q] = x[q] == ALL ? inf_of<TD>() : TD(x[q]);
    if constexpr (sizeof(TD) == 4) {
      reinterpret_cast<int4*>(d)[g] = make_int4(o[0], o[1], o[2], o[3]);
    } else {
      reinterpret_cast<longlong2*>(d)[2 * g] = make_longlong2(o[0], o[1]);
      reinterpret_cast<longlong2*>(d)[2 * g + 1] = make_longlong2(o[2], o[3]);
    }
  }
}

int dist_width(int64_t max_finite) {
  return max_finite >= 0 && max_finite <= 254 ? 1 : max_finite >= 0 && max_finite <= 65534 ? 2 : 0;
}

}  // namespace

void host_widen_dist(const void* src, int width, void* dst, bool wide, size_t cnt);   // hostwiden.cpp
bool host_narrow(const void* src, bool wide, void* dst, int width, size_t cnt);

// Uploads the n x n int32 (es 4) or int64 (es 8) cost matrix h into the contiguous device
// buffer d narrowed: host threads pack row chunks to u8 (or u16) while the previous chunks are
// on the wire, and one device pass widens them back (all-ones -> INF32 / INF_RAW). The width comes from the first
// rows; a later cell that does not fit aborts the packed upload (handled = false) and the caller
// copies the int32 matrix as is. The device-side scan then sees exactly the caller's matrix.
int upload_packed(int64_t n, const void* h, int es, void* d, cudaStream_t s, bool& handled, int& width) {
  handled = false;
  width = es;
  const bool wide = es == 8;
  const char* env = std::getenv("APSP_PACKED_UPLOAD");
  if (env && env[0] == '0') return 0;
  const int64_t cells = n * n;
  if (cells < (int64_t(1) << 22) || cells % 4) return 0;
  // width from the first rows (a bounded sample; the packing itself checks every cell)
  const int64_t sample = std::min<int64_t>(n, 64) * n;
  int64_t mx = 0;
  for (int64_t i = 0; i < sample; i++) {
    const int64_t v = wide ? static_cast<const int64_t*>(h)[i] : static_cast<const int32_t*>(h)[i];
    if (v == (wide ? INF_RAW : int64_t(INF32))) continue;
    if (v < 0) return 0;
    mx = std::max(mx, v);
  }
  const int w = mx <= 254 ? 1 : mx <= 65534 ? 2 : 0;
  if (!w) return 0;
  std::unique_lock<std::mutex> lk(g_up.mu);
  APSP_CUDA_TRY(g_up.reserve(size_t(cells) * w));
  char* st = static_cast<char*>(g_up.ptr);
  void* dev = nullptr;
  APSP_CUDA_TRY(cudaMallocAsync(&dev, size_t(cells) * w, s));
  const int64_t rows = chunk_rows(n);
  const int64_t nch = (n + rows - 1) / rows;
  const int T = host_workers();
  std::atomic<bool> abort{false};
  std::atomic<int> cuerr{0};
  std::vector<std::atomic<int>> pending(static_cast<size_t>(nch));
  for (auto& x : pending) x = T;
  auto work = [&](int t) {
    for (int64_t c = 0; c < nch && !abort; c++) {
      const int64_t r0 = c * rows, r1 = std::min(n, r0 + rows);
      const int64_t a = r0 + (r1 - r0) * t / T, b = r0 + (r1 - r0) * (t + 1) / T;
      if (a < b && !host_narrow(static_cast<const char*>(h) + size_t(a * n) * es, wide, st + size_t(a * n) * w, w,
                                size_t((b - a) * n))) {
        abort = true;
        return;
      }
      if (pending[size_t(c)].fetch_sub(1) == 1 && !abort) {   // last slice of the chunk: ship it
        const size_t off = size_t(r0 * n) * w, bytes = size_t((r1 - r0) * n) * w;
        if (cudaMemcpyAsync(static_cast<char*>(dev) + off, st + off, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
          cuerr = 1, abort = true;
      }
    }
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 1; t < T; t++) pool.emplace_back(work, t);
  work(0);
  for (auto& t : pool) t.join();
  const auto t1 = std::chrono::steady_clock::now();
  cudaError_t e = cuerr ? cudaErrorUnknown : cudaSuccess;
  if (!abort) {
    if (wide && w == 1) widen_costs_kernel<1><<<148 * 8, 256, 0, s>>>(dev, static_cast<int64_t*>(d), cells);
    else if (wide) widen_costs_kernel<2><<<148 * 8, 256, 0, s>>>(dev, static_cast<int64_t*>(d), cells);
    else if (w == 1) widen_costs_kernel<1><<<148 * 8, 256, 0, s>>>(dev, static_cast<int32_t*>(d), cells);
    else widen_costs_kernel<2><<<148 * 8, 256, 0, s>>>(dev, static_cast<int32_t*>(d), cells);
    e = cudaGetLastError();
    count_launches(1);
  }
  cudaFreeAsync(dev, s);
  // the staging buffer is reused by the next call: its copies must have landed
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = e2;
  if (std::getenv("APSP_READBACK_TRACE"))
    std::fprintf(stderr, "[upload] n=%lld w=%d threads=%d abort=%d host pack %.2f ms, pack+copies+widen %.2f ms\n",
                 (long long)n, w, T, int(abort.load()), std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  if (e != cudaSuccess) return set_cuda_error(e, "packed upload", __FILE__, __LINE__);
  handled = !abort;
  width = handled ? w : es;
  return 0;
}
void host_widen_pred(const uint16_t* src, void* dst, bool wide, size_t cnt);

int32_t readback_width(int64_t n, int64_t max_finite, int es, bool idx) {
  const int dw = dist_width(max_finite);
  return (dw ? dw : es) + (idx ? 2 : 0);
}

// Reads back n x n dist (int32 es 4 / int64 es 8) and the int32 pred (when idx_out; written as
// idx_dtype) from contiguous device buffers. handled = false when the packed path does not
// apply; the caller then does the plain copies.
int readback_packed(int64_t n, const void* d, int es, const int32_t* p, int64_t max_finite, void* dist_out,
                    void* idx_out, int idx_dtype, cudaStream_t s, bool& handled) {
  const bool wide = es == 8;
  handled = false;
  const char* env = std::getenv("APSP_PACKED_READBACK");
  if (env && env[0] == '0') return 0;
  const int64_t cells = n * n;
  if (cells < (int64_t(1) << 22) || cells % 4) return 0;              // small results: plain copies
  const int dw = dist_width(max_finite);
  const bool pk = idx_out && p && n < 65535;
  if ((idx_out && !pk) || (!dw && !pk)) return 0;

  const size_t dbytes = (size_t(cells) * dw + 255) & ~size_t(255), pbytes = pk ? size_t(cells) * 2 : 0;
  void* dev = nullptr;
  APSP_CUDA_TRY(cudaMallocAsync(&dev, dbytes + pbytes + 16, s));
  int* bad = reinterpret_cast<int*>(static_cast<char*>(dev) + dbytes + pbytes);
  uint16_t* ppk = reinterpret_cast<uint16_t*>(static_cast<char*>(dev) + dbytes);
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(int), s);
  if (e == cudaSuccess) {
    if (wide) launch_pack<int64_t>(dw, pk, d, p, cells, dev, ppk, bad, s);
    else launch_pack<int32_t>(dw, pk, d, p, cells, dev, ppk, bad, s);
    e = cudaGetLastError();
    count_launches(1);
  }
  std::unique_lock<std::mutex> lk(g_down.mu);
  if (e == cudaSuccess) e = g_down.reserve(dbytes + pbytes + 64);
  char* st = static_cast<char*>(g_down.ptr);
  volatile int* hbad = reinterpret_cast<volatile int*>(st + dbytes + pbytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync((void*)hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  const int64_t rows = chunk_rows(n);
  const int64_t nch = (n + rows - 1) / rows;
  std::vector<cudaEvent_t> ev(size_t(nch), nullptr);
  for (int64_t c = 0; e == cudaSuccess && c < nch; c++) {
    const size_t r0 = size_t(c * rows), rc = size_t(std::min(n, (c + 1) * rows) - c * rows);
    if (dw)
      e = cudaMemcpyAsync(st + r0 * n * dw, static_cast<char*>(dev) + r0 * n * dw, rc * n * dw,
                          cudaMemcpyDeviceToHost, s);
    else
      e = cudaMemcpyAsync(static_cast<char*>(dist_out) + r0 * n * es, static_cast<const char*>(d) + r0 * n * es,
                          rc * n * es, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && pk)
      e = cudaMemcpyAsync(st + dbytes + r0 * n * 2, ppk + r0 * n, rc * n * 2, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[size_t(c)], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev[size_t(c)], s);
  }
  if (e == cudaSuccess) {
    const int T = host_workers();
    std::atomic<int> err{0};
    auto work = [&](int w) {
      for (int64_t c = 0; c < nch; c++) {
        if (cudaEventSynchronize(ev[size_t(c)]) != cudaSuccess) { err = 1; return; }
        if (*hbad) return;
        const int64_t r0 = c * rows, r1 = std::min(n, r0 + rows);
        const int64_t a = r0 + (r1 - r0) * w / T, b = r0 + (r1 - r0) * (w + 1) / T;
        if (a == b) continue;
        const size_t off = size_t(a) * n, cnt = size_t(b - a) * n;
        if (dw) host_widen_dist(st + off * dw, dw, static_cast<char*>(dist_out) + off * es, wide, cnt);
        if (pk) {
          const uint16_t* src = reinterpret_cast<const uint16_t*>(st + dbytes) + off;
          const bool wide = idx_dtype == APSP_DTYPE_I64;
          host_widen_pred(src, static_cast<char*>(idx_out) + off * (wide ? 8 : 4), wide, cnt);
        }
      }
    };
    const bool trace = std::getenv("APSP_READBACK_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int w = 1; w < T; w++) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    if (trace) {
      // last chunk landed vs. widening done: the gap is the host tail
      const auto t1 = std::chrono::steady_clock::now();
      cudaEventSynchronize(ev.back());
      std::fprintf(stderr, "[readback] n=%lld dw=%d pred=%d chunks=%lld threads=%d host wait+widen %.2f ms\n",
                   (long long)n, dw, int(pk), (long long)nch, T,
                   std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    if (err) e = cudaErrorUnknown;
  }
  const bool flagged = e == cudaSuccess && *hbad;
  lk.unlock();
  for (cudaEvent_t x : ev)
    if (x) cudaEventDestroy(x);
  cudaFreeAsync(dev, s);
  if (e != cudaSuccess) return set_cuda_error(e, "packed readback", __FILE__, __LINE__);
  handled = !flagged;   // a value outside the promised width: the caller copies int32 as is
  return 0;
}

// ---- last-round streaming readback (blocked FW, u8 tier) ----------------------------------

namespace {

__global__ void pack_pred_rows_kernel(const int32_t* __restrict__ P, int64_t ldp, int64_t rows, int64_t n,
                                      uint16_t* __restrict__ out) {
  const int64_t q = n >> 2, total = rows * q;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < total; g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = g / q, j = 4 * (g - i * q);
    const int4 v = *reinterpret_cast<const int4*>(P + i * ldp + j);
    *reinterpret_cast<uint2*>(out + i * n + j) = make_uint2(uint32_t(v.x + 1) | uint32_t(v.y + 1) << 16,
                                                            uint32_t(v.z + 1) | uint32_t(v.w + 1) << 16);
  }
}

// The last FW round's row bands go to the host as they land: the u8 store rows are the dist
// readback as they are (255 = Infinity), pred rows are packed to u16 on a copy stream, and host
// workers widen each band into the caller's buffers while later bands are still computing.
// Valid only if the u8 attempt is the one that certifies; otherwise the caller reads back as
// usual and overwrites whatever was streamed.
class BandStream final : public BandSink {
 public:
  BandStream(int64_t n, int es, void* dist_out, void* idx_out, int idx_dtype, cudaStream_t s)
      : n_(n), es_(es), dist_out_(dist_out), idx_out_(idx_out), wide_idx_(idx_dtype == APSP_DTYPE_I64), lk_(g_down.mu) {
    pbase_ = (size_t(n) * n + 255) & ~size_t(255);
    if (g_down.reserve(pbase_ + size_t(n) * n * 2 + 64) != cudaSuccess) return;
    if (cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking) != cudaSuccess) return;
    if (cudaMallocAsync(&ppk_, size_t(n) * n * 2, s) != cudaSuccess) return;
    // the copy stream may use ppk_ only after its allocation on s
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return;
    cudaEventRecord(e, s);
    cudaStreamWaitEvent(cs_, e, 0);
    cudaEventDestroy(e);
    st_ = static_cast<char*>(g_down.ptr);
    const int T = host_workers();
    for (int t = 0; t < T; t++) pool_.emplace_back([this, t, T] { work(t, T); });
    ok_ = true;
  }
  ~BandStream() override { finish(); }

  bool ready() const { return ok_; }

  int band(int64_t r0, int64_t r1, const FwCtx& c, cudaStream_t s) override {
    r1 = std::min(r1, n_);
    if (!ok_ || r0 >= r1) return 0;
    if (c.store != STORE_U8 || !c.P) {   // not the u8 tier: these rows are not ours to stream
      invalid_ = true;
      return 0;
    }
    cudaEvent_t landed = nullptr, done = nullptr;
    APSP_CUDA_TRY(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming));
    // workers block on it (no spinning: 16 spinning threads would starve the launching thread)
    APSP_CUDA_TRY(cudaEventCreateWithFlags(&done, cudaEventDisableTiming | cudaEventBlockingSync));
    APSP_CUDA_TRY(cudaEventRecord(landed, s));
    APSP_CUDA_TRY(cudaStreamWaitEvent(cs_, landed, 0));
    cudaEventDestroy(landed);
    const int64_t rows = r1 - r0;
    APSP_CUDA_TRY(cudaMemcpy2DAsync(st_ + size_t(r0) * n_, size_t(n_), c.D + r0 * c.ld, size_t(c.ld), size_t(n_),
                                    size_t(rows), cudaMemcpyDeviceToHost, cs_));
    pack_pred_rows_kernel<<<148 * 4, 256, 0, cs_>>>(c.P + r0 * c.ldp, c.ldp, rows, n_, ppk_ + r0 * n_);
    APSP_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    APSP_CUDA_TRY(cudaMemcpyAsync(st_ + pbase_ + size_t(r0) * n_ * 2, ppk_ + r0 * n_, size_t(rows) * n_ * 2,
                                  cudaMemcpyDeviceToHost, cs_));
    APSP_CUDA_TRY(cudaEventRecord(done, cs_));
    {
      std::lock_guard<std::mutex> g(qm_);
      bands_.push_back({r0, r1, done});
      if (r1 == n_) covered_ = true;
    }
    qc_.notify_all();
    return 0;
  }

  // stops the workers; true when the streamed rows are the certified u8 result
  bool finish() {
    if (trace_)
      std::fprintf(stderr, "[bandstream] solve returned at %.2f ms (%zu bands)\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count(),
                   bands_.size());
    {
      std::lock_guard<std::mutex> g(qm_);
      if (finished_) return result_;
      finished_ = true;
    }
    qc_.notify_all();
    for (auto& t : pool_) t.join();
    pool_.clear();
    if (cs_) cudaStreamSynchronize(cs_);
    for (auto& b : bands_) cudaEventDestroy(b.ev);
    if (ppk_) cudaFreeAsync(ppk_, cs_);
    if (cs_) {
      cudaStreamSynchronize(cs_);
      cudaStreamDestroy(cs_);
    }
    cs_ = nullptr;
    ppk_ = nullptr;
    result_ = ok_ && !invalid_ && covered_ && !werr_;
    if (trace_)
      std::fprintf(stderr, "[bandstream] widened by %.2f ms, result %d\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count(),
                   int(result_));
    return result_;
  }

 private:
  struct Band { int64_t r0, r1; cudaEvent_t ev; };

  void work(int t, int T) {
    size_t next = 0;
    for (;;) {
      Band b;
      {
        std::unique_lock<std::mutex> g(qm_);
        qc_.wait(g, [&] { return next < bands_.size() || finished_; });
        if (next >= bands_.size()) return;   // finished and drained
        b = bands_[next++];
      }
      if (cudaEventSynchronize(b.ev) != cudaSuccess) { werr_ = true; continue; }
      if (t == 0 && trace_)
        std::fprintf(stderr, "[bandstream] rows %lld..%lld landed at %.2f ms\n", (long long)b.r0, (long long)b.r1,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0_).count());
      const int64_t a = b.r0 + (b.r1 - b.r0) * t / T, e = b.r0 + (b.r1 - b.r0) * (t + 1) / T;
      if (a >= e) continue;
      const size_t off = size_t(a) * n_, cnt = size_t(e - a) * n_;
      host_widen_dist(st_ + off, 1, static_cast<char*>(dist_out_) + off * es_, es_ == 8, cnt);
      host_widen_pred(reinterpret_cast<const uint16_t*>(st_ + pbase_) + off,
                      static_cast<char*>(idx_out_) + off * (wide_idx_ ? 8 : 4), wide_idx_, cnt);
    }
  }

  int64_t n_;
  int es_;
  void* dist_out_;
  void* idx_out_;
  bool wide_idx_;
  std::unique_lock<std::mutex> lk_;   // the readback staging is ours for the whole solve
  size_t pbase_ = 0;
  char* st_ = nullptr;
  cudaStream_t cs_ = nullptr;
  uint16_t* ppk_ = nullptr;
  std::vector<std::thread> pool_;
  std::mutex qm_;
  std::condition_variable qc_;
  std::vector<Band> bands_;
  bool finished_ = false, covered_ = false, ok_ = false, result_ = false;
  std::atomic<bool> invalid_{false}, werr_{false};
  const bool trace_ = std::getenv("APSP_READBACK_TRACE") != nullptr;
  const std::chrono::steady_clock::time_point t0_ = std::chrono::steady_clock::now();
};

}  // namespace

std::unique_ptr<BandSink> make_band_stream(int64_t n, int es, void* dist_out, void* idx_out, int idx_dtype,
                                           cudaStream_t s) {
  const char* env = std::getenv("APSP_STREAM_READBACK");
  if ((env && env[0] == '0') || !idx_out || n >= 65535 || n * n < (int64_t(1) << 22) || n % 4) return nullptr;
  auto b = std::make_unique<BandStream>(n, es, dist_out, idx_out, idx_dtype, s);
  if (!b->ready()) return nullptr;
  return b;
}

bool finish_band_stream(BandSink* b) { return b && static_cast<BandStream*>(b)->finish(); }

}  // namespace apsp
