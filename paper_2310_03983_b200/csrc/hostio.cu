// Host readback of apsp_solve_host (include/apsp_b200.h): the n x n int32 distances and
// predecessors leave the GPU narrowed, and host threads widen them into the caller's buffers.
//
// Over PCIe the readback of an int32 result is 8 bytes per cell (dist + pred). Most results need
// far fewer bits: a u8-tier result has max_finite <= 254, and predecessors are < n. One device
// pass packs dist to 1 or 2 bytes (INF32 -> all-ones) and pred to 2 bytes (p + 1, so -1 -> 0).
// The packed rows then come back in row chunks. Each chunk gets its own event, and a host worker
// pool widens chunk c while chunk c+1 is still on the wire. The pool writes with streaming stores,
// so the output lines are not read first. At n=16384 u8 this moves 768 MiB instead of 2 GiB.
//
// The pack kernel flags any value outside the promised width. A flagged result falls back to the
// plain int32 copies, so the output is always the exact device result.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>
#include <sched.h>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#include "engine.h"

namespace apsp {

namespace {

constexpr int32_t kInf32 = INF32;   // the API's int32 "no path" (core.py INF32)

template <int DW, bool PRED>
__global__ void pack_result_kernel(const int32_t* __restrict__ d, const int32_t* __restrict__ p, int64_t cells,
                                   void* __restrict__ dpk, uint16_t* __restrict__ ppk, int32_t lim,
                                   int* __restrict__ bad) {
  const int64_t groups = cells >> 2;
  int flag = 0;
  for (int64_t g = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; g < groups; g += int64_t(gridDim.x) * blockDim.x) {
    if (DW) {
      const int4 v = reinterpret_cast<const int4*>(d)[g];
      const int32_t x[4] = {v.x, v.y, v.z, v.w};
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const bool inf = x[q] == kInf32;
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

// ---- host widening (streaming stores where the target is 16-byte aligned) ------------------

template <typename T>
inline bool aligned16(const T* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void widen_dist(const void* src, int dw, int32_t* dst, size_t cnt) {
  size_t i = 0;
  if (dw == 1) {
    const uint8_t* s = static_cast<const uint8_t*>(src);
    for (; i < cnt && !aligned16(dst + i); i++) dst[i] = s[i] == 0xFF ? kInf32 : s[i];
#if defined(__SSE2__)
    const __m128i z = _mm_setzero_si128(), m = _mm_set1_epi32(0xFF), inf = _mm_set1_epi32(kInf32);
    for (; i + 16 <= cnt; i += 16) {
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i lo = _mm_unpacklo_epi8(b, z), hi = _mm_unpackhi_epi8(b, z);
      const __m128i w[4] = {_mm_unpacklo_epi16(lo, z), _mm_unpackhi_epi16(lo, z), _mm_unpacklo_epi16(hi, z),
                            _mm_unpackhi_epi16(hi, z)};
      for (int q = 0; q < 4; q++) {
        const __m128i e = _mm_cmpeq_epi32(w[q], m);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4 * q),
                         _mm_or_si128(_mm_andnot_si128(e, w[q]), _mm_and_si128(e, inf)));
      }
    }
#endif
    for (; i < cnt; i++) dst[i] = s[i] == 0xFF ? kInf32 : s[i];
  } else {
    const uint16_t* s = static_cast<const uint16_t*>(src);
    for (; i < cnt && !aligned16(dst + i); i++) dst[i] = s[i] == 0xFFFF ? kInf32 : s[i];
#if defined(__SSE2__)
    const __m128i z = _mm_setzero_si128(), m = _mm_set1_epi32(0xFFFF), inf = _mm_set1_epi32(kInf32);
    for (; i + 8 <= cnt; i += 8) {
      const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i w[2] = {_mm_unpacklo_epi16(h, z), _mm_unpackhi_epi16(h, z)};
      for (int q = 0; q < 2; q++) {
        const __m128i e = _mm_cmpeq_epi32(w[q], m);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4 * q),
                         _mm_or_si128(_mm_andnot_si128(e, w[q]), _mm_and_si128(e, inf)));
      }
    }
#endif
    for (; i < cnt; i++) dst[i] = s[i] == 0xFFFF ? kInf32 : s[i];
  }
}

template <typename T>
void widen_pred(const uint16_t* s, T* dst, size_t cnt) {
  size_t i = 0;
  for (; i < cnt && !aligned16(dst + i); i++) dst[i] = T(int32_t(s[i]) - 1);
#if defined(__SSE2__)
  const __m128i z = _mm_setzero_si128(), one = _mm_set1_epi32(1);
  for (; i + 8 <= cnt; i += 8) {
    const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i w[2] = {_mm_sub_epi32(_mm_unpacklo_epi16(h, z), one), _mm_sub_epi32(_mm_unpackhi_epi16(h, z), one)};
    for (int q = 0; q < 2; q++) {
      if (sizeof(T) == 4) {
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4 * q), w[q]);
      } else {
        const __m128i sg = _mm_srai_epi32(w[q], 31);
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4 * q), _mm_unpacklo_epi32(w[q], sg));
        _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 4 * q + 2), _mm_unpackhi_epi32(w[q], sg));
      }
    }
  }
#endif
  for (; i < cnt; i++) dst[i] = T(int32_t(s[i]) - 1);
}

// ---- pinned staging, grow-only, process-wide ------------------------------------------------

std::mutex g_stage_mu;
void* g_stage = nullptr;
size_t g_stage_bytes = 0;

int host_workers() {
  if (const char* e = std::getenv("APSP_HOST_THREADS")) return std::max(1, std::atoi(e));
  cpu_set_t set;
  int n = 0;
  if (sched_getaffinity(0, sizeof(set), &set) == 0) n = CPU_COUNT(&set);
  if (n <= 0) n = int(std::thread::hardware_concurrency());
  return std::clamp(n, 1, 16);
}

int dist_width(int64_t max_finite) {
  return max_finite >= 0 && max_finite <= 254 ? 1 : max_finite >= 0 && max_finite <= 65534 ? 2 : 0;
}

}  // namespace

int32_t readback_width(int64_t n, int64_t max_finite, bool idx, int idx_dtype) {
  const int dw = dist_width(max_finite);
  return (dw ? dw : 4) + (idx ? 2 : 0);
}

// Reads back n x n int32 dist (and int32 pred when idx_out) from contiguous device buffers.
// handled = false when the packed path does not apply; the caller then does the plain copies.
int readback_packed(int64_t n, const int32_t* d, const int32_t* p, int64_t max_finite, void* dist_out, void* idx_out,
                    int idx_dtype, cudaStream_t s, bool& handled) {
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
  const int grid = 148 * 8;
  const int32_t lim = dw == 1 ? 254 : 65534;
  if (e == cudaSuccess) {
    if (dw == 1 && pk) pack_result_kernel<1, true><<<grid, 256, 0, s>>>(d, p, cells, dev, ppk, lim, bad);
    else if (dw == 1) pack_result_kernel<1, false><<<grid, 256, 0, s>>>(d, p, cells, dev, ppk, lim, bad);
    else if (dw == 2 && pk) pack_result_kernel<2, true><<<grid, 256, 0, s>>>(d, p, cells, dev, ppk, lim, bad);
    else if (dw == 2) pack_result_kernel<2, false><<<grid, 256, 0, s>>>(d, p, cells, dev, ppk, lim, bad);
    else pack_result_kernel<0, true><<<grid, 256, 0, s>>>(d, p, cells, dev, ppk, lim, bad);
    e = cudaGetLastError();
    count_launches(1);
  }
  std::unique_lock<std::mutex> lk(g_stage_mu);
  const size_t need = dbytes + pbytes + 64;
  if (e == cudaSuccess && g_stage_bytes < need) {
    if (g_stage) cudaFreeHost(g_stage);
    g_stage = nullptr;
    g_stage_bytes = 0;
    e = cudaHostAlloc(&g_stage, need, cudaHostAllocPortable);
    if (e == cudaSuccess) g_stage_bytes = need;
  }
  char* st = static_cast<char*>(g_stage);
  volatile int* hbad = reinterpret_cast<volatile int*>(st + dbytes + pbytes);
  if (e == cudaSuccess) e = cudaMemcpyAsync((void*)hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  // row chunks: >= 16 of them, each at most 2048 rows
  const int64_t rows = std::min<int64_t>(2048, std::max<int64_t>(1, (n + 15) / 16));
  const int64_t nch = (n + rows - 1) / rows;
  std::vector<cudaEvent_t> ev(size_t(nch), nullptr);
  for (int64_t c = 0; e == cudaSuccess && c < nch; c++) {
    const size_t r0 = size_t(c * rows), rc = size_t(std::min(n, (c + 1) * rows) - c * rows);
    if (dw)
      e = cudaMemcpyAsync(st + r0 * n * dw, static_cast<char*>(dev) + r0 * n * dw, rc * n * dw,
                          cudaMemcpyDeviceToHost, s);
    else
      e = cudaMemcpyAsync(static_cast<int32_t*>(dist_out) + r0 * n, d + r0 * n, rc * n * 4, cudaMemcpyDeviceToHost, s);
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
        if (dw) widen_dist(st + off * dw, dw, static_cast<int32_t*>(dist_out) + off, cnt);
        if (pk) {
          const uint16_t* src = reinterpret_cast<const uint16_t*>(st + dbytes) + off;
          if (idx_dtype == APSP_DTYPE_I64) widen_pred(src, static_cast<int64_t*>(idx_out) + off, cnt);
          else widen_pred(src, static_cast<int32_t*>(idx_out) + off, cnt);
        }
      }
#if defined(__SSE2__)
      _mm_sfence();
#endif
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < T; w++) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
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

}  // namespace apsp
