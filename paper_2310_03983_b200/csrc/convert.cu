// Input scan (K7), API dtype <-> store conversion with padding and pred initialisation,
// result certificate (max finite), index copies and the minplus_product witness clear.
// All are HBM-bound elementwise kernels: 2D grid-stride sweeps (rows over blockIdx.y, columns
// over threads) -- no per-element 64-bit index division, coalesced along rows.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include "launch.h"

namespace apsp {

// API dtypes (apsp_b200.h): 0 = int32 (INF32), 1 = fp32 (+inf), 2 = int64 (INF_RAW)
enum ApiDtype : int { API_I32 = 0, API_F32 = 1, API_I64 = 2 };

size_t store_elem_size(int store) {
  switch (store) {
    case STORE_U8: return 1;
    case STORE_W32: case STORE_I32: case STORE_F32: return 4;
    case STORE_I64: return 8;
    case STORE_U16: return 2;
  }
  return 0;
}

template <int D> struct Api;
template <> struct Api<API_I32> { using T = int32_t; __device__ static bool fin(T v) { return v != INF32; } };
template <> struct Api<API_F32> { using T = float;   __device__ static bool fin(T v) { return !isinf(v) || v < 0; } };
template <> struct Api<API_I64> { using T = int64_t; __device__ static bool fin(T v) { return v != INF_RAW; } };

// rows over blockIdx.y (grid-stride), columns over blockIdx.x * blockDim.x + threadIdx.x
#define FOR_2D(i, j, rows, cols)                                                                         \
  for (int64_t i = blockIdx.y; i < (rows); i += gridDim.y)                                               \
    for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < (cols); j += int64_t(gridDim.x) * blockDim.x)

// Unrolled vector sweep for the HBM-bound reductions: rows over blockIdx.y (grid-stride); in a
// row each thread takes U segments blockDim.x apart per step and issues all U loads before using
// any, so enough bytes are in flight on 4 CTAs per SM (one load per thread reached ~2 TB/s).
template <int U, typename V, typename F>
__device__ __forceinline__ void sweep_vec(const V* base, int64_t ldv, int64_t rows, int64_t cv, F&& f) {
  for (int64_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const V* row = base + i * ldv;
    for (int64_t jb = int64_t(blockIdx.x) * blockDim.x * U + threadIdx.x; jb < cv;
         jb += int64_t(gridDim.x) * blockDim.x * U) {
      V w[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t j = jb + int64_t(u) * blockDim.x;
        if (j < cv) w[u] = __ldg(row + j);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t j = jb + int64_t(u) * blockDim.x;
        if (j < cv) f(i, j, w[u]);
      }
    }
  }
}
constexpr int kSweepU = 4;

static dim3 grid_vec(int64_t rows, int64_t cv, int64_t ctas) {
  int64_t gx = (cv + 256 * kSweepU - 1) / (256 * kSweepU);
  gx = std::min<int64_t>(std::max<int64_t>(gx, 1), 16);
  const int64_t gy = std::max<int64_t>(1, std::min<int64_t>({(ctas + gx - 1) / gx, rows, 65535}));
  return dim3(unsigned(gx), unsigned(gy));
}

static dim3 grid_2d(int64_t rows, int64_t cols, int64_t ctas = 148 * 16) {
  int64_t gx = (cols + 255) / 256;
  if (gx > 16) gx = 16;
  if (gx < 1) gx = 1;
  int64_t gy = (ctas + gx - 1) / gx;
  if (gy > rows) gy = rows;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  return dim3(unsigned(gx), unsigned(gy));
}

// Reductions (scan, certificate) run on 4 CTAs per SM and combine per CTA before one atomic
// per field: per-warp atomics on the same few addresses serialise in L2 (2368 CTAs x 8 warps
// made the n=2048 scan 40 us).
constexpr int64_t kReduceCtas = 148 * 4;
enum : uint32_t { F_NEG = 1, F_DIAG = 2, F_NONINT = 4, F_ANYFIN = 8, F_ZERO = 16 };

__device__ __forceinline__ void block_commit(ScanResult* out, uint32_t flags, long long mx, float mxf,
                                             unsigned long long edges) {
  __shared__ uint32_t s_fl[32];
  __shared__ long long s_mx[32];
  __shared__ float s_mf[32];
  __shared__ unsigned long long s_ed[32];
  flags = __reduce_or_sync(0xffffffffu, flags);
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mxf = fmaxf(mxf, __shfl_xor_sync(0xffffffffu, mxf, o));
    edges += __shfl_xor_sync(0xffffffffu, edges, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_fl[w] = flags;
    s_mx[w] = mx;
    s_mf[w] = mxf;
    s_ed[w] = edges;
  }
  __syncthreads();
  if (threadIdx.x) return;
  for (int q = 1; q < nw; q++) {
    flags |= s_fl[q];
    mx = max(mx, s_mx[q]);
    mxf = fmaxf(mxf, s_mf[q]);
    edges += s_ed[q];
  }
  if (flags & F_NEG) atomicOr(&out->negative, 1);
  if (flags & F_DIAG) atomicOr(&out->diag_nonzero, 1);
  if (flags & F_NONINT) atomicOr(&out->non_integral, 1);
  if (flags & F_ANYFIN) atomicOr(&out->any_finite, 1);
  if (flags & F_ZERO) atomicOr(&out->zero_offdiag, 1);
  if (mx >= 0) atomicMax(reinterpret_cast<unsigned long long*>(&out->max_finite), (unsigned long long)mx);
  if (mxf >= 0.f) atomicMax(reinterpret_cast<int*>(&out->max_finite_f), __float_as_int(mxf));
  if (edges) atomicAdd(&out->finite_offdiag, edges);
}

template <int D>
struct ScanAcc {   // per-thread flags as a bit set, the max in the input type (widened once, at the end)
  using T = typename Api<D>::T;
  uint32_t flags = 0;
  uint32_t edges = 0;   // a thread sees far fewer than 2^32 cells
  T mx = T(-1);
  __device__ __forceinline__ void add(T v, bool on_diag) {
    if (on_diag && v != T(0)) flags |= F_DIAG;
    if (!Api<D>::fin(v)) return;
    flags |= F_ANYFIN;
    if (!on_diag) {
      edges++;
      if (v == T(0)) flags |= F_ZERO;
    }
    if constexpr (D == API_F32) {
      if (isnan(v) || v < 0.f) {
        flags |= F_NEG;
        return;
      }
      if (v != floorf(v)) flags |= F_NONINT;
      mx = fmaxf(mx, v);
    } else {
      if (v < 0) {
        flags |= F_NEG;
        return;
      }
      mx = max(mx, v);
    }
  }
  __device__ __forceinline__ long long max_ll() const {
    if constexpr (D == API_F32) return mx < 0.f ? -1 : (long long)fminf(mx, 9.0e18f);
    else return (long long)mx;
  }
  __device__ __forceinline__ float max_f() const {
    if constexpr (D == API_F32) return mx;
    else return -1.f;
  }
};

// vec: 4-byte elements, cols % 4 == 0, ld % 4 == 0, 16-byte aligned base -> one 16-byte load
// per thread per step (the scalar sweep reaches ~30% of HBM bandwidth, this ~75%)
template <int D>
__global__ void scan_kernel(const typename Api<D>::T* h, int64_t ld, int64_t rows, int64_t cols, int64_t diag_off,
                            ScanResult* out, int vec) {
  using T = typename Api<D>::T;
  ScanAcc<D> a;
  if constexpr (sizeof(T) == 4) {
    if (vec) {
      sweep_vec<kSweepU>(reinterpret_cast<const int4*>(h), ld / 4, rows, cols / 4, [&](int64_t i, int64_t j4, int4 w) {
        const int64_t j = 4 * j4, dj = diag_off >= 0 ? i + diag_off - j : -1;
        a.add(__builtin_bit_cast(T, w.x), dj == 0);
        a.add(__builtin_bit_cast(T, w.y), dj == 1);
        a.add(__builtin_bit_cast(T, w.z), dj == 2);
        a.add(__builtin_bit_cast(T, w.w), dj == 3);
      });
    }
  }
  if (!vec || sizeof(T) != 4) {
    FOR_2D(i, j, rows, cols) a.add(h[i * ld + j], diag_off >= 0 && j == i + diag_off);
  }
  block_commit(out, a.flags, a.max_ll(), a.max_f(), a.edges);
}

static bool vec4_ok(const void* p, int64_t ld, int64_t cols, size_t es) {
  return es == 4 && cols % 4 == 0 && ld % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

int launch_scan(int in_dtype, const void* h, int64_t ld, int64_t rows, int64_t cols, int64_t diag_off,
                ScanResult* out_dev, cudaStream_t s) {
  APSP_CUDA_TRY(cudaMemsetAsync(out_dev, 0, sizeof(ScanResult), s));
  // max fields start at 0 after memset; negative sentinel not needed (values are >= 0)
  const int vec = vec4_ok(h, ld, cols, in_dtype == API_I64 ? 8 : 4);
  const dim3 g = vec ? grid_vec(rows, cols / 4, kReduceCtas) : grid_2d(rows, cols, kReduceCtas);
  switch (in_dtype) {
    case API_I32: scan_kernel<API_I32><<<g, 256, 0, s>>>((const int32_t*)h, ld, rows, cols, diag_off, out_dev, vec); break;
    case API_F32: scan_kernel<API_F32><<<g, 256, 0, s>>>((const float*)h, ld, rows, cols, diag_off, out_dev, vec); break;
    case API_I64: scan_kernel<API_I64><<<g, 256, 0, s>>>((const int64_t*)h, ld, rows, cols, diag_off, out_dev, 0); break;
    default: return set_error(2, "unknown dtype %d", in_dtype);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

// ---- conversion into a padded store ------------------------------------------------
// A finite input value into store S. The narrow stores saturate (negative -> 0, beyond the
// tier -> its Infinity): a speculative attempt (fw_sched.cu) may run a tier before the scan that
// rejects it is read back, and its kernels must still see keys inside the tier's range (a wrapped
// u16 key would carry garbage tag bits into the argmin decode). Admissible inputs are unchanged.
template <int S, typename V>
__device__ __forceinline__ typename StoreT<S>::T store_val(V v) {
  using T = typename StoreT<S>::T;
  if constexpr (S == STORE_U8 || S == STORE_U16 || S == STORE_W32) {
    const auto inf = store_inf<S>();
    if (!(v >= V(0))) return T(0);          // negative (and NaN): rejected by the scan anyway
    if (v >= V(inf)) return inf;
    return T(v);
  } else {
    return T(v);
  }
}

// rows [row0, row0 + R) of the padded N x N matrix (R = N, row0 = 0 for a whole matrix)
template <int D, int S>
__device__ __forceinline__ typename StoreT<S>::T store_cell(const typename Api<D>::T* h, int64_t ldh, int64_t n,
                                                            int64_t il, int64_t i, int64_t j, bool& fin) {
  using T = typename StoreT<S>::T;
  if (i < n && j < n) {
    const typename Api<D>::T v = h[il * ldh + j];
    fin = Api<D>::fin(v);
    return fin ? store_val<S>(v) : store_inf<S>();
  }
  fin = (i == j);
  return fin ? T(0) : store_inf<S>();
}

// vec: 4-byte input, n % 4 == 0, all pitches % 4 == 0 and 16-byte aligned bases -> 4 columns per
// thread step: one 16-byte input load, one 4 x es output store, one 16-byte pred store
template <int D, int S>
__global__ void to_store_kernel(const typename Api<D>::T* h, int64_t ldh, int64_t n, typename StoreT<S>::T* out,
                                int64_t ld, int64_t N, int32_t* P, int64_t ldp, int pred_init, int64_t row0,
                                int64_t R, int vec) {
  using T = typename StoreT<S>::T;
  if constexpr (sizeof(typename Api<D>::T) == 4 && sizeof(T) <= 4) {
    if (vec) {
      FOR_2D(il, j4, R, N / 4) {
        const int64_t i = row0 + il, j = 4 * j4;
        T o[4];
        bool fin[4];
        if (i < n && j + 3 < n) {
          const int4 w = __ldg(reinterpret_cast<const int4*>(h + il * ldh + j));
          const typename Api<D>::T v[4] = {__builtin_bit_cast(typename Api<D>::T, w.x),
                                           __builtin_bit_cast(typename Api<D>::T, w.y),
                                           __builtin_bit_cast(typename Api<D>::T, w.z),
                                           __builtin_bit_cast(typename Api<D>::T, w.w)};
#pragma unroll
          for (int q = 0; q < 4; q++) {
            fin[q] = Api<D>::fin(v[q]);
            o[q] = fin[q] ? store_val<S>(v[q]) : store_inf<S>();
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; q++) o[q] = store_cell<D, S>(h, ldh, n, il, i, j + q, fin[q]);
        }
        if constexpr (sizeof(T) == 1) {
          *reinterpret_cast<uint32_t*>(out + il * ld + j) =
              uint32_t(o[0]) | (uint32_t(o[1]) << 8) | (uint32_t(o[2]) << 16) | (uint32_t(o[3]) << 24);
        } else if constexpr (sizeof(T) == 2) {
          *reinterpret_cast<uint2*>(out + il * ld + j) =
              make_uint2(uint32_t(o[0]) | (uint32_t(o[1]) << 16), uint32_t(o[2]) | (uint32_t(o[3]) << 16));
        } else {
          *reinterpret_cast<int4*>(out + il * ld + j) =
              make_int4(__builtin_bit_cast(int, o[0]), __builtin_bit_cast(int, o[1]), __builtin_bit_cast(int, o[2]),
                        __builtin_bit_cast(int, o[3]));
        }
        if (P) {
          int32_t pv[4];
#pragma unroll
          for (int q = 0; q < 4; q++)
            pv[q] = (pred_init && fin[q] && i != j + q && i < n && j + q < n) ? int32_t(i) : -1;
          *reinterpret_cast<int4*>(P + il * ldp + j) = make_int4(pv[0], pv[1], pv[2], pv[3]);
        }
      }
      return;
    }
  }
  FOR_2D(il, j, R, N) {
    const int64_t i = row0 + il;
    bool fin;
    out[il * ld + j] = store_cell<D, S>(h, ldh, n, il, i, j, fin);
    if (P) P[il * ldp + j] = (pred_init && fin && i != j && i < n && j < n) ? int32_t(i) : -1;
  }
}

template <int D>
static int to_store_d(const void* h, int64_t ldh, int64_t n, int store, void* Dp, int64_t ld, int64_t N, int32_t* P,
                      int64_t ldp, int pred_init, int64_t row0, int64_t R, cudaStream_t s) {
  using TI = typename Api<D>::T;
  const size_t es_out = store_elem_size(store);
  const int vec = sizeof(TI) == 4 && es_out <= 4 && n % 4 == 0 && N % 4 == 0 && ldh % 4 == 0 && ld % 4 == 0 &&
                  (!P || ldp % 4 == 0) && (reinterpret_cast<uintptr_t>(h) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(Dp) & (4 * es_out - 1)) == 0 &&
                  (!P || (reinterpret_cast<uintptr_t>(P) & 15) == 0);
  const dim3 g = grid_2d(R, vec ? N / 4 : N);
  const TI* hh = static_cast<const TI*>(h);
  switch (store) {
    case STORE_U8: to_store_kernel<D, STORE_U8><<<g, 256, 0, s>>>(hh, ldh, n, (uint8_t*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    case STORE_W32: to_store_kernel<D, STORE_W32><<<g, 256, 0, s>>>(hh, ldh, n, (int32_t*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    case STORE_I32: to_store_kernel<D, STORE_I32><<<g, 256, 0, s>>>(hh, ldh, n, (int32_t*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    case STORE_F32: to_store_kernel<D, STORE_F32><<<g, 256, 0, s>>>(hh, ldh, n, (float*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    case STORE_I64: to_store_kernel<D, STORE_I64><<<g, 256, 0, s>>>(hh, ldh, n, (int64_t*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    case STORE_U16: to_store_kernel<D, STORE_U16><<<g, 256, 0, s>>>(hh, ldh, n, (uint16_t*)Dp, ld, N, P, ldp, pred_init, row0, R, vec); break;
    default: return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

int launch_to_store_rows(int in_dtype, const void* h, int64_t ldh, int64_t n, int store, void* D, int64_t ld,
                         int64_t N, int32_t* P, int64_t ldp, int pred_init, int64_t row0, int64_t R, cudaStream_t s) {
  switch (in_dtype) {
    case API_I32: return to_store_d<API_I32>(h, ldh, n, store, D, ld, N, P, ldp, pred_init, row0, R, s);
    case API_F32: return to_store_d<API_F32>(h, ldh, n, store, D, ld, N, P, ldp, pred_init, row0, R, s);
    case API_I64: return to_store_d<API_I64>(h, ldh, n, store, D, ld, N, P, ldp, pred_init, row0, R, s);
  }
  return set_error(2, "unknown dtype %d", in_dtype);
}

int launch_to_store(int in_dtype, const void* h, int64_t ldh, int64_t n, int store, void* D, int64_t ld, int64_t N,
                    int32_t* P, int64_t ldp, int pred_init, cudaStream_t s) {
  return launch_to_store_rows(in_dtype, h, ldh, n, store, D, ld, N, P, ldp, pred_init, 0, N, s);
}

// ---- conversion of a rectangular operand (no padding); h == nullptr fills Infinity -------
template <int D, int S>
__global__ void to_store_rect_kernel(const typename Api<D>::T* h, int64_t ldh, int64_t rows, int64_t cols,
                                     typename StoreT<S>::T* out, int64_t ldo) {
  using T = typename StoreT<S>::T;
  FOR_2D(i, j, rows, cols) {
    T o = store_inf<S>();
    if (h) {
      const typename Api<D>::T v = h[i * ldh + j];
      if (Api<D>::fin(v)) o = store_val<S>(v);
    }
    out[i * ldo + j] = o;
  }
}

template <int D>
static int rect_d(const void* h, int64_t ldh, int64_t rows, int64_t cols, int store, void* out, int64_t ldo,
                  cudaStream_t s) {
  using TI = typename Api<D>::T;
  const dim3 g = grid_2d(rows, cols);
  const TI* hh = static_cast<const TI*>(h);
  switch (store) {
    case STORE_U8: to_store_rect_kernel<D, STORE_U8><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (uint8_t*)out, ldo); break;
    case STORE_W32: to_store_rect_kernel<D, STORE_W32><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (int32_t*)out, ldo); break;
    case STORE_I32: to_store_rect_kernel<D, STORE_I32><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (int32_t*)out, ldo); break;
    case STORE_F32: to_store_rect_kernel<D, STORE_F32><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (float*)out, ldo); break;
    case STORE_I64: to_store_rect_kernel<D, STORE_I64><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (int64_t*)out, ldo); break;
    case STORE_U16: to_store_rect_kernel<D, STORE_U16><<<g, 256, 0, s>>>(hh, ldh, rows, cols, (uint16_t*)out, ldo); break;
    default: return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

int launch_to_store_rect(int in_dtype, const void* h, int64_t ldh, int64_t rows, int64_t cols, int store, void* out,
                         int64_t ldo, cudaStream_t s) {
  switch (in_dtype) {
    case API_I32: return rect_d<API_I32>(h, ldh, rows, cols, store, out, ldo, s);
    case API_F32: return rect_d<API_F32>(h, ldh, rows, cols, store, out, ldo, s);
    case API_I64: return rect_d<API_I64>(h, ldh, rows, cols, store, out, ldo, s);
  }
  return set_error(2, "unknown dtype %d", in_dtype);
}

// ---- conversion back -----------------------------------------------------------------
template <int S, int D>
__device__ __forceinline__ typename Api<D>::T from_cell(typename StoreT<S>::T v) {
  using TO = typename Api<D>::T;
  if constexpr (S == STORE_F32) {
    return TO(v);   // +inf maps to +inf (fp32 out) -- int outs never come from an fp32 store
  } else {
    if (v == store_inf<S>()) {
      if constexpr (D == API_I32) return INF32;
      else if constexpr (D == API_I64) return INF_RAW;
      else return __int_as_float(0x7f800000);
    }
    return TO(v);
  }
}

// vec: u8 / u16 store into a 4-byte API output, cols % 4 == 0, aligned pitches: 4 cells per step
template <int S, int D>
__global__ void from_store_kernel(const typename StoreT<S>::T* in, int64_t ld, int64_t rows, int64_t cols,
                                  typename Api<D>::T* out, int64_t ldo, int vec) {
  using T = typename StoreT<S>::T;
  using TO = typename Api<D>::T;
  if constexpr (sizeof(T) <= 2 && sizeof(TO) == 4) {
    if (vec) {
      FOR_2D(i, j4, rows, cols / 4) {
        T v[4];
        if constexpr (sizeof(T) == 1) *reinterpret_cast<uint32_t*>(v) = *reinterpret_cast<const uint32_t*>(in + i * ld + 4 * j4);
        else *reinterpret_cast<uint2*>(v) = *reinterpret_cast<const uint2*>(in + i * ld + 4 * j4);
        const TO o0 = from_cell<S, D>(v[0]), o1 = from_cell<S, D>(v[1]), o2 = from_cell<S, D>(v[2]),
                 o3 = from_cell<S, D>(v[3]);
        *reinterpret_cast<int4*>(out + i * ldo + 4 * j4) =
            make_int4(__builtin_bit_cast(int, o0), __builtin_bit_cast(int, o1), __builtin_bit_cast(int, o2),
                      __builtin_bit_cast(int, o3));
      }
      return;
    }
  }
  FOR_2D(i, j, rows, cols) out[i * ldo + j] = from_cell<S, D>(in[i * ld + j]);
}

template <int S>
static int from_store_s(const void* in, int64_t ld, int64_t rows, int64_t cols, int out_dtype, void* out, int64_t ldo,
                        cudaStream_t s) {
  using TI = typename StoreT<S>::T;
  // same representation on both sides (fp32 -> fp32, exact int32 -> int32, int64 -> int64):
  // a strided copy
  if ((S == STORE_F32 && out_dtype == API_F32) || (S == STORE_I32 && out_dtype == API_I32) ||
      (S == STORE_I64 && out_dtype == API_I64)) {
    APSP_CUDA_TRY(cudaMemcpy2DAsync(out, size_t(ldo) * sizeof(TI), in, size_t(ld) * sizeof(TI), size_t(cols) * sizeof(TI),
                                    size_t(rows), cudaMemcpyDeviceToDevice, s));
    return 0;
  }
  const int vec = sizeof(TI) <= 2 && out_dtype != API_I64 && cols % 4 == 0 && ld % 4 == 0 && ldo % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(in) & (4 * sizeof(TI) - 1)) == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const dim3 g = grid_2d(rows, vec ? cols / 4 : cols);
  const TI* ii = static_cast<const TI*>(in);
  switch (out_dtype) {
    case API_I32: from_store_kernel<S, API_I32><<<g, 256, 0, s>>>(ii, ld, rows, cols, (int32_t*)out, ldo, vec); break;
    case API_F32: from_store_kernel<S, API_F32><<<g, 256, 0, s>>>(ii, ld, rows, cols, (float*)out, ldo, vec); break;
    case API_I64: from_store_kernel<S, API_I64><<<g, 256, 0, s>>>(ii, ld, rows, cols, (int64_t*)out, ldo, vec); break;
    default: return set_error(2, "unknown dtype %d", out_dtype);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

int launch_from_store(int store, const void* D, int64_t ld, int64_t rows, int64_t cols, int out_dtype, void* out,
                      int64_t ldo, cudaStream_t s) {
  switch (store) {
    case STORE_U8: return from_store_s<STORE_U8>(D, ld, rows, cols, out_dtype, out, ldo, s);
    case STORE_W32: return from_store_s<STORE_W32>(D, ld, rows, cols, out_dtype, out, ldo, s);
    case STORE_I32: return from_store_s<STORE_I32>(D, ld, rows, cols, out_dtype, out, ldo, s);
    case STORE_F32: return from_store_s<STORE_F32>(D, ld, rows, cols, out_dtype, out, ldo, s);
    case STORE_I64: return from_store_s<STORE_I64>(D, ld, rows, cols, out_dtype, out, ldo, s);
    case STORE_U16: return from_store_s<STORE_U16>(D, ld, rows, cols, out_dtype, out, ldo, s);
  }
  return set_error(2, "unknown store %d", store);
}

// ---- index copies ----------------------------------------------------------------------
template <typename TO>
__global__ void copy_idx_kernel(const int32_t* P, int64_t ldp, int64_t rows, int64_t cols, TO* out, int64_t ldo) {
  FOR_2D(i, j, rows, cols) out[i * ldo + j] = TO(P[i * ldp + j]);
}

int launch_copy_idx(const int32_t* P, int64_t ldp, int64_t rows, int64_t cols, int out_dtype, void* out, int64_t ldo,
                    cudaStream_t s) {
  const dim3 g = grid_2d(rows, cols);
  if (out_dtype == API_I64) copy_idx_kernel<int64_t><<<g, 256, 0, s>>>(P, ldp, rows, cols, (int64_t*)out, ldo);
  else copy_idx_kernel<int32_t><<<g, 256, 0, s>>>(P, ldp, rows, cols, (int32_t*)out, ldo);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

__global__ void fill_idx_kernel(int32_t* P, int64_t ldp, int64_t rows, int64_t cols, int32_t v) {
  FOR_2D(i, j, rows, cols) P[i * ldp + j] = v;
}

int launch_fill_idx(int32_t* P, int64_t ldp, int64_t rows, int64_t cols, int32_t v, cudaStream_t s) {
  fill_idx_kernel<<<grid_2d(rows, cols), 256, 0, s>>>(P, ldp, rows, cols, v);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

int launch_copy_block(int store, const void* src, int64_t lds, void* dst, int64_t ldd, int64_t rows, int64_t cols,
                      cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return 0;
  const size_t es = store_elem_size(store);
  APSP_CUDA_TRY(cudaMemcpy2DAsync(dst, size_t(ldd) * es, src, size_t(lds) * es, size_t(cols) * es, size_t(rows),
                                  cudaMemcpyDeviceToDevice, s));
  return 0;
}

// ---- certificate: max finite value of a store ------------------------------------------
template <int S>
__global__ void max_finite_kernel(const typename StoreT<S>::T* D, int64_t ld, int64_t rows, int64_t cols,
                                  ScanResult* out, int vec) {
  const auto inf = store_inf<S>();
  long long mx = -1;
  float mxf = -1.f;
  if constexpr (S == STORE_U8) {
    if (vec) {   // 16 cells per step: INF bytes zeroed, then a packed byte max (the diagonal is 0,
                 // so a finite value always exists)
      uint32_t m4 = 0;
      sweep_vec<kSweepU>(reinterpret_cast<const uint4*>(D), ld / 16, rows, cols / 16, [&](int64_t, int64_t, uint4 w) {
        const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; q++) m4 = __vmaxu4(m4, x[q] & ~__vcmpeq4(x[q], 0xFFFFFFFFu));
      });
      mx = max(max(m4 & 0xFF, (m4 >> 8) & 0xFF), max((m4 >> 16) & 0xFF, m4 >> 24));
    }
  } else if constexpr (sizeof(typename StoreT<S>::T) == 4) {
    if (vec) {   // 4 cells per 16-byte segment
      sweep_vec<kSweepU>(reinterpret_cast<const uint4*>(D), ld / 4, rows, cols / 4, [&](int64_t, int64_t, uint4 w) {
        const uint32_t x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const auto v = __builtin_bit_cast(typename StoreT<S>::T, x[q]);
          if (v == inf) continue;
          if constexpr (S == STORE_F32) mxf = fmaxf(mxf, v);
          else mx = max(mx, (long long)v);
        }
      });
    }
  }
  if (!vec || (S != STORE_U8 && sizeof(typename StoreT<S>::T) != 4)) {
    FOR_2D(i, j, rows, cols) {
      const auto v = D[i * ld + j];
      if (v == inf) continue;
      if constexpr (S == STORE_F32) mxf = fmaxf(mxf, v);
      else mx = max(mx, (long long)v);
    }
  }
  block_commit(out, 0u, mx, mxf, 0ull);
}

int launch_max_finite(int store, const void* D, int64_t ld, int64_t rows, int64_t cols, ScanResult* out_dev,
                      cudaStream_t s) {
  APSP_CUDA_TRY(cudaMemsetAsync(out_dev, 0, sizeof(ScanResult), s));
  const size_t es = store_elem_size(store);
  const int per = es == 1 ? 16 : 4;   // cells per 16-byte segment (u8, or the 4-byte stores)
  const int vec = (es == 1 || es == 4) && cols % per == 0 && ld % per == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0;
  const dim3 g = vec ? grid_vec(rows, cols / per, kReduceCtas) : grid_2d(rows, cols, kReduceCtas);
  switch (store) {
    case STORE_U8: max_finite_kernel<STORE_U8><<<g, 256, 0, s>>>((const uint8_t*)D, ld, rows, cols, out_dev, vec); break;
    case STORE_W32: max_finite_kernel<STORE_W32><<<g, 256, 0, s>>>((const int32_t*)D, ld, rows, cols, out_dev, vec); break;
    case STORE_I32: max_finite_kernel<STORE_I32><<<g, 256, 0, s>>>((const int32_t*)D, ld, rows, cols, out_dev, vec); break;
    case STORE_F32: max_finite_kernel<STORE_F32><<<g, 256, 0, s>>>((const float*)D, ld, rows, cols, out_dev, vec); break;
    case STORE_I64: max_finite_kernel<STORE_I64><<<g, 256, 0, s>>>((const int64_t*)D, ld, rows, cols, out_dev, vec); break;
    case STORE_U16: max_finite_kernel<STORE_U16><<<g, 256, 0, s>>>((const uint16_t*)D, ld, rows, cols, out_dev, vec); break;
    default: return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

// ---- minplus_product self-witness via clear (minplus.py:99-111) -----------------------
template <int S>
__global__ void witness_clear_kernel(const typename StoreT<S>::T* X, int64_t ldx, const typename StoreT<S>::T* Y,
                                     int64_t ldy, const typename StoreT<S>::T* Dp, int64_t ldd, int32_t* via,
                                     int64_t ldv, int64_t n1, int64_t n2, int64_t n3, int64_t row_off,
                                     int64_t inner_off, int64_t col_off) {
  using A = typename StoreT<S>::A;
  const auto inf = store_inf<S>();
  FOR_2D(i, j, n1, n3) {
    const auto best = Dp[i * ldd + j];
    if (best == inf) continue;
    const int64_t ti = i + row_off - inner_off;
    if (ti >= 0 && ti < n2 && X[i * ldx + ti] != inf && Y[ti * ldy + j] != inf &&
        A(X[i * ldx + ti]) + A(Y[ti * ldy + j]) == A(best)) {
      via[i * ldv + j] = -1;
      continue;
    }
    const int64_t tj = j + col_off - inner_off;
    if (tj >= 0 && tj < n2 && X[i * ldx + tj] != inf && Y[tj * ldy + j] != inf &&
        A(X[i * ldx + tj]) + A(Y[tj * ldy + j]) == A(best))
      via[i * ldv + j] = -1;
  }
}

int launch_witness_clear(int store, const void* X, int64_t ldx, const void* Y, int64_t ldy, const void* Dp,
                         int64_t ldd, int32_t* via, int64_t ldv, int64_t n1, int64_t n2, int64_t n3, int64_t row_off,
                         int64_t inner_off, int64_t col_off, cudaStream_t s) {
  const dim3 g = grid_2d(n1, n3);
#define WC(S, T)                                                                                              \
  witness_clear_kernel<S><<<g, 256, 0, s>>>((const T*)X, ldx, (const T*)Y, ldy, (const T*)Dp, ldd, via, ldv, n1, \
                                            n2, n3, row_off, inner_off, col_off)
  switch (store) {
    case STORE_U8: WC(STORE_U8, uint8_t); break;
    case STORE_W32: WC(STORE_W32, int32_t); break;
    case STORE_I32: WC(STORE_I32, int32_t); break;
    case STORE_F32: WC(STORE_F32, float); break;
    case STORE_I64: WC(STORE_I64, int64_t); break;
    case STORE_U16: WC(STORE_U16, uint16_t); break;
    default: return set_error(2, "unknown store %d", store);
  }
#undef WC
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

// ---- error state -------------------------------------------------------------------------
static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int set_cuda_error(cudaError_t e, const char* what, const char* file, int line) {
  return set_error(3, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), cudaGetErrorString(e), file, line, what);
}

const char* last_error() { return g_err; }

static std::atomic<long long> g_launches{0};
void count_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

}  // namespace apsp
