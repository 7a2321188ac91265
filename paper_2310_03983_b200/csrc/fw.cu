// Floyd-Warshall kernels whose order of k matters: the classic per-k step (K1) and the
// diagonal-block closure (blocked phase 1 and the R-Kleene leaf).  Both use the
// strict-improvement rule of solvers.py:89-94 and write idx as pred[k][j] (FW rule) or as the
// global k (via rule, solvers.py:109-114).  Phase 2 runs as min-plus products against the
// closed diagonal block (minplus.cu).
//
// Race freedom: with a zero diagonal and nonnegative costs, row k and column k are invariant
// during step k (solvers.py:79-81), so one barrier per k suffices.
#include <algorithm>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include "launch.h"
#include "tiles.cuh"
#include "engine.h"

namespace apsp {

// ------------------------------------------------------------------------------------
// K1: one classic FW step over an n x n view (bit-exact with fw_classic)
// ------------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(256) fw_step_kernel(typename StoreT<S>::T* D, int64_t ld, int64_t n, int64_t k,
                                                      int32_t* idx, int64_t ldi, int mode, int64_t via_off,
                                                      Status* st) {
  using T = typename StoreT<S>::T;
  using A = typename StoreT<S>::A;
  const int64_t j = int64_t(blockIdx.x) * 32 + (threadIdx.x & 31);
  const int64_t ib = int64_t(blockIdx.y) * 32;
  __shared__ A dkj_s[32];
  __shared__ int32_t pkj_s[32];
  if (threadIdx.x < 32) {
    dkj_s[threadIdx.x] = j < n ? A(D[k * ld + j]) : A(store_inf<S>());
    pkj_s[threadIdx.x] = (j < n && idx && mode == IDX_PRED) ? idx[k * ldi + j] : -1;
  }
  __syncthreads();
  if (j >= n) return;
  const A dkj = dkj_s[threadIdx.x & 31];
  const int32_t pkj = pkj_s[threadIdx.x & 31];
  bool overflow = false, changed = false;
  for (int r = threadIdx.x >> 5; r < 32; r += 8) {
    const int64_t i = ib + r;
    if (i >= n) break;
    const A dik = A(D[i * ld + k]);
    const A c = dik + dkj;
    if (c < A(D[i * ld + j])) {
      overflow |= range_overflow<S>(c);
      changed = true;
      D[i * ld + j] = T(c);
      if (idx) idx[i * ldi + j] = (mode == IDX_PRED) ? pkj : int32_t(via_off + k);
    }
  }
  if (st) {
    if (overflow) st->overflow = 1;
    if (changed) st->changed = 1;
  }
}

// K1 for small n in ONE launch: a single 1024-thread CTA keeps the whole matrix in shared
// memory and runs the n classic steps with one barrier each (row and column k are invariant
// during step k, so the cells of a step are independent). Pred stays in global memory (L1/L2
// on this SM) and is touched only for improved cells: pred[i][j] <- pred[k][j], pred row k is
// invariant in step k too. Same strict-< rule as fw_step_kernel, so the result is bit-exact
// with fw_classic. n = 128 (u16): 0.65 -> 0.34 ms; n = 256 (u8): 2.0 -> 1.85 ms.
constexpr int K1CTA_THREADS = 1024;
constexpr size_t K1CTA_MAX_SMEM = 200 * 1024;

template <int S>
__global__ void __launch_bounds__(K1CTA_THREADS) fw_classic_cta_kernel(typename StoreT<S>::T* D, int64_t ld, int n,
                                                                       int32_t* idx, int64_t ldi, Status* st) {
  using T = typename StoreT<S>::T;
  using A = typename StoreT<S>::A;
  extern __shared__ __align__(16) unsigned char smraw_k1[];
  T* Ds = reinterpret_cast<T*>(smraw_k1);   // n x n, row pitch n
  int32_t* prow = reinterpret_cast<int32_t*>(smraw_k1 + ((size_t(n) * n * sizeof(T) + 15) / 16) * 16);
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  for (int e = t; e < n * n; e += K1CTA_THREADS) Ds[e] = D[int64_t(e / n) * ld + e % n];
  __syncthreads();
  bool overflow = false;
  for (int k = 0; k < n; k++) {
    if (idx) {   // pred row k (invariant in step k) into shared memory first
      for (int j = t; j < n; j += K1CTA_THREADS) prow[j] = idx[int64_t(k) * ldi + j];
      __syncthreads();
    }
    const T* rowk = Ds + k * n;
    for (int i = ty; i < n; i += 32) {
      const A dik = A(Ds[i * n + k]);
      if (dik == A(store_inf<S>())) continue;   // nothing through an unreachable k
      for (int j = tx; j < n; j += 32) {
        const A c = dik + A(rowk[j]);
        if (c < A(Ds[i * n + j])) {
          overflow |= range_overflow<S>(c);
          Ds[i * n + j] = T(c);
          if (idx) idx[int64_t(i) * ldi + j] = prow[j];
        }
      }
    }
    __syncthreads();
  }
  for (int e = t; e < n * n; e += K1CTA_THREADS) D[int64_t(e / n) * ld + e % n] = Ds[e];
  if (st && overflow) st->overflow = 1;
}

// The narrow stores (n even): cells as 16-bit values in shared memory, relaxed two at a time --
// one packed add (VADD2) and one packed compare per column pair, row k's pairs in registers.
// Sums stay below 2^16 (u8 <= 510, u16 <= 1022) and a stored sum is below the tier's Infinity,
// so there is nothing to flag. Same strict-< rule and pred copy as above.
template <int S>
__global__ void __launch_bounds__(K1CTA_THREADS) fw_classic_cta_packed_kernel(typename StoreT<S>::T* D, int64_t ld,
                                                                              int n, int32_t* idx, int64_t ldi) {
  using T = typename StoreT<S>::T;
  extern __shared__ __align__(16) unsigned char smraw_k1p[];
  uint16_t* Ds = reinterpret_cast<uint16_t*>(smraw_k1p);   // n x n, row pitch n (even)
  int32_t* prow = reinterpret_cast<int32_t*>(Ds + n * n);  // pred row k of the current step
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5, np = n >> 1;
  const uint32_t inf = uint32_t(store_inf<S>());
  for (int e = t; e < n * n; e += K1CTA_THREADS) Ds[e] = uint16_t(D[int64_t(e / n) * ld + e % n]);
  __syncthreads();
  for (int k = 0; k < n; k++) {
    // pred row k (invariant in step k) into shared memory first: an improved cell then copies
    // it from there instead of waiting on a global load (the loop was bound by those)
    if (idx) {
      for (int j = t; j < n; j += K1CTA_THREADS) prow[j] = idx[int64_t(k) * ldi + j];
      __syncthreads();
    }
    const uint32_t* rowk = reinterpret_cast<const uint32_t*>(Ds + k * n);
    for (int i = ty; i < n; i += 32) {
      const uint32_t dik = Ds[i * n + k];
      if (dik == inf) continue;   // nothing through an unreachable k
      const uint32_t dik2 = dik * 0x00010001u;
      uint32_t* rowi = reinterpret_cast<uint32_t*>(Ds + i * n);
      for (int q = tx; q < np; q += 32) {
        const uint32_t cur = rowi[q], cand = __vadd2(dik2, rowk[q]);
        const uint32_t lt = __vcmpltu2(cand, cur);   // 0xFFFF in each half that strictly improves
        if (lt) {
          rowi[q] = (cand & lt) | (cur & ~lt);
          if (idx) {
            const int64_t j = 2 * q;
            if (lt & 0xFFFFu) idx[int64_t(i) * ldi + j] = prow[j];
            if (lt >> 16) idx[int64_t(i) * ldi + j + 1] = prow[j + 1];
          }
        }
      }
    }
    __syncthreads();
  }
  for (int e = t; e < n * n; e += K1CTA_THREADS) D[int64_t(e / n) * ld + e % n] = T(Ds[e]);
}

// true (and launched) when the whole n x n store fits one CTA's shared memory
int launch_fw_classic_cta(int store, void* D, int64_t ld, int64_t n, int32_t* idx, int64_t ldi, Status* st,
                          cudaStream_t s, bool& done) {
  done = false;
  const size_t bytes = (size_t(n) * n * store_elem_size(store) + 15) / 16 * 16 + size_t(n) * 4;   // + pred row
  // one SM's issue rate bounds it: 2x the graph-replayed steps at n=128, ~8% at 256, slower above
  if (n < 2 || n > 256 || bytes > K1CTA_MAX_SMEM || getenv("APSP_K1_STEPS")) return 0;
  static std::atomic<unsigned long long> a8{0}, a16{0}, a32{0}, af{0}, a64{0}, aw{0}, p8{0}, p16{0};
  const int sb = int(bytes);
  if ((store == STORE_U8 || store == STORE_U16) && n % 2 == 0 && size_t(n) * n * 2 + size_t(n) * 4 <= K1CTA_MAX_SMEM &&
      !getenv("APSP_K1_SCALAR")) {
    const int sp = int(size_t(n) * n * 2 + size_t(n) * 4);
    if (store == STORE_U8) {
      APSP_CUDA_TRY(smem_optin(fw_classic_cta_packed_kernel<STORE_U8>, int(K1CTA_MAX_SMEM), p8));
      fw_classic_cta_packed_kernel<STORE_U8><<<1, K1CTA_THREADS, sp, s>>>(static_cast<uint8_t*>(D), ld, int(n), idx, ldi);
    } else {
      APSP_CUDA_TRY(smem_optin(fw_classic_cta_packed_kernel<STORE_U16>, int(K1CTA_MAX_SMEM), p16));
      fw_classic_cta_packed_kernel<STORE_U16><<<1, K1CTA_THREADS, sp, s>>>(static_cast<uint16_t*>(D), ld, int(n), idx,
                                                                            ldi);
    }
    APSP_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    done = true;
    return 0;
  }
  switch (store) {
#define K1CTA(ST, TT, ATTR)                                                                                  \
  case ST:                                                                                                   \
    APSP_CUDA_TRY(smem_optin(fw_classic_cta_kernel<ST>, int(K1CTA_MAX_SMEM), ATTR));                      \
    fw_classic_cta_kernel<ST><<<1, K1CTA_THREADS, sb, s>>>(static_cast<TT*>(D), ld, int(n), idx, ldi, st); \
    break;
    K1CTA(STORE_U8, uint8_t, a8)
    K1CTA(STORE_U16, uint16_t, a16)
    K1CTA(STORE_I32, int32_t, a32)
    K1CTA(STORE_F32, float, af)
    K1CTA(STORE_I64, int64_t, a64)
    K1CTA(STORE_W32, int32_t, aw)
#undef K1CTA
    default: return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  done = true;
  return 0;
}

// K1 for the narrow stores: HBM-bound, so each thread streams 16-byte row segments (16 u8 or
// 8 u16 cells) down a band of rows, four rows in flight. The cells are relaxed as packed
// 16-bit pairs with one VIADDMNMX.U16x2 (min(D[i][k] + D[k][j], D[i][j])) per two cells; the
// sums stay below 2^16 (u8: <= 510, u16: <= 1022). Row k's pairs stay in registers, column k is
// one broadcast byte per row, and a row whose D[i][k] is Infinity is skipped unread. Pred row k
// is read only for improved cells. Same strict-< rule and idx semantics as
// fw_step_kernel (row and column k are invariant during step k).
template <int S>
__device__ __forceinline__ void seg_to_pairs(const uint4& g, uint32_t (&p)[8 / sizeof(typename StoreT<S>::T)]) {
  const uint32_t w[4] = {g.x, g.y, g.z, g.w};
  if constexpr (sizeof(typename StoreT<S>::T) == 1) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      p[2 * q] = __byte_perm(w[q], 0, 0x4140);
      p[2 * q + 1] = __byte_perm(w[q], 0, 0x4342);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; q++) p[q] = w[q];
  }
}

template <int S>
__device__ __forceinline__ uint4 pairs_to_seg(const uint32_t (&p)[8 / sizeof(typename StoreT<S>::T)]) {
  if constexpr (sizeof(typename StoreT<S>::T) == 1)
    return make_uint4(__byte_perm(p[0], p[1], 0x6420), __byte_perm(p[2], p[3], 0x6420),
                      __byte_perm(p[4], p[5], 0x6420), __byte_perm(p[6], p[7], 0x6420));
  else
    return make_uint4(p[0], p[1], p[2], p[3]);
}

template <int S>
__global__ void __launch_bounds__(256, 3) fw_step_vec_kernel(typename StoreT<S>::T* D, int64_t ld, int64_t n, int64_t k,
                                                          int32_t* idx, int64_t ldi, int mode, int64_t via_off,
                                                          Status* st, int rows) {
  using T = typename StoreT<S>::T;
  constexpr int V = 16 / int(sizeof(T)), P = V / 2;
  const uint32_t INF = store_inf<S>();
  const int64_t j0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * V;
  if (j0 >= n) return;
  uint32_t dkj[P];
  seg_to_pairs<S>(*reinterpret_cast<const uint4*>(D + k * ld + j0), dkj);
  bool changed = false;
  const int64_t i1 = std::min<int64_t>(n, (int64_t(blockIdx.y) + 1) * rows);
  constexpr int R = 4;   // rows in flight per thread: their loads are issued before any store
  // column-k bytes run one batch ahead, so a batch's segment loads never wait on them
  uint32_t dnext[R];
  const int64_t ib = int64_t(blockIdx.y) * rows;
#pragma unroll
  for (int r = 0; r < R; r++) dnext[r] = ib + r < i1 ? uint32_t(D[(ib + r) * ld + k]) : INF;
  for (int64_t i0 = ib; i0 < i1; i0 += R) {
    uint32_t dik[R];
    uint4 seg[R];
#pragma unroll
    for (int r = 0; r < R; r++) dik[r] = dnext[r];
#pragma unroll
    for (int r = 0; r < R; r++)
      if (dik[r] != INF) seg[r] = *reinterpret_cast<const uint4*>(D + (i0 + r) * ld + j0);
#pragma unroll
    for (int r = 0; r < R; r++) dnext[r] = i0 + R + r < i1 ? uint32_t(D[(i0 + R + r) * ld + k]) : INF;
#pragma unroll
    for (int r = 0; r < R; r++) {
      if (dik[r] == INF) continue;
      uint32_t v[P], nv[P], diff = 0;
      seg_to_pairs<S>(seg[r], v);
      const uint32_t dik2 = dik[r] * 0x00010001u;
#pragma unroll
      for (int q = 0; q < P; q++) {
        nv[q] = __viaddmin_u16x2(dik2, dkj[q], v[q]);
        diff |= nv[q] ^ v[q];
      }
      if (!diff) continue;
      const int64_t i = i0 + r;
      changed = true;
      *reinterpret_cast<uint4*>(D + i * ld + j0) = pairs_to_seg<S>(nv);
      if (!idx) continue;
      const int32_t* pk = idx + k * ldi + j0;   // pred row k (invariant in step k; L1/L2-resident)
#pragma unroll
      for (int q = 0; q < P; q++) {
        const uint32_t x = nv[q] ^ v[q];
        if (x & 0xFFFFu) idx[i * ldi + j0 + 2 * q] = mode == IDX_PRED ? pk[2 * q] : int32_t(via_off + k);
        if (x >> 16) idx[i * ldi + j0 + 2 * q + 1] = mode == IDX_PRED ? pk[2 * q + 1] : int32_t(via_off + k);
      }
    }
  }
  if (st && changed) st->changed = 1;
}

int launch_fw_step(int store, void* D, int64_t ld, int64_t n, int64_t k, int32_t* idx, int64_t ldi, int mode,
                   int64_t via_off, Status* st, cudaStream_t s) {
  if ((store == STORE_U8 || store == STORE_U16) && !getenv("APSP_K1_SCALAR")) {
    const int es = int(store_elem_size(store)), V = 16 / es;
    if (n % V == 0 && (ld * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0) {
      const int64_t bx = (n / V + 255) / 256;
      // one full wave: 148 SMs x 3 resident CTAs (launch bounds), each streaming `rows` rows
      const int rows = int(std::max<int64_t>(8, (n * bx + 148 * 3 - 1) / (148 * 3)));
      const dim3 g(unsigned(bx), unsigned((n + rows - 1) / rows));
      if (store == STORE_U8)
        fw_step_vec_kernel<STORE_U8><<<g, 256, 0, s>>>((uint8_t*)D, ld, n, k, idx, ldi, mode, via_off, st, rows);
      else
        fw_step_vec_kernel<STORE_U16><<<g, 256, 0, s>>>((uint16_t*)D, ld, n, k, idx, ldi, mode, via_off, st, rows);
      APSP_CUDA_TRY(cudaGetLastError());
      count_launches(1);
      return 0;
    }
  }
  dim3 grid(unsigned((n + 31) / 32), unsigned((n + 31) / 32));
  switch (store) {
    case STORE_I32: fw_step_kernel<STORE_I32><<<grid, 256, 0, s>>>((int32_t*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    case STORE_F32: fw_step_kernel<STORE_F32><<<grid, 256, 0, s>>>((float*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    case STORE_I64: fw_step_kernel<STORE_I64><<<grid, 256, 0, s>>>((int64_t*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    case STORE_U16: fw_step_kernel<STORE_U16><<<grid, 256, 0, s>>>((uint16_t*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    case STORE_U8: fw_step_kernel<STORE_U8><<<grid, 256, 0, s>>>((uint8_t*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    case STORE_W32: fw_step_kernel<STORE_W32><<<grid, 256, 0, s>>>((int32_t*)D, ld, n, k, idx, ldi, mode, via_off, st); break;
    default: return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

// ------------------------------------------------------------------------------------
// Diagonal block closure, m <= 128, one CTA of 32x32 threads, block resident in smem.
// ------------------------------------------------------------------------------------
constexpr int MAXB = 128;

// Register-resident closure: 512 threads, thread (ty, tx) of 16x32 owns cells i = ty + 16a
// (a < 8), j = tx + 32c (c < 4).  Step k: the owners of row k / column k have published them
// into a double-buffered smem row/column (values, and pred for row k); one barrier; every
// thread relaxes its 32 cells; the owners of row / column k+1 publish them right away.
constexpr int CR = 8, CC = 4;
template <int S>
__global__ void __launch_bounds__(512) block_close_kernel(typename StoreT<S>::T* D, int64_t ld, int64_t lo, int m,
                                                          int32_t* idx, int64_t ldi, int mode, int64_t via_off,
                                                          Status* st) {
  using T = typename StoreT<S>::T;
  using A = typename StoreT<S>::A;
  __shared__ A rowk[2][MAXB];
  __shared__ A colk[2][MAXB];
  __shared__ int32_t prowk[2][MAXB];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const A inf = A(store_inf<S>());
  A v[CR][CC];
  int32_t p[CR][CC];
#pragma unroll
  for (int a = 0; a < CR; a++)
#pragma unroll
    for (int c = 0; c < CC; c++) {
      const int i = ty + 16 * a, j = tx + 32 * c;
      const bool in = i < m && j < m;
      v[a][c] = in ? A(D[(lo + i) * ld + lo + j]) : inf;
      p[a][c] = (in && idx) ? idx[(lo + i) * ldi + lo + j] : -1;
    }
// publish row / column KK of the register tile (select chains: no dynamic register indexing)
#define APSP_PUBLISH(KK, BUF)                                        \
  do {                                                               \
    const int pk_ = (KK), pb_ = (BUF);                               \
    if (ty == (pk_ & 15)) {                                          \
      const int sa_ = pk_ >> 4;                                      \
      _Pragma("unroll") for (int c = 0; c < CC; c++) {               \
        A rv_ = v[0][c];                                             \
        int32_t rp_ = p[0][c];                                       \
        _Pragma("unroll") for (int a = 1; a < CR; a++) {             \
          rv_ = (a == sa_) ? v[a][c] : rv_;                          \
          rp_ = (a == sa_) ? p[a][c] : rp_;                          \
        }                                                            \
        rowk[pb_][tx + 32 * c] = rv_;                                \
        prowk[pb_][tx + 32 * c] = rp_;                               \
      }                                                              \
    }                                                                \
    if (tx == (pk_ & 31)) {                                          \
      const int sc_ = pk_ >> 5;                                      \
      _Pragma("unroll") for (int a = 0; a < CR; a++) {               \
        A cv_ = v[a][0];                                             \
        _Pragma("unroll") for (int c = 1; c < CC; c++)               \
          cv_ = (c == sc_) ? v[a][c] : cv_;                          \
        colk[pb_][ty + 16 * a] = cv_;                                \
      }                                                              \
    }                                                                \
  } while (0)
  APSP_PUBLISH(0, 0);
  bool overflow = false;
  for (int k = 0; k < m; k++) {
    __syncthreads();
    const int b = k & 1;
    A dkj[CC], dik[CR];
    int32_t pkj[CC];
#pragma unroll
    for (int c = 0; c < CC; c++) {
      dkj[c] = rowk[b][tx + 32 * c];
      pkj[c] = prowk[b][tx + 32 * c];
    }
#pragma unroll
    for (int a = 0; a < CR; a++) dik[a] = colk[b][ty + 16 * a];
    const int32_t vk = int32_t(via_off + k);
#pragma unroll
    for (int a = 0; a < CR; a++)
#pragma unroll
      for (int c = 0; c < CC; c++) {
        const A cand = dik[a] + dkj[c];
        if (cand < v[a][c]) {
          overflow |= range_overflow<S>(cand);
          v[a][c] = cand;
          p[a][c] = (mode == IDX_PRED) ? pkj[c] : vk;
        }
      }
    if (k + 1 < m) APSP_PUBLISH(k + 1, b ^ 1);
  }
#pragma unroll
  for (int a = 0; a < CR; a++)
#pragma unroll
    for (int c = 0; c < CC; c++) {
      const int i = ty + 16 * a, j = tx + 32 * c;
      if (i < m && j < m) {
        D[(lo + i) * ld + lo + j] = T(v[a][c]);
        if (idx) idx[(lo + i) * ldi + lo + j] = p[a][c];
      }
    }
  if (st && overflow) st->overflow = 1;
}

// ------------------------------------------------------------------------------------
// u8 tier closure of an m <= 128 diagonal block: packed 16-bit DPX keys.
//   key = value << 7 | tag, tag = 1 + (k mod 64), decoded every 64 steps into the last
//   improving k per cell (8 bits, 1-based).  Row / column k are used tag-free.
//   pred is deferred: with k* the last improving step of (i,j), pred[k*][j] never changes after
//   step k* (else (i,j) would improve again), so pred_final[i][j] = pred_final[k*][j]; the
//   chains k* -> kst(k*, j) -> ... strictly decrease and are resolved by pointer jumping.
//   The result equals the classic in-block order exactly (values, pred and via).
// 512 threads: warp w owns columns 8w..8w+7 of every row, lane l owns rows 4l..4l+3, so a
// thread holds rows 4l + r (r < 4) x column pairs 8w + 2p (p < 4).  Row k of a warp's columns
// lives in lane k >> 2 of the same warp and is broadcast by shuffle; column k lives in warp
// k >> 3 (all lanes) and goes through shared memory, one 16-byte store per lane.  The k loop
// is unrolled by 8, so every register index is a compile-time constant (no select chains).
// ------------------------------------------------------------------------------------
struct CloseU8Smem {
  uint32_t colk[2][MAXB];     // column k as replicated tag-free keys, by row (16-byte lane slots)
  uint32_t colk1[2][MAXB];    // column k + 1 likewise (full blocks: two steps per barrier)
  int32_t P[MAXB][MAXB];      // pred resolution; prefetched by cp.async while the k loop runs
  uint8_t K[MAXB][MAXB];      // 1-based last improving k (0 = none); value staging before that
  uint8_t Kpad[MAXB][MAXB];   // second half of the u16 value staging
};

// Key formats of the packed closure: u8 values << 7 with 64-step tag windows, u16 values << 6
// with 32-step windows (INF + INF + tag < 2^16 in both).
template <int S> struct CloseKeys;
template <> struct CloseKeys<STORE_U8> {
  using T = uint8_t;
  static constexpr int TAG = 7, WIN = 64;
  static constexpr uint32_t INF = U8_INF;
};
template <> struct CloseKeys<STORE_U16> {
  using T = uint16_t;
  static constexpr int TAG = 6, WIN = 32;
  static constexpr uint32_t INF = U16_INF;
};

// The closure body is a device function so the persistent small-n kernel (fw_persist.cu) can
// run it as one of its tasks; block_close_dpx_kernel below is the stand-alone launch.
__device__ unsigned long long g_close128_phase[6];   // APSP_CLOSE_PROF: summed ns per phase + count
__device__ __forceinline__ unsigned long long close_gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}

template <int S, bool FULL>
__device__ __forceinline__ void close_dpx_body(typename CloseKeys<S>::T* D, int64_t ld, int64_t lo, int m,
                                               int32_t* idx, int64_t ldi, int mode, int64_t via_off,
                                               unsigned char* smraw_cu8, bool prof = false) {
  if (FULL) m = MAXB;   // every FW phase-1 block: the bounds checks fold away
  unsigned long long tp[5] = {};
  if (prof && threadIdx.x == 0) tp[0] = close_gtimer();
  using CK = CloseKeys<S>;
  using T = typename CK::T;
  constexpr int TAG = CK::TAG, WIN = CK::WIN, VB = int(sizeof(T));
  constexpr uint32_t TMASK2 = ((1u << TAG) - 1u) * 0x00010001u;   // tag bits of both halves
  constexpr uint32_t STRIP2 = ~TMASK2;
  CloseU8Smem& sm = *reinterpret_cast<CloseU8Smem*>(smraw_cu8);
  T (*stage)[MAXB] = reinterpret_cast<T (*)[MAXB]>(&sm.K[0][0]);   // value staging (aliases K, Kpad)
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t acc[4][4];   // [row r][pair p]: columns (8w + 2p, 8w + 2p + 1)
  uint32_t kst[4][2];   // byte 2 * (p & 1) + h of kst[r][p >> 1] = cell (r, 8w + 2p + h)
  // coalesced load through the K staging area (lanes over columns), then each thread picks
  // its 4 rows x 8 bytes
  constexpr int SEG = 16 / VB;   // values per 16-byte segment
  const bool vec = m == MAXB && ((reinterpret_cast<uintptr_t>(D + lo * ld + lo) | uintptr_t(ld * VB)) & 15) == 0;
  // the predecessors are needed only after the k loop: start their copy now
  const bool pre = FULL && idx && mode == IDX_PRED &&
                   ((reinterpret_cast<uintptr_t>(idx + lo * ldi + lo) | uintptr_t(ldi * 4)) & 15) == 0;
  if (pre) {
    for (int e = threadIdx.x; e < MAXB * MAXB / 4; e += blockDim.x) {
      const int i = e >> 5, j = 4 * (e & 31);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.P[i][j])),
                   "l"(idx + (lo + i) * ldi + lo + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  if (vec) {   // full aligned block (every FW phase 1): 16-byte row segments
    for (int e = threadIdx.x; e < MAXB * MAXB / SEG; e += blockDim.x) {
      const int i = e / (MAXB / SEG), j = SEG * (e % (MAXB / SEG));
      *reinterpret_cast<uint4*>(&stage[i][j]) = __ldcg(reinterpret_cast<const uint4*>(D + (lo + i) * ld + lo + j));
    }
  } else {
    for (int e = threadIdx.x; e < MAXB * MAXB; e += blockDim.x) {
      const int i = e >> 7, j = e & 127;
      stage[i][j] = (i < m && j < m) ? D[(lo + i) * ld + lo + j] : T(CK::INF);
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; r++) {
    kst[r][0] = kst[r][1] = 0;
    if constexpr (VB == 1) {
      const uint2 v = *reinterpret_cast<const uint2*>(&stage[4 * l + r][8 * w]);
      acc[r][0] = __byte_perm(v.x, 0, 0x4140) << TAG;
      acc[r][1] = __byte_perm(v.x, 0, 0x4342) << TAG;
      acc[r][2] = __byte_perm(v.y, 0, 0x4140) << TAG;
      acc[r][3] = __byte_perm(v.y, 0, 0x4342) << TAG;
    } else {
      const uint4 v = *reinterpret_cast<const uint4*>(&stage[4 * l + r][8 * w]);
      acc[r][0] = v.x << TAG;
      acc[r][1] = v.y << TAG;
      acc[r][2] = v.z << TAG;
      acc[r][3] = v.w << TAG;
    }
  }
  // column KC (its low 3 bits KL static) of the owner warp into buffer BUF
#define CU8_PUBCOL(OWN, KL, BUF)                                                                 \
  do {                                                                                           \
    if (OWN) {                                                                                   \
      const int pp_ = ((KL) & 7) >> 1;                                                       \
      const uint32_t sel_ = ((KL) & 1) ? 0x3232u : 0x1010u; /* replicate the half */        \
      *reinterpret_cast<uint4*>(&sm.colk[BUF][4 * l]) =                                          \
          make_uint4(__byte_perm(acc[0][pp_], 0, sel_) & STRIP2,                                 \
                     __byte_perm(acc[1][pp_], 0, sel_) & STRIP2,                                 \
                     __byte_perm(acc[2][pp_], 0, sel_) & STRIP2,                                 \
                     __byte_perm(acc[3][pp_], 0, sel_) & STRIP2);                                \
    }                                                                                            \
  } while (0)
  // tag window decode after step k: the last improving k per cell into kst
  auto decode = [&](int k) {
    const uint32_t wbase = uint32_t(k & ~(WIN - 1));
#pragma unroll
    for (int r = 0; r < 4; r++) {
#pragma unroll
      for (int p = 0; p < 4; p++) {
        const uint32_t tg = acc[r][p] & TMASK2;
        acc[r][p] ^= tg;
        const uint32_t tlo = tg & 0xFF, thi = tg >> 16;
        const int sh0 = 8 * (2 * (p & 1)), sh1 = sh0 + 8;
        uint32_t& ks = kst[r][p >> 1];
        if (tlo) ks = (ks & ~(0xFFu << sh0)) | ((wbase + tlo) << sh0);
        if (thi) ks = (ks & ~(0xFFu << sh1)) | ((wbase + thi) << sh1);
      }
    }
  };
  uint32_t tag2 = 0x00010001u;   // tag of step k: 1 + (k mod WIN) in both halves
  if (prof && threadIdx.x == 0) tp[1] = close_gtimer();
  if constexpr (FULL) {
    // Two steps per CTA barrier. Columns k and k + 1 (k even) form one key pair of one warp, so
    // the owner publishes the pair (after step k - 1) with a single 16-byte store per lane. Every
    // warp then advances column k + 1 through step k itself:
    //   D[i][k+1] <- min(D[i][k+1], D[i][k] + D[k][k+1])
    // (one packed add+min per row, with D[k][k+1] read from the published pair at row k) and
    // runs steps k and k + 1 back to back. Row k + 1 comes from the warp's own lanes after its
    // step k, as before. Only operands are computed redundantly; each cell is still updated by
    // its owner, so values, tags and k* are those of the one-step loop.
    // the pair goes out as two replicated, tag-free columns: colk[BUF] = column k,
    // colk1[BUF] = column k + 1 (both halves of every key equal)
#define CU8_PUBPAIR(OWN, KL, BUF)                                                                \
  do {                                                                                           \
    if (OWN) {                                                                                   \
      const int pp_ = ((KL) & 7) >> 1;                                                           \
      *reinterpret_cast<uint4*>(&sm.colk[BUF][4 * l]) = make_uint4(                              \
          __byte_perm(acc[0][pp_], 0, 0x1010) & STRIP2, __byte_perm(acc[1][pp_], 0, 0x1010) & STRIP2, \
          __byte_perm(acc[2][pp_], 0, 0x1010) & STRIP2, __byte_perm(acc[3][pp_], 0, 0x1010) & STRIP2); \
      *reinterpret_cast<uint4*>(&sm.colk1[BUF][4 * l]) = make_uint4(                             \
          __byte_perm(acc[0][pp_], 0, 0x3232) & STRIP2, __byte_perm(acc[1][pp_], 0, 0x3232) & STRIP2, \
          __byte_perm(acc[2][pp_], 0, 0x3232) & STRIP2, __byte_perm(acc[3][pp_], 0, 0x3232) & STRIP2); \
    }                                                                                            \
  } while (0)
    CU8_PUBPAIR(w == 0, 0, 0);
    for (int k0 = 0; k0 < MAXB; k0 += 8) {
      const bool own = w == (k0 >> 3), own_next = w == (k0 >> 3) + 1;
      const bool win_end = ((k0 >> 3) & (WIN / 8 - 1)) == WIN / 8 - 1;   // step k0 + 7 closes a window
#pragma unroll
      for (int kk = 0; kk < 8; kk += 2) {
        const int k = k0 + kk;
        const int buf = (kk >> 1) & 1;
        APSP_JITTER_POINT(k);
        __syncthreads();
        const uint4 c4 = *reinterpret_cast<const uint4*>(&sm.colk[buf][4 * l]);
        const uint4 c5 = *reinterpret_cast<const uint4*>(&sm.colk1[buf][4 * l]);
        const uint32_t dkk1 = sm.colk1[buf][k];   // D[k][k+1], replicated
        const uint32_t ck[4] = {c4.x, c4.y, c4.z, c4.w};
        uint32_t ck1[4] = {c5.x, c5.y, c5.z, c5.w};
#pragma unroll
        for (int r = 0; r < 4; r++) ck1[r] = __viaddmin_u16x2(ck[r], dkk1, ck1[r]);
        uint32_t dkj[4];
#pragma unroll
        for (int p = 0; p < 4; p++) dkj[p] = (__shfl_sync(0xffffffffu, acc[kk & 3][p], k >> 2) & STRIP2) | tag2;
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int p = 0; p < 4; p++) acc[r][p] = __viaddmin_u16x2(ck[r], dkj[p], acc[r][p]);
        tag2 += 0x00010001u;
#pragma unroll
        for (int p = 0; p < 4; p++)
          dkj[p] = (__shfl_sync(0xffffffffu, acc[(kk + 1) & 3][p], (k + 1) >> 2) & STRIP2) | tag2;
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int p = 0; p < 4; p++) acc[r][p] = __viaddmin_u16x2(ck1[r], dkj[p], acc[r][p]);
        const bool wend = kk == 6 && win_end;
        tag2 = wend ? 0x00010001u : tag2 + 0x00010001u;
        if (wend) decode(k + 1);
        if (k + 2 < MAXB) CU8_PUBPAIR(kk == 6 ? own_next : own, kk + 2, buf ^ 1);
      }
    }
#undef CU8_PUBPAIR
  } else {
  CU8_PUBCOL(w == 0, 0, 0);
  for (int k0 = 0; k0 < m; k0 += 8) {
    const bool own = w == (k0 >> 3), own_next = w == (k0 >> 3) + 1;
    const bool win_end = ((k0 >> 3) & (WIN / 8 - 1)) == WIN / 8 - 1;   // step k0 + 7 closes a window
#pragma unroll
    for (int kk = 0; kk < 8; kk++) {
      const int k = k0 + kk;
      if (FULL || k < m) {
        __syncthreads();
        const uint4 c4 = *reinterpret_cast<const uint4*>(&sm.colk[kk & 1][4 * l]);
        const uint32_t dik[4] = {c4.x, c4.y, c4.z, c4.w};
        uint32_t dkj[4];
#pragma unroll
        for (int p = 0; p < 4; p++) dkj[p] = (__shfl_sync(0xffffffffu, acc[kk & 3][p], k >> 2) & STRIP2) | tag2;
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int p = 0; p < 4; p++) acc[r][p] = __viaddmin_u16x2(dik[r], dkj[p], acc[r][p]);
        const bool wend = kk == 7 && win_end;
        tag2 = wend ? 0x00010001u : tag2 + 0x00010001u;
        if (wend || (!FULL && k + 1 == m)) decode(k);   // close this tag window
        if (k + 1 < m) CU8_PUBCOL(kk == 7 ? own_next : own, kk + 1, (kk + 1) & 1);
      }
    }
  }
  }
#undef CU8_PUBCOL
  // values back (through the staging area) and the 1-based k* bytes
  __syncthreads();   // every thread has read its cells and column k of the last step
  if (prof && threadIdx.x == 0) tp[2] = close_gtimer();
#pragma unroll
  for (int r = 0; r < 4; r++) {
    if constexpr (VB == 1) {
      const uint32_t v0 = __byte_perm(acc[r][0] >> TAG, acc[r][1] >> TAG, 0x6420);
      const uint32_t v1 = __byte_perm(acc[r][2] >> TAG, acc[r][3] >> TAG, 0x6420);
      *reinterpret_cast<uint2*>(&stage[4 * l + r][8 * w]) = make_uint2(v0, v1);
    } else {
      *reinterpret_cast<uint4*>(&stage[4 * l + r][8 * w]) =
          make_uint4(acc[r][0] >> TAG, acc[r][1] >> TAG, acc[r][2] >> TAG, acc[r][3] >> TAG);
    }
  }
  __syncthreads();
  if (vec) {
    for (int e = threadIdx.x; e < MAXB * MAXB / SEG; e += blockDim.x) {
      const int i = e / (MAXB / SEG), j = SEG * (e % (MAXB / SEG));
      *reinterpret_cast<uint4*>(D + (lo + i) * ld + lo + j) = *reinterpret_cast<const uint4*>(&stage[i][j]);
    }
  } else {
    for (int e = threadIdx.x; e < MAXB * MAXB; e += blockDim.x) {
      const int i = e >> 7, j = e & 127;
      if (i < m && j < m) D[(lo + i) * ld + lo + j] = stage[i][j];
    }
  }
  if (prof && threadIdx.x == 0) tp[3] = close_gtimer();
  if (!idx) return;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; r++)
    *reinterpret_cast<uint2*>(&sm.K[4 * l + r][8 * w]) = make_uint2(kst[r][0], kst[r][1]);
  __syncthreads();
  // pred / via resolution in a bank-conflict-free mapping: lanes over columns
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (mode == IDX_VIA) {
#pragma unroll
    for (int a = 0; a < 8; a++) {
      const int i = ty + 16 * a;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int j = tx + 32 * q;
        const uint32_t kk = sm.K[i][j];
        if (kk && i < m && j < m) idx[(lo + i) * ldi + lo + j] = int32_t(via_off + kk - 1);
      }
    }
    return;
  }
  if (pre) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {
#pragma unroll
    for (int a = 0; a < 8; a++) {
      const int i = ty + 16 * a;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int j = tx + 32 * q;
        sm.P[i][j] = (i < m && j < m) ? idx[(lo + i) * ldi + lo + j] : -1;
      }
    }
  }
  __syncthreads();
  for (int round = 0; round < 7; round++) {   // chains have length < 128 = 2^7
    int32_t np[8][4];
    uint8_t nk[8][4];
    bool live = false;
#pragma unroll
    for (int a = 0; a < 8; a++) {
      const int i = ty + 16 * a;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int j = tx + 32 * q;
        const uint8_t kk = sm.K[i][j];
        np[a][q] = sm.P[i][j];
        nk[a][q] = kk;
        if (kk) {
          np[a][q] = sm.P[kk - 1][j];
          nk[a][q] = sm.K[kk - 1][j];
          live |= nk[a][q] != 0;
        }
      }
    }
    // chains are usually a few hops long: stop as soon as none has a next hop left
    const bool more = __syncthreads_or(live);
#pragma unroll
    for (int a = 0; a < 8; a++) {
      const int i = ty + 16 * a;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const int j = tx + 32 * q;
        sm.P[i][j] = np[a][q];
        sm.K[i][j] = nk[a][q];
      }
    }
    __syncthreads();
    if (!more) break;
  }
  if (prof && threadIdx.x == 0) tp[4] = close_gtimer();
#pragma unroll
  for (int a = 0; a < 8; a++) {
    const int i = ty + 16 * a;
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int j = tx + 32 * q;
      if (i < m && j < m) idx[(lo + i) * ldi + lo + j] = sm.P[i][j];
    }
  }
  if (prof && threadIdx.x == 0) {   // load, k loop, values out, pred resolution, pred out
    const unsigned long long t5 = close_gtimer();
    atomicAdd(&g_close128_phase[0], tp[1] - tp[0]);
    atomicAdd(&g_close128_phase[1], tp[2] - tp[1]);
    atomicAdd(&g_close128_phase[2], tp[3] - tp[2]);
    atomicAdd(&g_close128_phase[3], tp[4] - tp[3]);
    atomicAdd(&g_close128_phase[4], t5 - tp[4]);
    atomicAdd(&g_close128_phase[5], 1ull);
  }
}

template <int S, bool FULL>
__global__ void __launch_bounds__(512) block_close_dpx_kernel(typename CloseKeys<S>::T* D, int64_t ld, int64_t lo,
                                                              int m, int32_t* idx, int64_t ldi, int mode,
                                                              int64_t via_off, int prof, const int* wait_count,
                                                              int wait_target, uint32_t* nxA, uint16_t* nxB,
                                                              int32_t* nxPred, int64_t nxPredLd) {
  extern __shared__ __align__(16) unsigned char smraw_cu8[];
  if (wait_count) {   // started ahead of its producer (fw_sched.cu): wait for the 3a count
    if (threadIdx.x == 0) {
      int v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(wait_count) : "memory");
        if (v >= wait_target) break;
        __nanosleep(64);
      }
    }
    __syncthreads();
  }
  close_dpx_body<S, FULL>(D, ld, lo, m, idx, ldi, mode, via_off, smraw_cu8, prof != 0);
  if constexpr (FULL) {
    if (nxA) {   // the closed block's layouts and pred rows for the next phase-2 launch (tiles.cuh)
      using T = typename CloseKeys<S>::T;
      __syncthreads();   // this CTA's value and pred stores are visible to all its threads
      const T* Dg = D + lo * ld + lo;
      auto get = [&](int r, int c0, T (&v)[16]) { load16_global(Dg + int64_t(r) * ld + c0, v); };
      constexpr int NCH = MAXB / SUB;
      const int64_t t0 = lo / MAXB;   // the diagonal tile's index in the panels
      emit_layout_a<T, NtFormat<S>::TAG, NCH, 512>(get, nxA + t0 * NCH * (SUB * MAXB));
      emit_layout_b<T, NtFormat<S>::TAG, NtFormat<S>::WIN, NCH, 512>(get, nxB + t0 * NCH * (SUB * MAXB));
      if (nxPred && idx) {
        CloseU8Smem& sm = *reinterpret_cast<CloseU8Smem*>(smraw_cu8);
        for (int e = threadIdx.x; e < MAXB * MAXB; e += blockDim.x) {
          const int i = e >> 7, j = e & 127;
          nxPred[int64_t(i) * nxPredLd + lo + j] = sm.P[i][j];
        }
      }
    }
  }
}

static bool close_prof_on() {
  static const bool on = getenv("APSP_CLOSE_PROF") != nullptr;
  return on;
}

// APSP_CLOSE_PROF=1: every 32nd u8 closure launch prints the mean phase split (syncs the device;
// diagnostics only)
static void close_prof_report() {
  static std::atomic<long long> calls{0};
  if (++calls % 32) return;
  unsigned long long ph[6] = {};
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpyFromSymbol(ph, g_close128_phase, sizeof(ph)) != cudaSuccess || !ph[5])
    return;
  fprintf(stderr, "[close128] mean ns over %llu: load %llu, k loop %llu, values out %llu, pred resolve %llu, pred out %llu\n",
          ph[5], ph[0] / ph[5], ph[1] / ph[5], ph[2] / ph[5], ph[3] / ph[5], ph[4] / ph[5]);
}

template <int S>
static int close_impl(void* D, int64_t ld, int64_t lo, int64_t m, int32_t* idx, int64_t ldi, int mode,
                      int64_t via_off, Status* st, cudaStream_t s) {
  block_close_kernel<S><<<1, 512, 0, s>>>(static_cast<typename StoreT<S>::T*>(D), ld, lo, int(m), idx, ldi, mode,
                                           via_off, st);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

int launch_block_close(int store, void* D, int64_t ld, int64_t lo, int64_t m, int32_t* idx, int64_t ldi, int mode,
                       int64_t via_off, Status* st, cudaStream_t s, const int* wait_count, int wait_target,
                       uint32_t* nxA, uint16_t* nxB, int32_t* nxPred, int64_t nxPredLd) {
  if (m <= 0) return 0;
  if ((wait_count || nxA) && !((store == STORE_U8 || store == STORE_U16) && m == MAXB && lo % MAXB == 0))
    return set_error(APSP_EINVAL, "device-signalled closure start needs a full u8 / u16 block");
  if (m > MAXB) {
    // classic order over a larger block: per-k steps on the sub-view
    for (int64_t k = 0; k < m; k++) {
      int rc = launch_fw_step(store, static_cast<char*>(D) + (lo * ld + lo) * store_elem_size(store), ld, m, k,
                              idx ? idx + lo * ldi + lo : nullptr, ldi, mode, via_off, st, s);
      if (rc) return rc;
    }
    return 0;
  }
  // pred mode on the 32-bit exact stores: the blocked in-CTA closure (close_blk.cu; distances
  // exact, pred a valid tree); via mode keeps the classic order (R-Kleene via is bit-exact)
  static const bool classic_close = getenv("APSP_CLASSIC_CLOSE") != nullptr;
  if (mode == IDX_PRED && close_blk_supported(store) && !classic_close)
    return launch_block_close_blk(store, D, ld, lo, m, idx, ldi, s);
  if ((wait_count || nxA) && getenv("APSP_SLOW_CLOSE"))
    return set_error(APSP_EINVAL, "device-signalled closure start needs the packed closure kernel");
  if ((store == STORE_U8 || store == STORE_U16) && !getenv("APSP_SLOW_CLOSE")) {
    static std::atomic<unsigned long long> attr8{0}, attr16{0};
    static std::atomic<unsigned long long> attr8f{0}, attr16f{0};
    const size_t sb = sizeof(CloseU8Smem);
    if (store == STORE_U8 && m == MAXB) {
      APSP_CUDA_TRY(smem_optin(block_close_dpx_kernel<STORE_U8, true>, int(sb), attr8f));
      block_close_dpx_kernel<STORE_U8, true><<<1, 512, sb, s>>>(static_cast<uint8_t*>(D), ld, lo, int(m), idx, ldi,
                                                                mode, via_off, int(close_prof_on()), wait_count,
                                                                wait_target, nxA, nxB, nxPred, nxPredLd);
      if (close_prof_on()) close_prof_report();
    } else if (store == STORE_U8) {
      APSP_CUDA_TRY(smem_optin(block_close_dpx_kernel<STORE_U8, false>, int(sb), attr8));
      block_close_dpx_kernel<STORE_U8, false><<<1, 512, sb, s>>>(static_cast<uint8_t*>(D), ld, lo, int(m), idx, ldi,
                                                                 mode, via_off, 0, nullptr, 0, nullptr, nullptr, nullptr, 0);
    } else if (m == MAXB) {
      APSP_CUDA_TRY(smem_optin(block_close_dpx_kernel<STORE_U16, true>, int(sb), attr16f));
      block_close_dpx_kernel<STORE_U16, true><<<1, 512, sb, s>>>(static_cast<uint16_t*>(D), ld, lo, int(m), idx,
                                                                 ldi, mode, via_off, 0, wait_count, wait_target, nxA, nxB,
                                                                 nxPred, nxPredLd);
    } else {
      APSP_CUDA_TRY(smem_optin(block_close_dpx_kernel<STORE_U16, false>, int(sb), attr16));
      block_close_dpx_kernel<STORE_U16, false><<<1, 512, sb, s>>>(static_cast<uint16_t*>(D), ld, lo, int(m), idx,
                                                                  ldi, mode, via_off, 0, nullptr, 0, nullptr, nullptr, nullptr, 0);
    }
    APSP_CUDA_TRY(cudaGetLastError());
    count_launches(1);
    return 0;
  }
  switch (store) {
    case STORE_U8: return close_impl<STORE_U8>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
    case STORE_W32: return close_impl<STORE_W32>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
    case STORE_I32: return close_impl<STORE_I32>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
    case STORE_F32: return close_impl<STORE_F32>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
    case STORE_I64: return close_impl<STORE_I64>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
    case STORE_U16: return close_impl<STORE_U16>(D, ld, lo, m, idx, ldi, mode, via_off, st, s);
  }
  return set_error(2, "unknown store %d", store);
}

#include "fw_persist.cuh"

}  // namespace apsp
