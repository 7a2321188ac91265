// Blocked closure of an m <= 128 diagonal block for the 32-bit exact stores (f32, w32, i32):
// FW phase 1 (pred mode) and the aligned R-Kleene pred leaves.
//
// The classic in-block loop (block_close_kernel, fw.cu) runs 128 dependent steps that each
// touch all 128 x 128 cells with a compare-select -- 115 us per f32 block, one SM. Here the
// block is closed as a blocked FW of 32-wide sub-blocks inside one CTA:
//   sub-round K:  (a) 4 warps close the 32 x 32 diagonal sub-block (32 steps, a named barrier
//                     per step, column k by shuffle, row k through shared memory);
//                 (b) all warps update the row and column panels against it;
//                 (c) all warps update the remaining cells with the new panels.
// (b) and (c) are min-plus products with FADD + FMNMX3 (values only, no per-update argmin).
// Each cell records only the last sub-round that strictly improved it. Afterwards a witness w
// of that sub-round with fl(d[i][w] + d[w][j]) == d[i][j] is searched (the last improving k is
// one: its operands were >= their final values and rounding is monotone), and
// pred[i][j] = pred[w][j] is resolved by pointer jumping (with positive costs d[w][j] <
// d[i][j], so the chains end). Distances equal the classic order exactly (exact closure);
// pred is a valid shortest-path tree, not necessarily the classic one -- FW phase 1 only needs
// that (the bit-exact classic pred is fw_classic(method="classic")); zero-cost edges never
// reach this kernel (fw_sched routes them to the classic order).
#include <cstdint>
#include <cstdlib>
#include "launch.h"
#include "tiles.cuh"

namespace apsp {

namespace {

constexpr int CB = 128;          // block
constexpr int SB = 32;           // sub-block
constexpr int CT = 512;          // threads

template <int S> struct BlkOps;
template <> struct BlkOps<STORE_F32> {
  using T = float;
  __device__ static T inf() { return __int_as_float(0x7f800000); }
  __device__ static T add(T a, T b) { return a + b; }
  __device__ static T min2(T a, T b) { return fminf(a, b); }
  __device__ static T min3(T a, T b, T c) { return fmin3(a, b, c); }
};
template <int S> struct BlkOpsI {
  using T = int32_t;
  __device__ static T inf() { return store_inf<S>(); }
  __device__ static T add(T a, T b) { return a + b; }   // INF + INF < 2^31 for both stores
  __device__ static T min2(T a, T b) { return min(a, b); }
  __device__ static T min3(T a, T b, T c) { return __vimin3_s32(a, b, c); }
};
template <> struct BlkOps<STORE_W32> : BlkOpsI<STORE_W32> {};
template <> struct BlkOps<STORE_I32> : BlkOpsI<STORE_I32> {};

template <typename T>
struct BlkSmem {
  T V[CB][CB];          // the block's values
  int32_t P[CB][CB];    // pred (input block, prefetched by cp.async), then resolved in place
  uint8_t K[CB][CB];    // 1 + last improving sub-round, then 1 + witness (0 = none)
  uint16_t Q[CB * CB];  // improved cells (witness search queue)
  int qn;
};

// other-index q (0..95) of sub-round K -> block index (skips [32K, 32K + 32))
__device__ __forceinline__ int other(int q, int K) { return q < SB * K ? q : q + SB; }

template <int S>
__global__ void __launch_bounds__(CT, 1) block_close_blk_kernel(typename StoreT<S>::T* D, int64_t ld, int64_t lo,
                                                                int m, int32_t* idx, int64_t ldi, int skip) {
  using O = BlkOps<S>;
  using T = typename O::T;
  extern __shared__ __align__(16) unsigned char smraw_blk[];
  BlkSmem<T>& sm = *reinterpret_cast<BlkSmem<T>*>(smraw_blk);
  const int t = threadIdx.x, l = t & 31, w = t >> 5;
  const T inf = O::inf();
  // input pred of the block: needed only at the end
  const bool pvec = idx && m == CB && ((reinterpret_cast<uintptr_t>(idx + lo * ldi + lo) | uintptr_t(ldi * 4)) & 15) == 0;
  if (pvec) {
    for (int e = t; e < CB * CB / 4; e += CT) {
      const int i = e >> 5, j = 4 * (e & 31);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.P[i][j])),
                   "l"(idx + (lo + i) * ldi + lo + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  } else if (idx) {
    for (int e = t; e < CB * CB; e += CT) {
      const int i = e >> 7, j = e & 127;
      sm.P[i][j] = (i < m && j < m) ? idx[(lo + i) * ldi + lo + j] : -1;
    }
  }
  if (m == CB && ((reinterpret_cast<uintptr_t>(D + lo * ld + lo) | uintptr_t(ld * 4)) & 15) == 0) {
    for (int e = t; e < CB * CB / 4; e += CT) {
      const int i = e >> 5, j = 4 * (e & 31);
      *reinterpret_cast<int4*>(&sm.V[i][j]) = *reinterpret_cast<const int4*>(D + (lo + i) * ld + lo + j);
    }
  } else {
    for (int e = t; e < CB * CB; e += CT) {
      const int i = e >> 7, j = e & 127;
      sm.V[i][j] = (i < m && j < m) ? D[(lo + i) * ld + lo + j] : (i == j ? T(0) : inf);
    }
  }
  for (int e = t; e < CB * CB / 16; e += CT) reinterpret_cast<uint4*>(&sm.K[0][0])[e] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const int nsub = (m + SB - 1) / SB;
  for (int K = 0; K < nsub; K++) {
    const int k0 = SB * K;
    const uint8_t tagK = uint8_t(K + 1);
    // (a) diagonal sub-block: warps 0..3, thread (w, l) owns column k0 + l, rows k0 + 8w + r
    if (w < 4 && !(skip & 2)) {
      T c[8], c0[8];
#pragma unroll
      for (int r = 0; r < 8; r++) c0[r] = c[r] = sm.V[k0 + 8 * w + r][k0 + l];
#pragma unroll
      for (int k = 0; k < SB; k++) {
        if (w == (k >> 3)) sm.V[k0 + k][k0 + l] = c[k & 7];   // publish row k (final for this step)
        APSP_JITTER_POINT(k0 + k);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const T rk = sm.V[k0 + k][k0 + l];
#pragma unroll
        for (int r = 0; r < 8; r++) c[r] = O::min2(c[r], O::add(__shfl_sync(0xffffffffu, c[r], k), rk));
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");   // every warp is done reading row 31
#pragma unroll
      for (int r = 0; r < 8; r++) {
        sm.V[k0 + 8 * w + r][k0 + l] = c[r];
        if (c[r] < c0[r]) sm.K[k0 + 8 * w + r][k0 + l] = tagK;
      }
    }
    __syncthreads();
    // (b) panels against the closed diagonal sub-block, computed into registers first (each
    // panel is also an operand of its own update):
    //   row panel:    rows k0 + 2w + {0,1}, other columns 3l + {0,1,2}
    //   column panel: other rows 6w + {0..5}, column k0 + l
    if (!(skip & 4)) {
      int rrow[2], rcol[3], crow[6];
#pragma unroll
      for (int a = 0; a < 2; a++) rrow[a] = k0 + 2 * w + a;
#pragma unroll
      for (int q = 0; q < 3; q++) rcol[q] = other(3 * l + q, K);
#pragma unroll
      for (int a = 0; a < 6; a++) crow[a] = other(6 * w + a, K);
      const int ccol = k0 + l;
      T ra[2][3], ca[6];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int q = 0; q < 3; q++) ra[a][q] = sm.V[rrow[a]][rcol[q]];
#pragma unroll
      for (int a = 0; a < 6; a++) ca[a] = sm.V[crow[a]][ccol];
      T ra0[2][3], ca0[6];
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int q = 0; q < 3; q++) ra0[a][q] = ra[a][q];
#pragma unroll
      for (int a = 0; a < 6; a++) ca0[a] = ca[a];
#pragma unroll 4
      for (int kr = 0; kr < SB; kr += 2) {
        T da[2][2], pb[2][3], pa[6][2], db[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
#pragma unroll
          for (int a = 0; a < 2; a++) da[a][h] = sm.V[rrow[a]][k0 + kr + h];      // Dg[row][kr]
#pragma unroll
          for (int q = 0; q < 3; q++) pb[h][q] = sm.V[k0 + kr + h][rcol[q]];      // row panel[kr][col]
#pragma unroll
          for (int a = 0; a < 6; a++) pa[a][h] = sm.V[crow[a]][k0 + kr + h];      // col panel[row][kr]
          db[h] = sm.V[k0 + kr + h][ccol];                                         // Dg[kr][col]
        }
#pragma unroll
        for (int a = 0; a < 2; a++)
#pragma unroll
          for (int q = 0; q < 3; q++)
            ra[a][q] = O::min3(ra[a][q], O::add(da[a][0], pb[0][q]), O::add(da[a][1], pb[1][q]));
#pragma unroll
        for (int a = 0; a < 6; a++) ca[a] = O::min3(ca[a], O::add(pa[a][0], db[0]), O::add(pa[a][1], db[1]));
      }
      APSP_JITTER_POINT(K + 500);
      __syncthreads();
#pragma unroll
      for (int a = 0; a < 2; a++)
#pragma unroll
        for (int q = 0; q < 3; q++)
          if (ra[a][q] < ra0[a][q]) {
            sm.V[rrow[a]][rcol[q]] = ra[a][q];
            sm.K[rrow[a]][rcol[q]] = tagK;
          }
#pragma unroll
      for (int a = 0; a < 6; a++)
        if (ca[a] < ca0[a]) {
          sm.V[crow[a]][ccol] = ca[a];
          sm.K[crow[a]][ccol] = tagK;
        }
    }
    __syncthreads();
    // (c) the rest: other rows 6w + {0..5} x other columns 3l + {0,1,2}, with the new panels
    if (!(skip & 8)) {
      int row[6], col[3];
#pragma unroll
      for (int a = 0; a < 6; a++) row[a] = other(6 * w + a, K);
#pragma unroll
      for (int q = 0; q < 3; q++) col[q] = other(3 * l + q, K);
      T acc[6][3], acc0[6][3];
#pragma unroll
      for (int a = 0; a < 6; a++)
#pragma unroll
        for (int q = 0; q < 3; q++) acc0[a][q] = acc[a][q] = sm.V[row[a]][col[q]];
#pragma unroll 4
      for (int kr = 0; kr < SB; kr += 2) {
        T pa[6][2], pb[2][3];
#pragma unroll
        for (int h = 0; h < 2; h++) {
#pragma unroll
          for (int a = 0; a < 6; a++) pa[a][h] = sm.V[row[a]][k0 + kr + h];
#pragma unroll
          for (int q = 0; q < 3; q++) pb[h][q] = sm.V[k0 + kr + h][col[q]];
        }
#pragma unroll
        for (int a = 0; a < 6; a++)
#pragma unroll
          for (int q = 0; q < 3; q++)
            acc[a][q] = O::min3(acc[a][q], O::add(pa[a][0], pb[0][q]), O::add(pa[a][1], pb[1][q]));
      }
      // no barrier needed before the stores: this step reads only panel cells and writes only
      // rest cells
#pragma unroll
      for (int a = 0; a < 6; a++)
#pragma unroll
        for (int q = 0; q < 3; q++)
          if (acc[a][q] < acc0[a][q]) {
            sm.V[row[a]][col[q]] = acc[a][q];
            sm.K[row[a]][col[q]] = tagK;
          }
    }
    __syncthreads();
  }
  if (idx && !(skip & 1)) {
    // witness of the last improving sub-round: the first w in it with d[i][w] + d[w][j] == d[i][j].
    // The improved cells are compacted into a queue first (warp-aggregated appends), then each
    // lane scans its cell's 32 candidates branch-free (independent loads, one select per w), so
    // the cost is the number of improved cells, without divergence.
    uint16_t* q = sm.Q;
    if (t == 0) sm.qn = 0;
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < CB * CB / CT; c++) {
      const int e = t + CT * c;
      const bool imp = sm.K[e >> 7][e & 127] != 0;
      const uint32_t bal = __ballot_sync(0xffffffffu, imp);
      if (!bal) continue;
      int base = 0;
      if (l == 0) base = atomicAdd(&sm.qn, __popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (imp) q[base + __popc(bal & ((1u << l) - 1u))] = uint16_t(e);
    }
    __syncthreads();
    const int qn = sm.qn;
    for (int it = t; it < qn; it += CT) {
      const int e = q[it], i = e >> 7, j = e & 127;
      const int w0 = SB * (sm.K[i][j] - 1);
      const int xi = i - w0, xj = j - w0;   // excluded candidates (outside [0, 32) if not in range)
      const T dij = sm.V[i][j];
      int found = 0;
#pragma unroll
      for (int x = SB - 1; x >= 0; x--) {
        const bool ok = O::add(sm.V[i][w0 + x], sm.V[w0 + x][j]) == dij;
        found = (ok && x != xi && x != xj) ? x + 1 : found;
      }
      sm.K[i][j] = uint8_t(found ? w0 + found : 0);   // 0 only if no witness exists (cannot happen)
    }
    if (pvec) asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // pointer jumping: pred[i][j] <- pred[w][j] until no cell has a pending witness
    for (int it = 0; it < 8; it++) {
      int32_t np[32];
      uint32_t nk[8];   // 4 pending witnesses per register
      bool live = false;
#pragma unroll
      for (int c = 0; c < 32; c++) {
        const int e = t + CT * c, i = e >> 7, j = e & 127;
        uint32_t kk = sm.K[i][j];
        np[c] = sm.P[i][j];
        if (kk) {
          np[c] = sm.P[kk - 1][j];
          kk = sm.K[kk - 1][j];
          live |= kk != 0;
        }
        if ((c & 3) == 0) nk[c >> 2] = 0;
        nk[c >> 2] |= kk << (8 * (c & 3));
      }
      const bool more = __syncthreads_or(live);
#pragma unroll
      for (int c = 0; c < 32; c++) {
        const int e = t + CT * c, i = e >> 7, j = e & 127;
        sm.P[i][j] = np[c];
        sm.K[i][j] = uint8_t(nk[c >> 2] >> (8 * (c & 3)));
      }
      __syncthreads();
      if (!more) break;
    }
  }
  if (m == CB && ((reinterpret_cast<uintptr_t>(D + lo * ld + lo) | uintptr_t(ld * 4)) & 15) == 0 && (!idx || pvec)) {
    for (int e = t; e < CB * CB / 4; e += CT) {
      const int i = e >> 5, j = 4 * (e & 31);
      *reinterpret_cast<int4*>(D + (lo + i) * ld + lo + j) = *reinterpret_cast<const int4*>(&sm.V[i][j]);
      if (idx) *reinterpret_cast<int4*>(idx + (lo + i) * ldi + lo + j) = *reinterpret_cast<const int4*>(&sm.P[i][j]);
    }
  } else {
    for (int e = t; e < CB * CB; e += CT) {
      const int i = e >> 7, j = e & 127;
      if (i < m && j < m) {
        D[(lo + i) * ld + lo + j] = sm.V[i][j];
        if (idx) idx[(lo + i) * ldi + lo + j] = sm.P[i][j];
      }
    }
  }
}

}  // namespace

bool close_blk_supported(int store) { return store == STORE_F32 || store == STORE_W32 || store == STORE_I32; }

int launch_block_close_blk(int store, void* D, int64_t ld, int64_t lo, int64_t m, int32_t* idx, int64_t ldi,
                           cudaStream_t s) {
  if (m <= 0) return 0;
  if (m > CB) return set_error(2, "blocked closure takes m <= %d", CB);
  const int sb = int(sizeof(BlkSmem<float>));
  // A/B timing only (results wrong): APSP_BLK_SKIP bits 1 witness, 2 diagonal, 4 panels, 8 rest
  static const int skip = getenv("APSP_BLK_SKIP") ? atoi(getenv("APSP_BLK_SKIP")) : 0;
  static std::atomic<unsigned long long> a0{0}, a1{0}, a2{0};
  switch (store) {
    case STORE_F32:
      APSP_CUDA_TRY(smem_optin(block_close_blk_kernel<STORE_F32>, sb, a0));
      block_close_blk_kernel<STORE_F32><<<1, CT, sb, s>>>(static_cast<float*>(D), ld, lo, int(m), idx, ldi, skip);
      break;
    case STORE_W32:
      APSP_CUDA_TRY(smem_optin(block_close_blk_kernel<STORE_W32>, sb, a1));
      block_close_blk_kernel<STORE_W32><<<1, CT, sb, s>>>(static_cast<int32_t*>(D), ld, lo, int(m), idx, ldi, skip);
      break;
    case STORE_I32:
      APSP_CUDA_TRY(smem_optin(block_close_blk_kernel<STORE_I32>, sb, a2));
      block_close_blk_kernel<STORE_I32><<<1, CT, sb, s>>>(static_cast<int32_t*>(D), ld, lo, int(m), idx, ldi, skip);
      break;
    default:
      return set_error(2, "blocked closure: store %d unsupported", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

}  // namespace apsp
