// Shared device helpers of the min-plus tile kernels (minplus.cu: register-staged and exact
// kernels plus the dispatch; minplus_bulk.cu: the bulk-staged kernels and their panel layouts).
#pragma once
#include <cstdint>
#include "launch.h"

namespace apsp {

constexpr int BM = 128, BN = 128, NT = 256;
#ifndef APSP_U8_UNROLL
#define APSP_U8_UNROLL 32
#endif
constexpr int kU8Unroll = APSP_U8_UNROLL;
#ifndef APSP_ROW_DECODE
#define APSP_ROW_DECODE 1
#endif

// Tile origin of this CTA.  Full grid: (blockIdx.y, blockIdx.x).  Cross-list mode
// (only_lo < only_hi): blockIdx.x enumerates the tiles of rows band + cols band [lo, hi)
// (band width w tiles): first the w full tile rows, then the remaining rows of the w columns.
__device__ __forceinline__ void tile_origin(const MinplusArgs& p, int bm, int bn, int64_t& i0, int64_t& j0) {
  if (p.only_lo < p.only_hi) {   // tile counts fit 32 bits: 32-bit division (a 64-bit one is ~100 instr)
    const int wr = int((p.only_hi - p.only_lo) / bm), lo_r = int(p.only_lo / bm);   // row band, in row tiles
    const int wc = int((p.only_hi - p.only_lo) / bn), lo_c = int(p.only_lo / bn);   // col band, in col tiles
    const int nt_c = int((p.n + bn - 1) / bn);
    const int id = int(blockIdx.x) >> (p.split_rows ? 1 : 0);   // half-row CTAs: two per tile
    if (id < wr * nt_c) {
      i0 = int64_t(lo_r + id / nt_c) * bm;
      j0 = int64_t(id % nt_c) * bn;
    } else {
      const int id2 = id - wr * nt_c, rr = id2 / wc, cc = id2 % wc;
      i0 = int64_t(rr < lo_r ? rr : rr + wr) * bm;
      j0 = int64_t(lo_c + cc) * bn;
    }
  } else if (p.first_lo < p.first_hi) {   // 1D: the cross of [first_lo, first_hi) first, then the rest
    const int wr = int((p.first_hi - p.first_lo) / bm), lo_r = int(p.first_lo / bm);
    const int wc = int((p.first_hi - p.first_lo) / bn), lo_c = int(p.first_lo / bn);
    const int nt_r = int((p.m + bm - 1) / bm), nt_c = int((p.n + bn - 1) / bn);
    const int id = (int(blockIdx.x) >> (p.split_rows ? 1 : 0)) + p.id_begin, ncross = wr * nt_c + (nt_r - wr) * wc;
    if (id < ncross) {
      if (id < wr * nt_c) {
        i0 = int64_t(lo_r + id / nt_c) * bm;
        j0 = int64_t(id % nt_c) * bn;
      } else {
        const int id2 = id - wr * nt_c, rr = id2 / wc, cc = id2 % wc;
        i0 = int64_t(rr < lo_r ? rr : rr + wr) * bm;
        j0 = int64_t(lo_c + cc) * bn;
      }
    } else {
      const int id3 = id - ncross, rr = id3 / (nt_c - wc), cc = id3 % (nt_c - wc);
      i0 = int64_t(rr < lo_r ? rr : rr + wr) * bm;
      j0 = int64_t(cc < lo_c ? cc : cc + wc) * bn;
    }
  } else if (p.raster > 1) {
    // Grouped rasterisation: CTAs launch in linear blockIdx order, so consecutive CTAs take the
    // tiles of `raster` row tiles column by column -- the row panels of the group stay hot in L2
    // while each column panel is read once per group instead of once per row tile.
    const int nt_c = int(gridDim.x), nt_r = int(gridDim.y), g = p.raster;
    const int id = int(blockIdx.y) * nt_c + int(blockIdx.x);
    const int grp = id / (g * nt_c), r0 = grp * g, gs = min(nt_r - r0, g), in = id - grp * g * nt_c;
    i0 = int64_t(r0 + in % gs) * bm;
    j0 = int64_t(in / gs) * bn;
  } else {
    i0 = int64_t(blockIdx.y) * bm;
    j0 = int64_t(blockIdx.x) * bn;
  }
}

__device__ __forceinline__ bool tile_skipped(const MinplusArgs& p, int64_t i0, int64_t j0, int bm, int bn) {
  const bool rin = i0 >= p.skip_row_lo && i0 + bm <= p.skip_row_hi;
  const bool cin = j0 >= p.skip_col_lo && j0 + bn <= p.skip_col_hi;
  const bool r2 = i0 >= p.skip2_lo && i0 + bm <= p.skip2_hi;
  const bool c2 = j0 >= p.skip2_lo && j0 + bn <= p.skip2_hi;
  const bool r3 = i0 >= p.skip3_lo && i0 + bm <= p.skip3_hi;
  const bool c3 = j0 >= p.skip3_lo && j0 + bn <= p.skip3_hi;
  return rin || cin || r2 || c2 || r3 || c3;
}

// key format of the bulk-staged narrow tiles (minplus_bulk.cu Narrow<S>): key = v << TAG | tag,
// tags 1..32*WIN per decode window
template <int S> struct NtFormat;
template <> struct NtFormat<STORE_U8> { static constexpr int TAG = 7, WIN = 3; };
template <> struct NtFormat<STORE_U16> { static constexpr int TAG = 6, WIN = 1; };

// ---- next-round operand layouts written by their producers (FW b = 128, u8 / u16) ----------
// The phase-2 cross launch of round K+1 reads the column and row panels of pivot K+1 in the
// prep_pair_kernel formats. All of them but the diagonal block are final when 3a(K) writes
// them, the diagonal when the closure does; so the producers lay them out directly and the
// separate prep launch (which waited for SM slots behind 3b) goes away. get(r, c) returns the
// tile value at row r, column c (0..127); the layouts are those of prep_nt_a_body /
// prep_nt_b_body: A = replicated key pairs [chunk][k][row], B = tagged keys [chunk][k][col].
// load16(r, c0, v) fills v[0..15] with the tile row r, columns c0..c0+15 (c0 % 16 == 0).
// NCH chunks of 32 k; every thread first loads all its segments (global sources: the loads
// overlap instead of one L2 round trip per segment), then stores them
// ROWS = 128 (whole tile) or 64 (rows [row_lo, row_lo + 64) of it: a half-tile CTA). For B the
// tile rows are the k index, so a half covers chunks [row_lo / 32, row_lo / 32 + NCH / 2).
template <typename T, int TAG, int NCH, int NTHR, int ROWS = 128, typename L>
__device__ __forceinline__ void emit_layout_a(L&& load16, uint32_t* Atile, int row_lo = 0) {
  constexpr int PER = NCH * 2 * ROWS / NTHR;   // items: chunk x row x 16-k half
  T v[PER][16];
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int e = threadIdx.x + u * NTHR, c = e / (2 * ROWS), tt = e % (2 * ROWS);
    const int r = row_lo + tt % ROWS, kb = 16 * (tt / ROWS);
    load16(r, c * SUB + kb, v[u]);
  }
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int e = threadIdx.x + u * NTHR, c = e / (2 * ROWS), tt = e % (2 * ROWS);
    const int r = row_lo + tt % ROWS, kb = 16 * (tt / ROWS);
    uint32_t* dst = Atile + int64_t(c) * (SUB * 128);
#pragma unroll
    for (int q = 0; q < 16; q++) dst[(kb + q) * 128 + r] = (uint32_t(v[u][q]) << TAG) * 0x00010001u;
  }
}
template <typename T, int TAG, int WIN, int NCH, int NTHR, int ROWS = 128, typename L>
__device__ __forceinline__ void emit_layout_b(L&& load16, uint16_t* Btile, int row_lo = 0) {
  constexpr int PER = NCH * 256 * ROWS / 128 / NTHR;
  const int c0 = row_lo / SUB;
  T v[PER][16];
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int e = threadIdx.x + u * NTHR, c = c0 + (e >> 8), tt = e & 255, kk = tt >> 3, cb = 16 * (tt & 7);
    load16(c * SUB + kk, cb, v[u]);
  }
#pragma unroll
  for (int u = 0; u < PER; u++) {
    const int e = threadIdx.x + u * NTHR, c = c0 + (e >> 8), tt = e & 255, kk = tt >> 3, cb = 16 * (tt & 7);
    const uint32_t tag = uint32_t(SUB * (c % WIN) + kk + 1);
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 8; q++)
      o[q] = ((uint32_t(v[u][2 * q]) << TAG) | tag) | (((uint32_t(v[u][2 * q + 1]) << TAG) | tag) << 16);
    uint4* dst = reinterpret_cast<uint4*>(Btile + int64_t(c) * (SUB * 128) + kk * 128 + cb);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
}
// 16 values of a row-major tile in global memory (16-byte aligned rows), for load16
template <typename T>
__device__ __forceinline__ void load16_global(const T* row, T (&v)[16]) {
  const uint4* src = reinterpret_cast<const uint4*>(row);
  reinterpret_cast<uint4*>(v)[0] = src[0];
  if constexpr (sizeof(T) == 2) reinterpret_cast<uint4*>(v)[1] = src[1];
}

__device__ __forceinline__ void emit_idx(const MinplusArgs& p, int64_t i, int64_t j, uint32_t kk) {
  if (p.idx == nullptr) return;
  int32_t v = (p.mode == IDX_PRED) ? __ldg(p.predB + int64_t(kk) * p.ldp + j) : int32_t(p.inner_off + kk);
  p.idx[i * p.ldi + j] = v;
}

// u8 tier keys: 16-bit UNSIGNED, key = value << 7 | tag, tag = 1..64 over a 64-k decode window
// (two 32-k chunks).  INF key = 255 << 7 = 32640; the largest sum INF + INF + tag = 65407 < 2^16.
constexpr int U8_TAG = 7;
constexpr uint32_t U8_KINF = uint32_t(U8_INF) << U8_TAG;
constexpr uint32_t U8_TAGMASK2 = 0x007F007Fu;

__device__ __forceinline__ uint32_t viaddmin_u16x2(uint32_t a, uint32_t b, uint32_t c) {
  return __viaddmin_u16x2(a, b, c);
}

// 0xFFFF in each 16-bit half whose bit 15 is set, else 0 (PTX prmt sign replication; the
// CUDA __byte_perm intrinsic masks selectors to 3 bits and cannot express it).
__device__ __forceinline__ uint32_t prmt_sign_halves(uint32_t x) {
  uint32_t d;
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(d) : "r"(x));
  return d;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps until the phase completes instead
// of re-issuing the probe (a spinning producer warp steals issue slots from the ALU-bound
// consumers on its SM sub-partition)
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

inline dim3 grid_for(const MinplusArgs& a, int bm, int bn) {
  if (a.only_lo < a.only_hi) {   // the cross of rows and columns [lo, hi) (tile_origin's enumeration)
    const int64_t wr = (a.only_hi - a.only_lo) / bm, wc = (a.only_hi - a.only_lo) / bn;
    const int64_t nt_r = (a.m + bm - 1) / bm, nt_c = (a.n + bn - 1) / bn;
    return dim3(unsigned((wr * nt_c + (nt_r - wr) * wc) << (a.split_rows ? 1 : 0)), 1);
  }
  if (a.first_lo < a.first_hi) {
    const int64_t total = ((a.n + bn - 1) / bn) * ((a.m + bm - 1) / bm);
    const int64_t cnt = a.id_count > 0 ? a.id_count : total - a.id_begin;
    return dim3(unsigned(cnt << (a.split_rows ? 1 : 0)), 1);
  }
  return dim3(unsigned((a.n + bn - 1) / bn), unsigned((a.m + bm - 1) / bm));
}

// Race stress (the debug build libapsp_b200_jitter.so, -DAPSP_JITTER; tools/race_stress.py):
// at the synchronisation points of the barrier-free rings and the closures a pseudo-random
// eighth of the warps sleep up to ~4 us, so every ordering the code relies on gets exercised
// with warps far apart. compute-sanitizer is not available on the GPU pool; this plus the
// oracle comparison is the race evidence. Compiles to nothing in the product build.
#ifdef APSP_JITTER
__device__ __forceinline__ void jitter_point(uint32_t salt) {
  uint32_t h = (blockIdx.x * 73856093u) ^ (blockIdx.y * 19349663u) ^ ((threadIdx.x >> 5) * 83492791u) ^
               (salt * 2654435761u) ^ uint32_t(clock());
  h ^= h >> 13;
  h *= 0x5bd1e995u;
  h ^= h >> 15;
  if ((h & 7u) == 0u) __nanosleep(h & 4095u);
}
#define APSP_JITTER_POINT(salt) ::apsp::jitter_point(salt)
#else
#define APSP_JITTER_POINT(salt) ((void)0)
#endif

// 3-input fp32 min (FMNMX3 on sm_100)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// packed fp32x2 add (FADD2 on sm_100; a scalar operand packed as {x, x} folds into the
// instruction's .F32 broadcast form): two correctly rounded sums per instruction
__device__ __forceinline__ unsigned long long pack_f2(float x, float y) {
  unsigned long long d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(x), "f"(y));
  return d;
}
__device__ __forceinline__ float2 fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}

// bulk-staged launchers (minplus_bulk.cu)
template <int S> int launch_nt(const MinplusArgs& a, cudaStream_t s);
int launch_w32nt(const MinplusArgs& a, cudaStream_t s);
int launch_f32nt(const MinplusArgs& a, cudaStream_t s);
int launch_f32dm(const MinplusArgs& a, cudaStream_t s);
bool f32_deferred();

}  // namespace apsp
