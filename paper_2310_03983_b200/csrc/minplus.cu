// Min-plus tile kernels:  C <- min(C, A (x) B)  with argmin -> idx on strict improvement.
//
// This is the bulk of the work for both solvers: FW phases 2-3 and every block product of the
// R-Kleene recursion.  Keyed tiers carry the argmin inside the value: key(x) = x << tag_bits,
// the right operand carries tag = 1 + (k mod window); the min over keys is the lexicographic
// (value, smallest k) min and an untagged (old) key wins ties, so a tag survives only on
// strict improvement (minplus.py:80-82,128-133).  Tags are decoded into a 16-bit k index per
// cell once per window and cleared.
//
//  * minplus_bulk.cu: the bulk-staged kernels on pre-laid-out panels (u8/u16 VIADDMNMX.U16x2,
//    w32 VIADDMNMX.U32, exact fp32 deferred-argmin and compare-select) and the panel layouts.
//  * here: register-staged kernels for unaligned shapes (u8, w32), the exact compare-select
//    kernel (int32 / fp32 / int64) and the launch dispatch.
#include <algorithm>
#include <cstdlib>
#include "tiles.cuh"

namespace apsp {

// ------------------------------------------------------------------------------------
// narrow tier: uint8 store, packed 16-bit keys
// ------------------------------------------------------------------------------------
struct SmemU8 {
  uint32_t As[2][SUB][BM];   // replicated key pair (k0 | k0 << 16) per row
  uint16_t Bs[2][SUB][BN];   // tagged key per column
  uint8_t Cs[BM][BN];        // old values of the tile (cp.async prefetch)
};

__device__ __forceinline__ void u8_load_chunk(const MinplusArgs& p, int64_t i0, int64_t j0, int64_t kc,
                                              bool fast, uint4& ra, uint4& rb) {
  const int t = threadIdx.x;
  const uint8_t* A = static_cast<const uint8_t*>(p.A);
  const uint8_t* B = static_cast<const uint8_t*>(p.B);
  {  // A: row r = t & 127, 16 k starting at kc + 16*(t>>7)
    int64_t i = i0 + (t & 127), k = kc + 16 * (t >> 7);
    if (fast) {
      ra = __ldg(reinterpret_cast<const uint4*>(A + i * p.lda + k));
    } else {
      uint8_t b[16];
#pragma unroll
      for (int q = 0; q < 16; q++)
        b[q] = (i < p.m && k + q < p.k) ? A[i * p.lda + k + q] : uint8_t(U8_INF);
      ra = *reinterpret_cast<uint4*>(b);
    }
  }
  {  // B: row kk = t >> 3, 16 columns starting at j0 + 16*(t&7)
    int64_t k = kc + (t >> 3), j = j0 + 16 * (t & 7);
    if (fast) {
      rb = __ldg(reinterpret_cast<const uint4*>(B + k * p.ldb + j));
    } else {
      uint8_t b[16];
#pragma unroll
      for (int q = 0; q < 16; q++)
        b[q] = (k < p.k && j + q < p.n) ? B[k * p.ldb + j + q] : uint8_t(U8_INF);
      rb = *reinterpret_cast<uint4*>(b);
    }
  }
}

__device__ __forceinline__ void u8_store_chunk(SmemU8& sm, int buf, const uint4& ra, const uint4& rb, int tagbase) {
  const int t = threadIdx.x;
  {
    const int r = t & 127, kb = 16 * (t >> 7);
    uint32_t w[4] = {ra.x, ra.y, ra.z, ra.w};
#pragma unroll
    for (int q = 0; q < 16; q++) {
      uint32_t v = (w[q >> 2] >> (8 * (q & 3))) & 0xFF;
      sm.As[buf][kb + q][r] = v * 0x00800080u;   // (v<<7) in both halves
    }
  }
  {
    const int kk = t >> 3, cb = 16 * (t & 7);
    const uint32_t tag = uint32_t(tagbase + kk + 1) * 0x00010001u;
    uint32_t w[4] = {rb.x, rb.y, rb.z, rb.w};
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      o[2 * q] = (__byte_perm(w[q], 0, 0x4140) << U8_TAG) | tag;
      o[2 * q + 1] = (__byte_perm(w[q], 0, 0x4342) << U8_TAG) | tag;
    }
    uint4* dst = reinterpret_cast<uint4*>(&sm.Bs[buf][kk][cb]);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

__global__ void __launch_bounds__(NT, 2) minplus_u8_kernel(MinplusArgs p) {
  extern __shared__ __align__(16) unsigned char smraw_u8[];
  SmemU8& sm = *reinterpret_cast<SmemU8*>(smraw_u8);
  int64_t i0, j0;
  tile_origin(p, BM, BN, i0, j0);
  if (tile_skipped(p, i0, j0, BM, BN)) return;
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;

  uint32_t acc[8][4];   // [row][pair]: pairs = cols {4tx,4tx+1},{4tx+2,4tx+3},{64+4tx..},{..}
  uint32_t kst[8][4];   // packed 16-bit k index (KNONE = untouched)
  const uint8_t* C = static_cast<const uint8_t*>(p.C);
  const bool cfast = (i0 + BM <= p.m) && (j0 + BN <= p.n) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) &&
                     ((p.ldc & 15) == 0);
  {  // old values -> smem asynchronously (cp.async); merged after the first chunk
    const int r = t >> 1, cb = 64 * (t & 1);
    if (cfast) {
      const uint8_t* src = C + (i0 + r) * p.ldc + j0 + cb;
      const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&sm.Cs[r][cb]));
#pragma unroll
      for (int q = 0; q < 4; q++)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 16 * q), "l"(src + 16 * q));
      asm volatile("cp.async.commit_group;\n" ::);
    } else {
      for (int q = 0; q < 64; q++) {
        const int64_t i = i0 + r, j = j0 + cb + q;
        sm.Cs[r][cb + q] = (i < p.m && j < p.n) ? C[i * p.ldc + j] : uint8_t(U8_INF);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      acc[r][q] = U8_KINF * 0x00010001u;
      kst[r][q] = 0u;
    }

  const bool abfast_base = ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0) && ((p.lda & 15) == 0) &&
                           ((reinterpret_cast<uintptr_t>(p.B) & 15) == 0) && ((p.ldb & 15) == 0) &&
                           (i0 + BM <= p.m) && (j0 + BN <= p.n);
  const int64_t nchunks = (p.k + SUB - 1) / SUB;
  uint4 ra, rb;
  u8_load_chunk(p, i0, j0, 0, abfast_base && SUB <= p.k, ra, rb);
  u8_store_chunk(sm, 0, ra, rb, 0);
  __syncthreads();
  for (int64_t c = 0; c < nchunks; c++) {
    const int buf = int(c & 1);
    const bool more = c + 1 < nchunks;
    if (more) u8_load_chunk(p, i0, j0, (c + 1) * SUB, abfast_base && (c + 2) * SUB <= p.k, ra, rb);
#pragma unroll kU8Unroll
    for (int kk = 0; kk < SUB; kk++) {
      const uint4 a0 = *reinterpret_cast<const uint4*>(&sm.As[buf][kk][4 * ty]);
      const uint4 a1 = *reinterpret_cast<const uint4*>(&sm.As[buf][kk][64 + 4 * ty]);
      const uint2 b0 = *reinterpret_cast<const uint2*>(&sm.Bs[buf][kk][4 * tx]);
      const uint2 b1 = *reinterpret_cast<const uint2*>(&sm.Bs[buf][kk][64 + 4 * tx]);
      const uint32_t a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const uint32_t b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[r][q] = viaddmin_u16x2(a[r], b[q], acc[r][q]);
    }
    if (c == 0) {
      // merge the (prefetched) old values: an untagged old key wins value ties, so only a
      // strictly improving candidate keeps its tag (strict-improvement rule)
      asm volatile("cp.async.wait_all;\n" ::);
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 8; r++) {
        const int ri = r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4;
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const uint32_t w = *reinterpret_cast<const uint32_t*>(&sm.Cs[ri][64 * h + 4 * tx]);
          acc[r][2 * h] = __vminu2(acc[r][2 * h], __byte_perm(w, 0, 0x4140) << U8_TAG);
          acc[r][2 * h + 1] = __vminu2(acc[r][2 * h + 1], __byte_perm(w, 0, 0x4342) << U8_TAG);
        }
      }
    }
    // decode the tags of the 64-k window (after every second chunk and the last one) into
    // 1-based k indices (0 = untouched), branch-free:
    //   tg   = tags of the pair;  tg + 0x7FFF per half sets bit 15 iff the tag is nonzero
    //   mask = PRMT sign-replication of bytes 1/3 -> 0xFFFF per half with a tag
    //   kst  = mask ? (window base + tg) : kst   (one LOP3; no cross-half carry: all >= 0)
    if ((c & 1) || !more) {
      uint32_t any = 0;
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) any |= acc[r][q];
      if (__any_sync(0xffffffffu, any & U8_TAGMASK2)) {
        const uint32_t kb2 = uint32_t((c & ~int64_t(1)) * SUB) * 0x00010001u;
#pragma unroll
        for (int r = 0; r < 8; r++)
#pragma unroll
          for (int q = 0; q < 4; q++) {
            const uint32_t tg = acc[r][q] & U8_TAGMASK2;
            const uint32_t mask = prmt_sign_halves(tg + 0x7FFF7FFFu);
            kst[r][q] = (kst[r][q] & ~mask) | ((tg + kb2) & mask);
            acc[r][q] ^= tg;
          }
      }
    }
    if (more) u8_store_chunk(sm, buf ^ 1, ra, rb, int((c + 1) & 1) * SUB);
    __syncthreads();
  }

  // epilogue: values of improved row segments, then idx of improved cells.  The pred gathers
  // of a row are issued back to back (restrict: idx rows never alias the predB rows a tile
  // reads -- the pivot cross is skipped / snapshotted), then stored, 16B when all 4 improved.
  bool changed = false;
  uint8_t* Cw = static_cast<uint8_t*>(p.C);
  const int32_t* __restrict__ pb = p.predB;
  int32_t* __restrict__ out = p.idx;
  const bool idx_vec = out && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((p.ldi & 3) == 0);
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const int64_t i = i0 + (r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4);
    int32_t pv[2][4];
    uint32_t ks[2][4];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t k0 = kst[r][2 * h], k1 = kst[r][2 * h + 1];
      ks[h][0] = k0 & 0xFFFF; ks[h][1] = k0 >> 16; ks[h][2] = k1 & 0xFFFF; ks[h][3] = k1 >> 16;
      const int64_t j = j0 + 64 * h + 4 * tx;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        pv[h][q] = 0;
        if (out && ks[h][q] != 0u && i < p.m && j + q < p.n)
          pv[h][q] = (p.mode == IDX_PRED) ? __ldg(pb + int64_t(ks[h][q] - 1u) * p.ldp + j + q)
                                          : int32_t(p.inner_off + ks[h][q] - 1u);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t k0 = kst[r][2 * h], k1 = kst[r][2 * h + 1];
      if ((k0 | k1) == 0u) continue;
      changed = true;
      const int64_t j = j0 + 64 * h + 4 * tx;
      const uint32_t w = __byte_perm(acc[r][2 * h] >> U8_TAG, acc[r][2 * h + 1] >> U8_TAG, 0x6420);
      if (cfast) {
        *reinterpret_cast<uint32_t*>(Cw + i * p.ldc + j) = w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (i < p.m && j + q < p.n) Cw[i * p.ldc + j + q] = uint8_t(w >> (8 * q));
      }
      if (!out || i >= p.m) continue;
      const bool all4 = ks[h][0] && ks[h][1] && ks[h][2] && ks[h][3];
      if (all4 && idx_vec && cfast) {
        *reinterpret_cast<int4*>(out + i * p.ldi + j) = make_int4(pv[h][0], pv[h][1], pv[h][2], pv[h][3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (ks[h][q] != 0u && j + q < p.n) out[i * p.ldi + j + q] = pv[h][q];
      }
    }
  }
  if (p.status && p.track_changed && __syncthreads_or(changed) && t == 0) p.status->changed = 1;
}

// ------------------------------------------------------------------------------------
// wide tier: int32 store (< 2^24), int32 keys, VIADD + VIMNMX3 over k pairs
// ------------------------------------------------------------------------------------
struct SmemW32 {
  int32_t As[2][SUB][BM];
  int32_t Bs[2][SUB][BN];
};

__device__ __forceinline__ void w32_load_chunk(const MinplusArgs& p, int64_t i0, int64_t j0, int64_t kc,
                                               bool fast, int4 (&ra)[4], int4 (&rb)[4]) {
  const int t = threadIdx.x;
  const int32_t* A = static_cast<const int32_t*>(p.A);
  const int32_t* B = static_cast<const int32_t*>(p.B);
  {
    int64_t i = i0 + (t & 127), k = kc + 16 * (t >> 7);
    if (fast) {
#pragma unroll
      for (int q = 0; q < 4; q++) ra[q] = __ldg(reinterpret_cast<const int4*>(A + i * p.lda + k) + q);
    } else {
      int32_t* v = reinterpret_cast<int32_t*>(ra);
#pragma unroll
      for (int q = 0; q < 16; q++) v[q] = (i < p.m && k + q < p.k) ? A[i * p.lda + k + q] : W32_INF;
    }
  }
  {
    int64_t k = kc + (t >> 3), j = j0 + 16 * (t & 7);
    if (fast) {
#pragma unroll
      for (int q = 0; q < 4; q++) rb[q] = __ldg(reinterpret_cast<const int4*>(B + k * p.ldb + j) + q);
    } else {
      int32_t* v = reinterpret_cast<int32_t*>(rb);
#pragma unroll
      for (int q = 0; q < 16; q++) v[q] = (k < p.k && j + q < p.n) ? B[k * p.ldb + j + q] : W32_INF;
    }
  }
}

__device__ __forceinline__ void w32_store_chunk(SmemW32& sm, int buf, const int4 (&ra)[4], const int4 (&rb)[4]) {
  const int t = threadIdx.x;
  {
    const int r = t & 127, kb = 16 * (t >> 7);
    const int32_t* v = reinterpret_cast<const int32_t*>(ra);
#pragma unroll
    for (int q = 0; q < 16; q++) sm.As[buf][kb + q][r] = v[q] << TAG_BITS;
  }
  {
    const int kk = t >> 3, cb = 16 * (t & 7);
    const int32_t tag = kk + 1;
    const int32_t* v = reinterpret_cast<const int32_t*>(rb);
    int4* dst = reinterpret_cast<int4*>(&sm.Bs[buf][kk][cb]);
#pragma unroll
    for (int q = 0; q < 4; q++)
      dst[q] = make_int4((v[4 * q] << TAG_BITS) | tag, (v[4 * q + 1] << TAG_BITS) | tag,
                         (v[4 * q + 2] << TAG_BITS) | tag, (v[4 * q + 3] << TAG_BITS) | tag);
  }
}

__global__ void __launch_bounds__(NT, 1) minplus_w32_kernel(MinplusArgs p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  SmemW32& sm = *reinterpret_cast<SmemW32*>(smraw);
  int64_t i0, j0;
  tile_origin(p, BM, BN, i0, j0);
  if (tile_skipped(p, i0, j0, BM, BN)) return;
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;

  int32_t acc[8][8];
  uint32_t kst[8][4];
  const int32_t* C = static_cast<const int32_t*>(p.C);
  const bool cfast = (i0 + BM <= p.m) && (j0 + BN <= p.n) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0) &&
                     ((p.ldc & 3) == 0);
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const int64_t i = i0 + (r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int64_t j = j0 + 64 * h + 4 * tx;
      if (cfast) {
        int4 v = *reinterpret_cast<const int4*>(C + i * p.ldc + j);
        acc[r][4 * h] = v.x << TAG_BITS; acc[r][4 * h + 1] = v.y << TAG_BITS;
        acc[r][4 * h + 2] = v.z << TAG_BITS; acc[r][4 * h + 3] = v.w << TAG_BITS;
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++)
          acc[r][4 * h + q] = ((i < p.m && j + q < p.n) ? C[i * p.ldc + j + q] : W32_INF) << TAG_BITS;
      }
      kst[r][2 * h] = 0xFFFFFFFFu;
      kst[r][2 * h + 1] = 0xFFFFFFFFu;
    }
  }

  const bool abfast_base = ((reinterpret_cast<uintptr_t>(p.A) & 15) == 0) && ((p.lda & 3) == 0) &&
                           ((reinterpret_cast<uintptr_t>(p.B) & 15) == 0) && ((p.ldb & 3) == 0) &&
                           (i0 + BM <= p.m) && (j0 + BN <= p.n);
  const int64_t nchunks = (p.k + SUB - 1) / SUB;
  int4 ra[4], rb[4];
  w32_load_chunk(p, i0, j0, 0, abfast_base && SUB <= p.k, ra, rb);
  w32_store_chunk(sm, 0, ra, rb);
  __syncthreads();
  for (int64_t c = 0; c < nchunks; c++) {
    const int buf = int(c & 1);
    const bool more = c + 1 < nchunks;
    if (more) w32_load_chunk(p, i0, j0, (c + 1) * SUB, abfast_base && (c + 2) * SUB <= p.k, ra, rb);
#pragma unroll 2
    for (int kk = 0; kk < SUB; kk += 2) {
      int32_t a0[8], a1[8], b0[8], b1[8];
      {
        const int4 x0 = *reinterpret_cast<const int4*>(&sm.As[buf][kk][4 * ty]);
        const int4 x1 = *reinterpret_cast<const int4*>(&sm.As[buf][kk][64 + 4 * ty]);
        const int4 y0 = *reinterpret_cast<const int4*>(&sm.As[buf][kk + 1][4 * ty]);
        const int4 y1 = *reinterpret_cast<const int4*>(&sm.As[buf][kk + 1][64 + 4 * ty]);
        a0[0] = x0.x; a0[1] = x0.y; a0[2] = x0.z; a0[3] = x0.w; a0[4] = x1.x; a0[5] = x1.y; a0[6] = x1.z; a0[7] = x1.w;
        a1[0] = y0.x; a1[1] = y0.y; a1[2] = y0.z; a1[3] = y0.w; a1[4] = y1.x; a1[5] = y1.y; a1[6] = y1.z; a1[7] = y1.w;
      }
      {
        const int4 x0 = *reinterpret_cast<const int4*>(&sm.Bs[buf][kk][4 * tx]);
        const int4 x1 = *reinterpret_cast<const int4*>(&sm.Bs[buf][kk][64 + 4 * tx]);
        const int4 y0 = *reinterpret_cast<const int4*>(&sm.Bs[buf][kk + 1][4 * tx]);
        const int4 y1 = *reinterpret_cast<const int4*>(&sm.Bs[buf][kk + 1][64 + 4 * tx]);
        b0[0] = x0.x; b0[1] = x0.y; b0[2] = x0.z; b0[3] = x0.w; b0[4] = x1.x; b0[5] = x1.y; b0[6] = x1.z; b0[7] = x1.w;
        b1[0] = y0.x; b1[1] = y0.y; b1[2] = y0.z; b1[3] = y0.w; b1[4] = y1.x; b1[5] = y1.y; b1[6] = y1.z; b1[7] = y1.w;
      }
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int q = 0; q < 8; q++) acc[r][q] = vimin3(acc[r][q], a0[r] + b0[q], a1[r] + b1[q]);
    }
    int32_t any = 0;
#pragma unroll
    for (int r = 0; r < 8; r++)
#pragma unroll
      for (int q = 0; q < 8; q++) any |= acc[r][q];
    if (any & 0x3F) {
      const uint32_t kb = uint32_t(c * SUB) - 1u;
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int q = 0; q < 8; q++) {
          const uint32_t tg = uint32_t(acc[r][q]) & 0x3F;
          if (tg) {
            acc[r][q] ^= int32_t(tg);
            uint32_t& ks = kst[r][q >> 1];
            if (q & 1) ks = (ks & 0x0000FFFFu) | ((kb + tg) << 16);
            else ks = (ks & 0xFFFF0000u) | ((kb + tg) & 0xFFFF);
          }
        }
    }
    if (more) w32_store_chunk(sm, buf ^ 1, ra, rb);
    __syncthreads();
  }

  bool changed = false;
  int32_t* Cw = static_cast<int32_t*>(p.C);
#pragma unroll
  for (int r = 0; r < 8; r++) {
    const int64_t i = i0 + (r < 4 ? 4 * ty + r : 64 + 4 * ty + r - 4);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t k0 = kst[r][2 * h], k1 = kst[r][2 * h + 1];
      if ((k0 & k1) == 0xFFFFFFFFu) continue;
      changed = true;
      const int64_t j = j0 + 64 * h + 4 * tx;
      int32_t v[4];
#pragma unroll
      for (int q = 0; q < 4; q++) v[q] = acc[r][4 * h + q] >> TAG_BITS;
      if (cfast) {
        *reinterpret_cast<int4*>(Cw + i * p.ldc + j) = make_int4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (i < p.m && j + q < p.n) Cw[i * p.ldc + j + q] = v[q];
      }
      if (i < p.m) {
        const uint32_t ks[4] = {k0 & 0xFFFF, k0 >> 16, k1 & 0xFFFF, k1 >> 16};
#pragma unroll
        for (int q = 0; q < 4; q++)
          if (ks[q] != KNONE && j + q < p.n) emit_idx(p, i, j + q, ks[q]);
      }
    }
  }
  if (p.status && p.track_changed && __syncthreads_or(changed) && t == 0) p.status->changed = 1;
}

// ------------------------------------------------------------------------------------
// exact tier: compare-select over any store (int32 API, fp32, int64)
// ------------------------------------------------------------------------------------
constexpr int EM = 64, EN = 64;   // 256 threads, 4x4 cells each

template <int S>
__global__ void __launch_bounds__(NT) minplus_exact_kernel(MinplusArgs p) {
  using T = typename StoreT<S>::T;
  __shared__ T As[SUB][EM + 1];
  __shared__ T Bs[SUB][EN];
  int64_t i0, j0;
  tile_origin(p, EM, EN, i0, j0);
  if (tile_skipped(p, i0, j0, EM, EN)) return;
  const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
  const T inf = store_inf<S>();
  const T* A = static_cast<const T*>(p.A);
  const T* B = static_cast<const T*>(p.B);
  T* C = static_cast<T*>(p.C);

  T acc[4][4];
  int32_t kid[4][4];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int64_t i = i0 + ty + 16 * r, j = j0 + tx + 16 * q;
      acc[r][q] = (i < p.m && j < p.n) ? C[i * p.ldc + j] : inf;
      kid[r][q] = -1;
    }
  bool overflow = false;
  for (int64_t kc = 0; kc < p.k; kc += SUB) {
    for (int e = t; e < SUB * EM; e += NT) {
      const int r = e / SUB, kk = e % SUB;
      const int64_t i = i0 + r, k = kc + kk;
      As[kk][r] = (i < p.m && k < p.k) ? A[i * p.lda + k] : inf;
      const int kb = e / EN, c = e % EN;
      const int64_t kb_ = kc + kb, j = j0 + c;
      Bs[kb][c] = (kb_ < p.k && j < p.n) ? B[kb_ * p.ldb + j] : inf;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < SUB; kk++) {
      T a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; r++) a[r] = As[kk][ty + 16 * r];
#pragma unroll
      for (int q = 0; q < 4; q++) b[q] = Bs[kk][tx + 16 * q];
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const T s = a[r] + b[q];
          if (s < acc[r][q]) {
            overflow |= range_overflow<S>(s);
            acc[r][q] = s;
            kid[r][q] = int32_t(kc + kk);
          }
        }
    }
    __syncthreads();
  }
  bool changed = false;
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int64_t i = i0 + ty + 16 * r, j = j0 + tx + 16 * q;
      if (kid[r][q] >= 0 && i < p.m && j < p.n) {
        changed = true;
        C[i * p.ldc + j] = acc[r][q];
        emit_idx(p, i, j, uint32_t(kid[r][q]));
      }
    }
  if (p.status) {
    if (overflow) p.status->overflow = 1;
    if (p.track_changed && __syncthreads_or(changed) && t == 0) p.status->changed = 1;
  }
}

int launch_minplus(int store, const MinplusArgs& a, cudaStream_t s) {
  if (a.m <= 0 || a.n <= 0) return 0;
  if (a.npeers < 0 || a.npeers > MAX_PEERS) return set_error(2, "npeers %d outside [0, %d]", a.npeers, MAX_PEERS);
  if (a.npeers && !(a.Aprep && a.Bprep && (store == STORE_U8 || store == STORE_U16 || store == STORE_W32)))
    return set_error(2, "fused peer stores need a bulk-staged tier (u8 / u16 / w32) with prepared panels");
  if (a.push_all && !(a.npeers && (store == STORE_U8 || store == STORE_U16 || store == STORE_W32)))
    return set_error(2, "whole-panel peer pushes need a bulk-staged tier (u8 / u16 / w32) and peers");
  if (a.k <= 0) return 0;
  if (a.k > 65535) return set_error(2, "min-plus inner dimension %lld exceeds 65535", (long long)a.k);
  if (a.only_lo < a.only_hi) {
    const int tb = (store == STORE_U8 || store == STORE_W32) ? BM : EM;
    if (a.only_lo % tb || a.only_hi % tb || a.m != a.n)
      return set_error(2, "cross-list mode needs tile-aligned bands on a square view");
  }
  switch (store) {
    case STORE_U8: {
      if (a.Aprep && a.Bprep) {
        const int rc = launch_nt<STORE_U8>(a, s);
        if (rc) return rc;
        break;
      }
      static std::atomic<unsigned long long> attr{0};
      APSP_CUDA_TRY(smem_optin(minplus_u8_kernel, int(sizeof(SmemU8)), attr));
      minplus_u8_kernel<<<grid_for(a, BM, BN), NT, sizeof(SmemU8), s>>>(a);
      break;
    }
    case STORE_W32: {
      if (a.Aprep && a.Bprep) {
        const int rc = launch_w32nt(a, s);
        if (rc) return rc;
        break;
      }
      static std::atomic<unsigned long long> attr{0};
      APSP_CUDA_TRY(smem_optin(minplus_w32_kernel, int(sizeof(SmemW32)), attr));
      minplus_w32_kernel<<<grid_for(a, BM, BN), NT, sizeof(SmemW32), s>>>(a);
      break;
    }
    case STORE_U16: {
      if (!(a.Aprep && a.Bprep)) return set_error(2, "the u16 tier needs pre-laid-out panels (aligned products)");
      const int rc = launch_nt<STORE_U16>(a, s);
      if (rc) return rc;
      break;
    }
    case STORE_F32:
      if (a.Aprep && a.Bprep) {
        const int rc = f32_deferred() ? launch_f32dm(a, s) : launch_f32nt(a, s);
        if (rc) return rc;
        break;
      }
      [[fallthrough]];
    case STORE_I32:
    case STORE_I64: {
      const dim3 grid = grid_for(a, EM, EN);
      if (store == STORE_I32) minplus_exact_kernel<STORE_I32><<<grid, NT, 0, s>>>(a);
      else if (store == STORE_F32) minplus_exact_kernel<STORE_F32><<<grid, NT, 0, s>>>(a);
      else minplus_exact_kernel<STORE_I64><<<grid, NT, 0, s>>>(a);
      break;
    }
    default:
      return set_error(2, "unknown store %d", store);
  }
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return 0;
}

}  // namespace apsp
