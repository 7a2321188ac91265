// Host-side halves of the narrowed transfers (hostio.cu): widening of the readback (u8/u16
// distances -> int32, all-ones -> INF32; u16 predecessors p + 1 -> int32/int64) and narrowing
// of the int32 cost upload (int32 -> u8/u16 when every cell fits). Compiled by the host compiler (not
// nvcc) so the AVX-512 variant can be selected at run time. All variants use streaming stores
// once the destination is aligned, so the output lines are written without being read first.
#include <cstddef>
#include <cstdint>
#include <immintrin.h>

namespace apsp {

namespace {

constexpr int32_t kInf32 = 0x3FFFFFFF;   // common.cuh INF32

constexpr long long kInfRaw = 1LL << 61;   // common.cuh INF_RAW

template <typename S, typename D = int32_t>
inline D dist_of(S v) { return v == S(~S(0)) ? (sizeof(D) == 4 ? D(kInf32) : D(kInfRaw)) : D(v); }

// ---- AVX-512 -----------------------------------------------------------------------------

template <typename S, typename D>
__attribute__((target("avx512f,avx512bw"))) void widen_dist_avx512(const S* s, D* d, size_t cnt) {
  size_t i = 0;
  for (; i < cnt && (reinterpret_cast<uintptr_t>(d + i) & 63); i++) d[i] = dist_of<S, D>(s[i]);
  if constexpr (sizeof(D) == 4) {
    const __m512i all = _mm512_set1_epi32(int(S(~S(0)))), inf = _mm512_set1_epi32(kInf32);
    for (; i + 16 <= cnt; i += 16) {
      __m512i v;
      if (sizeof(S) == 1) v = _mm512_cvtepu8_epi32(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i)));
      else v = _mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i)));
      v = _mm512_mask_mov_epi32(v, _mm512_cmpeq_epi32_mask(v, all), inf);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), v);
    }
  } else {
    const __m512i all = _mm512_set1_epi64((long long)S(~S(0))), inf = _mm512_set1_epi64(kInfRaw);
    for (; i + 8 <= cnt; i += 8) {
      __m512i v;
      if (sizeof(S) == 1) v = _mm512_cvtepu8_epi64(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + i)));
      else v = _mm512_cvtepu16_epi64(_mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i)));
      v = _mm512_mask_mov_epi64(v, _mm512_cmpeq_epi64_mask(v, all), inf);
      _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), v);
    }
  }
  for (; i < cnt; i++) d[i] = dist_of<S, D>(s[i]);
  _mm_sfence();
}

template <typename T>
__attribute__((target("avx512f,avx512bw"))) void widen_pred_avx512(const uint16_t* s, T* d, size_t cnt) {
  size_t i = 0;
  for (; i < cnt && (reinterpret_cast<uintptr_t>(d + i) & 63); i++) d[i] = T(int32_t(s[i]) - 1);
  const __m512i one = _mm512_set1_epi32(1);
  for (; i + 16 <= cnt; i += 16) {
    const __m512i v =
        _mm512_sub_epi32(_mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i))), one);
    if (sizeof(T) == 4) {
      _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), v);
    } else {
      _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i), _mm512_cvtepi32_epi64(_mm512_castsi512_si256(v)));
      _mm512_stream_si512(reinterpret_cast<__m512i*>(d + i + 8),
                          _mm512_cvtepi32_epi64(_mm512_extracti64x4_epi64(v, 1)));
    }
  }
  for (; i < cnt; i++) d[i] = T(int32_t(s[i]) - 1);
  _mm_sfence();
}

// ---- SSE2 baseline -----------------------------------------------------------------------

template <typename S>
void widen_dist_scalar64(const S* s, int64_t* d, size_t cnt) {
  for (size_t i = 0; i < cnt; i++) d[i] = dist_of<S, int64_t>(s[i]);
}

template <typename S>
void widen_dist_sse2(const S* s, int32_t* d, size_t cnt) {
  size_t i = 0;
  for (; i < cnt && (reinterpret_cast<uintptr_t>(d + i) & 15); i++) d[i] = dist_of(s[i]);
  const __m128i z = _mm_setzero_si128(), all = _mm_set1_epi32(int(S(~S(0)))), inf = _mm_set1_epi32(kInf32);
  for (; i + 8 <= cnt; i += 8) {
    __m128i w[2];
    if (sizeof(S) == 1) {
      const __m128i b = _mm_unpacklo_epi8(_mm_loadl_epi64(reinterpret_cast<const __m128i*>(s + i)), z);
      w[0] = _mm_unpacklo_epi16(b, z);
      w[1] = _mm_unpackhi_epi16(b, z);
    } else {
      const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      w[0] = _mm_unpacklo_epi16(h, z);
      w[1] = _mm_unpackhi_epi16(h, z);
    }
    for (int q = 0; q < 2; q++) {
      const __m128i e = _mm_cmpeq_epi32(w[q], all);
      _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4 * q),
                       _mm_or_si128(_mm_andnot_si128(e, w[q]), _mm_and_si128(e, inf)));
    }
  }
  for (; i < cnt; i++) d[i] = dist_of(s[i]);
  _mm_sfence();
}

template <typename T>
void widen_pred_sse2(const uint16_t* s, T* d, size_t cnt) {
  size_t i = 0;
  for (; i < cnt && (reinterpret_cast<uintptr_t>(d + i) & 15); i++) d[i] = T(int32_t(s[i]) - 1);
  const __m128i z = _mm_setzero_si128(), one = _mm_set1_epi32(1);
  for (; i + 8 <= cnt; i += 8) {
    const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i w[2] = {_mm_sub_epi32(_mm_unpacklo_epi16(h, z), one), _mm_sub_epi32(_mm_unpackhi_epi16(h, z), one)};
    for (int q = 0; q < 2; q++) {
      if (sizeof(T) == 4) {
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4 * q), w[q]);
      } else {
        const __m128i sg = _mm_srai_epi32(w[q], 31);
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4 * q), _mm_unpacklo_epi32(w[q], sg));
        _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 4 * q + 2), _mm_unpackhi_epi32(w[q], sg));
      }
    }
  }
  for (; i < cnt; i++) d[i] = T(int32_t(s[i]) - 1);
  _mm_sfence();
}

// int32 / int64 costs -> u8/u16 (INF -> all-ones). Returns false at the first cell that is
// neither INF nor in [0, lim]; the caller then uploads the matrix as is.
template <typename S>
__attribute__((target("avx512f,avx512bw"))) bool narrow_avx512(const int32_t* s, S* d, size_t cnt, int32_t lim) {
  size_t i = 0;
  const __m512i inf = _mm512_set1_epi32(kInf32), all = _mm512_set1_epi32(int(S(~S(0)))), l = _mm512_set1_epi32(lim);
  for (; i + 16 <= cnt; i += 16) {
    const __m512i v = _mm512_loadu_si512(s + i);
    const __mmask16 isinf = _mm512_cmpeq_epi32_mask(v, inf);
    if (_mm512_mask_cmpgt_epu32_mask(~isinf, v, l)) return false;   // unsigned: negatives fail too
    const __m512i w = _mm512_mask_mov_epi32(v, isinf, all);
    if (sizeof(S) == 1) _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi32_epi8(w));
    else _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i), _mm512_cvtepi32_epi16(w));
  }
  for (; i < cnt; i++) {
    if (s[i] == kInf32) d[i] = S(~S(0));
    else if (uint32_t(s[i]) > uint32_t(lim)) return false;
    else d[i] = S(s[i]);
  }
  return true;
}

template <typename S>
__attribute__((target("avx512f,avx512bw"))) bool narrow_avx512(const int64_t* s, S* d, size_t cnt, int32_t lim) {
  size_t i = 0;
  const __m512i inf = _mm512_set1_epi64(kInfRaw), all = _mm512_set1_epi64((long long)S(~S(0))),
                l = _mm512_set1_epi64(lim);
  for (; i + 8 <= cnt; i += 8) {
    const __m512i v = _mm512_loadu_si512(s + i);
    const __mmask8 isinf = _mm512_cmpeq_epi64_mask(v, inf);
    if (_mm512_mask_cmpgt_epu64_mask(__mmask8(~isinf), v, l)) return false;
    const __m512i w = _mm512_mask_mov_epi64(v, isinf, all);
    if (sizeof(S) == 1) _mm_storel_epi64(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi64_epi8(w));
    else _mm_storeu_si128(reinterpret_cast<__m128i*>(d + i), _mm512_cvtepi64_epi16(w));
  }
  for (; i < cnt; i++) {
    if (s[i] == kInfRaw) d[i] = S(~S(0));
    else if (uint64_t(s[i]) > uint64_t(lim)) return false;
    else d[i] = S(s[i]);
  }
  return true;
}

template <typename T, typename S>
bool narrow_scalar(const T* s, S* d, size_t cnt, int32_t lim) {
  const T inf = sizeof(T) == 4 ? T(kInf32) : T(kInfRaw);
  for (size_t i = 0; i < cnt; i++) {
    if (s[i] == inf) d[i] = S(~S(0));
    else if (s[i] < 0 || s[i] > T(lim)) return false;
    else d[i] = S(s[i]);
  }
  return true;
}

bool has_avx512() {
  static const bool ok = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw");
  return ok;
}

}  // namespace

void host_widen_dist(const void* src, int width, void* dst, bool wide, size_t cnt) {
  if (wide) {
    if (width == 1) {
      if (has_avx512()) widen_dist_avx512(static_cast<const uint8_t*>(src), static_cast<int64_t*>(dst), cnt);
      else widen_dist_scalar64(static_cast<const uint8_t*>(src), static_cast<int64_t*>(dst), cnt);
    } else {
      if (has_avx512()) widen_dist_avx512(static_cast<const uint16_t*>(src), static_cast<int64_t*>(dst), cnt);
      else widen_dist_scalar64(static_cast<const uint16_t*>(src), static_cast<int64_t*>(dst), cnt);
    }
    return;
  }
  if (width == 1) {
    if (has_avx512()) widen_dist_avx512(static_cast<const uint8_t*>(src), static_cast<int32_t*>(dst), cnt);
    else widen_dist_sse2(static_cast<const uint8_t*>(src), static_cast<int32_t*>(dst), cnt);
  } else {
    if (has_avx512()) widen_dist_avx512(static_cast<const uint16_t*>(src), static_cast<int32_t*>(dst), cnt);
    else widen_dist_sse2(static_cast<const uint16_t*>(src), static_cast<int32_t*>(dst), cnt);
  }
}

void host_widen_pred(const uint16_t* src, void* dst, bool wide, size_t cnt) {
  if (wide) {
    if (has_avx512()) widen_pred_avx512(src, static_cast<int64_t*>(dst), cnt);
    else widen_pred_sse2(src, static_cast<int64_t*>(dst), cnt);
  } else {
    if (has_avx512()) widen_pred_avx512(src, static_cast<int32_t*>(dst), cnt);
    else widen_pred_sse2(src, static_cast<int32_t*>(dst), cnt);
  }
}

template <typename T>
static bool narrow_any(const T* src, void* dst, int width, size_t cnt) {
  if (width == 1)
    return has_avx512() ? narrow_avx512(src, static_cast<uint8_t*>(dst), cnt, 254)
                        : narrow_scalar(src, static_cast<uint8_t*>(dst), cnt, 254);
  return has_avx512() ? narrow_avx512(src, static_cast<uint16_t*>(dst), cnt, 65534)
                      : narrow_scalar(src, static_cast<uint16_t*>(dst), cnt, 65534);
}

bool host_narrow(const void* src, bool wide, void* dst, int width, size_t cnt) {
  return wide ? narrow_any(static_cast<const int64_t*>(src), dst, width, cnt)
              : narrow_any(static_cast<const int32_t*>(src), dst, width, cnt);
}

}  // namespace apsp
