// Shared definitions for the APSP sm_100a kernels.
//
// Value domains ("stores").  Every kernel works on one of these in-HBM formats; the
// sentinel of each is chosen so that INF + INF never overflows the arithmetic type, which
// makes "strict c < d" saturate at Infinity with no branch (the reference gets the same
// effect from INF_RAW = 2^61, core.py:19-20):
//
//   STORE_U8    uint8_t  finite 0..254, INF 255      narrow tier (16-bit keys, 7-bit tags, u16x2 DPX)
//   STORE_U16   uint16_t finite 0..510, INF 511      narrow tier (16-bit keys, 6-bit tags, u16x2 DPX)
//   STORE_W32   int32_t  finite 0..2^24-2, INF 2^24-1 wide tier   (keys are 32-bit)
//   STORE_I32   int32_t  finite 0..2^30-2, INF 0x3FFFFFFF   exact int32 (API format)
//   STORE_F32   float    finite >= 0, INF +inf             exact fp32 (API format)
//   STORE_I64   int64_t  finite 0..2^60-1, INF 2^61        exact int64 (reference format)
//
// Keyed tiers (U8/W32) carry the argmin inside the value: key = value << 6 | tag, where
// tag = 1 + (k mod 32) is attached to the right operand.  A plain integer min over keys is
// then the lexicographic (value, smallest k) argmin the reference uses
// (minplus.py:80-82, strict improvement = untagged old key wins ties).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apsp {

enum Store : int { STORE_U8 = 0, STORE_W32 = 1, STORE_I32 = 2, STORE_F32 = 3, STORE_I64 = 4, STORE_U16 = 5 };

constexpr int32_t INF32 = 0x3FFFFFFF;
constexpr int64_t INF_RAW = int64_t(1) << 61;
constexpr int64_t MAX_FINITE_COST = (int64_t(1) << 60) - 1;

constexpr int TAG_BITS = 6;
constexpr int SUB = 32;                 // k-steps between argmin decodes (tags 1..32)
constexpr int U8_INF = 255;
constexpr int U16_INF = 511;
constexpr int32_t W32_INF = 0x00FFFFFF;
constexpr uint32_t K16_INF = uint32_t(U8_INF) << TAG_BITS;      // 16320; 2*K16_INF+32 < 2^15
constexpr int32_t K32_INF = W32_INF << TAG_BITS;                 // 0x3FFFFFC0
constexpr uint32_t TAGMASK2 = 0x003F003Fu;                      // tags of a packed key pair
constexpr uint16_t KNONE = 0xFFFF;                               // "not improved" k index

template <int S> struct StoreT;
template <> struct StoreT<STORE_U8>  { using T = uint8_t;  using A = int32_t; static constexpr bool keyed = true; };
template <> struct StoreT<STORE_W32> { using T = int32_t;  using A = int32_t; static constexpr bool keyed = true; };
template <> struct StoreT<STORE_I32> { using T = int32_t;  using A = int32_t; static constexpr bool keyed = false; };
template <> struct StoreT<STORE_F32> { using T = float;    using A = float;   static constexpr bool keyed = false; };
template <> struct StoreT<STORE_I64> { using T = int64_t;  using A = int64_t; static constexpr bool keyed = false; };
template <> struct StoreT<STORE_U16> { using T = uint16_t; using A = int32_t; static constexpr bool keyed = true; };

template <int S> __host__ __device__ inline typename StoreT<S>::T store_inf();
template <> __host__ __device__ inline uint8_t store_inf<STORE_U8>() { return U8_INF; }
template <> __host__ __device__ inline int32_t store_inf<STORE_W32>() { return W32_INF; }
template <> __host__ __device__ inline int32_t store_inf<STORE_I32>() { return INF32; }
template <> __host__ __device__ inline float store_inf<STORE_F32>() { return __builtin_huge_valf(); }
template <> __host__ __device__ inline int64_t store_inf<STORE_I64>() { return INF_RAW; }
template <> __host__ __device__ inline uint16_t store_inf<STORE_U16>() { return U16_INF; }

// Overflow rule of the int64 domain (solvers.py:91-92): a strictly improving finite sum
// above MAX_FINITE_COST is a range error.  The narrower domains never report it: their
// sums saturate to "no improvement" and the host certificate (fw.cu) decides exactness.
template <int S> __device__ __forceinline__ bool range_overflow(typename StoreT<S>::A c) { return false; }
template <> __device__ __forceinline__ bool range_overflow<STORE_I64>(int64_t c) { return c > MAX_FINITE_COST; }

// Index output of a min-plus update (the reference's two artifacts):
//   IDX_PRED  idx[i][j] <- pred_right[k*][j]   (FW rule, solvers.py:94)
//   IDX_VIA   idx[i][j] <- inner_off + k*      (global via, minplus.py:91-97)
enum IdxMode : int { IDX_PRED = 0, IDX_VIA = 1 };

struct Status {            // device-side status word, one per solve
  int32_t overflow;        // int64 domain left the finite range
  int32_t changed;         // any strict improvement (fw_squaring convergence)
};

__device__ __forceinline__ uint32_t viaddmin16x2(uint32_t a, uint32_t b, uint32_t c) {
  return __viaddmin_s16x2(a, b, c);
}
__device__ __forceinline__ int32_t vimin3(int32_t a, int32_t b, int32_t c) { return __vimin3_s32(a, b, c); }

#define APSP_CUDA_TRY(expr)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return ::apsp::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
  } while (0)

int set_cuda_error(cudaError_t e, const char* what, const char* file, int line);
int set_error(int code, const char* fmt, ...);
void count_launches(long long k);   // process-wide kernel launch counter (apsp_launch_count)

}  // namespace apsp
