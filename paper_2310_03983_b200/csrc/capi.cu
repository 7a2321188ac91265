// C ABI (include/apsp_b200.h): thin extern "C" wrappers over the engine, plus the host-level
// entry point.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include "engine.h"

using namespace apsp;

// =============================================================================================
extern "C" {

const char* apsp_last_error(void) { return apsp::last_error(); }
void apsp_set_profiling(int on) { g_prof.on = on != 0; }
long long apsp_launch_count(void) { return apsp::launch_count(); }
int apsp_profile_read(double* kernel_ms, int32_t* launches) {
  apsp_info info{};
  APSP_CUDA_TRY(cudaDeviceSynchronize());
  g_prof.collect(&info);
  g_prof.reset();
  if (kernel_ms) *kernel_ms = info.kernel_ms;
  if (launches) *launches = info.kernel_launches;
  return 0;
}

int apsp_scan(int dtype, const void* h, int64_t ld, int64_t rows, int64_t cols, int64_t diag_off,
              apsp_scan_result* out, void* stream) {
  static_assert(sizeof(apsp_scan_result) == sizeof(ScanResult), "scan result layout");
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, sizeof(ScanResult), s);
  if (rc) return rc;
  rc = launch_scan(dtype, h, ld, rows, cols, diag_off, static_cast<ScanResult*>(sc.base), s);
  if (rc) return rc;
  APSP_CUDA_TRY(cudaMemcpyAsync(out, sc.base, sizeof(ScanResult), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  return 0;
}

size_t apsp_shard_scratch_bytes(int tier, int64_t N, int64_t rows, int block) {
  const int store = tier_store(tier);
  return shard_scratch_bytes(N, rows, block, store < 0 ? 8 : store_elem_size(store));
}

int apsp_shard_prepare(int dtype, int tier, int64_t n, int64_t N, int64_t row0, int64_t rows, const void* h,
                       int64_t ldh, void* D, int64_t ld, int32_t* P, int64_t ldp, void* stream) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  return launch_to_store_rows(dtype, h, ldh, n, store, D, ld, N, P, ldp, 1, row0, rows, (cudaStream_t)stream);
}

int apsp_shard_pivot(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, void* stream) {
  return shard_pivot_impl(tier, N, block, D, ld, P, ldp, lrow, k0, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_shard_update(int tier, int64_t N, int block, int64_t row_lo, int64_t row_hi, void* D, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, void* stream) {
  return shard_update_impl(tier, N, block, row_lo, row_hi, D, ld, P, ldp, panel, ldpv, ppanel, ldpp, k0, skip_lo,
                           skip_hi, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_shard_pivot_fused(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                           int64_t k0, int npeers, const int64_t* peer_dv, const int64_t* peer_dp, void* scratch,
                           size_t scratch_bytes, void* stream) {
  return shard_pivot_impl(tier, N, block, D, ld, P, ldp, lrow, k0, scratch, scratch_bytes, (cudaStream_t)stream,
                          npeers, peer_dv, peer_dp);
}

void* apsp_side_stream(void) { return side_stream(); }

int apsp_shard_finish(int tier, int dtype, int64_t rows, int64_t n, const void* D, int64_t ld, const int32_t* P,
                      int64_t ldp, void* dist, int64_t ldd, int32_t* pred, int64_t ldpo, int64_t* max_finite,
                      void* stream) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  cudaStream_t s = (cudaStream_t)stream;
  Scratch sc;
  int rc = sc.acquire(nullptr, 0, sizeof(ScanResult), s);
  if (rc) return rc;
  ScanResult* r = static_cast<ScanResult*>(sc.base);
  if (rows > 0) {
    rc = launch_max_finite(store, D, ld, rows, n, r, s);
    if (!rc && dist) rc = launch_from_store(store, D, ld, rows, n, dtype, dist, ldd, s);
    if (!rc && pred && P) rc = launch_copy_idx(P, ldp, rows, n, APSP_DTYPE_I32, pred, ldpo, s);
    if (rc) return rc;
  } else {
    APSP_CUDA_TRY(cudaMemsetAsync(r, 0, sizeof(ScanResult), s));
  }
  ScanResult h{};
  APSP_CUDA_TRY(cudaMemcpyAsync(&h, r, sizeof(ScanResult), cudaMemcpyDeviceToHost, s));
  APSP_CUDA_TRY(cudaStreamSynchronize(s));
  if (max_finite) *max_finite = rows > 0 && h.max_finite >= 0 ? h.max_finite : -1;
  return 0;
}

size_t apsp_rk_shard_scratch_bytes(int64_t N, int thr) { return rk_shard_scratch_bytes(N, thr); }

int apsp_rk_shard_product_fused(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                                int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                                int64_t k, int64_t inner_off, int64_t N, int thr, int npeers, const int64_t* peer_dc,
                                const int64_t* peer_di, void* scratch, size_t scratch_bytes, void* stream) {
  return rk_shard_product_impl(tier, A, lda, B, ldb, C, ldc, idx, ldi, pred_b, ldpb, m, n, k, inner_off, N, thr,
                               scratch, scratch_bytes, (cudaStream_t)stream, npeers, peer_dc, peer_di);
}

int apsp_rk_shard_leaf(int tier, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, void* stream) {
  return rk_shard_leaf_impl(tier, D, ld, P, ldp, lo, m, thr, scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_rk_shard_product(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          void* stream) {
  return rk_shard_product_impl(tier, A, lda, B, ldb, C, ldc, idx, ldi, pred_b, ldpb, m, n, k, inner_off, N, thr,
                               scratch, scratch_bytes, (cudaStream_t)stream);
}

int apsp_abi_version(void) { return APSP_ABI_VERSION; }

size_t apsp_workspace_bytes(int algorithm, int dtype, int64_t n, int block) {
  switch (algorithm) {
    case APSP_ALG_FW_BLOCKED: return fw_ws_bytes(dtype, n, block > 0 ? block : default_block(n));
    case APSP_ALG_RKLEENE: return std::max(rk_ws_bytes(dtype, n, 1, 1 << 30), rk_ws_bytes(dtype, n, 0));
    case APSP_ALG_FW_SQUARING: return sq_ws_bytes(dtype, n);
    case APSP_ALG_FW_CLASSIC: return 0;
  }
  return 0;
}

int apsp_fw_blocked(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, int block, int tier,
                    void* ws, size_t ws_bytes, void* stream, apsp_info* info) {
  return fw_blocked_impl(dtype, n, dist, ld, pred, ldp, block, tier, ws, ws_bytes, (cudaStream_t)stream, info);
}

int apsp_fw_classic(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, void* stream,
                    apsp_info* info) {
  return fw_classic_impl(dtype, n, dist, ld, pred, ldp, (cudaStream_t)stream, info);
}

int apsp_rkleene(int dtype, int64_t n, void* dist, int64_t ld, int32_t* idx, int64_t ldi, int idx_mode,
                 int base_threshold, int aligned, int tier, void* ws, size_t ws_bytes, void* stream, apsp_info* info) {
  return rkleene_impl(dtype, n, dist, ld, idx, ldi, idx_mode, base_threshold, aligned, tier, ws, ws_bytes,
                      (cudaStream_t)stream, info);
}

int apsp_fw_squaring(int dtype, int64_t n, void* dist, int64_t ld, int32_t* via, int64_t ldv, int tier, void* ws,
                     size_t ws_bytes, void* stream, apsp_info* info) {
  return squaring_impl(dtype, n, dist, ld, via, ldv, tier, ws, ws_bytes, (cudaStream_t)stream, info);
}

int apsp_minplus(int dtype, int accumulate, int64_t n1, int64_t n2, int64_t n3, const void* x, int64_t ldx,
                 const void* y, int64_t ldy, void* z, int64_t ldz, int32_t* via, int64_t ldv, int64_t row_off,
                 int64_t inner_off, int64_t col_off, int tier, void* stream, apsp_info* info) {
  return minplus_impl(dtype, accumulate, n1, n2, n3, x, ldx, y, ldy, z, ldz, via, ldv, row_off, inner_off, col_off,
                      tier, (cudaStream_t)stream, info);
}

int apsp_solve_host(int algorithm, int dtype, int64_t n, const void* h, void* dist_out, void* idx_out, int idx_dtype,
                    int idx_mode, int block, int base_threshold, int aligned, int tier, int device, apsp_info* info) {
  if (n < 1) return set_error(APSP_EDIMENSION, "cost matrix must be non-empty");
  if (idx_dtype != APSP_DTYPE_I32 && idx_dtype != APSP_DTYPE_I64)
    return set_error(APSP_EINVAL, "index dtype must be int32 or int64");
  APSP_CUDA_TRY(cudaSetDevice(device));
  keep_pool();
  cudaStream_t s;
  APSP_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const size_t es = dtype == APSP_DTYPE_I64 ? 8 : 4;
  const size_t bytes = size_t(n) * n * es;
  void* d = nullptr;
  int32_t* p = nullptr;
  void* pw = nullptr;
  int rc = 0;
  auto fail = [&](int code) {
    if (d) cudaFreeAsync(d, s);
    if (p) cudaFreeAsync(p, s);
    if (pw) cudaFreeAsync(pw, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return code;
  };
  cudaError_t e = cudaMallocAsync(&d, bytes, s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&p, size_t(n) * n * 4, s);
  if (e == cudaSuccess && idx_dtype == APSP_DTYPE_I64 && idx_out) e = cudaMallocAsync(&pw, size_t(n) * n * 8, s);
  if (e != cudaSuccess) return fail(set_cuda_error(e, "host staging", __FILE__, __LINE__));
  bool up = false;
  int up_width = int(es);
  if (dtype == APSP_DTYPE_I32 || dtype == APSP_DTYPE_I64) {   // integer costs: narrowed upload
    rc = upload_packed(n, h, int(es), d, s, up, up_width);
    if (rc) return fail(rc);
  }
  if (!up) e = cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return fail(set_cuda_error(e, "host staging", __FILE__, __LINE__));
  apsp_info local{};
  local.max_finite = -1;   // stays -1 (no packed readback) unless the solver reports it
  // blocked FW: the last round's row bands stream to the host while the rest computes
  std::unique_ptr<BandSink> bands;
  if (algorithm == APSP_ALG_FW_BLOCKED && (dtype == APSP_DTYPE_I32 || dtype == APSP_DTYPE_I64))
    bands = make_band_stream(n, int(es), dist_out, idx_out, idx_dtype, s);
  switch (algorithm) {
    case APSP_ALG_FW_BLOCKED:
      rc = fw_blocked_impl(dtype, n, d, n, p, n, block, tier, nullptr, 0, s, &local, bands.get());
      break;
    case APSP_ALG_FW_CLASSIC: rc = fw_classic_impl(dtype, n, d, n, p, n, s, &local); break;
    case APSP_ALG_RKLEENE:
      rc = rkleene_impl(dtype, n, d, n, p, n, idx_mode, base_threshold, aligned, tier, nullptr, 0, s, &local);
      break;
    case APSP_ALG_FW_SQUARING: rc = squaring_impl(dtype, n, d, n, p, n, tier, nullptr, 0, s, &local); break;
    default: rc = set_error(APSP_EINVAL, "unknown algorithm %d", algorithm);
  }
  local.h2d_bytes_per_cell = up ? up_width : int32_t(es);
  if (info) *info = local;
  if (bands) {   // the streamed rows stand only if the u8 attempt certified
    const bool streamed = finish_band_stream(bands.get()) && rc == 0 && local.tier == APSP_TIER_U8;
    bands.reset();   // releases the readback staging
    if (streamed) {
      if (info) info->d2h_bytes_per_cell = 1 + 2;
      return fail(0);
    }
  }
  if (rc) return fail(rc);
  if (dtype == APSP_DTYPE_I32 || dtype == APSP_DTYPE_I64) {   // integer results: narrowed readback
    bool done = false;
    rc = readback_packed(n, d, int(es), idx_out ? p : nullptr, local.max_finite, dist_out, idx_out, idx_dtype, s,
                         done);
    if (rc) return fail(rc);
    if (done) {
      if (info) info->d2h_bytes_per_cell = readback_width(n, local.max_finite, int(es), idx_out != nullptr);
      return fail(0);
    }
  }
  if (info) info->d2h_bytes_per_cell = int32_t(es + (idx_out ? (idx_dtype == APSP_DTYPE_I64 ? 8 : 4) : 0));
  e = cudaMemcpyAsync(dist_out, d, bytes, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess && idx_out) {
    if (idx_dtype == APSP_DTYPE_I64) {
      rc = launch_copy_idx(p, n, n, n, APSP_DTYPE_I64, pw, n, s);
      if (rc) return fail(rc);
      e = cudaMemcpyAsync(idx_out, pw, size_t(n) * n * 8, cudaMemcpyDeviceToHost, s);
    } else {
      e = cudaMemcpyAsync(idx_out, p, size_t(n) * n * 4, cudaMemcpyDeviceToHost, s);
    }
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(set_cuda_error(e, "host readback", __FILE__, __LINE__));
  return fail(0);
}

}  // extern "C"
