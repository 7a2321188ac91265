/*
 * apsp_b200.h -- C ABI of the B200-native dense APSP engine (libapsp_b200.so).
 *
 * Drop-in boundary for the reference's hot path (apsp 0.1.0, /root/reference/pkg/src/apsp):
 * each entry point below replaces one reference function; the Python package
 * paper_2310_03983_b200 binds them with ctypes and keeps the reference's Python API
 * (fw_classic / rkleene / fw_squaring / minplus_product / minplus_accumulate).
 *
 * Conventions
 *   - dtype: APSP_DTYPE_I32 (Infinity = 0x3FFFFFFF), APSP_DTYPE_F32 (Infinity = +inf),
 *            APSP_DTYPE_I64 (Infinity = 2^61 = the reference's INF_RAW, core.py:19).
 *   - index matrices (pred / via) are int32 on the device, -1 = None (core.py:233-272);
 *     the host-level call can widen them to int64 like the reference's PredMatrix/ViaMatrix.
 *   - matrices are row-major with a leading dimension (elements).
 *   - device-level calls take device pointers and a cudaStream_t (NULL = legacy default
 *     stream).  They are stream-ordered except for the small host reads the solver needs
 *     to pick and certify a value tier (documented per call).  ws may be NULL: the library
 *     then allocates stream-ordered scratch itself.
 *   - every call returns an apsp_status; apsp_last_error() holds a thread-local message.
 */
#ifndef APSP_B200_H
#define APSP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define APSP_ABI_VERSION 2

typedef enum {
  APSP_OK = 0,
  APSP_ERANGE = 1,      /* -> CostRangeError      (solvers.py:91-92,146-147; minplus.py:158-163) */
  APSP_EINVAL = 2,      /* -> ParameterError      (solvers.py:131-132,227-230; minplus.py:181-183) */
  APSP_ECUDA = 3,       /* CUDA runtime failure */
  APSP_ENCCL = 4,       /* collective failure (multi-GPU path) */
  APSP_ENEGATIVE = 5,   /* -> NegativeWeightError (solvers.py:70-71; minplus.py:153-155) */
  APSP_EDIAGONAL = 6,   /* -> MalformedGraphError (solvers.py:72-73) */
  APSP_EDIMENSION = 7,  /* -> DimensionError      (minplus.py:179-180,221-228) */
  APSP_ECONVERGE = 8    /* -> ApspError           (solvers.py:195-196) */
} apsp_status;

typedef enum { APSP_DTYPE_I32 = 0, APSP_DTYPE_F32 = 1, APSP_DTYPE_I64 = 2 } apsp_dtype;

/* Value tiers (in-HBM store formats); AUTO picks the narrowest exact one and certifies it. */
typedef enum {
  APSP_TIER_AUTO = -1,
  APSP_TIER_U8 = 0,   /* uint8 store (values < 255), 16-bit packed keys, VIADDMNMX.U16x2 */
  APSP_TIER_W32 = 1,  /* int32 store (< 2^24), 32-bit keys, VIADD + VIMNMX3 */
  APSP_TIER_I32 = 2,  /* exact int32 compare-select */
  APSP_TIER_F32 = 3,  /* exact fp32 compare-select (continuous weights) */
  APSP_TIER_I64 = 4,  /* exact int64 compare-select (full reference range) */
  APSP_TIER_U16 = 5   /* uint16 store (values < 511), 16-bit packed keys, VIADDMNMX.U16x2 (aligned products) */
} apsp_tier;

typedef enum { APSP_IDX_PRED = 0, APSP_IDX_VIA = 1 } apsp_idx_mode;

typedef enum {
  APSP_ALG_FW_BLOCKED = 0,  /* blocked 3-phase FW (replaces fw_classic, solvers.py:118) */
  APSP_ALG_FW_CLASSIC = 1,  /* classic k-order FW, bit-exact pred (solvers.py:118-155) */
  APSP_ALG_RKLEENE = 2,     /* recursive closure (solvers.py:207-296) */
  APSP_ALG_FW_SQUARING = 3  /* repeated min-plus squaring (solvers.py:167-204) */
} apsp_algorithm;

typedef struct apsp_info {
  int32_t tier;         /* tier that produced the returned result */
  int32_t tiers_tried;  /* bitmask over apsp_tier values */
  int32_t iterations;   /* fw_squaring rounds (solvers.py:186-194); 0 otherwise */
  int32_t launches;     /* kernels launched by the call */
  int64_t max_finite;   /* largest finite distance of the result (integer tiers) */
  int64_t relaxations;  /* exact candidate count, the reference's relaxation_count */
  double device_ms;     /* CUDA-event time of the solve (device-level calls) */
  int32_t flags;        /* bit 0: zero-cost edges -> classic k order used for predecessors */
  int32_t kernel_launches; /* profiled min-plus tile launches (apsp_set_profiling(1)) */
  double kernel_ms;     /* summed CUDA-event time of those launches */
  int32_t block;        /* pivot block used by the blocked FW (0 otherwise) */
  int32_t d2h_bytes_per_cell; /* apsp_solve_host: result bytes per cell read back (dist + idx) */
  int32_t h2d_bytes_per_cell; /* apsp_solve_host: cost bytes per cell uploaded */
  int32_t reserved;
} apsp_info;

const char* apsp_last_error(void);
int apsp_abi_version(void);

/* Profiling switch (process-wide): when on, every min-plus tile launch (FW phase 3, R-Kleene
 * and squaring products) is bracketed by CUDA events on its stream and apsp_info reports
 * their count and summed duration.  Off by default; costs two event records per launch. */
void apsp_set_profiling(int on);

/* Number of kernels this library has launched in the process (all devices, all calls). */
long long apsp_launch_count(void);
/* Profiled min-plus tile launches recorded on this host thread since the last read (the shard
 * entry points below have no apsp_info): their count and summed CUDA-event time. Synchronises
 * with the recorded events; resets the record. */
int apsp_profile_read(double* kernel_ms, int32_t* launches);

/* Scratch bytes the device-level calls need when ws != NULL. */
size_t apsp_workspace_bytes(int algorithm, int dtype, int64_t n, int block);

/* Blocked three-phase Floyd-Warshall, in place on dist; pred (int32, n x n, ldp) receives
 * predecessors (pred[i][j] = last vertex before j, -1 = None).
 * Replaces fw_classic (solvers.py:118-155): same distances bit-exactly, pred a valid
 * shortest-path tree (equal-length ties may pick another predecessor).
 * block: pivot block size (0 = by n).  Host syncs: after the input scan and after the
 * certificate; a repeated call of the same shape starts the tier that certified last time
 * right behind the scan and syncs once.  dist is written only on success; on an error
 * return the contents of pred are unspecified. */
int apsp_fw_blocked(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, int block,
                    int tier, void* ws, size_t ws_bytes, void* stream, apsp_info* info);

/* Classic k-order Floyd-Warshall (one launch per k), in place; bit-exact dist and pred with
 * fw_classic (solvers.py:77-95,134-147).  dtype = storage of dist (no tiering). */
int apsp_fw_classic(int dtype, int64_t n, void* dist, int64_t ld, int32_t* pred, int64_t ldp, void* stream,
                    apsp_info* info);

/* R-Kleene recursive closure (solvers.py:207-296), in place on dist; idx receives via (global
 * intermediate vertex, APSP_IDX_VIA) or pred (APSP_IDX_PRED).
 * aligned = 0: floor split and classic leaves at base_threshold -> via bit-exact with rkleene.
 * aligned = 1: splits on 128-multiples, leaves of <= base_threshold closed by blocked FW. */
int apsp_rkleene(int dtype, int64_t n, void* dist, int64_t ld, int32_t* idx, int64_t ldi, int idx_mode,
                 int base_threshold, int aligned, int tier, void* ws, size_t ws_bytes, void* stream, apsp_info* info);

/* Repeated squaring H <- min(H, H (x) H) until unchanged (solvers.py:167-204); via folded. */
int apsp_fw_squaring(int dtype, int64_t n, void* dist, int64_t ld, int32_t* via, int64_t ldv, int tier, void* ws,
                     size_t ws_bytes, void* stream, apsp_info* info);

/* minplus_product (accumulate = 0; minplus.py:166-203, offsets = (row, inner, col)) and
 * minplus_accumulate (accumulate = 1; minplus.py:206-252, z and via are the seeds).
 * x: n1 x n2, y: n2 x n3, z: n1 x n3 (out; in for accumulate), via: n1 x n3 (out; in for accumulate). */
int apsp_minplus(int dtype, int accumulate, int64_t n1, int64_t n2, int64_t n3, const void* x, int64_t ldx,
                 const void* y, int64_t ldy, void* z, int64_t ldz, int32_t* via, int64_t ldv, int64_t row_off,
                 int64_t inner_off, int64_t col_off, int tier, void* stream, apsp_info* info);

/* Host-level call (reference-facing): host input h (n x n, dense, dtype), host outputs
 * dist_out (dtype) and idx_out (idx_dtype = APSP_DTYPE_I32 or APSP_DTYPE_I64).  Copies in,
 * solves on `device`, copies out; synchronous like the reference solvers.
 * algorithm: apsp_algorithm; idx_mode: APSP_IDX_PRED / APSP_IDX_VIA (rkleene only). */
int apsp_solve_host(int algorithm, int dtype, int64_t n, const void* h, void* dist_out, void* idx_out, int idx_dtype,
                    int idx_mode, int block, int base_threshold, int aligned, int tier, int device, apsp_info* info);

/* ---- building blocks: input scan and row-band shards of the blocked FW (multi-GPU) ----------
 * The sharded solver (paper_2310_03983_b200.distributed) runs one process per GPU; rank r owns
 * rows [row0, row0 + rows) of the N x N padded matrix (rows a multiple of block).  Per pivot
 * block k0 the owner calls apsp_shard_pivot, broadcasts the b x N row panel (values + pred)
 * with NCCL, and every rank calls apsp_shard_update with the received panel.  tier must be the
 * same on all ranks (chosen from the all-reduced apsp_scan results). */
typedef struct apsp_scan_result {
  int32_t negative;      /* a finite cost < 0 (or NaN) */
  int32_t diag_nonzero;  /* a diagonal cell != 0 */
  int32_t non_integral;  /* fp32 input with a non-integral finite cost */
  int32_t any_finite;
  int64_t max_finite;    /* largest finite cost (integer view) */
  float max_finite_f;    /* largest finite cost (fp32 input) */
  int32_t zero_offdiag;  /* a zero-cost edge off the diagonal */
  uint64_t finite_offdiag; /* number of finite off-diagonal cells (edges) */
} apsp_scan_result;

/* diag_off: cell (i, i + diag_off) is diagonal (0 whole matrix, row0 for a shard, -1 none). Syncs. */
int apsp_scan(int dtype, const void* h, int64_t ld, int64_t rows, int64_t cols, int64_t diag_off,
              apsp_scan_result* out, void* stream);
size_t apsp_shard_scratch_bytes(int tier, int64_t N, int64_t rows, int block);
int apsp_shard_prepare(int dtype, int tier, int64_t n, int64_t N, int64_t row0, int64_t rows, const void* h,
                       int64_t ldh, void* D, int64_t ld, int32_t* P, int64_t ldp, void* stream);
int apsp_shard_pivot(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, void* stream);
/* Fused variant: the pivot's row-panel product also stores the whole b x N panel (values and
 * pred, every cell) into npeers (<= 7) peer receive slots -- address + peer_dv[r] / peer_dp[r]
 * bytes from the local panel rows, IPC-mapped over NVLink -- replacing the NCCL broadcast with
 * the kernel's own peer stores.  u8 / u16 tiers. */
int apsp_shard_pivot_fused(int tier, int64_t N, int block, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                           int64_t k0, int npeers, const int64_t* peer_dv, const int64_t* peer_dp, void* scratch,
                           size_t scratch_bytes, void* stream);
/* Updates local rows [row_lo, row_hi) with the received panel; rows [skip_lo, skip_hi) (the
 * caller's own pivot rows, -1 if none) are left alone. */
int apsp_shard_update(int tier, int64_t N, int block, int64_t row_lo, int64_t row_hi, void* D, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, void* stream);
/* The library's high-priority side stream of the current device (lookahead pivots). */
void* apsp_side_stream(void);
/* Converts rows x n back to dtype (dist) and copies pred; *max_finite = largest finite local
 * distance (for the cross-rank certificate), -1 if none.  Syncs. */
int apsp_shard_finish(int tier, int dtype, int64_t rows, int64_t n, const void* D, int64_t ld, const int32_t* P,
                      int64_t ldp, void* dist, int64_t ldd, int32_t* pred, int64_t ldpo, int64_t* max_finite,
                      void* stream);

/* ---- sharded R-Kleene: replicated matrix, products split by output row bands --
 * Every rank holds the whole padded N x N store matrix D and pred P (apsp_shard_prepare with
 * row0 = 0, rows = N; N a multiple of 128).  The host recursion (distributed.py run_rkleene,
 * the order of solvers.py:239-286 with the 128-aligned split) calls apsp_rk_shard_leaf for the
 * diagonal leaves (every rank, redundantly) and apsp_rk_shard_product for its band of output
 * rows of each block product C <- min(C, A (x) B) (pred <- pred_b[k*][j]); the caller then
 * all-gathers the bands.  Replaces the band loop of rkleene (solvers.py:239-286) across GPUs. */
size_t apsp_rk_shard_scratch_bytes(int64_t N, int thr);
int apsp_rk_shard_leaf(int tier, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, void* stream);
int apsp_rk_shard_product(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          void* stream);
/* Fused exchange: the same product, whose epilogue also stores every improved C / pred segment
 * at the same position of npeers (<= 7) peer replicas -- address + peer_dc[r] / peer_di[r]
 * bytes, peer memory mapped into this process (CUDA IPC over NVLink) -- so the band reaches every
 * GPU while the other tiles still compute; the caller then only needs a barrier instead of an
 * all-gather.  u8 / u16 / w32 tiers (bulk-staged tiles) only. */
int apsp_rk_shard_product_fused(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                                int32_t* idx, int64_t ldi, const int32_t* pred_b, int64_t ldpb, int64_t m, int64_t n,
                                int64_t k, int64_t inner_off, int64_t N, int thr, int npeers, const int64_t* peer_dc,
                                const int64_t* peer_di, void* scratch, size_t scratch_bytes, void* stream);

/* ---- host-side matrix wire format of the reference (textio.py:70-119), multi-threaded ----------
 * apsp_format_matrix_i64: writes "n\n" + n rows of n fields (integer or INF) into out; returns
 * the byte count, or the required capacity when out is NULL / cap is too small, -2 for a
 * negative cell.  apsp_parse_matrix_i64: parses the n body lines (after the header) into out;
 * 0 ok, -(1 + row) for a malformed row (*bad_col = field), -(1 + n) for a wrong line count. */
int64_t apsp_format_matrix_i64(const int64_t* m, int64_t n, char* out, int64_t cap);
int64_t apsp_parse_matrix_i64(const char* text, int64_t len, int64_t n, int64_t* out, int64_t* bad_col);

#ifdef __cplusplus
}
#endif
#endif /* APSP_B200_H */
