// Host-side launchers for the sm_100a kernels (one translation unit per kernel family).
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace apsp {

// Opt a kernel into more than 48 KB of dynamic shared memory, once per device (the attribute is
// per device; a process may drive several GPUs through apsp_solve_host's device argument).
template <typename K>
inline cudaError_t smem_optin(K* kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kernel), cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// One min-plus tile update  C <- min(C, A (x) B)  with strict-improvement lexicographic
// (value, smallest k) argmin, written to idx on improvement only.  Covers FW phase 3
// (skip_row/col_tile = the pivot block) and every R-Kleene block product
// (solvers.py:250-286; minplus.py:114-133).
constexpr int MAX_PEERS = 7;      // 8 GPUs per NVSwitch node

struct MinplusArgs {
  const void* A; int64_t lda;     // m x k
  const void* B; int64_t ldb;     // k x n
  void* C; int64_t ldc;           // m x n, in/out
  int32_t* idx; int64_t ldi;      // m x n, written where C strictly improves (may be null)
  const int32_t* predB; int64_t ldp;  // k x n, IDX_PRED source rows (pred of B's rows)
  int64_t m, n, k;
  int64_t inner_off;              // IDX_VIA: global vertex of k = 0
  int mode;                       // IdxMode
  int64_t skip_row_lo, skip_row_hi;  // rows [lo,hi) and cols [lo,hi) form the FW pivot cross;
  int64_t skip_col_lo, skip_col_hi;  // tiles entirely inside either band are skipped
  int64_t skip2_lo, skip2_hi;     // a second cross (rows and cols [lo,hi)) to skip (lookahead rest)
  int64_t skip3_lo, skip3_hi;     // a third cross to skip (two-deep lookahead rest)
  int64_t only_lo, only_hi;       // if lo < hi: the grid enumerates only the tiles of this cross
  Status* status;                 // optional: overflow flag (+ changed flag if track_changed)
  int track_changed;              // set status->changed on any strict improvement (squaring)
  // u8 / u16 / w32 tiers: operand panels pre-laid-out by launch_prep_bulk (bulk-copy staging);
  // null = off.  Bprep is uint16 keys for u8/u16 and uint32 keys for w32.
  const uint32_t* Aprep;          // [m/128][k/32][32][128] keys (u8/u16: replicated into both halves)
  const void* Bprep;              // [n/128][k/32][32][128] tagged keys
  // Fused exchange (bulk-staged kernels only): every improved C / idx segment is also stored at
  // the same position of up to MAX_PEERS peer replicas -- address + peer_dC[r] / peer_dI[r]
  // bytes (peer memory mapped over NVLink), so the product's output reaches every GPU while the
  // remaining tiles compute.
  int npeers;
  int64_t peer_dC[MAX_PEERS];
  int64_t peer_dI[MAX_PEERS];
  int push_all;                   // peer-store every cell of each tile, not only improved ones
  // Programmatic dependent launch: this launch has no data dependency on the kernel queued
  // right before it on the stream (FW phase 3b after 3a: disjoint tiles), so its CTAs may start
  // while that kernel's last wave drains.
  int pdl;
  // Exact fp32 deferred-argmin kernel: detect improvements (and rescan) every 8 k instead of
  // every 32 -- cheaper when many cells improve per chunk (early FW rounds).
  int fine;
  // Optional exit count (u8 / u16 bulk-staged kernels): every CTA, skipped or not, adds 1 here
  // after its stores are fenced, so a kernel on another stream can start on the device as soon
  // as this launch's count is reached (the FW closure after the 3a cross, fw_sched.cu).
  int* exit_count;
  // Optional next-round layouts (FW 3a with b = 128, u8 / u16 bulk kernel): the tiles of the
  // cross [only_lo, only_hi) other than the diagonal also write themselves in the prep formats
  // of the next phase-2 launch -- column-band tiles as A row tile i0/128 of nxA, row-band tiles
  // as B column tile j0/128 of nxB plus their final pred rows into nxPred (ld nxPredLd).
  uint32_t* nxA;
  uint16_t* nxB;
  int32_t* nxPred;
  int64_t nxPredLd;
  // Optional (same kernels): the CTA of the cross's diagonal tile stores diag_value to diag_flag
  // (release) right after its own stores, ahead of the rest of the launch; and every CTA waits
  // (acquire) until *wait_count >= wait_target before reading anything.
  int* diag_flag;
  int diag_value;
  const int* wait_count;
  int wait_target;
  // Optional per-tile round flags (FW b = 128 device-signalled chain, u8 / u16 bulk kernel): the
  // CTA of tile (I, J) waits until tile_flags[I * tile_ld + J] >= tile_round (the previous round
  // has updated it), and releases tile_round + 1 after its stores. Lets a launch start while the
  // previous round's last wave drains.
  int* tile_flags;
  int tile_ld;
  int tile_round;
  // Full-grid launches: if first_lo < first_hi the (1D) grid enumerates the tiles of the cross
  // [first_lo, first_hi) first, then the rest row-major (FW 3b: the next 3a's inputs first).
  int64_t first_lo, first_hi;
  // Cross-list launches of the u8 / u16 bulk kernel: two CTAs per tile, each owning 64 rows
  // (half the work each: the latency-bound FW 3a / cross launches use twice the SMs). Round
  // flags and the diagonal flag then count halves: a whole-tile CTA adds 2, a half adds 1.
  int split_rows;
  // First-mode launches (first_lo < first_hi): this launch covers CTA ids [id_begin, id_begin +
  // grid) of the enumeration (a launch split in two: whole tiles, then the tail as half rows)
  int id_begin;
  int id_count;   // 0: to the end of the enumeration
  // Full-grid launches: grouped tile order (row tiles per group; <= 1: row-major), see tile_origin
  int raster;
};

// Lay the u8 operand panels out in the tile kernel's shared-memory format, once per product:
// A (m x k) -> replicated 16-bit key pairs, B (k x n) -> tagged 16-bit keys.  m, n multiples of
// 128 and k a multiple of 32 (the FW phase-3 case).
size_t prep_bytes(int64_t m, int64_t n, int64_t k);
int launch_prep_bulk(int store, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t m, int64_t n,
                     int64_t k, uint32_t* Aprep, void* Bprep, cudaStream_t s, const int32_t* psrc = nullptr,
                     int64_t lds = 0, int32_t* pdst = nullptr, int64_t ldd = 0, int64_t pcols = 0,
                     int* exit_count = nullptr, int* ctas = nullptr);

// Row tiles per rasterisation group of full-grid launches (APSP_RASTER_G, default 1 = row-major).
int raster_group();

// Default-initialised args: nothing skipped, full grid.
inline MinplusArgs minplus_args() {
  MinplusArgs a{};
  a.skip_row_lo = a.skip_row_hi = a.skip_col_lo = a.skip_col_hi = -1;
  a.skip2_lo = a.skip2_hi = -1;
  a.skip3_lo = a.skip3_hi = -1;
  a.only_lo = a.only_hi = -1;
  a.first_lo = a.first_hi = -1;
  a.raster = raster_group();
  return a;
}

int launch_minplus(int store, const MinplusArgs& a, cudaStream_t s);

// Closure of the diagonal block [lo, lo+m) (m <= 128) in classic k order, one CTA:
// FW phase 1 and the R-Kleene leaf (_fw_via_block, solvers.py:98-115).
// Small-n u8 blocked FW in one persistent launch (fw_persist.cuh, in fw.cu)
bool fw_persist_enabled(int store, int64_t N);
size_t fw_persist_scratch_bytes(int64_t N);
int launch_fw_persist(uint8_t* D, int64_t ld, int32_t* P, int64_t ldp, int64_t N, void* scratch, cudaStream_t s);
bool fw_persist64_enabled(int store, int64_t N);
size_t fw_persist64_scratch_bytes(int64_t N);
int launch_fw_persist64(int store, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t N, void* scratch,
                        cudaStream_t s);
// Blocked in-CTA closure for the 32-bit exact stores, pred mode (close_blk.cu)
bool close_blk_supported(int store);
int launch_block_close_blk(int store, void* D, int64_t ld, int64_t lo, int64_t m, int32_t* idx, int64_t ldi,
                           cudaStream_t s);
// wait_count (u8 / u16 full 128-blocks only): the closure kernel starts on the device once
// *wait_count >= wait_target (acquire), instead of behind a stream event
// nx* (same conditions): the closed block also writes its layouts / pred rows for the next
// phase-2 launch (see MinplusArgs::nxA)
int launch_block_close(int store, void* D, int64_t ld, int64_t lo, int64_t m,
                       int32_t* idx, int64_t ldi, int mode, int64_t via_off, Status* st,
                       cudaStream_t s, const int* wait_count = nullptr, int wait_target = 0,
                       uint32_t* nxA = nullptr, uint16_t* nxB = nullptr, int32_t* nxPred = nullptr,
                       int64_t nxPredLd = 0);

// K1 for small n: all n classic steps in one single-CTA launch (the store in shared memory);
// done = false (nothing launched) when the matrix does not fit
int launch_fw_classic_cta(int store, void* D, int64_t ld, int64_t n, int32_t* idx, int64_t ldi, Status* st,
                          cudaStream_t s, bool& done);

// Classic per-k Floyd-Warshall step (K1): bit-exact pred/via parity with fw_classic
// (solvers.py:77-95).  One launch per k; row k / column k are invariant in step k.
int launch_fw_step(int store, void* D, int64_t ld, int64_t n, int64_t k, int32_t* idx,
                   int64_t ldi, int mode, int64_t via_off, Status* st, cudaStream_t s);

// Input scan (K7): negatives, nonzero diagonal, max finite, non-integral fp32.
struct ScanResult {
  int32_t negative;
  int32_t diag_nonzero;
  int32_t non_integral;
  int32_t any_finite;
  int64_t max_finite;      // integer domains (fp32: floor of max)
  float max_finite_f;      // fp32 domain
  int32_t zero_offdiag;    // a finite zero cost off the diagonal (zero-weight edge)
  unsigned long long finite_offdiag;   // number of finite off-diagonal cells (edges)
};
// diag_off: cell (i, i + diag_off) is a diagonal cell (0 for a whole matrix, row0 for a
// row shard, -1: no diagonal check)
int launch_scan(int in_dtype, const void* h, int64_t ld, int64_t rows, int64_t cols,
                int64_t diag_off, ScanResult* out_dev, cudaStream_t s);

// API dtype <-> store conversion, with padding to N (pad vertices are isolated) and the
// FW pred initialisation pred[i][j] = i where h[i][j] finite and i != j (solvers.py:135-137).
int launch_to_store(int in_dtype, const void* h, int64_t ldh, int64_t n, int store, void* D,
                    int64_t ld, int64_t N, int32_t* P, int64_t ldp, int pred_init, cudaStream_t s);
// the same for rows [row0, row0 + R) of the padded matrix (h holds those rows of the input)
// rectangular operand (no padding, no pred); h == nullptr fills Infinity
int launch_to_store_rect(int in_dtype, const void* h, int64_t ldh, int64_t rows, int64_t cols, int store, void* out,
                         int64_t ldo, cudaStream_t s);
int launch_to_store_rows(int in_dtype, const void* h, int64_t ldh, int64_t n, int store, void* D, int64_t ld,
                         int64_t N, int32_t* P, int64_t ldp, int pred_init, int64_t row0, int64_t R, cudaStream_t s);
int launch_from_store(int store, const void* D, int64_t ld, int64_t rows, int64_t cols,
                      int out_dtype, void* out, int64_t ldo, cudaStream_t s);
int launch_copy_idx(const int32_t* P, int64_t ldp, int64_t rows, int64_t cols, int out_dtype,
                    void* out, int64_t ldo, cudaStream_t s);
int launch_fill_idx(int32_t* P, int64_t ldp, int64_t rows, int64_t cols, int32_t v, cudaStream_t s);
int launch_copy_block(int store, const void* src, int64_t lds, void* dst, int64_t ldd,
                      int64_t rows, int64_t cols, cudaStream_t s);
int launch_max_finite(int store, const void* D, int64_t ld, int64_t rows, int64_t cols,
                      ScanResult* out_dev, cudaStream_t s);
// Self-witness via clear of minplus_product (minplus.py:99-111).
int launch_witness_clear(int store, const void* X, int64_t ldx, const void* Y, int64_t ldy,
                         const void* Dp, int64_t ldd, int32_t* via, int64_t ldv, int64_t n1,
                         int64_t n2, int64_t n3, int64_t row_off, int64_t inner_off,
                         int64_t col_off, cudaStream_t s);

size_t store_elem_size(int store);

}  // namespace apsp
