// Multi-GPU building blocks: row-band FW shards and sharded R-Kleene products.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "engine.h"

namespace apsp {

// ---- row-band shards of a blocked FW (multi-GPU building blocks) ---------------------------
//
// Rank r owns rows [row0, row0 + R) of the padded N x N matrix (R a multiple of b).  Per
// pivot block [k0, k0 + b) with owner o (local pivot rows [lrow, lrow + b) on o):
//   owner:     shard_pivot  = phase 1 on the diagonal block + row panel <- Dg (x) row panel
//   broadcast  row panel values (b x N) and pred (b x N) from o        (NCCL, caller)
//   everyone:  shard_update = column panel <- colpanel (x) Dg; phase 3 on the local rows
// The arithmetic is exactly the single-GPU schedule, so results are bit-identical to one GPU
// at the same b.
size_t shard_scratch_bytes(int64_t N, int64_t R, int b, size_t es) {
  size_t v = size_t(b) * N * 4 + 256;                                         // pred row-panel snapshot
  if (b > TILE_ALIGN) v += size_t(b) * N * es + size_t(R) * b * es + 512;     // value snapshots
  v += std::max(prep_bytes(b, N, b), prep_bytes(std::max<int64_t>(R, b), N, b)) + 256;   // panel layouts
  if (b > TILE_ALIGN) v += fw_scratch_bytes(b, TILE_ALIGN, es) + 256;        // phase-1 sub-run
  return v;
}

struct ShardScratch {
  int32_t* predsnap;
  char* rowsnap;
  char* colsnap;
  char* prep;
  char* sub;
};

ShardScratch shard_carve(void* scratch, int64_t N, int64_t R, int b, size_t es) {
  ShardScratch c{};
  char* p = static_cast<char*>(scratch);
  c.predsnap = reinterpret_cast<int32_t*>(p);
  p += size_t(b) * N * 4 + 256;
  if (b > TILE_ALIGN) {
    c.rowsnap = p;
    c.colsnap = p + size_t(b) * N * es + 256;
    p += size_t(b) * N * es + size_t(R) * b * es + 512;
  }
  c.prep = p;
  p += std::max(prep_bytes(b, N, b), prep_bytes(std::max<int64_t>(R, b), N, b)) + 256;
  if (b > TILE_ALIGN) c.sub = p;
  return c;
}

int shard_pivot_impl(int tier, int64_t N, int b, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lrow,
                     int64_t k0, void* scratch, size_t scratch_bytes, cudaStream_t s, int npeers,
                     const int64_t* peer_dv, const int64_t* peer_dp) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  const size_t es = store_elem_size(store);
  if (scratch_bytes < shard_scratch_bytes(N, b, b, es)) return set_error(APSP_EINVAL, "shard scratch too small");
  const ShardScratch sc = shard_carve(scratch, N, b, b, es);
  char* D = static_cast<char*>(Dv);
  FwCtx c;
  c.store = store; c.es = es;
  c.D = D + (lrow * ld + k0) * es; c.ld = ld;
  c.P = P ? P + lrow * ldp + k0 : nullptr; c.ldp = ldp;
  c.m = b; c.b = b; c.mode = IDX_PRED; c.via_off = k0;
  c.predsnap = sc.predsnap;
  c.sub = sc.sub;
  int rc = fw_phase1(c, 0, s);                           // diagonal block, classic order
  if (rc) return rc;
  char* rowp = D + lrow * ld * es;
  const bool nt = bulk_store(store, b);
  const bool snap = !nt && b > TILE_ALIGN;
  if (P) APSP_CUDA_TRY(cudaMemcpy2DAsync(sc.predsnap, size_t(N) * 4, P + lrow * ldp, size_t(ldp) * 4, size_t(N) * 4,
                                         size_t(b), cudaMemcpyDeviceToDevice, s));
  if (snap && (rc = launch_copy_block(store, rowp, ld, sc.rowsnap, N, b, N, s))) return rc;
  MinplusArgs a = minplus_args();
  a.A = c.D; a.lda = ld;
  a.B = snap ? sc.rowsnap : rowp; a.ldb = snap ? N : ld;
  a.C = rowp; a.ldc = ld;
  a.idx = P ? P + lrow * ldp : nullptr; a.ldi = ldp;
  a.predB = sc.predsnap; a.ldp = N;
  a.m = b; a.n = N; a.k = b; a.inner_off = k0; a.mode = IDX_PRED;
  if (npeers > 0) {
    // fused panel push: the product also covers the diagonal tiles (Dg (x) Dg never improves a
    // closed block) and stores every cell of the b x N panel, values and pred, into each
    // peer's receive slot (address + peer_dv / peer_dp bytes, IPC-mapped over NVLink)
    if (!nt || !(store == STORE_U8 || store == STORE_U16 || store == STORE_W32))
      return set_error(APSP_EINVAL, "the fused panel push needs a bulk-staged tier (u8 / u16 / w32)");
    if (npeers > MAX_PEERS) return set_error(APSP_EINVAL, "npeers %d outside [0, %d]", npeers, MAX_PEERS);
    a.npeers = npeers;
    a.push_all = 1;
    for (int r = 0; r < npeers; r++) {
      a.peer_dC[r] = peer_dv[r];
      a.peer_dI[r] = peer_dp[r];
    }
  } else {
    a.skip_col_lo = k0; a.skip_col_hi = k0 + b;
  }
  if (nt) {
    if ((rc = launch_prep_bulk(store, c.D, ld, rowp, ld, b, N, b, prep_a(sc.prep), prep_b(sc.prep, b, b), s)))
      return rc;
    a.Aprep = prep_a(sc.prep);
    a.Bprep = prep_b(sc.prep, b, b);
  }
  return launch_minplus(store, a, s);
}

int shard_update_impl(int tier, int64_t N, int b, int64_t row_lo, int64_t row_hi, void* Dv, int64_t ld, int32_t* P,
                      int64_t ldp, const void* panel, int64_t ldpv, const int32_t* ppanel, int64_t ldpp, int64_t k0,
                      int64_t skip_lo, int64_t skip_hi, void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  const int64_t R = row_hi - row_lo;
  if (R <= 0) return 0;
  const size_t es = store_elem_size(store);
  if (scratch_bytes < shard_scratch_bytes(N, R, b, es)) return set_error(APSP_EINVAL, "shard scratch too small");
  const ShardScratch sc = shard_carve(scratch, N, R, b, es);
  char* D = static_cast<char*>(Dv) + row_lo * ld * es;      // the processed row range
  int32_t* Pr = P ? P + row_lo * ldp : nullptr;
  const char* pv = static_cast<const char*>(panel);
  const bool nt = bulk_store(store, b);
  const bool snap = !nt && b > TILE_ALIGN;
  const bool skip = skip_lo >= 0 && skip_hi > skip_lo;
  int rc = 0;
  if (snap && (rc = launch_copy_block(store, D + k0 * es, ld, sc.colsnap, b, R, b, s))) return rc;
  // column panel of the rows against the (received) closed diagonal block
  MinplusArgs q = minplus_args();
  q.A = snap ? sc.colsnap : D + k0 * es; q.lda = snap ? b : ld;
  q.B = pv + k0 * es; q.ldb = ldpv;
  q.C = D + k0 * es; q.ldc = ld;
  q.idx = Pr ? Pr + k0 : nullptr; q.ldi = ldp;
  q.predB = ppanel ? ppanel + k0 : nullptr; q.ldp = ldpp;
  q.m = R; q.n = b; q.k = b; q.inner_off = k0; q.mode = IDX_PRED;
  if (skip) { q.skip_row_lo = skip_lo - row_lo; q.skip_row_hi = skip_hi - row_lo; }
  if (nt) {
    if ((rc = launch_prep_bulk(store, D + k0 * es, ld, pv + k0 * es, ldpv, R, b, b, prep_a(sc.prep),
                                 prep_b(sc.prep, R, b), s)))
      return rc;
    q.Aprep = prep_a(sc.prep);
    q.Bprep = prep_b(sc.prep, R, b);
  }
  if ((rc = launch_minplus(store, q, s))) return rc;
  // phase 3 of the rows
  MinplusArgs a = minplus_args();
  a.A = D + k0 * es; a.lda = ld;
  a.B = pv; a.ldb = ldpv;
  a.C = D; a.ldc = ld;
  a.idx = Pr; a.ldi = ldp;
  a.predB = ppanel; a.ldp = ldpp;
  a.m = R; a.n = N; a.k = b; a.inner_off = k0; a.mode = IDX_PRED;
  if (skip) { a.skip_row_lo = skip_lo - row_lo; a.skip_row_hi = skip_hi - row_lo; }
  a.skip_col_lo = k0; a.skip_col_hi = k0 + b;
  if (nt) {
    if ((rc = launch_prep_bulk(store, D + k0 * es, ld, pv, ldpv, R, N, b, prep_a(sc.prep), prep_b(sc.prep, R, b),
                                 s)))
      return rc;
    a.Aprep = prep_a(sc.prep);
    a.Bprep = prep_b(sc.prep, R, b);
  }
  return timed_minplus(store, a, s);
}

// ---- sharded R-Kleene: replicated matrix, every block product split by output row bands ----
// Every rank holds the whole N x N store matrix (N a multiple of 128, aligned split).  The host
// schedule (distributed.py run_rkleene) mirrors RK::close; each of the six block products is
// computed by every rank on its band of output rows (rk_shard_product) and the bands are then
// all-gathered; the diagonal leaves are closed redundantly on every rank (rk_shard_leaf), so all
// replicas stay bit-identical to the single-GPU aligned R-Kleene.
size_t rk_shard_scratch_bytes(int64_t N, int thr) {
  const int64_t h = rk_half(N, 1);
  const int64_t leaf = std::max<int64_t>(round_up(std::min<int64_t>(thr, N), TILE_ALIGN), TILE_ALIGN);
  return 256 + prep_bytes(h, h, h) + 512 + fw_scratch_bytes(leaf, TILE_ALIGN, 4) + 512;
}

int rk_shard_leaf_impl(int tier, void* Dv, int64_t ld, int32_t* P, int64_t ldp, int64_t lo, int64_t m, int thr,
                       void* scratch, size_t scratch_bytes, cudaStream_t s) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  if (lo % TILE_ALIGN || m % TILE_ALIGN || m <= 0) return set_error(APSP_EINVAL, "leaf blocks must be 128-aligned");
  const int64_t N = ld;
  if (scratch_bytes < rk_shard_scratch_bytes(N, thr)) return set_error(APSP_EINVAL, "rk shard scratch too small");
  Status* st = static_cast<Status*>(scratch);
  char* leafws = static_cast<char*>(scratch) + 256 + ((prep_bytes(rk_half(N, 1), rk_half(N, 1), rk_half(N, 1)) + 511) / 256) * 256;
  char* D = static_cast<char*>(Dv);
  const size_t es = store_elem_size(store);
  int launches = 0;
  if (m > TILE_ALIGN)
    return fw_blocked_view(store, D + (lo * ld + lo) * es, ld, P + lo * ldp + lo, ldp, m, DEFAULT_BLOCK, IDX_PRED, lo,
                           st, s, &launches, nullptr, leafws, getenv("APSP_NO_LOOKAHEAD") ? nullptr : side_stream());
  return launch_block_close(store, D, ld, lo, m, P, ldp, IDX_PRED, lo, st, s);
}

int rk_shard_product_impl(int tier, const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                          int32_t* idx, int64_t ldi, const int32_t* predB, int64_t ldpb, int64_t m, int64_t n,
                          int64_t k, int64_t inner_off, int64_t N, int thr, void* scratch, size_t scratch_bytes,
                          cudaStream_t s, int npeers, const int64_t* peer_dc,
                          const int64_t* peer_di) {
  const int store = tier_store(tier);
  if (store < 0) return set_error(APSP_EINVAL, "unknown tier %d", tier);
  if (m <= 0 || n <= 0 || k <= 0) return 0;
  if (scratch_bytes < rk_shard_scratch_bytes(N, thr)) return set_error(APSP_EINVAL, "rk shard scratch too small");
  char* prep = static_cast<char*>(scratch) + 256;
  MinplusArgs a = minplus_args();
  a.A = A; a.lda = lda; a.B = B; a.ldb = ldb;
  a.C = C; a.ldc = ldc;
  a.idx = idx; a.ldi = ldi;
  a.predB = predB; a.ldp = ldpb;
  a.m = m; a.n = n; a.k = k;
  a.inner_off = inner_off;
  a.mode = IDX_PRED;
  a.status = static_cast<Status*>(scratch);
  if (npeers < 0 || npeers > MAX_PEERS) return set_error(APSP_EINVAL, "npeers %d outside [0, %d]", npeers, MAX_PEERS);
  a.npeers = npeers;
  for (int r = 0; r < npeers; r++) {
    a.peer_dC[r] = peer_dc[r];
    a.peer_dI[r] = peer_di[r];
  }
  if (bulk_store(store, k) && m % TILE_ALIGN == 0 && n % TILE_ALIGN == 0 && k % 32 == 0) {   // as RK::mp
    int rc = launch_prep_bulk(store, A, lda, B, ldb, m, n, k, prep_a(prep), prep_b(prep, m, k), s);
    if (rc) return rc;
    a.Aprep = prep_a(prep);
    a.Bprep = prep_b(prep, m, k);
  }
  return timed_minplus(store, a, s);
}


}  // namespace apsp
