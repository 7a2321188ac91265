#include <type_traits>
// Small-n blocked Floyd-Warshall in ONE persistent launch (u8 tier), included by fw.cu.
//
// For N <= a few thousand the launch-based schedule is bound by its per-round chain -- closure
// (one CTA) -> panel layouts -> panels -> layouts -> the next pivot's cross -- each a separate
// launch of a few dozen CTAs (n=1024: ~85 us per round, 8 rounds). Here one CTA per SM pulls
// tasks from a static dataflow order and waits only for the tiles it reads:
//
//   C(K)    close the diagonal tile (K,K)                    (the DPX closure body, fw.cu)
//   R(K,J)  row panel    D_KJ <- min(D_KJ, D_KK (x) D_KJ)    J != K
//   L(I,K)  column panel D_IK <- min(D_IK, D_IK (x) D_KK)    I != K
//   U(K,I,J) D_IJ <- min(D_IJ, D_IK (x) D_KJ)                I, J != K
//
// done[I][J] counts the rounds a tile has completed. A task of round K waits until its operand
// tiles reached K+1 (panels) and its own tile reached K, then publishes K+1 (release after a CTA
// barrier; acquire spin by one thread; all tile data is read through L2, ld.global.cg / cp.async.cg,
// so no SM reads a stale L1 line). The claim order
//     C(0) P(0) A(0) | C(1) P(1) B'(0) A(1) B''(0) | C(2) P(2) B'(1) A(2) B''(1) | ... | B(nb-1)
// (P = the panels, A(K) = the round-K updates of the tiles in the cross of K+1, B(K) = the rest,
// split into B'(K), its tiles in the cross of K+2, and B''(K), the others)
// is the lookahead schedule, and every dependency of a task is claimed before it. Tasks are
// claimed only by CTAs that are running (an atomic counter), and a running CTA finishes its task,
// so by induction over the claim order every spin-wait ends -- whether or not every CTA of the
// grid is resident (the grid is sized to the SMs / occupancy only to use them all).
//
// Tile tasks use 512 threads on a 128 x 128 tile (4 rows x 8 columns each), k = 128 in four
// 32-k chunks staged through registers into shared memory as packed 16-bit keys
// (v << 7 | tag, tags 1..96 per 3-chunk window) and relaxed with VIADDMNMX.U16x2, the same
// arithmetic and argmin semantics as minplus_nt_kernel: strict improvement, smallest k, pred
// gathered from the B rows' pred for improved cells only. The row-panel task reads its own tile
// as B and its pred rows, so every gather of a task completes before any of its stores (barrier).

// APSP_PERSIST_TRACE: summed globaltimer ns of the 64-wide closure's phases (load, k loop, pred
// resolution, stores) over all closure tasks, printed with the trace
__device__ unsigned long long g_close64_phase[5];

namespace persist {

constexpr int PT = 512;            // threads
constexpr int PB = 128;            // tile
constexpr uint32_t KINF2 = (uint32_t(U8_INF) << 7) * 0x00010001u;
constexpr uint32_t TMASK2 = 0x007F007Fu;
// T_UCLOSE(K): round K-1's update of the diagonal tile (K,K) fused into its closure -- one task
// hop fewer on the per-round chain (closure -> panel -> cross tile -> closure)
enum Task : int { T_CLOSE = 0, T_ROW = 1, T_COL = 2, T_UPD = 3, T_UCLOSE = 4 };

struct TileSmem {
  uint32_t As[2][SUB][PB];   // replicated key pairs (v << 7 in both halves), by k then row
  uint16_t Bs[2][SUB][PB];   // tagged keys, by k then column
};
union Smem {
  TileSmem tile;
  CloseU8Smem close;
};

__device__ __forceinline__ int acquire_ld(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void release_st(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_at_least(const int* p, int v) {
  while (acquire_ld(p) < v) __nanosleep(64);
}

// chunk c (k in [32c, 32c + 32)) of A (rows of the tile, 128 x 32 bytes) and B (32 x 128 bytes):
// 8 bytes of each per thread, through L2
__device__ __forceinline__ void load_chunk(const uint8_t* A, int64_t lda, const uint8_t* B, int64_t ldb, int c,
                                           uint2& ra, uint2& rb) {
  const int t = threadIdx.x;
  ra = __ldcg(reinterpret_cast<const uint2*>(A + int64_t(t >> 2) * lda + SUB * c + 8 * (t & 3)));
  rb = __ldcg(reinterpret_cast<const uint2*>(B + int64_t(SUB * c + (t >> 4)) * ldb + 8 * (t & 15)));
}

__device__ __forceinline__ void store_chunk(TileSmem& sm, int buf, const uint2& ra, const uint2& rb, int tagbase) {
  const int t = threadIdx.x;
  {
    const int r = t >> 2, kb = 8 * (t & 3);
    const uint32_t w[2] = {ra.x, ra.y};
#pragma unroll
    for (int q = 0; q < 8; q++) sm.As[buf][kb + q][r] = ((w[q >> 2] >> (8 * (q & 3))) & 0xFFu) * 0x00800080u;
  }
  {
    const int kk = t >> 4, cb = 8 * (t & 15);
    const uint32_t tag = uint32_t(tagbase + kk + 1) * 0x00010001u;
    const uint32_t w[2] = {rb.x, rb.y};
    uint32_t o[4];
#pragma unroll
    for (int q = 0; q < 2; q++) {
      o[2 * q] = (__byte_perm(w[q], 0, 0x4140) << 7) | tag;
      o[2 * q + 1] = (__byte_perm(w[q], 0, 0x4342) << 7) | tag;
    }
    *reinterpret_cast<uint4*>(&sm.Bs[buf][kk][cb]) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// C <- min(C, A (x) B) on one 128 x 128 tile, k = 128; pred[i][j] <- predB[k*][j] on strict
// improvement. Thread t: rows 4*(t>>4) + r, columns 4*(t&15) + {0..3} and 64 + 4*(t&15) + {0..3}.
__device__ void tile_task(TileSmem& sm, uint8_t* C, int64_t ldc, const uint8_t* A, int64_t lda, const uint8_t* B,
                          int64_t ldb, int32_t* P, int64_t ldp, const int32_t* PB_, int64_t ldpb) {
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  uint32_t acc[4][4], kst[4][4];
  // the old values, untagged keys (they win ties: strict improvement)
#pragma unroll
  for (int r = 0; r < 4; r++) {
    const uint8_t* row = C + int64_t(4 * ty + r) * ldc;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const uint32_t w = __ldcg(reinterpret_cast<const unsigned int*>(row + 64 * h + 4 * tx));
      acc[r][2 * h] = __byte_perm(w, 0, 0x4140) << 7;
      acc[r][2 * h + 1] = __byte_perm(w, 0, 0x4342) << 7;
      kst[r][2 * h] = kst[r][2 * h + 1] = 0u;
    }
  }
  uint2 ra, rb;
  load_chunk(A, lda, B, ldb, 0, ra, rb);
  store_chunk(sm, 0, ra, rb, 0);
  __syncthreads();
#pragma unroll 1
  for (int c = 0; c < 4; c++) {
    const int buf = c & 1;
    if (c < 3) load_chunk(A, lda, B, ldb, c + 1, ra, rb);
#pragma unroll 8
    for (int kk = 0; kk < SUB; kk++) {
      const uint4 a = *reinterpret_cast<const uint4*>(&sm.As[buf][kk][4 * ty]);
      const uint2 b0 = *reinterpret_cast<const uint2*>(&sm.Bs[buf][kk][4 * tx]);
      const uint2 b1 = *reinterpret_cast<const uint2*>(&sm.Bs[buf][kk][64 + 4 * tx]);
      const uint32_t av[4] = {a.x, a.y, a.z, a.w};
      const uint32_t bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) acc[r][q] = __viaddmin_u16x2(av[r], bv[q], acc[r][q]);
    }
    if (c == 2 || c == 3) {   // close a tag window: chunks 0-2 (tags 1..96), then chunk 3 (1..32)
      const uint32_t kb2 = uint32_t(c == 2 ? 0 : 3 * SUB) * 0x00010001u;
#pragma unroll
      for (int r = 0; r < 4; r++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const uint32_t tg = acc[r][q] & TMASK2;
          const uint32_t mask = prmt_sign_halves(tg + 0x7FFF7FFFu);
          kst[r][q] = (kst[r][q] & ~mask) | ((tg + kb2) & mask);
          acc[r][q] -= tg;
        }
    }
    if (c < 3) store_chunk(sm, buf ^ 1, ra, rb, c == 2 ? 0 : (c + 1) * SUB);
    __syncthreads();
  }
  // every gather before any store: the row-panel task's B rows / pred rows are its own tile
  int32_t pv[4][8];
#pragma unroll
  for (int r = 0; r < 4; r++)
#pragma unroll
    for (int q = 0; q < 4; q++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t k1 = (kst[r][q] >> (16 * h)) & 0xFFFFu;
        const int j = (q < 2 ? 0 : 64) + 4 * tx + 2 * (q & 1) + h;
        pv[r][2 * q + h] = (P && k1) ? __ldcg(PB_ + int64_t(k1 - 1) * ldpb + j) : 0;
      }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; r++) {
    uint8_t* row = C + int64_t(4 * ty + r) * ldc;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if ((kst[r][2 * h] | kst[r][2 * h + 1]) == 0u) continue;
      *reinterpret_cast<uint32_t*>(row + 64 * h + 4 * tx) =
          __byte_perm(acc[r][2 * h] >> 7, acc[r][2 * h + 1] >> 7, 0x6420);
      if (!P) continue;
      int32_t* prow = P + int64_t(4 * ty + r) * ldp + 64 * h + 4 * tx;
#pragma unroll
      for (int q = 0; q < 2; q++)
#pragma unroll
        for (int hh = 0; hh < 2; hh++)
          if ((kst[r][2 * h + q] >> (16 * hh)) & 0xFFFFu) prow[2 * q + hh] = pv[r][4 * h + 2 * q + hh];
    }
  }
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}

__global__ void __launch_bounds__(PT, 1) fw_persist_kernel(uint8_t* D, int64_t ld, int32_t* P, int64_t ldp, int nb,
                                                           const int4* items, int nitems, int* done, int* counter,
                                                           unsigned long long* trace) {
  extern __shared__ __align__(16) unsigned char smraw_persist[];
  Smem& sm = *reinterpret_cast<Smem*>(smraw_persist);
  __shared__ int s_item;
  const int t = threadIdx.x;
  for (;;) {
    if (t == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) break;
    const int4 w = items[it];   // (task, K, I, J)
    const int K = w.y, I = w.z, J = w.w;
    unsigned long long t_claim = 0, t_ready = 0;
    if (trace && t == 0) t_claim = gtimer();
    if (t == 0) {
      if (w.x == T_CLOSE) {
        wait_at_least(&done[K * nb + K], K);
      } else if (w.x == T_UCLOSE) {
        wait_at_least(&done[K * nb + K - 1], K);
        wait_at_least(&done[(K - 1) * nb + K], K);
        wait_at_least(&done[K * nb + K], K - 1);
      } else if (w.x == T_ROW) {
        wait_at_least(&done[K * nb + K], K + 1);
        wait_at_least(&done[K * nb + J], K);
      } else if (w.x == T_COL) {
        wait_at_least(&done[K * nb + K], K + 1);
        wait_at_least(&done[I * nb + K], K);
      } else {
        wait_at_least(&done[I * nb + K], K + 1);
        wait_at_least(&done[K * nb + J], K + 1);
        wait_at_least(&done[I * nb + J], K);
      }
    }
    __syncthreads();
    if (trace && t == 0) t_ready = gtimer();
    const int64_t k0 = int64_t(K) * PB;
    if (w.x == T_CLOSE || w.x == T_UCLOSE) {
      if (w.x == T_UCLOSE) {   // round K-1 on the tile first (pivot block K-1)
        const int64_t kp = k0 - PB;
        tile_task(sm.tile, D + k0 * ld + k0, ld, D + k0 * ld + kp, ld, D + kp * ld + k0, ld,
                  P ? P + k0 * ldp + k0 : nullptr, ldp, P ? P + kp * ldp + k0 : nullptr, ldp);
        __syncthreads();
      }
      close_dpx_body<STORE_U8, true>(D, ld, k0, PB, P, ldp, IDX_PRED, k0,
                                     reinterpret_cast<unsigned char*>(&sm.close));
    } else {
      const int64_t i0 = int64_t(w.x == T_ROW ? K : I) * PB, j0 = int64_t(w.x == T_COL ? K : J) * PB;
      tile_task(sm.tile, D + i0 * ld + j0, ld, D + i0 * ld + k0, ld, D + k0 * ld + j0, ld, P ? P + i0 * ldp + j0 : nullptr,
                ldp, P ? P + k0 * ldp + j0 : nullptr, ldp);
    }
    __syncthreads();   // the task's stores precede the release
    if (t == 0) {
      __threadfence();
      const int ti = (w.x == T_CLOSE || w.x == T_UCLOSE || w.x == T_ROW) ? K : I;
      const int tj = (w.x == T_CLOSE || w.x == T_UCLOSE || w.x == T_COL) ? K : J;
      release_st(&done[ti * nb + tj], K + 1);
      if (trace) {   // APSP_PERSIST_TRACE: claim / dependencies met / done (globaltimer ns), SM
        unsigned int smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        trace[4 * it] = t_claim;
        trace[4 * it + 1] = t_ready;
        trace[4 * it + 2] = gtimer();
        trace[4 * it + 3] = smid;
      }
    }
  }
}

}  // namespace persist

// The claim order of the persistent schedule (see above), built once per (device, block count).
static const int4* persist_items(int nb, int* nitems, bool fuse_diag) {
  struct Entry { int dev, nb, fuse, n; int4* d; };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.dev == dev && e.nb == nb && e.fuse == int(fuse_diag)) {
      *nitems = e.n;
      return e.d;
    }
  std::vector<int4> v;
  // round-K updates inside (part 0) / outside (part 1) the cross of K+1; part 1 optionally only
  // the tiles in (sel = 1) or outside (sel = 2) the cross of K+2, so the rest of round K-1 that
  // the next cross needs is claimed before that cross, and the remainder after it
  auto updates = [&](int K, bool next_cross, int sel = 0) {
    for (int I = 0; I < nb; I++)
      for (int J = 0; J < nb; J++) {
        if (I == K || J == K) continue;
        const bool nx = K + 1 < nb && (I == K + 1 || J == K + 1);
        if (nx != next_cross) continue;
        const bool nx2 = K + 2 < nb && (I == K + 2 || J == K + 2);
        if ((sel == 1 && !nx2) || (sel == 2 && nx2)) continue;
        if (fuse_diag && I == K + 1 && J == K + 1) continue;   // fused into T_UCLOSE(K+1)
        v.push_back(make_int4(persist::T_UPD, K, I, J));
      }
  };
  auto close_and_panels = [&](int K) {
    v.push_back(make_int4(K && fuse_diag ? persist::T_UCLOSE : persist::T_CLOSE, K, K, K));
    for (int q = 1; q < nb; q++) {   // the next pivot's panel tiles first
      const int X = (K + q) % nb;
      v.push_back(make_int4(persist::T_ROW, K, K, X));
      v.push_back(make_int4(persist::T_COL, K, X, K));
    }
  };
  close_and_panels(0);
  updates(0, true);
  for (int K = 1; K < nb; K++) {
    close_and_panels(K);
    updates(K - 1, false, 1);   // round K-1 tiles of the cross of K+1 (needed by A(K))
    updates(K, true);           // A(K): round K on the cross of K+1 (needed by the next closure)
    updates(K - 1, false, 2);   // the rest of round K-1
  }
  updates(nb - 1, false);
  int4* d = nullptr;
  if (cudaMalloc(&d, v.size() * sizeof(int4)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, v.data(), v.size() * sizeof(int4), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  cache.push_back({dev, nb, int(fuse_diag), int(v.size()), d});
  *nitems = int(v.size());
  return d;
}

static int persist_dump_trace(unsigned long long* trace, const int4* items, int nitems, cudaStream_t s);

size_t fw_persist_scratch_bytes(int64_t N) {
  const int64_t nb = N / TILE_ALIGN;
  return size_t(nb * nb + 64) * sizeof(int);
}

// Up to 2560: beyond it the launch-based device-signalled chain (fw_sched.cu) is faster
// (n=2816: 1.79 vs 1.71 ms, 3072: 2.17 vs 1.87 ms).
bool fw_persist_enabled(int store, int64_t N) {
  static const int64_t max_n = getenv("APSP_PERSIST_MAX_N") ? atoll(getenv("APSP_PERSIST_MAX_N")) : 2560;
  return store == STORE_U8 && N % TILE_ALIGN == 0 && N <= max_n && N >= TILE_ALIGN;
}

// co-resident CTAs of a persistent kernel on the current device (SMs x CTAs per SM), cached per
// (device, kernel): the occupancy query is not free on a small-n call path
template <typename K>
static cudaError_t persist_slots(K kernel, int threads, int smem, int& slots) {
  struct Entry { int dev; const void* fn; int slots; };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const void* fn = reinterpret_cast<const void*>(kernel);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry& c : cache)
      if (c.dev == dev && c.fn == fn) {
        slots = c.slots;
        return cudaSuccess;
      }
  }
  int sms = 0, per_sm = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (e != cudaSuccess) return e;
  slots = sms * per_sm;
  std::lock_guard<std::mutex> lock(mu);
  cache.push_back({dev, fn, slots});
  return cudaSuccess;
}

// One persistent launch for the whole u8 blocked FW of an N x N view (N a multiple of 128).
int launch_fw_persist(uint8_t* D, int64_t ld, int32_t* P, int64_t ldp, int64_t N, void* scratch, cudaStream_t s) {
  const int nb = int(N / TILE_ALIGN);
  int nitems = 0;
  // (the 128-wide closure is long: fusing the diagonal update into it measured slower at n=3072)
  const int4* items = persist_items(nb, &nitems, false);
  if (!items) return set_error(APSP_ECUDA, "persistent schedule table allocation failed");
  int* done = static_cast<int*>(scratch);
  int* counter = done + nb * nb;
  APSP_CUDA_TRY(cudaMemsetAsync(scratch, 0, fw_persist_scratch_bytes(N), s));
  static std::atomic<unsigned long long> attr{0};
  const int sb = int(sizeof(persist::Smem));
  APSP_CUDA_TRY(smem_optin(persist::fw_persist_kernel, sb, attr));
  int sms = 0;
  APSP_CUDA_TRY(persist_slots(persist::fw_persist_kernel, persist::PT, sb, sms));
  const int grid = std::min(sms, nitems);
  unsigned long long* trace = nullptr;
  if (getenv("APSP_PERSIST_TRACE")) APSP_CUDA_TRY(cudaMalloc(&trace, size_t(nitems) * 4 * sizeof(unsigned long long)));
  persist::fw_persist_kernel<<<grid, persist::PT, sb, s>>>(D, ld, P, ldp, nb, items, nitems, done, counter, trace);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return persist_dump_trace(trace, items, nitems, s);
}

// APSP_PERSIST_TRACE=file: per task (kind, K, I, J, claim, ready, done ns, SM) as CSV, for the
// schedule's critical path (tools/persist_trace.py)
static int persist_dump_trace(unsigned long long* trace, const int4* items, int nitems, cudaStream_t s) {
  const char* tpath = getenv("APSP_PERSIST_TRACE");
  if (trace) {
    std::vector<unsigned long long> h(size_t(nitems) * 4);
    std::vector<int4> it(nitems);
    APSP_CUDA_TRY(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
    APSP_CUDA_TRY(cudaMemcpyAsync(it.data(), items, it.size() * sizeof(int4), cudaMemcpyDeviceToHost, s));
    APSP_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(trace);
    if (FILE* f = fopen(tpath, "w")) {
      unsigned long long ph[5] = {};
      if (cudaMemcpyFromSymbol(ph, g_close64_phase, sizeof(ph)) == cudaSuccess && ph[4])
        fprintf(stderr, "[persist64] close64 phases (mean ns over %llu): load %llu, k loop %llu, pred %llu, store %llu\n",
                ph[4], ph[0] / ph[4], ph[1] / ph[4], ph[2] / ph[4], ph[3] / ph[4]);
      fprintf(f, "kind,K,I,J,claim,ready,done,sm\n");
      for (int i = 0; i < nitems; i++)
        fprintf(f, "%d,%d,%d,%d,%llu,%llu,%llu,%llu\n", it[i].x, it[i].y, it[i].z, it[i].w, h[4 * i], h[4 * i + 1],
                h[4 * i + 2], h[4 * i + 3]);
      fclose(f);
    }
  }
  return 0;
}

// ------------------------------------------------------------------------------------------
// 64-wide pivot blocks (N <= APSP_PERSIST64_MAX_N): the per-round chain is what bounds small n,
// and a 64 x 64 closure is ~8x cheaper than a 128 x 128 one (64 steps over 4096 cells instead
// of 128 over 16384), so halving b halves the chain even though the rounds double. Same
// dataflow schedule and semantics as above with 64 x 64 tiles: 256-thread CTAs, several per SM
// (grid = occupancy x SMs), k = 64 per task in one shot (tags 1..64, one decode).
// ------------------------------------------------------------------------------------------
namespace persist64 {

constexpr int QT = 256;   // threads
constexpr int QB = 64;    // tile / pivot block

// Key formats: u8 values << 7 with one 64-k tag window per task; u16 values (<= 510) << 6 with
// two 32-k windows (INF + INF + tag < 2^16 in both), decoded after k = 31.
template <int S> struct K64;
template <> struct K64<STORE_U8> {
  using T = uint8_t;
  static constexpr int TAG = 7, WIN = 64;
};
template <> struct K64<STORE_U16> {
  using T = uint16_t;
  static constexpr int TAG = 6, WIN = 32;
};
// w32: unsigned 32-bit keys v << 7 | tag, one per cell, one 64-k window (INF + INF + tag < 2^32)
template <> struct K64<STORE_W32> {
  using T = int32_t;
  static constexpr int TAG = 7, WIN = 64;
};
template <int S> __device__ __forceinline__ constexpr uint32_t tmask2() {
  return ((1u << K64<S>::TAG) - 1u) * 0x00010001u;
}
// 8 consecutive cells (16-byte aligned for u16, 8 for u8) as 4 key pairs
template <int S>
__device__ __forceinline__ void load_pairs(const typename K64<S>::T* src, uint32_t (&a)[4]) {
  constexpr int TAG = K64<S>::TAG;
  if constexpr (S == STORE_U8) {
    const uint2 v = __ldcg(reinterpret_cast<const uint2*>(src));
    a[0] = __byte_perm(v.x, 0, 0x4140) << TAG;
    a[1] = __byte_perm(v.x, 0, 0x4342) << TAG;
    a[2] = __byte_perm(v.y, 0, 0x4140) << TAG;
    a[3] = __byte_perm(v.y, 0, 0x4342) << TAG;
  } else {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src));
    a[0] = v.x << TAG;
    a[1] = v.y << TAG;
    a[2] = v.z << TAG;
    a[3] = v.w << TAG;
  }
}
// 4 tag-free key pairs back as 8 cells
template <int S>
__device__ __forceinline__ void store_pairs(typename K64<S>::T* dst, const uint32_t (&a)[4]) {
  constexpr int TAG = K64<S>::TAG;
  if constexpr (S == STORE_U8) {
    *reinterpret_cast<uint2*>(dst) = make_uint2(__byte_perm(a[0] >> TAG, a[1] >> TAG, 0x6420),
                                                __byte_perm(a[2] >> TAG, a[3] >> TAG, 0x6420));
  } else {
    *reinterpret_cast<uint4*>(dst) = make_uint4(a[0] >> TAG, a[1] >> TAG, a[2] >> TAG, a[3] >> TAG);
  }
}
// close a tag window: the last improving k (1-based, window base wb) of each half into kst
__device__ __forceinline__ void decode_pair(uint32_t& acc, uint32_t& kst, uint32_t tmask, uint32_t wb) {
  const uint32_t tg = acc & tmask;
  acc -= tg;
  if (tg & 0xFFFFu) kst = (kst & 0xFFFF0000u) | ((tg & 0xFFFFu) + wb);
  if (tg >> 16) kst = (kst & 0x0000FFFFu) | (((tg >> 16) + wb) << 16);
}

struct TileSmem {
  uint32_t As[QB][QB];    // [k][row] replicated key pairs
  uint16_t Bs[QB][QB];    // [k][col] tagged keys
  int32_t Pb[QB][QB];     // pred rows of B (cp.async during the k loop: the gathers hit smem)
};
struct CloseSmem {
  uint32_t colk[2][QB];   // column k as replicated tag-free keys, by row
  uint32_t colk1[2][QB];  // column k+1 likewise (two steps per barrier)
  int32_t P[QB][QB];      // pred resolution
  uint8_t K[QB][QB];      // 1-based last improving k (0 = none)
};
union Smem {
  TileSmem tile;
  CloseSmem close;
};
struct TileSmemW {        // w32 tile task: 32-bit keys for both operands
  uint32_t As[QB][QB];    // [k][row]
  uint32_t Bs[QB][QB];    // [k][col] tagged
  int32_t Pb[QB][QB];
};
union SmemW {
  TileSmemW tile;
  CloseSmem close;
};

// 64 x 64 closure in classic k order (values, pred bit-exact with the classic in-block loop).
// Warp w owns columns 8w..8w+7 (4 key pairs), lane l rows 2l, 2l+1: row k comes by shuffle from
// lane k/2 of the same warp, column k from its owner warp through shared memory (double
// buffered, one barrier per step). The last improving k rides in the 7-bit tag (k + 1 <= 64).
template <int S>
__device__ void close64(CloseSmem& sm, typename K64<S>::T* D, int64_t ld, int32_t* P, int64_t ldp, bool prof) {
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  unsigned long long tp0 = prof && t == 0 ? persist::gtimer() : 0, tp1 = 0, tp2 = 0, tp3 = 0;
  constexpr uint32_t TMASK2 = tmask2<S>(), STRIP2 = ~TMASK2;
  constexpr int WIN = K64<S>::WIN;
  uint32_t acc[2][4];
  uint32_t kst[2][4] = {};
#pragma unroll
  for (int r = 0; r < 2; r++) load_pairs<S>(D + int64_t(2 * l + r) * ld + 8 * w, acc[r]);
  if (P) {   // the input pred block, for the resolution after the k loop: in flight meanwhile
    for (int e = t; e < QB * QB / 4; e += QT) {
      const int i = e >> 4, j = 4 * (e & 15);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.P[i][j])),
                   "l"(P + int64_t(i) * ldp + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // Two steps per barrier: columns k and k+1 (k even) are one key pair of one warp, published
  // together as two replicated tag-free columns; every warp advances column k+1 through step k
  // itself, D[i][k+1] <- min(D[i][k+1], D[i][k] + D[k][k+1]), then runs steps k and k+1 back to
  // back (row k+1 comes from its owner lane after that lane's own step-k update). Each cell is
  // still updated by its owner in k order, so values and tags are those of the one-step loop.
#define P64_PUBPAIR(PP, BUF)                                                                \
  do {                                                                                      \
    *reinterpret_cast<uint2*>(&sm.colk[BUF][2 * l]) =                                       \
        make_uint2(__byte_perm(acc[0][PP], 0, 0x1010) & STRIP2, __byte_perm(acc[1][PP], 0, 0x1010) & STRIP2); \
    *reinterpret_cast<uint2*>(&sm.colk1[BUF][2 * l]) =                                      \
        make_uint2(__byte_perm(acc[0][PP], 0, 0x3232) & STRIP2, __byte_perm(acc[1][PP], 0, 0x3232) & STRIP2); \
  } while (0)
  if (w == 0) P64_PUBPAIR(0, 0);
  if (prof) {
    __syncthreads();
    if (t == 0) tp1 = persist::gtimer();
  }
#pragma unroll 1
  for (int k0 = 0; k0 < QB; k0 += 8) {
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      const int k = k0 + kk, buf = (kk >> 1) & 1;
      __syncthreads();
      const uint2 c2 = *reinterpret_cast<const uint2*>(&sm.colk[buf][2 * l]);
      const uint2 c3 = *reinterpret_cast<const uint2*>(&sm.colk1[buf][2 * l]);
      const uint32_t dkk1 = sm.colk1[buf][k];   // D[k][k+1], replicated
      const uint32_t ck1x = __viaddmin_u16x2(c2.x, dkk1, c3.x), ck1y = __viaddmin_u16x2(c2.y, dkk1, c3.y);
      uint32_t dkj[4];
      const uint32_t tag2 = uint32_t(k % WIN + 1) * 0x00010001u;
#pragma unroll
      for (int p = 0; p < 4; p++) dkj[p] = (__shfl_sync(0xffffffffu, acc[0][p], k >> 1) & STRIP2) | tag2;
#pragma unroll
      for (int p = 0; p < 4; p++) {
        acc[0][p] = __viaddmin_u16x2(c2.x, dkj[p], acc[0][p]);
        acc[1][p] = __viaddmin_u16x2(c2.y, dkj[p], acc[1][p]);
      }
#pragma unroll
      for (int p = 0; p < 4; p++) dkj[p] = (__shfl_sync(0xffffffffu, acc[1][p], (k + 1) >> 1) & STRIP2) | (tag2 + 0x00010001u);
#pragma unroll
      for (int p = 0; p < 4; p++) {
        acc[0][p] = __viaddmin_u16x2(ck1x, dkj[p], acc[0][p]);
        acc[1][p] = __viaddmin_u16x2(ck1y, dkj[p], acc[1][p]);
      }
      if (WIN < QB && k + 2 == WIN) {   // u16: the first 32-k window closes after step k + 1
#pragma unroll
        for (int r = 0; r < 2; r++)
#pragma unroll
          for (int p = 0; p < 4; p++) decode_pair(acc[r][p], kst[r][p], TMASK2, 0u);
      }
      // the next pair (k+2, k+3): pair ((kk+2) & 7) >> 1 of warp (k+2) >> 3
      if (k + 2 < QB) {
        if (kk == 6) {
          if (w == (k0 >> 3) + 1) P64_PUBPAIR(0, buf ^ 1);
        } else if (w == (k0 >> 3)) {
          P64_PUBPAIR(((kk + 2) & 7) >> 1, buf ^ 1);
        }
      }
    }
  }
#undef P64_PUBPAIR
  __syncthreads();   // every warp is past its last read of colk
  if (prof && t == 0) tp2 = persist::gtimer();
  // the (last) window: its tag is k* + 1 - base (0 = no improvement in it)
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int p = 0; p < 4; p++) decode_pair(acc[r][p], kst[r][p], TMASK2, uint32_t(QB - WIN));
  // values back (improved pairs only change; writing all is simpler and equally final)
#pragma unroll
  for (int r = 0; r < 2; r++) store_pairs<S>(D + int64_t(2 * l + r) * ld + 8 * w, acc[r]);
  if (!P) return;
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int p = 0; p < 4; p++) {
      sm.K[2 * l + r][8 * w + 2 * p] = uint8_t(kst[r][p] & 0xFFu);
      sm.K[2 * l + r][8 * w + 2 * p + 1] = uint8_t(kst[r][p] >> 16);
    }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // pred[i][j] = pred_final[k*][j]: pointer jumping (chains strictly shorten: < 64 = 2^6 hops)
  for (int round = 0; round < 6; round++) {
    int32_t np[16];
    uint8_t nk[16];
    bool live = false;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int e = t + QT * c, i = e >> 6, j = e & 63;
      const uint8_t kk = sm.K[i][j];
      np[c] = sm.P[i][j];
      nk[c] = kk;
      if (kk) {
        np[c] = sm.P[kk - 1][j];
        nk[c] = sm.K[kk - 1][j];
        live |= nk[c] != 0;
      }
    }
    const bool more = __syncthreads_or(live);
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int e = t + QT * c, i = e >> 6, j = e & 63;
      sm.P[i][j] = np[c];
      sm.K[i][j] = nk[c];
    }
    __syncthreads();
    if (!more) break;
  }
  if (prof && t == 0) tp3 = persist::gtimer();
  for (int e = t; e < QB * QB / 4; e += QT) {
    const int i = e >> 4, j = 4 * (e & 15);
    *reinterpret_cast<int4*>(P + int64_t(i) * ldp + j) = *reinterpret_cast<const int4*>(&sm.P[i][j]);
  }
  if (prof && t == 0) {
    const unsigned long long tp4 = persist::gtimer();
    atomicAdd(&g_close64_phase[0], tp1 - tp0);
    atomicAdd(&g_close64_phase[1], tp2 - tp1);
    atomicAdd(&g_close64_phase[2], tp3 - tp2);
    atomicAdd(&g_close64_phase[3], tp4 - tp3);
    atomicAdd(&g_close64_phase[4], 1ull);
  }
}

// C <- min(C, A (x) B) on a 64 x 64 tile, k = 64. Thread t: rows 2*(t>>3) + {0,1}, columns
// 8*(t&7) .. + 7 (4 key pairs).
template <int S>
__device__ void tile64(TileSmem& sm, typename K64<S>::T* C, int64_t ldc, const typename K64<S>::T* A, int64_t lda,
                       const typename K64<S>::T* B, int64_t ldb, int32_t* P, int64_t ldp, const int32_t* PB_,
                       int64_t ldpb) {
  using T = typename K64<S>::T;
  constexpr int TAG = K64<S>::TAG, WIN = K64<S>::WIN;
  constexpr uint32_t TMASK2 = tmask2<S>();
  const int t = threadIdx.x, ty = t >> 3, tx = t & 7;
  if (P) {   // B's pred rows, in flight while the tile computes (L2 only: cp.async.cg)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int e = t + QT * q, i = e >> 4, j = 4 * (e & 15);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.Pb[i][j])),
                   "l"(PB_ + int64_t(i) * ldpb + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  {  // stage A (64 rows x 64 k) and B (64 k x 64 cols): 16 values of each per thread
    const int ra = t >> 2, ka = 16 * (t & 3);
    T va[16];
    reinterpret_cast<uint4*>(va)[0] = __ldcg(reinterpret_cast<const uint4*>(A + int64_t(ra) * lda + ka));
    if constexpr (sizeof(T) == 2)
      reinterpret_cast<uint4*>(va)[1] = __ldcg(reinterpret_cast<const uint4*>(A + int64_t(ra) * lda + ka) + 1);
#pragma unroll
    for (int q = 0; q < 16; q++) sm.As[ka + q][ra] = (uint32_t(va[q]) << TAG) * 0x00010001u;
    const int kb = t >> 2, cb = 16 * (t & 3);
    T vb[16];
    reinterpret_cast<uint4*>(vb)[0] = __ldcg(reinterpret_cast<const uint4*>(B + int64_t(kb) * ldb + cb));
    if constexpr (sizeof(T) == 2)
      reinterpret_cast<uint4*>(vb)[1] = __ldcg(reinterpret_cast<const uint4*>(B + int64_t(kb) * ldb + cb) + 1);
    const uint32_t tag = uint32_t(kb % WIN + 1);
    uint32_t o[8];
#pragma unroll
    for (int q = 0; q < 8; q++)
      o[q] = ((uint32_t(vb[2 * q]) << TAG) | tag) | (((uint32_t(vb[2 * q + 1]) << TAG) | tag) << 16);
    uint4* dst = reinterpret_cast<uint4*>(&sm.Bs[kb][cb]);
    dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
    dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
  uint32_t acc[2][4];
#pragma unroll
  for (int r = 0; r < 2; r++) load_pairs<S>(C + int64_t(2 * ty + r) * ldc + 8 * tx, acc[r]);
  __syncthreads();
  uint32_t kst[2][4] = {};
#pragma unroll
  for (int w0 = 0; w0 < QB; w0 += WIN) {   // one tag window per WIN k
#pragma unroll 16
    for (int k = w0; k < w0 + WIN; k++) {
      const uint2 a = *reinterpret_cast<const uint2*>(&sm.As[k][2 * ty]);
      const uint4 b = *reinterpret_cast<const uint4*>(&sm.Bs[k][8 * tx]);
      const uint32_t bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int p = 0; p < 4; p++) {
        acc[0][p] = __viaddmin_u16x2(a.x, bv[p], acc[0][p]);
        acc[1][p] = __viaddmin_u16x2(a.y, bv[p], acc[1][p]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; r++)
#pragma unroll
      for (int p = 0; p < 4; p++) decode_pair(acc[r][p], kst[r][p], TMASK2, uint32_t(w0));
  }
  // the gathers read the smem snapshot of B's pred rows (taken before any store of this task,
  // so the row-panel task, whose B is its own tile, needs no barrier before its stores)
  if (P) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  int32_t pv[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const uint32_t k1 = (kst[r][p] >> (16 * h)) & 0xFFFFu;
        pv[r][2 * p + h] = (P && k1) ? sm.Pb[k1 - 1][8 * tx + 2 * p + h] : 0;
      }
#pragma unroll
  for (int r = 0; r < 2; r++) {
    if ((kst[r][0] | kst[r][1] | kst[r][2] | kst[r][3]) == 0u) continue;
    store_pairs<S>(C + int64_t(2 * ty + r) * ldc + 8 * tx, acc[r]);
    if (!P) continue;
    int32_t* prow = P + int64_t(2 * ty + r) * ldp + 8 * tx;
#pragma unroll
    for (int p = 0; p < 4; p++)
#pragma unroll
      for (int h = 0; h < 2; h++)
        if ((kst[r][p] >> (16 * h)) & 0xFFFFu) prow[2 * p + h] = pv[r][2 * p + h];
  }
}

// ---- w32 tier: one unsigned 32-bit key per cell (v << 7 | tag), VIADDMNMX.U32 ----------------
// Same thread mapping as the packed tasks: a thread owns 2 rows x 8 columns, now 16 keys.
constexpr uint32_t W_TMASK = 0x7Fu, W_STRIP = ~0x7Fu;

__device__ __forceinline__ void load8_w32(const int32_t* src, uint32_t (&a)[8]) {
  const uint4 v0 = __ldcg(reinterpret_cast<const uint4*>(src)), v1 = __ldcg(reinterpret_cast<const uint4*>(src) + 1);
  a[0] = v0.x << 7; a[1] = v0.y << 7; a[2] = v0.z << 7; a[3] = v0.w << 7;
  a[4] = v1.x << 7; a[5] = v1.y << 7; a[6] = v1.z << 7; a[7] = v1.w << 7;
}
__device__ __forceinline__ void store8_w32(int32_t* dst, const uint32_t (&a)[8]) {
  reinterpret_cast<uint4*>(dst)[0] = make_uint4(a[0] >> 7, a[1] >> 7, a[2] >> 7, a[3] >> 7);
  reinterpret_cast<uint4*>(dst)[1] = make_uint4(a[4] >> 7, a[5] >> 7, a[6] >> 7, a[7] >> 7);
}

// 64 x 64 w32 closure, classic k order, two steps per barrier (as close64): warp w owns columns
// 8w..8w+7, lane l rows 2l, 2l+1; the tag (k + 1, one window) is the last improving k.
__device__ void close64_w32(CloseSmem& sm, int32_t* D, int64_t ld, int32_t* P, int64_t ldp) {
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  uint32_t acc[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++) load8_w32(D + int64_t(2 * l + r) * ld + 8 * w, acc[r]);
  if (P) {
    for (int e = t; e < QB * QB / 4; e += QT) {
      const int i = e >> 4, j = 4 * (e & 15);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.P[i][j])),
                   "l"(P + int64_t(i) * ldp + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  // columns k, k+1 (tag-free) of the owner warp into buffer BUF
#define W64_PUB(C0, BUF)                                                                            \
  do {                                                                                              \
    *reinterpret_cast<uint2*>(&sm.colk[BUF][2 * l]) = make_uint2(acc[0][C0] & W_STRIP, acc[1][C0] & W_STRIP); \
    *reinterpret_cast<uint2*>(&sm.colk1[BUF][2 * l]) =                                              \
        make_uint2(acc[0][(C0) + 1] & W_STRIP, acc[1][(C0) + 1] & W_STRIP);                         \
  } while (0)
  if (w == 0) W64_PUB(0, 0);
#pragma unroll 1
  for (int k0 = 0; k0 < QB; k0 += 8) {
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      const int k = k0 + kk, buf = (kk >> 1) & 1;
      __syncthreads();
      const uint2 c2 = *reinterpret_cast<const uint2*>(&sm.colk[buf][2 * l]);
      const uint2 c3 = *reinterpret_cast<const uint2*>(&sm.colk1[buf][2 * l]);
      const uint32_t dkk1 = sm.colk1[buf][k];   // D[k][k+1]
      const uint32_t ck1x = min(c3.x, c2.x + dkk1), ck1y = min(c3.y, c2.y + dkk1);
      uint32_t dkj[8];
#pragma unroll
      for (int c = 0; c < 8; c++) dkj[c] = (__shfl_sync(0xffffffffu, acc[kk & 1][c], k >> 1) & W_STRIP) | uint32_t(k + 1);
#pragma unroll
      for (int c = 0; c < 8; c++) {
        acc[0][c] = min(acc[0][c], c2.x + dkj[c]);
        acc[1][c] = min(acc[1][c], c2.y + dkj[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; c++)
        dkj[c] = (__shfl_sync(0xffffffffu, acc[(kk + 1) & 1][c], (k + 1) >> 1) & W_STRIP) | uint32_t(k + 2);
#pragma unroll
      for (int c = 0; c < 8; c++) {
        acc[0][c] = min(acc[0][c], ck1x + dkj[c]);
        acc[1][c] = min(acc[1][c], ck1y + dkj[c]);
      }
      if (k + 2 < QB) {
        if (kk == 6) {
          if (w == (k0 >> 3) + 1) W64_PUB(0, buf ^ 1);
        } else if (w == (k0 >> 3)) {
          W64_PUB((kk + 2) & 7, buf ^ 1);
        }
      }
    }
  }
#undef W64_PUB
  __syncthreads();
  uint32_t kst[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) {
      kst[r][c] = acc[r][c] & W_TMASK;
      acc[r][c] -= kst[r][c];
    }
#pragma unroll
  for (int r = 0; r < 2; r++) store8_w32(D + int64_t(2 * l + r) * ld + 8 * w, acc[r]);
  if (!P) return;
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) sm.K[2 * l + r][8 * w + c] = uint8_t(kst[r][c]);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  for (int round = 0; round < 6; round++) {
    int32_t np[16];
    uint8_t nk[16];
    bool live = false;
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int e = t + QT * c, i = e >> 6, j = e & 63;
      const uint8_t kk = sm.K[i][j];
      np[c] = sm.P[i][j];
      nk[c] = kk;
      if (kk) {
        np[c] = sm.P[kk - 1][j];
        nk[c] = sm.K[kk - 1][j];
        live |= nk[c] != 0;
      }
    }
    const bool more = __syncthreads_or(live);
#pragma unroll
    for (int c = 0; c < 16; c++) {
      const int e = t + QT * c, i = e >> 6, j = e & 63;
      sm.P[i][j] = np[c];
      sm.K[i][j] = nk[c];
    }
    __syncthreads();
    if (!more) break;
  }
  for (int e = t; e < QB * QB / 4; e += QT) {
    const int i = e >> 4, j = 4 * (e & 15);
    *reinterpret_cast<int4*>(P + int64_t(i) * ldp + j) = *reinterpret_cast<const int4*>(&sm.P[i][j]);
  }
}

// C <- min(C, A (x) B) on a 64 x 64 w32 tile, k = 64 (one tag window)
__device__ void tile64_w32(TileSmemW& sm, int32_t* C, int64_t ldc, const int32_t* A, int64_t lda, const int32_t* B,
                           int64_t ldb, int32_t* P, int64_t ldp, const int32_t* PB_, int64_t ldpb) {
  const int t = threadIdx.x, ty = t >> 3, tx = t & 7;
  if (P) {
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int e = t + QT * q, i = e >> 4, j = 4 * (e & 15);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(&sm.Pb[i][j])),
                   "l"(PB_ + int64_t(i) * ldpb + j) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  {  // A (64 rows x 64 k) transposed to [k][row]; B (64 k x 64 cols) tagged: 16 values each per thread
    const int ra = t >> 2, ka = 16 * (t & 3);
#pragma unroll
    for (int q4 = 0; q4 < 4; q4++) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(A + int64_t(ra) * lda + ka) + q4);
      sm.As[ka + 4 * q4][ra] = v.x << 7;
      sm.As[ka + 4 * q4 + 1][ra] = v.y << 7;
      sm.As[ka + 4 * q4 + 2][ra] = v.z << 7;
      sm.As[ka + 4 * q4 + 3][ra] = v.w << 7;
    }
    const int kb = t >> 2, cb = 16 * (t & 3);
    const uint32_t tag = uint32_t(kb + 1);
#pragma unroll
    for (int q4 = 0; q4 < 4; q4++) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(B + int64_t(kb) * ldb + cb) + q4);
      reinterpret_cast<uint4*>(&sm.Bs[kb][cb])[q4] =
          make_uint4((v.x << 7) | tag, (v.y << 7) | tag, (v.z << 7) | tag, (v.w << 7) | tag);
    }
  }
  uint32_t acc[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++) load8_w32(C + int64_t(2 * ty + r) * ldc + 8 * tx, acc[r]);
  __syncthreads();
#pragma unroll 8
  for (int k = 0; k < QB; k++) {
    const uint2 a = *reinterpret_cast<const uint2*>(&sm.As[k][2 * ty]);
    const uint4 b0 = reinterpret_cast<const uint4*>(&sm.Bs[k][8 * tx])[0];
    const uint4 b1 = reinterpret_cast<const uint4*>(&sm.Bs[k][8 * tx])[1];
    const uint32_t bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int c = 0; c < 8; c++) {
      acc[0][c] = min(acc[0][c], a.x + bv[c]);
      acc[1][c] = min(acc[1][c], a.y + bv[c]);
    }
  }
  uint32_t kst[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) {
      kst[r][c] = acc[r][c] & W_TMASK;
      acc[r][c] -= kst[r][c];
    }
  if (P) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  int32_t pv[2][8];
#pragma unroll
  for (int r = 0; r < 2; r++)
#pragma unroll
    for (int c = 0; c < 8; c++) pv[r][c] = (P && kst[r][c]) ? sm.Pb[kst[r][c] - 1][8 * tx + c] : 0;
#pragma unroll
  for (int r = 0; r < 2; r++) {
    uint32_t any = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) any |= kst[r][c];
    if (!any) continue;
    store8_w32(C + int64_t(2 * ty + r) * ldc + 8 * tx, acc[r]);
    if (!P) continue;
    int32_t* prow = P + int64_t(2 * ty + r) * ldp + 8 * tx;
#pragma unroll
    for (int c = 0; c < 8; c++)
      if (kst[r][c]) prow[c] = pv[r][c];
  }
}

template <int S>
__global__ void __launch_bounds__(QT, 3) fw_persist64_kernel(typename K64<S>::T* D, int64_t ld, int32_t* P, int64_t ldp, int nb,
                                                             const int4* items, int nitems, int* done, int* counter,
                                                             unsigned long long* trace) {
  using SmemT = typename std::conditional<S == STORE_W32, SmemW, Smem>::type;
  extern __shared__ __align__(16) unsigned char smraw_p64[];   // sizeof(SmemT) (w32: 48 KB, opt-in)
  SmemT& sm = *reinterpret_cast<SmemT*>(smraw_p64);
  __shared__ int s_item;
  const int t = threadIdx.x;
  auto tile = [&](typename K64<S>::T* C, int64_t ldc, const typename K64<S>::T* A, const typename K64<S>::T* B,
                  int32_t* Pc, const int32_t* Pb_) {
    if constexpr (S == STORE_W32) tile64_w32(sm.tile, C, ldc, A, ld, B, ld, Pc, ldp, Pb_, ldp);
    else tile64<S>(sm.tile, C, ldc, A, ld, B, ld, Pc, ldp, Pb_, ldp);
  };
  for (;;) {
    if (t == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= nitems) break;
    const int4 w = items[it];   // (task, K, I, J)
    const int K = w.y, I = w.z, J = w.w;
    unsigned long long t_claim = 0, t_ready = 0;
    if (trace && t == 0) t_claim = persist::gtimer();
    if (t == 0) {
      if (w.x == persist::T_CLOSE) {
        persist::wait_at_least(&done[K * nb + K], K);
      } else if (w.x == persist::T_UCLOSE) {
        persist::wait_at_least(&done[K * nb + K - 1], K);
        persist::wait_at_least(&done[(K - 1) * nb + K], K);
        persist::wait_at_least(&done[K * nb + K], K - 1);
      } else if (w.x == persist::T_ROW) {
        persist::wait_at_least(&done[K * nb + K], K + 1);
        persist::wait_at_least(&done[K * nb + J], K);
      } else if (w.x == persist::T_COL) {
        persist::wait_at_least(&done[K * nb + K], K + 1);
        persist::wait_at_least(&done[I * nb + K], K);
      } else {
        persist::wait_at_least(&done[I * nb + K], K + 1);
        persist::wait_at_least(&done[K * nb + J], K + 1);
        persist::wait_at_least(&done[I * nb + J], K);
      }
    }
    __syncthreads();
    if (trace && t == 0) t_ready = persist::gtimer();
    const int64_t k0 = int64_t(K) * QB;
    if (w.x == persist::T_CLOSE || w.x == persist::T_UCLOSE) {
      if (w.x == persist::T_UCLOSE) {   // round K-1 on the tile first (pivot block K-1)
        const int64_t kp = k0 - QB;
        tile(D + k0 * ld + k0, ld, D + k0 * ld + kp, D + kp * ld + k0, P ? P + k0 * ldp + k0 : nullptr,
             P ? P + kp * ldp + k0 : nullptr);
        __syncthreads();
      }
      if constexpr (S == STORE_W32) close64_w32(sm.close, D + k0 * ld + k0, ld, P ? P + k0 * ldp + k0 : nullptr, ldp);
      else close64<S>(sm.close, D + k0 * ld + k0, ld, P ? P + k0 * ldp + k0 : nullptr, ldp, trace != nullptr);
    } else {
      const int64_t i0 = int64_t(w.x == persist::T_ROW ? K : I) * QB;
      const int64_t j0 = int64_t(w.x == persist::T_COL ? K : J) * QB;
      tile(D + i0 * ld + j0, ld, D + i0 * ld + k0, D + k0 * ld + j0, P ? P + i0 * ldp + j0 : nullptr,
           P ? P + k0 * ldp + j0 : nullptr);
    }
    __syncthreads();
    if (t == 0) {
      __threadfence();
      const bool cl = w.x == persist::T_CLOSE || w.x == persist::T_UCLOSE;
      const int ti = (cl || w.x == persist::T_ROW) ? K : I;
      const int tj = (cl || w.x == persist::T_COL) ? K : J;
      persist::release_st(&done[ti * nb + tj], K + 1);
      if (trace) {
        unsigned int smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        trace[4 * it] = t_claim;
        trace[4 * it + 1] = t_ready;
        trace[4 * it + 2] = persist::gtimer();
        trace[4 * it + 3] = smid;
      }
    }
  }
}

}  // namespace persist64

bool fw_persist64_enabled(int store, int64_t N) {
  static const int64_t max_n = getenv("APSP_PERSIST64_MAX_N") ? atoll(getenv("APSP_PERSIST64_MAX_N")) : 2048;
  // N = 128 is one classic-order closure (pred bit-exact with the reference, test-pinned): the
  // 128-wide schedule handles it
  return (store == STORE_U8 || store == STORE_U16 || store == STORE_W32) && N % 64 == 0 && N <= max_n && N >= 256;
}

size_t fw_persist64_scratch_bytes(int64_t N) {
  const int64_t nb = N / 64;
  return size_t(nb * nb + 64) * sizeof(int);
}

int launch_fw_persist64(int store, void* D, int64_t ld, int32_t* P, int64_t ldp, int64_t N, void* scratch,
                        cudaStream_t s) {
  if (store != STORE_U8 && store != STORE_U16 && store != STORE_W32)
    return set_error(APSP_EINVAL, "the 64-wide schedule is u8 / u16 / w32");
  const int nb = int(N / 64);
  int nitems = 0;
  const int4* items = persist_items(nb, &nitems, true);
  if (!items) return set_error(APSP_ECUDA, "persistent schedule table allocation failed");
  int* done = static_cast<int*>(scratch);
  int* counter = done + nb * nb;
  APSP_CUDA_TRY(cudaMemsetAsync(scratch, 0, fw_persist64_scratch_bytes(N), s));
  int slots = 0;
  constexpr int sb = int(sizeof(persist64::Smem)), sbw = int(sizeof(persist64::SmemW));
  static std::atomic<unsigned long long> a8{0}, a16{0}, a32{0};
  if (store == STORE_U8) {
    APSP_CUDA_TRY(smem_optin(persist64::fw_persist64_kernel<STORE_U8>, sb, a8));
    APSP_CUDA_TRY(persist_slots(persist64::fw_persist64_kernel<STORE_U8>, persist64::QT, sb, slots));
  } else if (store == STORE_U16) {
    APSP_CUDA_TRY(smem_optin(persist64::fw_persist64_kernel<STORE_U16>, sb, a16));
    APSP_CUDA_TRY(persist_slots(persist64::fw_persist64_kernel<STORE_U16>, persist64::QT, sb, slots));
  } else {
    APSP_CUDA_TRY(smem_optin(persist64::fw_persist64_kernel<STORE_W32>, sbw, a32));
    APSP_CUDA_TRY(persist_slots(persist64::fw_persist64_kernel<STORE_W32>, persist64::QT, sbw, slots));
  }
  if (slots < 1) return set_error(APSP_ECUDA, "persistent kernel does not fit an SM");
  const int grid = std::min(slots, nitems);
  unsigned long long* trace = nullptr;
  if (getenv("APSP_PERSIST_TRACE")) APSP_CUDA_TRY(cudaMalloc(&trace, size_t(nitems) * 4 * sizeof(unsigned long long)));
  if (store == STORE_U8)
    persist64::fw_persist64_kernel<STORE_U8><<<grid, persist64::QT, sb, s>>>(static_cast<uint8_t*>(D), ld, P, ldp, nb,
                                                                            items, nitems, done, counter, trace);
  else if (store == STORE_U16)
    persist64::fw_persist64_kernel<STORE_U16><<<grid, persist64::QT, sb, s>>>(static_cast<uint16_t*>(D), ld, P, ldp,
                                                                             nb, items, nitems, done, counter, trace);
  else
    persist64::fw_persist64_kernel<STORE_W32><<<grid, persist64::QT, sbw, s>>>(static_cast<int32_t*>(D), ld, P, ldp,
                                                                             nb, items, nitems, done, counter, trace);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  return persist_dump_trace(trace, items, nitems, s);
}
