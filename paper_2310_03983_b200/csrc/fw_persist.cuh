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
//     C(0) P(0) A(0) | C(1) P(1) B(0) A(1) | C(2) P(2) B(1) A(2) | ... | B(nb-1)
// (P = the panels, A(K) = the round-K updates of the tiles in the cross of K+1, B(K) = the rest)
// is the lookahead schedule, and every dependency of a task is claimed before it: with every CTA
// resident (grid = SM count, one CTA per SM), the spin-waits always end.
//
// Tile tasks use 512 threads on a 128 x 128 tile (4 rows x 8 columns each), k = 128 in four
// 32-k chunks staged through registers into shared memory as packed 16-bit keys
// (v << 7 | tag, tags 1..96 per 3-chunk window) and relaxed with VIADDMNMX.U16x2, the same
// arithmetic and argmin semantics as minplus_nt_kernel: strict improvement, smallest k, pred
// gathered from the B rows' pred for improved cells only. The row-panel task reads its own tile
// as B and its pred rows, so every gather of a task completes before any of its stores (barrier).

namespace persist {

constexpr int PT = 512;            // threads
constexpr int PB = 128;            // tile
constexpr uint32_t KINF2 = (uint32_t(U8_INF) << 7) * 0x00010001u;
constexpr uint32_t TMASK2 = 0x007F007Fu;
enum Task : int { T_CLOSE = 0, T_ROW = 1, T_COL = 2, T_UPD = 3 };

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
    if (w.x == T_CLOSE) {
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
      const int ti = w.x == T_CLOSE ? K : w.x == T_ROW ? K : I;
      const int tj = w.x == T_CLOSE ? K : w.x == T_COL ? K : J;
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
static const int4* persist_items(int nb, int* nitems) {
  struct Entry { int dev, nb, n; int4* d; };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : cache)
    if (e.dev == dev && e.nb == nb) {
      *nitems = e.n;
      return e.d;
    }
  std::vector<int4> v;
  auto updates = [&](int K, bool next_cross) {   // round-K updates in / outside the cross of K+1
    for (int I = 0; I < nb; I++)
      for (int J = 0; J < nb; J++) {
        if (I == K || J == K) continue;
        const bool nx = K + 1 < nb && (I == K + 1 || J == K + 1);
        if (nx == next_cross) v.push_back(make_int4(persist::T_UPD, K, I, J));
      }
  };
  auto close_and_panels = [&](int K) {
    v.push_back(make_int4(persist::T_CLOSE, K, K, K));
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
    updates(K - 1, false);
    updates(K, true);
  }
  updates(nb - 1, false);
  int4* d = nullptr;
  if (cudaMalloc(&d, v.size() * sizeof(int4)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, v.data(), v.size() * sizeof(int4), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  cache.push_back({dev, nb, int(v.size()), d});
  *nitems = int(v.size());
  return d;
}

size_t fw_persist_scratch_bytes(int64_t N) {
  const int64_t nb = N / TILE_ALIGN;
  return size_t(nb * nb + 64) * sizeof(int);
}

bool fw_persist_enabled(int store, int64_t N) {
  static const int64_t max_n = getenv("APSP_PERSIST_MAX_N") ? atoll(getenv("APSP_PERSIST_MAX_N")) : 3072;
  return store == STORE_U8 && N % TILE_ALIGN == 0 && N <= max_n && N >= TILE_ALIGN;
}

// One persistent launch for the whole u8 blocked FW of an N x N view (N a multiple of 128).
int launch_fw_persist(uint8_t* D, int64_t ld, int32_t* P, int64_t ldp, int64_t N, void* scratch, cudaStream_t s) {
  const int nb = int(N / TILE_ALIGN);
  int nitems = 0;
  const int4* items = persist_items(nb, &nitems);
  if (!items) return set_error(APSP_ECUDA, "persistent schedule table allocation failed");
  int* done = static_cast<int*>(scratch);
  int* counter = done + nb * nb;
  APSP_CUDA_TRY(cudaMemsetAsync(scratch, 0, fw_persist_scratch_bytes(N), s));
  static std::atomic<unsigned long long> attr{0};
  const int sb = int(sizeof(persist::Smem));
  APSP_CUDA_TRY(smem_optin(persist::fw_persist_kernel, sb, attr));
  int dev = 0, sms = 0;
  APSP_CUDA_TRY(cudaGetDevice(&dev));
  APSP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int grid = std::min(sms, nitems);
  // APSP_PERSIST_TRACE=file: per task (kind, K, I, J, claim, ready, done ns, SM) as CSV, for the
  // schedule's critical path (tools/persist_trace.py)
  const char* tpath = getenv("APSP_PERSIST_TRACE");
  unsigned long long* trace = nullptr;
  if (tpath) APSP_CUDA_TRY(cudaMalloc(&trace, size_t(nitems) * 4 * sizeof(unsigned long long)));
  persist::fw_persist_kernel<<<grid, persist::PT, sb, s>>>(D, ld, P, ldp, nb, items, nitems, done, counter, trace);
  APSP_CUDA_TRY(cudaGetLastError());
  count_launches(1);
  if (trace) {
    std::vector<unsigned long long> h(size_t(nitems) * 4);
    std::vector<int4> it(nitems);
    APSP_CUDA_TRY(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s));
    APSP_CUDA_TRY(cudaMemcpyAsync(it.data(), items, it.size() * sizeof(int4), cudaMemcpyDeviceToHost, s));
    APSP_CUDA_TRY(cudaStreamSynchronize(s));
    cudaFree(trace);
    if (FILE* f = fopen(tpath, "w")) {
      fprintf(f, "kind,K,I,J,claim,ready,done,sm\n");
      for (int i = 0; i < nitems; i++)
        fprintf(f, "%d,%d,%d,%d,%llu,%llu,%llu,%llu\n", it[i].x, it[i].y, it[i].z, it[i].w, h[4 * i], h[4 * i + 1],
                h[4 * i + 2], h[4 * i + 3]);
      fclose(f);
    }
  }
  return 0;
}
