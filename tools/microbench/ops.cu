// Issue-rate microbenchmark for the min-plus inner-loop instruction candidates on sm_100a.
// Each thread runs R rounds over U independent accumulators; we report updates/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define U 16
#define R 4096

__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d; asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ unsigned long long pack2(float x, float y) {
  unsigned long long d; asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(x), "f"(y)); return d;
}
__device__ __forceinline__ void unpack2(unsigned long long v, float& x, float& y) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(v));
}

// A: FADD + FMNMX (2 ops per update)
__global__ void k_fadd_fmnmx(float* out, float b0, float step) {
  float acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 1e30f; a[i] = threadIdx.x * 0.5f + i; }
  float b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = fminf(acc[i], a[i] + b);
    b += step;
  }
  float s = 0; for (int i = 0; i < U; i++) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}
// B: FADD2 + FMNMX3: 2 updates per (FADD2 + FMNMX3)
__global__ void k_fadd2_fmnmx3(float* out, float b0, float step) {
  float acc[U]; unsigned long long a2[U];
  for (int i = 0; i < U; i++) { acc[i] = 1e30f; a2[i] = pack2(threadIdx.x * 0.5f + i, threadIdx.x * 0.25f + i); }
  float b = b0;
  for (int r = 0; r < R; r++) {
    unsigned long long bb = pack2(b, b + 1.0f);
#pragma unroll
    for (int i = 0; i < U; i++) {
      float x, y; unpack2(fadd2(a2[i], bb), x, y);
      acc[i] = fmin3(acc[i], x, y);
    }
    b += step;
  }
  float s = 0; for (int i = 0; i < U; i++) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}
// B2: FADD + FMNMX3 (scalar adds, 3-input min)
__global__ void k_fadd_fmnmx3(float* out, float b0, float step) {
  float acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 1e30f; a[i] = threadIdx.x * 0.5f + i; }
  float b = b0;
  for (int r = 0; r < R; r++) {
    float b1 = b + 1.0f;
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = fmin3(acc[i], a[i] + b, a[i] + b1);
    b += step;
  }
  float s = 0; for (int i = 0; i < U; i++) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}
// C: int IADD + IMNMX
__global__ void k_iadd_imnmx(int* out, int b0, int step) {
  int acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 0x3fffffff; a[i] = threadIdx.x * 3 + i; }
  int b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = min(acc[i], a[i] + b);
    b += step;
  }
  int s = 0; for (int i = 0; i < U; i++) s ^= acc[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// D: DPX viaddmin s32
__global__ void k_viaddmin(int* out, int b0, int step) {
  int acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 0x3fffffff; a[i] = threadIdx.x * 3 + i; }
  int b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = __viaddmin_s32(a[i], b, acc[i]);
    b += step;
  }
  int s = 0; for (int i = 0; i < U; i++) s ^= acc[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// E: DPX viaddmin s16x2 (2 updates per instr)
__global__ void k_viaddmin16x2(int* out, int b0, int step) {
  unsigned acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 0x3fff3fffu; a[i] = (threadIdx.x * 3 + i) * 0x10001u; }
  unsigned b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = __viaddmin_s16x2(a[i], b, acc[i]);
    b += step;
  }
  unsigned s = 0; for (int i = 0; i < U; i++) s ^= acc[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// F: IADD + 3-input int min (vimin3)
__global__ void k_iadd_vimin3(int* out, int b0, int step) {
  int acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 0x3fffffff; a[i] = threadIdx.x * 3 + i; }
  int b = b0;
  for (int r = 0; r < R; r++) {
    int b1 = b + 7;
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = __vimin3_s32(acc[i], a[i] + b, a[i] + b1);
    b += step;
  }
  int s = 0; for (int i = 0; i < U; i++) s ^= acc[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// G: exact argmin fp32: FADD, FSETP, FSEL, SEL
__global__ void k_argmin_f32(float* out, float b0, float step) {
  float acc[U], a[U]; int idx[U];
  for (int i = 0; i < U; i++) { acc[i] = 1e30f; a[i] = threadIdx.x * 0.5f + i; idx[i] = -1; }
  float b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) { float s = a[i] + b; bool p = s < acc[i]; acc[i] = p ? s : acc[i]; idx[i] = p ? r : idx[i]; }
    b -= step;
  }
  float s = 0; for (int i = 0; i < U; i++) s += acc[i] + idx[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}
// G2: exact argmin int32 (the i32 tier's register-staged compare-select): IADD, ISETP, min, SEL
__global__ void k_argmin_i32(int* out, int b0, int step) {
  int acc[U], a[U], idx[U];
  for (int i = 0; i < U; i++) { acc[i] = 0x3fffffff; a[i] = threadIdx.x * 3 + i; idx[i] = -1; }
  int b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) { int s = a[i] + b; bool p = s < acc[i]; acc[i] = min(acc[i], s); idx[i] = p ? r : idx[i]; }
    b -= step;
  }
  int s = 0; for (int i = 0; i < U; i++) s ^= acc[i] + idx[i];
  if (s == 12345) out[threadIdx.x] = s;
}
// H: FFMA reference (peak issue)
__global__ void k_ffma(float* out, float b0, float step) {
  float acc[U], a[U];
  for (int i = 0; i < U; i++) { acc[i] = 0.f; a[i] = threadIdx.x * 0.5f + i; }
  float b = b0;
  for (int r = 0; r < R; r++) {
#pragma unroll
    for (int i = 0; i < U; i++) acc[i] = fmaf(a[i], b, acc[i]);
    b += step;
  }
  float s = 0; for (int i = 0; i < U; i++) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <typename K, typename T>
void run(const char* name, K kern, T* out, T b0, T step, double upd_per_inner, int blocks, int threads, int clk_mhz) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) kern<<<blocks, threads>>>(out, b0, step);
  cudaEventRecord(e0);
  int reps = 5;
  for (int w = 0; w < reps; w++) kern<<<blocks, threads>>>(out, b0, step);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
  double upd = (double)blocks * threads * R * U * upd_per_inner;
  double rate = upd / (ms * 1e-3);
  printf("%-18s %8.3f ms  %8.2f T upd/s  %6.1f upd/clk/SM @%dMHz\n", name, ms, rate / 1e12,
         rate / (148.0 * clk_mhz * 1e6), clk_mhz);
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
}

int main() {
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); clk /= 1000;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d clock %d MHz\n", sms, clk);
  float* f; int* i; cudaMalloc(&f, 4096); cudaMalloc(&i, 4096);
  int blocks = sms * 8, threads = 256;
  for (int pass = 0; pass < 2; pass++) {
  run("fadd+fmnmx", k_fadd_fmnmx, f, 1.f, 0.001f, 1.0, blocks, threads, clk);
  run("fadd2+fmnmx3", k_fadd2_fmnmx3, f, 1.f, 0.001f, 2.0, blocks, threads, clk);
  run("fadd+fmnmx3", k_fadd_fmnmx3, f, 1.f, 0.001f, 2.0, blocks, threads, clk);
  run("iadd+imnmx", k_iadd_imnmx, i, 1, 1, 1.0, blocks, threads, clk);
  run("viaddmin_s32", k_viaddmin, i, 1, 1, 1.0, blocks, threads, clk);
  run("viaddmin_s16x2", k_viaddmin16x2, i, 1, 1, 2.0, blocks, threads, clk);
  run("iadd+vimin3", k_iadd_vimin3, i, 1, 1, 2.0, blocks, threads, clk);
  run("argmin_f32", k_argmin_f32, f, 1.f, 0.001f, 1.0, blocks, threads, clk);
  run("argmin_i32", k_argmin_i32, i, 1, 1, 1.0, blocks, threads, clk);
  run("ffma(1 op)", k_ffma, f, 1.f, 0.001f, 1.0, blocks, threads, clk);
  }
  return 0;
}
