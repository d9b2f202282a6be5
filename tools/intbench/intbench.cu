// INT/FP64 pipe throughput microbenchmark for the roofline denominators used in
// DESIGN.md (the INT peak is not in MEASURED_PEAKS.json).  Each kernel runs a
// long chain of independent ops per thread (8 independent accumulators) over a
// full grid (148 SMs x 8 CTAs x 256 threads), timed with CUDA events.
// Reports ops/s and ops/clk/SM at the measured SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_imad_wide(const int32_t* __restrict__ w, int64_t* out, int n) {
  int32_t a = w[threadIdx.x & 31], b = w[(threadIdx.x + 7) & 31];
  int64_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      int32_t x = a + i;
      acc[i] += (int64_t)x * (int64_t)b;  // IMAD.WIDE
    }
    b ^= it;
  }
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x123456789) out[0] = s;
}

__global__ void k_imad32(const int32_t* __restrict__ w, int64_t* out, int n) {
  int32_t a = w[threadIdx.x & 31], b = w[(threadIdx.x + 7) & 31];
  int32_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = acc[i] * a + b;  // IMAD
    b ^= it;
  }
  int32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x12345) out[0] = s;
}

__global__ void k_mulhi64(const int32_t* __restrict__ w, int64_t* out, int n) {
  uint64_t a = (uint64_t)w[threadIdx.x & 31] * 0x9E3779B97F4A7C15ull;
  uint64_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = a + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = __umul64hi(acc[i], a) + acc[i];
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x123456789) out[0] = s;
}

__global__ void k_dfma(const int32_t* __restrict__ w, int64_t* out, int n) {
  double a = w[threadIdx.x & 31], b = w[(threadIdx.x + 7) & 31];
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 1.2345) out[0] = (int64_t)s;
}

__global__ void k_iadd3(const int32_t* __restrict__ w, int64_t* out, int n) {
  uint32_t a = w[threadIdx.x & 31], b = w[(threadIdx.x + 7) & 31];
  uint32_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = (acc[i] + a + b) ^ (acc[i] >> 3);
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x12345) out[0] = s;
}

// 64-bit Shoup modular product x * w mod q (in [0, 2q)), the unit of every "alu" roofline in
// bench.py: 8 independent chains per thread
__global__ void k_shoup(const int32_t* __restrict__ w, int64_t* out, int n) {
  const uint64_t q = 0xfffffffffffc001ull;
  const uint64_t wv = 0x0123456789abcdeull + (uint64_t)w[threadIdx.x & 31];
  const uint64_t wsh = (uint64_t)(((unsigned __int128)wv << 64) / q);
  uint64_t acc[8];
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = (uint64_t)w[(threadIdx.x + i) & 31] * 0x9E3779B97F4A7C15ull;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) acc[i] = acc[i] * wv - __umul64hi(acc[i], wsh) * q;
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  if (s == 0x123456789) out[0] = s;
}

typedef void (*kfn)(const int32_t*, int64_t*, int);

static void run(const char* name, kfn f, double ops_per_inner, int* w, int64_t* o) {
  int sms = 148, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 3; r++) f<<<blocks, threads>>>(w, o, 0);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; r++) f<<<blocks, threads>>>(w, o, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * ITERS * 8 * ops_per_inner * reps;
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double per_s = ops / (ms * 1e-3);
  printf("{\"op\": \"%s\", \"ops_per_s\": %.4e, \"ms\": %.3f, \"per_clk_per_sm_at_maxclk\": %.2f}\n", name, per_s,
         ms / reps, per_s / (sms * (double)clk_khz * 1e3));
}

int main() {
  int* w;
  int64_t* o;
  cudaMalloc(&w, 128);
  cudaMemset(w, 1, 128);
  cudaMalloc(&o, 64);
  run("imad_wide_s32", k_imad_wide, 1, w, o);
  run("imad_s32", k_imad32, 1, w, o);
  run("umul64hi", k_mulhi64, 1, w, o);
  run("dfma", k_dfma, 1, w, o);
  run("shoup_modmul64", k_shoup, 1, w, o);
  run("iadd_xor_shift(3 ops)", k_iadd3, 3, w, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
