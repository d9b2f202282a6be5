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

// tcgen05 int8 tensor-core throughput (the roofline of the byte-plane MAC's tensor side): one CTA
// per SM, one thread issues back-to-back kind::i8 UMMAs M=128 N=256 K=32 (the MAC kernels' shape)
// from fixed shared-memory tiles into one TMEM accumulator, then waits on the commit.
#define MMA_ITERS 8192
__global__ void __launch_bounds__(128) k_umma_i8(const int32_t* __restrict__ w, int64_t* out, int n) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[256 * 32];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 32; e += 128) sA[e] = (uint8_t)(e * 37 + w[e & 31]);
  for (int e = tid; e < 256 * 32; e += 128) sB[e] = (uint8_t)(e * 91 + 3);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  auto desc = [](uint32_t saddr) {
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(128 >> 4) << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    return d;
  };
  if (tid == 0) {
    const uint32_t id = (2u << 4) | (1u << 7) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t da = desc((uint32_t)__cvta_generic_to_shared(sA)), db = desc((uint32_t)__cvta_generic_to_shared(sB));
    for (int it = 0; it < MMA_ITERS; it++)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(it));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mb) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r0;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (r0 == 0x12345u) out[0] = r0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

typedef void (*kfn)(const int32_t*, int64_t*, int);

static void run(const char* name, kfn f, double ops_per_inner, int* w, int64_t* o, int blocks = 148 * 8,
                int threads = 256, double ops_per_thread = 0) {
  int sms = 148;
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
  double ops = ops_per_thread > 0 ? (double)blocks * ops_per_thread * reps
                                 : (double)blocks * threads * ITERS * 8 * ops_per_inner * reps;
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
  // per CTA: MMA_ITERS UMMAs of 2 * 128 * 256 * 32 int8 ops
  run("tcgen05_i8_ops", k_umma_i8, 0, w, o, 148, 128, (double)MMA_ITERS * 2 * 128 * 256 * 32);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
