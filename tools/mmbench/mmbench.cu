// Modular-arithmetic formulation microbenchmark (design evidence for the INT-bound kernels): the
// Harvey NTT butterfly and the lazy key-switching term in several formulations, 8 independent
// chains per thread over 148 SMs x 8 CTAs x 256 threads, CUDA events; each variant is first checked
// against exact 128-bit arithmetic on random inputs.  Prints one JSON line per variant:
//   bfly_*: Harvey CT butterflies/clk/SM;  ks_*: key-switching products (d w mod q, lazy)/clk/SM.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;
#define ITERS 2048

__device__ __forceinline__ u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

// ---- hi64(x * w) variants ----
__device__ __forceinline__ u64 hi_c(u64 x, u64 w) { return __umul64hi(x, w); }
// exact, explicit 32-bit multiply-adds with carries
__device__ __forceinline__ u64 hi_ptx(u64 x, u64 w) {
  uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32);
  uint32_t t0, c1, c2, c3;
  asm("mul.hi.u32 %0, %4, %6;\n\t"
      "mad.lo.cc.u32 %1, %4, %7, %0;\n\t"
      "madc.hi.u32 %2, %4, %7, 0;\n\t"
      "mad.lo.cc.u32 %1, %5, %6, %1;\n\t"
      "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
      "addc.u32 %3, 0, 0;\n\t"
      "mad.lo.cc.u32 %2, %5, %7, %2;\n\t"
      "madc.hi.u32 %3, %5, %7, %3;"
      : "=&r"(t0), "=&r"(c1), "=&r"(c2), "=&r"(c3)
      : "r"(x0), "r"(x1), "r"(w0), "r"(w1));
  return ((u64)c3 << 32) | c2;
}
// approximate: x1 w1 + hi(x1 w0) + hi(x0 w1); hi_exact - 3 <= result <= hi_exact
__device__ __forceinline__ u64 hi_apx(u64 x, u64 w) {
  uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32);
  const uint32_t a = __umulhi(x1, w0), b = __umulhi(x0, w1);
  return (u64)x1 * w1 + a + b;
}
// lo64(h * q) for q = 1 + q1 2^32 (q0 == 1)
__device__ __forceinline__ u64 mulq_sp(u64 h, uint32_t q1) {
  return h + ((u64)((uint32_t)h * q1) << 32);
}

template <int V>
__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wsh, u64 q) {
  if constexpr (V == 0) return x * w - hi_c(x, wsh) * q;
  if constexpr (V == 1) return x * w - hi_ptx(x, wsh) * q;
  if constexpr (V == 2) return x * w - hi_apx(x, wsh) * q;                      // [0, 5q)
  if constexpr (V == 3) return x * w - mulq_sp(hi_c(x, wsh), (uint32_t)(q >> 32));
  if constexpr (V == 4) return x * w - mulq_sp(hi_apx(x, wsh), (uint32_t)(q >> 32));
  return 0;
}

__device__ __forceinline__ void bfly_ptx_full(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 q2);
// Harvey CT butterfly, [0, 4q) -> [0, 4q) (exact quotient variants)
template <int V>
__device__ __forceinline__ void bfly(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 q2) {
  if constexpr (V == 9) {
    bfly_ptx_full(x, y, w, wsh, q, q2);
    return;
  }
  const u64 X = csub(x, q2);
  const u64 T = shoup<V>(y, w, wsh, q);
  x = X + T;
  y = X - T + q2;
}

// whole Harvey CT butterfly in PTX on 32-bit halves (exact Shoup quotient)
__device__ __forceinline__ void bfly_ptx_full(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 q2) {
  uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), y0 = (uint32_t)y, y1 = (uint32_t)(y >> 32);
  const uint32_t w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32), s0 = (uint32_t)wsh, s1 = (uint32_t)(wsh >> 32);
  const uint32_t q0 = (uint32_t)q, q1 = (uint32_t)(q >> 32), p0 = (uint32_t)q2, p1 = (uint32_t)(q2 >> 32);
  asm("{\n\t.reg .u32 a, b, c, h0, h1, t0, t1, u0, u1, v0, v1;\n\t.reg .pred p;\n\t"
      // X = x >= 2q ? x - 2q : x
      "sub.cc.u32 v0, %0, %10;\n\tsubc.cc.u32 v1, %1, %11;\n\tsubc.u32 a, 0, 0;\n\t"
      "setp.eq.u32 p, a, 0;\n\t@p mov.u32 %0, v0;\n\t@p mov.u32 %1, v1;\n\t"
      // h = hi64(y * wsh)
      "mul.hi.u32 a, %2, %6;\n\t"
      "mad.lo.cc.u32 a, %2, %7, a;\n\tmadc.hi.u32 b, %2, %7, 0;\n\t"
      "mad.lo.cc.u32 a, %3, %6, a;\n\tmadc.hi.cc.u32 b, %3, %6, b;\n\taddc.u32 c, 0, 0;\n\t"
      "mad.lo.cc.u32 h0, %3, %7, b;\n\tmadc.hi.u32 h1, %3, %7, c;\n\t"
      // T = y w - h q (mod 2^64)
      "mul.lo.u32 t0, %2, %4;\n\tmul.hi.u32 t1, %2, %4;\n\tmad.lo.u32 t1, %2, %5, t1;\n\tmad.lo.u32 t1, %3, %4, t1;\n\t"
      "mul.lo.u32 u0, h0, %8;\n\tmul.hi.u32 u1, h0, %8;\n\tmad.lo.u32 u1, h0, %9, u1;\n\tmad.lo.u32 u1, h1, %8, u1;\n\t"
      "sub.cc.u32 t0, t0, u0;\n\tsubc.u32 t1, t1, u1;\n\t"
      // y' = X - T + 2q, x' = X + T
      "sub.cc.u32 v0, %0, t0;\n\tsubc.u32 v1, %1, t1;\n\tadd.cc.u32 %2, v0, %10;\n\taddc.u32 %3, v1, %11;\n\t"
      "add.cc.u32 %0, %0, t0;\n\taddc.u32 %1, %1, t1;\n\t}"
      : "+r"(x0), "+r"(x1), "+r"(y0), "+r"(y1)
      : "r"(w0), "r"(w1), "r"(s0), "r"(s1), "r"(q0), "r"(q1), "r"(p0), "r"(p1));
  x = ((u64)x1 << 32) | x0;
  y = ((u64)y1 << 32) | y0;
}

template <int V>
__global__ void k_bfly(const u64* __restrict__ prm, u64* out) {
  const u64 q = prm[0], w = prm[1] + threadIdx.x, wsh = (u64)(((u128)w << 64) / q);
  const u64 q2 = 2 * q;
  u64 a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; i++) {
    a[i] = (prm[2] * (threadIdx.x + 17 * i)) % q;
    b[i] = (prm[3] * (threadIdx.x + 29 * i)) % q;
  }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      bfly<V>(a[i], b[i], w, wsh, q, q2);
      bfly<V>(a[i + 1], b[i + 1], w, wsh, q, q2);
      bfly<V>(a[i], a[i + 1], w, wsh, q, q2);
      bfly<V>(b[i], b[i + 1], w, wsh, q, q2);
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += a[i] ^ b[i];
  if (s == 0x1234567) out[0] = s;
}

// lazy key-switching term as in ksmac_v2: r += d w (mod 2^64), h += hi(d w'); one h q per 3 terms
template <int V>
__global__ void k_ks(const u64* __restrict__ prm, u64* out) {
  const u64 q = prm[0];
  u64 kv[3], ks[3];
#pragma unroll
  for (int i = 0; i < 3; i++) {
    kv[i] = (prm[1] + threadIdx.x * 7 + i) % q;
    ks[i] = (u64)(((u128)kv[i] << 64) / q);
  }
  u64 d[8];
#pragma unroll
  for (int t = 0; t < 8; t++) d[t] = (prm[2] * (threadIdx.x + 13 * t)) % q;
  u64 acc = 0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int t = 0; t < 8; t++) {
      u64 r = d[t], h = 0;
#pragma unroll
      for (int i = 0; i < 3; i++) {
        const u64 di = d[t] ^ (u64)i;  // three different digits
        r += di * kv[i];
        if constexpr (V == 0 || V == 3) h += hi_c(di, ks[i]);
        else if constexpr (V == 1) h += hi_ptx(di, ks[i]);
        else h += hi_apx(di, ks[i]);
      }
      if constexpr (V >= 3) r -= mulq_sp(h, (uint32_t)(q >> 32));
      else r -= h * q;
      d[t] = r & 0x0fffffffffffffffull;
      acc += r;
    }
  }
  if (acc == 0x1234567) out[0] = acc;
}

// ---- checks against exact arithmetic ----
template <int V>
__global__ void k_check(const u64* __restrict__ prm, const u64* xs, int n, int* bad) {
  const u64 q = prm[0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 x = xs[3 * i], w = xs[3 * i + 1] % q;
    const u64 wsh = (u64)(((u128)w << 64) / q);
    const u64 r = shoup<V>(x, w, wsh, q);
    const u64 lim = (V == 2 || V == 4) ? 5 * q : 2 * q;
    if (r >= lim || r % q != (u64)(((u128)x * w) % q)) atomicAdd(bad, 1);
    const u64 y = xs[3 * i + 2];
    if (hi_ptx(x, y) != __umul64hi(x, y)) atomicAdd(bad + 1, 1);
    const u64 ha = hi_apx(x, y), he = __umul64hi(x, y);
    if (ha > he || he - ha > 3) atomicAdd(bad + 2, 1);
  }
}

__global__ void k_check_bfly(const u64* __restrict__ prm, const u64* xs, int n, int* bad) {
  const u64 q = prm[0], q2 = 2 * q;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const u64 x = xs[3 * i] % (4 * q), y = xs[3 * i + 1] % (4 * q), w = xs[3 * i + 2] % q;
    const u64 wsh = (u64)(((u128)w << 64) / q);
    u64 a = x, b = y, c = x, d = y;
    bfly<0>(a, b, w, wsh, q, q2);
    bfly<9>(c, d, w, wsh, q, q2);
    if (a != c || b != d) atomicAdd(bad, 1);
  }
}

typedef void (*kfn)(const u64*, u64*);

static void run(const char* name, kfn f, double ops_per_thread, const u64* prm, u64* o) {
  const int blocks = 148 * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 3; r++) f<<<blocks, threads>>>(prm, o);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; r++) f<<<blocks, threads>>>(prm, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * ops_per_thread * reps;
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double per_s = ops / (ms * 1e-3);
  printf("{\"op\": \"%s\", \"ops_per_s\": %.4e, \"per_clk_per_sm_at_maxclk\": %.3f}\n", name, per_s,
         per_s / (148 * (double)clk_khz * 1e3));
}

int main(int argc, char** argv) {
  // q: a 60-bit prime = 1 mod 2^32 when argv[1] == "sp", else the round-1 style q = 1 mod 2^14
  const bool sp = argc > 1 && argv[1][0] == 's';
  u64 h_prm[4] = {sp ? 0xfffffa000000001ull : 0xfffffffffffc001ull, 0x0123456789abcdeull, 0x9E3779B97F4A7C15ull,
                  0xC2B2AE3D27D4EB4Full};
  u64 *prm, *o, *xs;
  int* bad;
  cudaMalloc(&prm, sizeof h_prm);
  cudaMemcpy(prm, h_prm, sizeof h_prm, cudaMemcpyHostToDevice);
  cudaMalloc(&o, 64);
  const int n = 1 << 22;
  u64* hx = (u64*)malloc(3 * (size_t)n * 8);
  u64 s = 88172645463325252ull;
  for (size_t i = 0; i < 3 * (size_t)n; i++) {
    s ^= s << 13, s ^= s >> 7, s ^= s << 17;
    hx[i] = (i % 97 == 0) ? ~0ull - (s & 0xff) : s;  // include values near 2^64
  }
  cudaMalloc(&xs, 3 * (size_t)n * 8);
  cudaMemcpy(xs, hx, 3 * (size_t)n * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&bad, 12);
  int hb[3];
#define CHECK(V)                                                                                     \
  cudaMemset(bad, 0, 12);                                                                            \
  k_check<V><<<592, 256>>>(prm, xs, n, bad);                                                         \
  cudaMemcpy(hb, bad, 12, cudaMemcpyDeviceToHost);                                                   \
  printf("{\"check\": \"shoup<%d>\", \"q\": \"%llx\", \"bad\": %d, \"bad_hi_ptx\": %d, \"bad_hi_apx\": %d}\n", V, \
         (unsigned long long)h_prm[0], hb[0], hb[1], hb[2]);
  CHECK(0) CHECK(1) CHECK(2)
  if (sp) { CHECK(3) CHECK(4) }
  cudaMemset(bad, 0, 12);
  k_check_bfly<<<592, 256>>>(prm, xs, n, bad);
  cudaMemcpy(hb, bad, 12, cudaMemcpyDeviceToHost);
  printf("{\"check\": \"bfly_ptx_full == bfly_c\", \"bad\": %d}\n", hb[0]);
  const double nb = (double)ITERS * 16, nk = (double)ITERS * 8 * 3;
  run("bfly_ptx_full", k_bfly<9>, nb, prm, o);
  run("bfly_c", k_bfly<0>, nb, prm, o);
  run("bfly_ptx", k_bfly<1>, nb, prm, o);
  run("ks_c", k_ks<0>, nk, prm, o);
  run("ks_ptx", k_ks<1>, nk, prm, o);
  run("ks_apx", k_ks<2>, nk, prm, o);
  if (sp) {
    run("bfly_sp", k_bfly<3>, nb, prm, o);
    run("ks_sp", k_ks<3>, nk, prm, o);
    run("ks_apx_sp", k_ks<4>, nk, prm, o);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
