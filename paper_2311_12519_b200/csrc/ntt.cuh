// Negacyclic NTT / INTT over Z_q[X]/(X^N+1) per RNS limb, q < 2^60 (fits Harvey's [0,4q) lazy range).
//
// Why an NTT at all: the paper's HRot is key switching, whose polynomial products the
// paper's SEAL baseline performs in NTT form ("decomposing ciphertext and converting them
// to NTT space", PAPER.md:1472 [app]; NTT requires q = 1 mod 2n).
//
// Schedule (one CTA per polynomial-limb, N/16 threads, 16 coefficients per thread):
//   forward  (Cooley-Tukey, natural order in -> bit-reversed order out): stages with span
//            t = N/2, N/4, ..., 1 processed in register groups of 4 stages (radix-16);
//            a remainder group of LOGN % 4 stages handles the smallest spans.
//   inverse  (Gentleman-Sande, bit-reversed in -> natural out): the mirror schedule,
//            followed by the N^{-1} scaling.
// Between groups the coefficients are exchanged through shared memory padded by one word
// per 16 (index k -> k + k/16) so the small-span groups are bank-conflict free.
// Output slot k of the forward transform holds a(psi^{2 bitrev(k) + 1}).
//
// Twiddles: psi_rev[m + i] = psi^{bitrev(m + i)} with Shoup companions (per limb tables).
// Butterflies keep Harvey's lazy ranges: forward values in [0, 4q), inverse in [0, 2q).
#pragma once

#include "hy_common.cuh"

struct LimbConsts {
  LimbConst lc[HY_MAX_LIMBS];
};

__device__ __forceinline__ int smem_pad(int k) { return k + (k >> 4); }

__device__ __forceinline__ void ct_bfly(u64& x, u64& y, u64 w, u64 wsh, u64 q, u64 q2) {
  // Harvey CT butterfly: x, y in [0, 4q) -> x + w y, x - w y in [0, 4q)
  u64 X = csub(x, q2);
  u64 T = shoup_mul(y, w, wsh, q);
  x = X + T;
  y = X - T + q2;
}

__device__ __forceinline__ void gs_bfly(u64& x, u64& y, u64 w, u64 wsh, u64 q2) {
  // Harvey GS butterfly: x, y in [0, 2q) -> x + y, (x - y) w in [0, 2q)
  u64 U = csub(x + y, q2);
  u64 V = x - y + q2;
  y = shoup_mul(V, w, wsh, q2 >> 1);
  x = U;
}

// ---------------------------------------------------------------------------------------
// forward transform; Job: bind(block) sets `limb`; load(k) returns a value in [0, 4q);
// store(k, v) receives canonical v in [0, q).
// ---------------------------------------------------------------------------------------
template <int LOGN, class Job>
__global__ void __launch_bounds__((1 << LOGN) / 16) ntt_fwd_kernel(Job job, DevTables tab, LimbConsts L) {
  constexpr int N = 1 << LOGN;
  constexpr int T = N / 16;
  constexpr int FULL = LOGN / 4;
  constexpr int REM = LOGN % 4;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  Job jb = job;
  jb.bind(blockIdx.x);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const u64* __restrict__ W = tab.psi_rev + (size_t)l * N;
  const u64* __restrict__ Ws = tab.psi_rev_sh + (size_t)l * N;
  u64 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = jb.load(tid + r * T);

  int thi = N / 2;
#pragma unroll
  for (int gi = 0; gi < FULL; gi++) {
    const int delta = thi >> 3;
    const int base = (tid / delta) * (16 * delta) + (tid % delta);
    if (gi > 0) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = sm[smem_pad(base + r * delta)];
    }
#pragma unroll
    for (int s = 0; s < 4; s++) {
      const int t = thi >> s;
      const int step = 8 >> s;
      const int m = N / (2 * t);
#pragma unroll
      for (int r = 0; r < 16; r++) {
        if ((r & step) == 0) {
          const int j = base + r * delta;
          const int widx = m + j / (2 * t);
          ct_bfly(v[r], v[r + step], __ldg(W + widx), __ldg(Ws + widx), q, q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; r++) sm[smem_pad(base + r * delta)] = v[r];
    __syncthreads();
    thi >>= 4;
  }
  if constexpr (REM > 0) {
    // spans 2^{REM-1} .. 1 over 16 consecutive coefficients per thread
    const int base = 16 * tid;
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = sm[smem_pad(base + r)];
#pragma unroll
    for (int s = 0; s < REM; s++) {
      const int t = (1 << (REM - 1)) >> s;
      const int m = N / (2 * t);
#pragma unroll
      for (int r = 0; r < 16; r++) {
        if ((r & t) == 0) {
          const int j = base + r;
          const int widx = m + j / (2 * t);
          ct_bfly(v[r], v[r + t], __ldg(W + widx), __ldg(Ws + widx), q, q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; r++) sm[smem_pad(base + r)] = v[r];
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = tid + r * T;
    u64 x = sm[smem_pad(k)];
    x = csub(x, q2);
    x = csub(x, q);
    jb.store(k, x);
  }
}

// ---------------------------------------------------------------------------------------
// inverse transform; Job: bind(block) sets `limb`; load(k) returns a value in [0, 2q);
// store(k, v) receives canonical v in [0, q).
// ---------------------------------------------------------------------------------------
template <int LOGN, class Job>
__global__ void __launch_bounds__((1 << LOGN) / 16) ntt_inv_kernel(Job job, DevTables tab, LimbConsts L) {
  constexpr int N = 1 << LOGN;
  constexpr int T = N / 16;
  constexpr int FULL = LOGN / 4;
  constexpr int REM = LOGN % 4;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  Job jb = job;
  jb.bind(blockIdx.x);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const u64* __restrict__ W = tab.ipsi_rev + (size_t)l * N;
  const u64* __restrict__ Ws = tab.ipsi_rev_sh + (size_t)l * N;
  u64 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k = tid + r * T;
    sm[smem_pad(k)] = jb.load(k);
  }
  __syncthreads();

  int tlo = 1;
  if constexpr (REM > 0) {
    const int base = 16 * tid;
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = sm[smem_pad(base + r)];
#pragma unroll
    for (int s = 0; s < REM; s++) {
      const int t = 1 << s;
      const int h = N / (2 * t);
#pragma unroll
      for (int r = 0; r < 16; r++) {
        if ((r & t) == 0) {
          const int j = base + r;
          const int widx = h + j / (2 * t);
          gs_bfly(v[r], v[r + t], __ldg(W + widx), __ldg(Ws + widx), q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 16; r++) sm[smem_pad(base + r)] = v[r];
    __syncthreads();
    tlo = 1 << REM;
  }
#pragma unroll
  for (int gi = 0; gi < FULL; gi++) {
    const int delta = tlo;  // thi / 8 with thi = 8 tlo
    const int base = (tid / delta) * (16 * delta) + (tid % delta);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = sm[smem_pad(base + r * delta)];
#pragma unroll
    for (int s = 0; s < 4; s++) {
      const int t = tlo << s;
      const int step = 1 << s;
      const int h = N / (2 * t);
#pragma unroll
      for (int r = 0; r < 16; r++) {
        if ((r & step) == 0) {
          const int j = base + r * delta;
          const int widx = h + j / (2 * t);
          gs_bfly(v[r], v[r + step], __ldg(W + widx), __ldg(Ws + widx), q2);
        }
      }
    }
    if (gi + 1 < FULL) {
#pragma unroll
      for (int r = 0; r < 16; r++) sm[smem_pad(base + r * delta)] = v[r];
      __syncthreads();
    } else {
      // last group: delta = N/16, base = tid -> coefficient tid + r N/16; scale by N^{-1}
      const u64 ni = L.lc[l].ninv, nis = L.lc[l].ninv_sh;
#pragma unroll
      for (int r = 0; r < 16; r++) {
        u64 x = shoup_mul(v[r], ni, nis, q);
        jb.store(base + r * delta, csub(x, q));
      }
    }
    tlo <<= 4;
  }
}

// ---------------------------------------------------------------------------------------
// automorphism X -> X^g in the bit-reversed NTT domain:
// out[k] = in[perm(k)], 2 bitrev(perm(k)) + 1 = (2 bitrev(k) + 1) g  (mod 2N)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int auto_perm(int k, uint32_t g, int logN) {
  const uint32_t twoN_mask = (2u << logN) - 1u;
  uint32_t e = ((__brev((uint32_t)k) >> (32 - logN)) * 2u + 1u) * g & twoN_mask;
  return (int)(__brev((e - 1u) >> 1) >> (32 - logN));
}

template <int LOGN>
inline size_t ntt_smem_bytes() {
  return (size_t)((1 << LOGN) + (1 << LOGN) / 16) * sizeof(u64);
}
