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
// Butterfly position k of the forward transform holds a(psi^{2 bitrev(k) + 1}); the kernels
// store (and the inverse loads) in SLOT ORDER instead: global position j holds the evaluation
// at psi^{e_j}, e_j = 3^j (j < N/2) or -3^{j-N/2} (j >= N/2) mod 2N, through the table
// k_of_slot (the permutation is applied between shared memory and HBM, so it is free).  In slot
// order every Galois automorphism X -> X^{(+/-)3^s} is a cyclic shift by s inside each half,
// plus a half exchange for the minus sign — PermAuto reads become streams.
//
// Twiddles: psi_rev[m + i] = psi^{bitrev(m + i)} with Shoup companions (per limb tables).
// Butterflies keep Harvey's lazy ranges: forward values in [0, 4q), inverse in [0, 2q).
#pragma once

#include <cooperative_groups.h>

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
// Kernel geometry.  A transform of N = S * B coefficients runs on S CTAs of T = B / 8 threads
// (B = min(N, 4096), 8 values per thread, radix-8 register groups between shared-memory
// exchanges).  Forward (Cooley-Tukey, natural in): after its first log2(S) stages the array
// splits into S independent blocks, so CTA h recomputes those stages for block h only from the S
// inputs x[r + h'B] (one extra Shoup product per value at S = 2) and then transforms its block
// alone.  Inverse (Gentleman-Sande, slot order in): CTA h transforms block h, then the S CTAs of
// a thread-block cluster exchange through distributed shared memory for the last log2(S)
// stages.  Splitting halves (S = 2) the single-transform latency at N = 8192 and keeps every
// CTA at 512 threads x <= 64 registers (3 CTAs / SM by registers).
// ---------------------------------------------------------------------------------------
template <int LOGN>
struct NttCfg {
  static constexpr int LOGS = LOGN > 12 ? LOGN - 12 : 0;
  static constexpr int S = 1 << LOGS;
  static constexpr int LOGB = LOGN - LOGS;
  static constexpr int B = 1 << LOGB;
  static constexpr int LOGV = 3;
  static constexpr int V = 1 << LOGV;
  static constexpr int T = B / V;
  static constexpr int FULL = LOGB / LOGV;
  static constexpr int REM = LOGB % LOGV;
};

// ---------------------------------------------------------------------------------------
// forward transform; Job: bind(poly) sets `limb`; load(k) (coefficient k) returns a value in
// [0, 4q); store(j, v) receives canonical v in [0, q) for slot-order position j.
// tab.own_j / own_k: slot positions owned by block h (ascending) and their in-block butterfly
// position, [S][B] each.
// ---------------------------------------------------------------------------------------
template <int LOGN, class Job>
__global__ void __launch_bounds__(NttCfg<LOGN>::T) ntt_fwd_kernel(Job job, DevTables tab, LimbConsts L) {
  pdl_begin();
  using C = NttCfg<LOGN>;
  constexpr int S = C::S, B = C::B, V = C::V, T = C::T;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  const int h = blockIdx.x % S;
  Job jb = job;
  jb.bind(blockIdx.x / S);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const u64* __restrict__ W = tab.psi_rev + ((size_t)l << LOGN);
  const u64* __restrict__ Ws = tab.psi_rev_sh + ((size_t)l << LOGN);
  u64 v[V];
#pragma unroll
  for (int r = 0; r < V; r++) {
    const int rr = tid + r * T;
    if constexpr (S == 1) {
      v[r] = jb.load(rr);
    } else {
      u64 y[S];
#pragma unroll
      for (int g = 0; g < S; g++) y[g] = jb.load(rr + g * B);
#pragma unroll
      for (int st = 0; st < C::LOGS; st++) {
        const int m = 1 << st, span = S / (2 * m);
#pragma unroll
        for (int g = 0; g < S; g++)
          if ((g & span) == 0) {
            const int widx = m + g / (2 * span);
            ct_bfly(y[g], y[g + span], __ldg(W + widx), __ldg(Ws + widx), q, q2);
          }
      }
      v[r] = y[0];
#pragma unroll
      for (int g = 1; g < S; g++)
        if (g == h) v[r] = y[g];
    }
  }
  // local stages: global stage with m = S m_loc blocks uses twiddle m_loc (S + h) + i_loc
  int thi = B / 2;
#pragma unroll
  for (int gi = 0; gi < C::FULL; gi++) {
    const int delta = thi >> (C::LOGV - 1);
    const int base = (tid / delta) * (V * delta) + (tid % delta);
    if (gi > 0) {
#pragma unroll
      for (int r = 0; r < V; r++) v[r] = sm[smem_pad(base + r * delta)];
    }
#pragma unroll
    for (int s = 0; s < C::LOGV; s++) {
      const int t = thi >> s;
      const int step = (V / 2) >> s;
      const int mloc = B / (2 * t);
#pragma unroll
      for (int r = 0; r < V; r++) {
        if ((r & step) == 0) {
          const int j = base + r * delta;
          const int widx = mloc * (S + h) + j / (2 * t);
          ct_bfly(v[r], v[r + step], __ldg(W + widx), __ldg(Ws + widx), q, q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < V; r++) sm[smem_pad(base + r * delta)] = v[r];
    __syncthreads();
    thi >>= C::LOGV;
  }
  if constexpr (C::REM > 0) {
    const int base = V * tid;
#pragma unroll
    for (int r = 0; r < V; r++) v[r] = sm[smem_pad(base + r)];
#pragma unroll
    for (int s = 0; s < C::REM; s++) {
      const int t = (1 << (C::REM - 1)) >> s;
      const int mloc = B / (2 * t);
#pragma unroll
      for (int r = 0; r < V; r++) {
        if ((r & t) == 0) {
          const int j = base + r;
          const int widx = mloc * (S + h) + j / (2 * t);
          ct_bfly(v[r], v[r + t], __ldg(W + widx), __ldg(Ws + widx), q, q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < V; r++) sm[smem_pad(base + r)] = v[r];
    __syncthreads();
  }
  const int32_t* __restrict__ oj = tab.own_j + h * B;
  const int32_t* __restrict__ ok = tab.own_k + h * B;
#pragma unroll
  for (int r = 0; r < V; r++) {
    const int idx = tid + r * T;
    u64 x = sm[smem_pad(__ldg(ok + idx))];
    x = csub(x, q2);
    x = csub(x, q);
    jb.store(__ldg(oj + idx), x);
  }
}

// ---------------------------------------------------------------------------------------
// inverse transform; Job: bind(poly) sets `limb`; load(j) (slot order) returns a value in
// [0, 2q); store(k, v) receives canonical v in [0, q) for coefficient k.  Launched in clusters
// of S CTAs.
// ---------------------------------------------------------------------------------------
template <int LOGN, class Job>
__global__ void __launch_bounds__(NttCfg<LOGN>::T) ntt_inv_kernel(Job job, DevTables tab, LimbConsts L) {
  pdl_begin();
  using C = NttCfg<LOGN>;
  constexpr int S = C::S, B = C::B, V = C::V, T = C::T;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  const int h = blockIdx.x % S;
  Job jb = job;
  jb.bind(blockIdx.x / S);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const u64* __restrict__ W = tab.ipsi_rev + ((size_t)l << LOGN);
  const u64* __restrict__ Ws = tab.ipsi_rev_sh + ((size_t)l << LOGN);
  u64 v[V];
  {
    const int32_t* __restrict__ oj = tab.own_j + h * B;
    const int32_t* __restrict__ ok = tab.own_k + h * B;
#pragma unroll
    for (int r = 0; r < V; r++) {
      const int idx = tid + r * T;
      sm[smem_pad(__ldg(ok + idx))] = jb.load(__ldg(oj + idx));
    }
  }
  __syncthreads();

  // local stages: span t < B; global twiddle index (B / 2t)(S + h) + j / 2t
  int tlo = 1;
  if constexpr (C::REM > 0) {
    const int base = V * tid;
#pragma unroll
    for (int r = 0; r < V; r++) v[r] = sm[smem_pad(base + r)];
#pragma unroll
    for (int s = 0; s < C::REM; s++) {
      const int t = 1 << s;
      const int mloc = B / (2 * t);
#pragma unroll
      for (int r = 0; r < V; r++) {
        if ((r & t) == 0) {
          const int j = base + r;
          const int widx = mloc * (S + h) + j / (2 * t);
          gs_bfly(v[r], v[r + t], __ldg(W + widx), __ldg(Ws + widx), q2);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < V; r++) sm[smem_pad(base + r)] = v[r];
    __syncthreads();
    tlo = 1 << C::REM;
  }
#pragma unroll
  for (int gi = 0; gi < C::FULL; gi++) {
    const int delta = tlo;
    const int base = (tid / delta) * (V * delta) + (tid % delta);
#pragma unroll
    for (int r = 0; r < V; r++) v[r] = sm[smem_pad(base + r * delta)];
#pragma unroll
    for (int s = 0; s < C::LOGV; s++) {
      const int t = tlo << s;
      const int step = 1 << s;
      const int mloc = B / (2 * t);
#pragma unroll
      for (int r = 0; r < V; r++) {
        if ((r & step) == 0) {
          const int j = base + r * delta;
          const int widx = mloc * (S + h) + j / (2 * t);
          gs_bfly(v[r], v[r + step], __ldg(W + widx), __ldg(Ws + widx), q2);
        }
      }
    }
    if (S > 1 || gi + 1 < C::FULL) {
#pragma unroll
      for (int r = 0; r < V; r++) sm[smem_pad(base + r * delta)] = v[r];
      __syncthreads();
    } else {
      // last group of an unsplit transform: delta = B / V, base = tid -> coefficient tid + r T
      const u64 ni = L.lc[l].ninv, nis = L.lc[l].ninv_sh;
#pragma unroll
      for (int r = 0; r < V; r++) {
        u64 x = shoup_mul(v[r], ni, nis, q);
        jb.store(base + r * delta, csub(x, q));
      }
    }
    tlo <<= C::LOGV;
  }
  if constexpr (S > 1) {
    // cross-block stages (span t = span_b B): values of the S blocks at offset r through DSMEM
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    u64* peer[S];
#pragma unroll
    for (int g = 0; g < S; g++) peer[g] = cl.map_shared_rank(sm, g);
    const u64 ni = L.lc[l].ninv, nis = L.lc[l].ninv_sh;
#pragma unroll
    for (int r = 0; r < V; r++) {
      const int rr = tid + r * T;
      u64 y[S];
#pragma unroll
      for (int g = 0; g < S; g++) y[g] = peer[g][smem_pad(rr)];
#pragma unroll
      for (int st = 0; st < C::LOGS; st++) {
        const int span = 1 << st;
#pragma unroll
        for (int g = 0; g < S; g++)
          if ((g & span) == 0) {
            const int widx = S / (2 * span) + g / (2 * span);
            gs_bfly(y[g], y[g + span], __ldg(W + widx), __ldg(Ws + widx), q2);
          }
      }
      u64 x = y[0];
#pragma unroll
      for (int g = 1; g < S; g++)
        if (g == h) x = y[g];
      x = shoup_mul(x, ni, nis, q);
      jb.store(h * B + rr, csub(x, q));
    }
    cl.sync();  // peers may still read this CTA's shared memory
  }
}

// ---------------------------------------------------------------------------------------
// automorphism X -> X^g on a slot-ordered NTT vector: out[j] = in[galois_perm(j)]
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int galois_perm(int j, GaloisAct a, int half) {
  return ((j + (int)a.shift) & (half - 1)) | ((j & half) ^ (a.swap ? half : 0));
}

template <int LOGN>
inline size_t ntt_smem_bytes() {
  constexpr int B = NttCfg<LOGN>::B;
  return (size_t)(B + B / 16) * sizeof(u64);
}

// =======================================================================================
// One-CTA-per-transform NTT for N = 4096 / 8192 (the ring degrees of every N <= 8192 config):
// T = N / 32 threads x 32 coefficients per thread, three register groups of butterfly stages
// (5 + 5 + LOGN - 10 stages) separated by two shared-memory exchanges, plus one exchange that
// applies the slot-order permutation.  Compared with ntt_fwd_kernel: no recomputed first stage,
// 2 (not 4) exchanges, twiddles (w, w') as one 16-byte load, uniform (broadcast) twiddles in the
// first group, and an XOR swizzle instead of padding (every exchange pattern is bank-conflict
// free for 64-bit words, checked exhaustively for both N).
//   group A (stages 0..4):  thread tid holds coefficients j = tid + T r           (r < 32)
//   group B (stages 5..9):  j = (tid / D) 32 D + tid % D + D r,  D = N / 1024
//   group C (stages 10..):  j = D (tid + T q) + r',  q < 32 / D, r' < D (D-point sub-blocks)
// Twiddles: psi2[l][m + i] = (psi^{bitrev(m + i)}, Shoup companion) for the butterflies of block i
// of stage log2 m (inverse: ipsi2 with psi^{-1}).  Forward values stay in Harvey's [0, 4q); the
// inverse keeps [0, 2q) and folds N^{-1} into its last stage.
// =======================================================================================
#ifndef NTT2_APX
#define NTT2_APX 0
#endif
#ifndef NTT2_PTX
#define NTT2_PTX 1
#endif
#ifndef NTT2_Q1
#define NTT2_Q1 0
#endif
#ifndef NTT2_LAZY  // forward transform: conditional subtraction on every other stage only (needs NTT2_PTX, not NTT2_APX); bit-exact, measured no faster (C4 S1 4.39 vs 4.37 ms): off
#define NTT2_LAZY 0
#endif
#ifndef NTT2_MINB  // resident CTAs per SM asked of ptxas at N = 8192 (2: 128 registers; 3: 80 registers, spills)
#define NTT2_MINB 2
#endif
#ifndef NTT2_EXP  // timing experiments only (wrong results), bit mask: 1 = no butterfly arithmetic, 2 = no global loads / stores, 4 = no twiddle loads
#define NTT2_EXP 0
#endif
// Butterflies on 32-bit halves (inline PTX).  The C form compiled to ~40 SASS per butterfly (register
// moves on the FMA pipe, IMAD.X adds, compare + select pairs); these are ~21: the exact Shoup
// quotient H = hi64(y w') from four 32-bit partial products, T = y w + H (2^64 - q) (mod 2^64) as
// accumulating multiply-adds, and every conditional subtraction as subtract-with-borrow + LOP3 select.
//   CT (forward, Harvey): x, y in [0, 4q) -> x' = X + T, y' = X - T + 2q, X = x mod' 2q, T in [0, 2q)
//   GS (inverse):         x, y in [0, 2q) -> x' = (x + y) mod' 2q, y' = Shoup(x - y + 2q) in [0, 2q)
#if NTT2_APX  // approximate quotient y1 s1 + hi32(y1 s0) + hi32(y0 s1): undershoots by <= 3, T in [0, 5q)
#define NTT2_SHOUP_H(Y0, Y1)                                       \
  "mul.lo.u32 h0, " Y1 ", s1;\n\t"                                \
  "mul.hi.u32 h1, " Y1 ", s1;\n\t"                                \
  "mad.hi.cc.u32 h0, " Y1 ", s0, h0;\n\t"                         \
  "addc.u32 h1, h1, 0;\n\t"                                       \
  "mad.hi.cc.u32 h0, " Y0 ", s1, h0;\n\t"                         \
  "addc.u32 h1, h1, 0;\n\t"
#else
#define NTT2_SHOUP_H(Y0, Y1)                                       \
  "mul.hi.u32 a0, " Y0 ", s0;\n\t"                                \
  "mad.lo.cc.u32 a0, " Y0 ", s1, a0;\n\t"                         \
  "madc.hi.u32 a1, " Y0 ", s1, 0;\n\t"                            \
  "mad.lo.cc.u32 a0, " Y1 ", s0, a0;\n\t"                         \
  "madc.hi.cc.u32 a1, " Y1 ", s0, a1;\n\t"                        \
  "addc.u32 a2, 0, 0;\n\t"                                        \
  "mad.lo.cc.u32 h0, " Y1 ", s1, a1;\n\t"                         \
  "madc.hi.u32 h1, " Y1 ", s1, a2;\n\t"
#endif
#if NTT2_Q1  // q = 1 mod 2^32: H q = H + (H0 q1) 2^32 (mod 2^64); n1 = -q1 mod 2^32
#define NTT2_SHOUP_T(Y0, Y1)                                       \
  NTT2_SHOUP_H(Y0, Y1)                                             \
  "mul.lo.u32 T0, " Y0 ", w0;\n\t"                                \
  "mul.hi.u32 T1, " Y0 ", w0;\n\t"                                \
  "mad.lo.u32 T1, " Y0 ", w1, T1;\n\t"                            \
  "mad.lo.u32 T1, " Y1 ", w0, T1;\n\t"                            \
  "sub.cc.u32 T0, T0, h0;\n\t"                                    \
  "subc.u32 T1, T1, h1;\n\t"                                      \
  "mad.lo.u32 T1, h0, n1, T1;\n\t"
#else
#define NTT2_SHOUP_T(Y0, Y1)                                       \
  NTT2_SHOUP_H(Y0, Y1)                                             \
  "mul.lo.u32 T0, " Y0 ", w0;\n\t"                                \
  "mul.hi.u32 T1, " Y0 ", w0;\n\t"                                \
  "mad.lo.u32 T1, " Y0 ", w1, T1;\n\t"                            \
  "mad.lo.u32 T1, " Y1 ", w0, T1;\n\t"                            \
  "mad.lo.cc.u32 T0, h0, n0, T0;\n\t"                             \
  "madc.hi.u32 T1, h0, n0, T1;\n\t"                               \
  "mad.lo.u32 T1, h0, n1, T1;\n\t"                                \
  "mad.lo.u32 T1, h1, n0, T1;\n\t"
#endif
// nq operand: 2^64 - q (generic), or (-q1 mod 2^32) << 32 (NTT2_Q1)
__device__ __forceinline__ u64 ntt2_nq(u64 q) {
#if NTT2_Q1
  return (u64)(0u - (uint32_t)(q >> 32)) << 32;
#else
  return 0 - q;
#endif
}

__device__ __forceinline__ void ntt2_ct_ptx(u64& x, u64& y, u64 w, u64 ws, u64 nq, u64 q2) {
  asm("{\n\t.reg .u32 x0, x1, y0, y1, w0, w1, s0, s1, n0, n1, t0, t1, a0, a1, a2, h0, h1, T0, T1, d0, d1, m;\n\t"
      "mov.b64 {x0, x1}, %0;\n\tmov.b64 {y0, y1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\tmov.b64 {t0, t1}, %5;\n\t"
      NTT2_SHOUP_T("y0", "y1")
      "sub.cc.u32 d0, x0, t0;\n\tsubc.cc.u32 d1, x1, t1;\n\tsubc.u32 m, 0, 0;\n\t"
      "lop3.b32 x0, m, x0, d0, 0xCA;\n\tlop3.b32 x1, m, x1, d1, 0xCA;\n\t"
      "add.cc.u32 d0, x0, t0;\n\taddc.u32 d1, x1, t1;\n\t"
      "sub.cc.u32 y0, d0, T0;\n\tsubc.u32 y1, d1, T1;\n\t"
      "add.cc.u32 x0, x0, T0;\n\taddc.u32 x1, x1, T1;\n\t"
      "mov.b64 %0, {x0, x1};\n\tmov.b64 %1, {y0, y1};\n\t}"
      : "+l"(x), "+l"(y)
      : "l"(w), "l"(ws), "l"(nq), "l"(q2));
}

// Forward butterfly with the conditional subtraction on every other stage only (NTT2_LAZY): a Shoup
// product takes any 64-bit y, so the values may grow by 2q per stage: [0, 4q) in, no correction in
// stages 0, 1 and every odd stage (values < 8q < 2^63), x mod' 4q in the even stages >= 2 (values
// back below 6q); the output is normalised from [0, 8q).  cs is a compile-time constant after unrolling.
__device__ __forceinline__ void ntt2_ct_lazy(u64& x, u64& y, u64 w, u64 ws, u64 nq, u64 q2, u64 q4, bool cs) {
  if (cs) {
    asm("{\n\t.reg .u32 x0, x1, y0, y1, w0, w1, s0, s1, n0, n1, t0, t1, f0, f1, a0, a1, a2, h0, h1, T0, T1, d0, d1, m;\n\t"
        "mov.b64 {x0, x1}, %0;\n\tmov.b64 {y0, y1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\tmov.b64 {t0, t1}, %5;\n\tmov.b64 {f0, f1}, %6;\n\t"
        NTT2_SHOUP_T("y0", "y1")
        "sub.cc.u32 d0, x0, f0;\n\tsubc.cc.u32 d1, x1, f1;\n\tsubc.u32 m, 0, 0;\n\t"
        "lop3.b32 x0, m, x0, d0, 0xCA;\n\tlop3.b32 x1, m, x1, d1, 0xCA;\n\t"
        "add.cc.u32 d0, x0, t0;\n\taddc.u32 d1, x1, t1;\n\t"
        "sub.cc.u32 y0, d0, T0;\n\tsubc.u32 y1, d1, T1;\n\t"
        "add.cc.u32 x0, x0, T0;\n\taddc.u32 x1, x1, T1;\n\t"
        "mov.b64 %0, {x0, x1};\n\tmov.b64 %1, {y0, y1};\n\t}"
        : "+l"(x), "+l"(y)
        : "l"(w), "l"(ws), "l"(nq), "l"(q2), "l"(q4));
  } else {
    asm("{\n\t.reg .u32 x0, x1, y0, y1, w0, w1, s0, s1, n0, n1, t0, t1, a0, a1, a2, h0, h1, T0, T1, d0, d1;\n\t"
        "mov.b64 {x0, x1}, %0;\n\tmov.b64 {y0, y1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\t"
        "mov.b64 {n0, n1}, %4;\n\tmov.b64 {t0, t1}, %5;\n\t"
        NTT2_SHOUP_T("y0", "y1")
        "add.cc.u32 d0, x0, t0;\n\taddc.u32 d1, x1, t1;\n\t"
        "sub.cc.u32 y0, d0, T0;\n\tsubc.u32 y1, d1, T1;\n\t"
        "add.cc.u32 x0, x0, T0;\n\taddc.u32 x1, x1, T1;\n\t"
        "mov.b64 %0, {x0, x1};\n\tmov.b64 %1, {y0, y1};\n\t}"
        : "+l"(x), "+l"(y)
        : "l"(w), "l"(ws), "l"(nq), "l"(q2));
  }
}

__device__ __forceinline__ void ntt2_gs_ptx(u64& x, u64& y, u64 w, u64 ws, u64 nq, u64 q2) {
  asm("{\n\t.reg .u32 x0, x1, y0, y1, w0, w1, s0, s1, n0, n1, t0, t1, a0, a1, a2, h0, h1, T0, T1, d0, d1, v0, v1, m;\n\t"
      "mov.b64 {x0, x1}, %0;\n\tmov.b64 {y0, y1}, %1;\n\tmov.b64 {w0, w1}, %2;\n\tmov.b64 {s0, s1}, %3;\n\t"
      "mov.b64 {n0, n1}, %4;\n\tmov.b64 {t0, t1}, %5;\n\t"
      "add.cc.u32 v0, x0, t0;\n\taddc.u32 v1, x1, t1;\n\t"
      "sub.cc.u32 v0, v0, y0;\n\tsubc.u32 v1, v1, y1;\n\t"
      "add.cc.u32 x0, x0, y0;\n\taddc.u32 x1, x1, y1;\n\t"
      "sub.cc.u32 d0, x0, t0;\n\tsubc.cc.u32 d1, x1, t1;\n\tsubc.u32 m, 0, 0;\n\t"
      "lop3.b32 x0, m, x0, d0, 0xCA;\n\tlop3.b32 x1, m, x1, d1, 0xCA;\n\t"
      NTT2_SHOUP_T("v0", "v1")
      "mov.b64 %0, {x0, x1};\n\tmov.b64 %1, {T0, T1};\n\t}"
      : "+l"(x), "+l"(y)
      : "l"(w), "l"(ws), "l"(nq), "l"(q2));
}

#if NTT2_EXP & 4
#define NTT2_TW(p) make_ulonglong2((u64)(size_t)(p), 12345)
#else
#define NTT2_TW(p) __ldg(p)
#endif
#ifndef NTT2_PRE  // 1: L1 prefetch of the next register group's twiddles before each barrier (measured slower: S1 4.37 -> 4.49 ms)
#define NTT2_PRE 0
#endif
__device__ __forceinline__ void ntt2_pf(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// twiddles of group B (stages 5..9) of block `blk`: 2^{s-5} consecutive entries per stage, shared by the
// D threads of the block -> lane d of the block prefetches one 128-byte line
template <int LOGN>
__device__ __forceinline__ void ntt2_pf_groupB(const ulonglong2* W, int tid) {
  constexpr int D = 1 << (LOGN - 10);
  const int blk = tid / D, d = tid % D;
  if (d < 2) ntt2_pf(W + (1 << 9) + (blk << 4) + 8 * d);
  else if (d == 2) ntt2_pf(W + (1 << 8) + (blk << 3));
  else if (d == 3) ntt2_pf(W + (1 << 7) + (blk << 2));
  if (D <= 4 || d == 4) ntt2_pf(W + (1 << 6) + (blk << 1));
  if (D <= 4 || d == 5) ntt2_pf(W + (1 << 5) + blk);
}
// twiddles of group C (stages 10..LOGN-1) of this thread's sub-blocks
template <int LOGN>
__device__ __forceinline__ void ntt2_pf_groupC(const ulonglong2* W, int tid) {
  constexpr int T = 1 << (LOGN - 5), D = 1 << (LOGN - 10), QN = 32 / D;
#pragma unroll
  for (int s = 10; s < LOGN; s++)
#pragma unroll
    for (int qq = 0; qq < QN; qq++) ntt2_pf(W + (1 << s) + ((tid + T * qq) << (s - 10)));
}
template <int LOGN>
struct Ntt2Cfg {
  static constexpr int LOGV = 5, V = 32;
  static constexpr int LOGT = LOGN - LOGV, T = 1 << LOGT;
  static constexpr int LOGD = LOGN - 2 * LOGV, D = 1 << LOGD;
  static constexpr int QN = V / D;  // sub-blocks per thread in group C
};

template <int LOGN>
__device__ __forceinline__ int ntt2_sw(int k) {
  if constexpr (LOGN == 13) return k ^ ((k >> 4) & 7) ^ (((k >> 8) & 1) << 3);
  else return k ^ ((k >> 4) & 3) ^ (((k >> 7) & 3) << 2);
}

struct Ntt2Tables {
  const ulonglong2* tw;   // [L][N] (w, w') forward (psi) or inverse (psi^{-1})
  const int32_t* kos;     // [N] bit-reversed butterfly position of slot j
};

__device__ __forceinline__ u64 csub2(u64 x, u64 m) { return x >= m ? x - m : x; }

template <int LOGN, class Job>
__global__ void __launch_bounds__(Ntt2Cfg<LOGN>::T, (LOGN == 13 ? NTT2_MINB : 2 * NTT2_MINB))
    ntt2_fwd_kernel(Job job, Ntt2Tables tb, LimbConsts L) {
  pdl_begin();
  using C = Ntt2Cfg<LOGN>;
  constexpr int N = 1 << LOGN, T = C::T, V = C::V, D = C::D;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  Job jb = job;
  jb.bind(blockIdx.x);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const ulonglong2* __restrict__ W = tb.tw + ((size_t)l << LOGN);
  u64 v[V];
#pragma unroll
  for (int r = 0; r < V; r++) v[r] = (NTT2_EXP & 2) ? (u64)(tid + T * r) * q : jb.load(tid + T * r);
#if NTT2_EXP & 1
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w, int) { x ^= y + w.x; y ^= w.y; };
#elif NTT2_PTX && NTT2_LAZY && !NTT2_APX
  const u64 nq = ntt2_nq(q), q4 = 4 * q;
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w, int st) {
    ntt2_ct_lazy(x, y, w.x, w.y, nq, q2, q4, st >= 2 && (st & 1) == 0);
  };
#elif NTT2_PTX
  const u64 nq = ntt2_nq(q), qb = (NTT2_APX ? 5 : 2) * q;  // values in [0, 2 qb)
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w, int) { ntt2_ct_ptx(x, y, w.x, w.y, nq, qb); };
#elif NTT2_APX
  // approximate Shoup quotient (umulhi_apx: Tt in [0, 5q)): values stay in [0, 10q) < 2^64 (q < 2^60)
  const u64 qb = 5 * q;
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w, int) {  // CT: [0, 10q) -> [0, 10q)
    const u64 X = csub2(x, qb);
    const u64 Tt = y * w.x - umulhi_apx(y, w.y) * q;
    x = X + Tt;
    y = X - Tt + qb;
  };
#else
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w, int) {  // Harvey CT: [0, 4q) -> [0, 4q)
    const u64 X = csub2(x, q2);
    const u64 Tt = shoup_mul(y, w.x, w.y, q);
    x = X + Tt;
    y = X - Tt + q2;
  };
#endif
  // ---- group A: stages 0..4, twiddles uniform over the CTA ----
#pragma unroll
  for (int s = 0; s < 5; s++) {
    const int h = 16 >> s;
#pragma unroll
    for (int r = 0; r < V; r++)
      if ((r & h) == 0) bfly(v[r], v[r + h], NTT2_TW(W + (1 << s) + (r >> (5 - s))), s);
  }
#pragma unroll
  for (int r = 0; r < V; r++) sm[ntt2_sw<LOGN>(tid + T * r)] = v[r];
  if (NTT2_PRE == 1) ntt2_pf_groupB<LOGN>(W, tid);
  __syncthreads();
  // ---- group B: stages 5..9 ----
  const int blk = tid / D, baseB = blk * (D * V) + tid % D;
#pragma unroll
  for (int r = 0; r < V; r++) v[r] = sm[ntt2_sw<LOGN>(baseB + D * r)];
#pragma unroll
  for (int s = 5; s < 10; s++) {
    const int h = 16 >> (s - 5);
    const int sh = LOGN - s;  // log2 of the block size of stage s
#pragma unroll
    for (int r = 0; r < V; r++)
      if ((r & h) == 0) bfly(v[r], v[r + h], NTT2_TW(W + (1 << s) + (blk << (s - 5)) + ((D * r) >> sh)), s);
  }
  // (every thread rewrites exactly the positions it read: no barrier before the write-back)
#pragma unroll
  for (int r = 0; r < V; r++) sm[ntt2_sw<LOGN>(baseB + D * r)] = v[r];
  if (NTT2_PRE == 1) ntt2_pf_groupC<LOGN>(W, tid);
  __syncthreads();
  // ---- group C: stages 10..LOGN-1 inside D-point sub-blocks ----
#pragma unroll
  for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
    for (int rr = 0; rr < D; rr++) v[qq * D + rr] = sm[ntt2_sw<LOGN>(D * (tid + T * qq) + rr)];
#pragma unroll
  for (int s = 10; s < LOGN; s++) {
    const int h = D >> (s - 9);
#pragma unroll
    for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
      for (int rr = 0; rr < D; rr++)
        if ((rr & h) == 0)
          bfly(v[qq * D + rr], v[qq * D + rr + h],
               NTT2_TW(W + (1 << s) + ((tid + T * qq) << (s - 10)) + (rr >> (LOGN - s))), s);
  }
#pragma unroll
  for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
    for (int rr = 0; rr < D; rr++) {
#if NTT2_APX
      const u64 x = csub2(csub2(csub2(csub2(v[qq * D + rr], 8 * q), 4 * q), q2), q);
#elif NTT2_PTX && NTT2_LAZY
      const u64 x = csub2(csub2(csub2(v[qq * D + rr], 4 * q), q2), q);
#else
      const u64 x = csub2(csub2(v[qq * D + rr], q2), q);
#endif
      sm[ntt2_sw<LOGN>(D * (tid + T * qq) + rr)] = x;
    }
  __syncthreads();
  // ---- slot-order output: position j holds butterfly position kos[j] (coalesced stores) ----
#pragma unroll 8
  for (int r = 0; r < V; r++) {
    const int j = tid + T * r;
    const u64 x = sm[ntt2_sw<LOGN>(__ldg(tb.kos + j))];
    if (!(NTT2_EXP & 2) || x == 0x123456789abcdefull) jb.store(j, x);
  }
}

template <int LOGN, class Job>
__global__ void __launch_bounds__(Ntt2Cfg<LOGN>::T, (LOGN == 13 ? NTT2_MINB : 2 * NTT2_MINB))
    ntt2_inv_kernel(Job job, Ntt2Tables tb, LimbConsts L) {
  pdl_begin();
  using C = Ntt2Cfg<LOGN>;
  constexpr int N = 1 << LOGN, T = C::T, V = C::V, D = C::D;
  extern __shared__ u64 sm[];
  const int tid = threadIdx.x;
  Job jb = job;
  jb.bind(blockIdx.x);
  const int l = jb.limb;
  const u64 q = L.lc[l].q, q2 = L.lc[l].two_q;
  const ulonglong2* __restrict__ W = tb.tw + ((size_t)l << LOGN);
  // ---- slot-order input -> butterfly positions ----
  if (NTT2_PRE == 1) ntt2_pf_groupC<LOGN>(W, tid);
#pragma unroll 8
  for (int r = 0; r < V; r++) {
    const int j = tid + T * r;
    sm[ntt2_sw<LOGN>(__ldg(tb.kos + j))] = jb.load(j);
  }
  __syncthreads();
  u64 v[V];
#if NTT2_PTX
  const u64 qb = (NTT2_APX ? 5 : 2) * q, nq = ntt2_nq(q);  // values in [0, qb)
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w) { ntt2_gs_ptx(x, y, w.x, w.y, nq, qb); };
#elif NTT2_APX
  const u64 qb = 5 * q;  // approximate quotients: values in [0, 5q)
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w) {  // GS: [0, 5q) -> [0, 5q)
    const u64 U = csub2(x + y, qb);
    const u64 Vv = x - y + qb;
    y = Vv * w.x - umulhi_apx(Vv, w.y) * q;
    x = U;
  };
#else
  const u64 qb = q2;
  auto bfly = [&](u64& x, u64& y, const ulonglong2 w) {  // Harvey GS: [0, 2q) -> [0, 2q)
    const u64 U = csub2(x + y, q2);
    const u64 Vv = x - y + q2;
    y = shoup_mul(Vv, w.x, w.y, q);
    x = U;
  };
#endif
  // ---- group C (stages LOGN-1 .. 10) ----
#pragma unroll
  for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
    for (int rr = 0; rr < D; rr++) v[qq * D + rr] = sm[ntt2_sw<LOGN>(D * (tid + T * qq) + rr)];
#pragma unroll
  for (int s = LOGN - 1; s >= 10; s--) {
    const int h = D >> (s - 9);
#pragma unroll
    for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
      for (int rr = 0; rr < D; rr++)
        if ((rr & h) == 0)
          bfly(v[qq * D + rr], v[qq * D + rr + h],
               __ldg(W + (1 << s) + ((tid + T * qq) << (s - 10)) + (rr >> (LOGN - s))));
  }
#pragma unroll
  for (int qq = 0; qq < C::QN; qq++)
#pragma unroll
    for (int rr = 0; rr < D; rr++) sm[ntt2_sw<LOGN>(D * (tid + T * qq) + rr)] = v[qq * D + rr];
  if (NTT2_PRE == 1) ntt2_pf_groupB<LOGN>(W, tid);
  __syncthreads();
  // ---- group B (stages 9 .. 5) ----
  const int blk = tid / D, baseB = blk * (D * V) + tid % D;
#pragma unroll
  for (int r = 0; r < V; r++) v[r] = sm[ntt2_sw<LOGN>(baseB + D * r)];
#pragma unroll
  for (int s = 9; s >= 5; s--) {
    const int h = 16 >> (s - 5);
    const int sh = LOGN - s;
#pragma unroll
    for (int r = 0; r < V; r++)
      if ((r & h) == 0) bfly(v[r], v[r + h], __ldg(W + (1 << s) + (blk << (s - 5)) + ((D * r) >> sh)));
  }
#pragma unroll
  for (int r = 0; r < V; r++) sm[ntt2_sw<LOGN>(baseB + D * r)] = v[r];
  __syncthreads();
  // ---- group A (stages 4 .. 0), N^{-1} folded into stage 0 ----
#pragma unroll
  for (int r = 0; r < V; r++) v[r] = sm[ntt2_sw<LOGN>(tid + T * r)];
#pragma unroll
  for (int s = 4; s >= 1; s--) {
    const int h = 16 >> s;
#pragma unroll
    for (int r = 0; r < V; r++)
      if ((r & h) == 0) bfly(v[r], v[r + h], __ldg(W + (1 << s) + (r >> (5 - s))));
  }
  {
    const u64 ni = L.lc[l].ninv, nis = L.lc[l].ninv_sh;
    const ulonglong2 wn = __ldg(W);  // slot 0 of the inverse table: psi^{-1}-twiddle of stage 0 times N^{-1}
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const u64 x = v[r], y = v[r + 16];
      const u64 a0 = csub2(shoup_mul(x + y, ni, nis, q), q);
      const u64 a1 = csub2(shoup_mul(x - y + qb, wn.x, wn.y, q), q);
      jb.store(tid + T * r, a0);
      jb.store(tid + T * (r + 16), a1);
    }
  }
}

template <int LOGN>
inline size_t ntt2_smem_bytes() {
  return (size_t)(1 << LOGN) * sizeof(u64);
}
