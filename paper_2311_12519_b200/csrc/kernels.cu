// Device kernels of the Hyena hot path and their launchers.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "hy_common.cuh"
#include "ntt.cuh"

namespace {

LimbConsts limb_consts(const hy_params* p) {
  LimbConsts L;
  for (uint32_t l = 0; l < p->L; l++) L.lc[l] = p->lc[l];
  return L;
}

struct QArr {
  u64 q[HY_MAX_LIMBS];
};

QArr qarr(const hy_params* p) {
  QArr a;
  for (uint32_t l = 0; l < p->L; l++) a.q[l] = p->q[l];
  return a;
}

QArr onesh_arr(const hy_params* p) {  // floor(2^64 / q_l): x mod q_l in [0, 2 q_l) by one Shoup product
  QArr a;
  for (uint32_t l = 0; l < p->L; l++) a.q[l] = p->lc[l].one_sh;
  return a;
}

// ------------------------------------------------------------------------------------------
// NTT jobs
// ------------------------------------------------------------------------------------------
struct PolyJob {  // src/dst [n][L][N]; `src_stride_polys` lets a job walk every other poly
  const u64* src;
  u64* dst;
  int L, N;
  int limb;
  const u64* s;
  u64* d;
  __device__ void bind(int b) {
    limb = b % L;
    s = src + (size_t)b * N;
    d = dst + (size_t)b * N;
  }
  __device__ u64 load(int k) const { return s[k]; }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// S1 PermDecomp (PAPER.md:375-377, :1472 [app]): per input ct, digits d_i = [c1]_{q_i} lifted to
// every limb l and NTT'd (L*L jobs), plus NTT(c0) per limb (L jobs).  (c0_only: the L NTT(c0) jobs
// alone, for the no-hoisting ablation; PermDecompSubJob: the sub-digit base variant.)
struct PermDecompJob {
  const u64* ct;
  u64* D;
  u64* C0;
  int L, N;
  QArr qa;
  size_t ct_stride;  // words between consecutive input cts (0 = 2 L N, contiguous)
  int limb;
  const u64* s;
  u64* d;
  u64 qd;
  bool red;
  bool c0_only = false;
  __device__ void bind(int b) {
    const int nd = c0_only ? 0 : L;
    const int per = nd * L + L;
    const int c = b / per, r = b % per;
    const u64* cb = ct + (size_t)c * (ct_stride ? ct_stride : (size_t)2 * L * N);
    if (r < nd * L) {
      const int i = r / L;
      limb = r % L;
      s = cb + ((size_t)L + i) * N;
      d = D + ((size_t)(c * L + i) * L + limb) * N;
      qd = qa.q[limb];
      red = qa.q[i] / 4 >= qa.q[limb];  // digit may exceed the lazy [0, 4 q_l) input range
    } else {
      limb = r - nd * L;
      s = cb + (size_t)limb * N;
      d = C0 + ((size_t)c * L + limb) * N;
      qd = qa.q[limb];
      red = false;
    }
  }
  __device__ u64 load(int k) const {
    u64 x = s[k];
    return red ? x % qd : x;
  }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// PermDecomp with a sub-digit base 2^w (hy_params_create2, NEXT-4): digit dd = i V + v of limb i is
// floor([c1]_{q_i} / 2^{w v}) mod 2^w (< q_l), NTT'd into every limb l (ND*L jobs) + NTT(c0) (L jobs)
struct PermDecompSubJob {
  const u64* ct;
  u64* D;
  u64* C0;
  int L, N, ND, V, wd;
  size_t ct_stride;
  int limb;
  const u64* s;
  u64* d;
  int sh;  // -1: c0 (whole residue)
  __device__ void bind(int b) {
    const int per = ND * L + L;
    const int c = b / per, r = b % per;
    const u64* cb = ct + (size_t)c * (ct_stride ? ct_stride : (size_t)2 * L * N);
    if (r < ND * L) {
      const int dd = r / L;
      limb = r % L;
      s = cb + ((size_t)L + dd / V) * N;
      d = D + ((size_t)(c * ND + dd) * L + limb) * N;
      sh = wd * (dd % V);
    } else {
      limb = r - ND * L;
      s = cb + (size_t)limb * N;
      d = C0 + ((size_t)c * L + limb) * N;
      sh = -1;
    }
  }
  __device__ u64 load(int k) const {
    const u64 x = s[k];
    return sh >= 0 ? (x >> sh) & ((1ull << wd) - 1) : x;
  }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// row-swap step (a): digits of P_{g,1}.c1 back to coefficient form (INTT per limb i)
struct StridedInvJob {
  const u64* base;  // poly (o, i) at base + o*ostride + i*N
  size_t ostride;
  u64* dst;         // [o][L][N]
  int L, N;
  int limb;
  const u64* s;
  u64* d;
  __device__ void bind(int b) {
    const int o = b / L;
    limb = b % L;
    s = base + (size_t)o * ostride + (size_t)limb * N;
    d = dst + ((size_t)o * L + limb) * N;
  }
  __device__ u64 load(int k) const { return s[k]; }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// row-swap step (b): NTT_l of digit i (coefficient form, in [0, q_i)) for l != i (RNS digits: digit i
// in limb i is the ct's own NTT(c1) limb i); with a sub-digit base every (digit dd, limb l) pair
struct DigitLiftJob {
  const u64* dig;  // [o][L][N]
  u64* D2;         // [o][ND digit][L limb][N]
  int L, N;
  QArr qa;
  QArr osh{};  // floor(2^64 / q_l) per limb (onesh_arr)
  int limb;
  const u64* s;
  u64* d;
  u64 qd;
  bool red;
  int ND = 0, V = 1, wd = 0;
  int sh = 0;
  __device__ void bind(int b) {
    if (ND) {  // sub-digits: all ND * L jobs
      const int per = ND * L;
      const int o = b / per, r = b % per;
      const int dd = r / L, i = dd / V;
      limb = r % L;
      s = dig + ((size_t)o * L + i) * N;
      d = D2 + (((size_t)o * ND + dd) * L + limb) * N;
      qd = qa.q[limb];
      sh = wd * (dd % V);
      red = false;
      return;
    }
    const int per = L * (L - 1);
    const int o = b / per, r = b % per;
    const int i = r / (L - 1), lj = r % (L - 1);
    limb = lj < i ? lj : lj + 1;
    s = dig + ((size_t)o * L + i) * N;
    d = D2 + (((size_t)o * L + i) * L + limb) * N;
    qd = qa.q[limb];
    red = qa.q[i] / 4 >= qa.q[limb];
  }
  __device__ u64 load(int k) const {
    u64 x = s[k];
    if (ND) return (x >> sh) & ((1ull << wd) - 1);
    return red ? reduce_2q(x, osh.q[limb], qd) : x;  // [0, 2 q_l): inside the NTT's [0, 4q) input
  }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// Key switching of whole ciphertexts (hy_rotate, S4 alignment), elementwise in the slot-order
// NTT domain, one thread per (output, limb, position):
//   X.c0[j] = c0[perm(j)] + sum_i D_i[perm(j)] b_i[j] (+ add.c0[j]),  X.c1[j] = sum_i D_i[perm(j)] a_i[j] (+ add.c1[j])
// digit i in limb l is read from `diag` (the ct's own c1 limb, already NTT(d_l) in limb l) when
// given.  The result is then brought back to coefficient form by a plain inverse transform.
struct KsApplyArgs {
  const u64* c0;
  size_t c0_stride;
  const u64* D;  // [o][L digit][L limb][N]
  size_t D_stride;
  const u64* diag;
  size_t diag_stride;
  const u64* add;  // [o][2][L][N] or null
  size_t add_stride;
  const u64* key;
  GaloisAct act;
  u64* out;  // [o][2][L][N] NTT form
  int L, logN;
  size_t total;  // nout * L * N
  LimbConsts lcs;
  int ND = 0;    // gadget digits (0: ND = L, one per limb); D is [o][ND][L][N], keys [ND][2][L][N]
  int d_rot = 0; // 1: D holds the digits of the already ROTATED c1 (no-hoisting ablation): read at j
};

template <int LT>
__global__ void __launch_bounds__(256) ks_apply_kernel(KsApplyArgs a) {
  pdl_begin();
  const size_t idx = (size_t)blockIdx.x * 256 + threadIdx.x;
  if (idx >= a.total) return;
  const int N = 1 << a.logN, L = LT > 0 ? LT : a.L;
  const int ND = LT > 0 ? LT : (a.ND ? a.ND : a.L);
  const int j = (int)(idx & (N - 1));
  const size_t ol = idx >> a.logN;
  const int l = (int)(ol % L);
  const size_t o = ol / L;
  const LimbConst& c = a.lcs.lc[l];
  const u64 q = c.q, q2 = c.two_q;
  const int jp = galois_perm(j, a.act, N >> 1);
  const size_t LN = (size_t)L * N, kblk = 2 * ND * LN;
  const u64* D = a.D + o * a.D_stride;
  const u64* kb = a.key + (size_t)l * N + j;
  u64 a0 = __ldg(a.c0 + o * a.c0_stride + (size_t)l * N + jp), a1 = 0;
  for (int i = 0; i < ND; i++) {
    const u64 dv = (a.diag && ND == L && i == l) ? __ldg(a.diag + o * a.diag_stride + (size_t)i * N + jp)
                                                 : __ldg(D + ((size_t)i * L + l) * N + (a.d_rot ? j : jp));
    const u64* k0 = kb + (size_t)(2 * i) * LN;
    const u64* k1 = k0 + LN;
    a0 = csub(a0 + shoup_mul(dv, __ldg(k0), __ldg(k0 + kblk), q), q2);
    a1 = csub(a1 + shoup_mul(dv, __ldg(k1), __ldg(k1 + kblk), q), q2);
  }
  if (a.add) {
    const u64* ad = a.add + o * a.add_stride + (size_t)l * N + j;
    a0 = csub(a0 + __ldg(ad), q2);
    a1 = csub(a1 + __ldg(ad + LN), q2);
  }
  u64* dst = a.out + o * 2 * LN + (size_t)l * N + j;
  dst[0] = csub(a0, q);
  dst[LN] = csub(a1, q);
}

hy_status launch_ks_apply(const KsApplyArgs& a, cudaStream_t s) {
  if (!a.total) return HY_OK;
  const unsigned blocks = (unsigned)((a.total + 255) / 256);
  switch (a.ND && a.ND != a.L ? 0 : a.L) {  // compile-time digit count: all loads of a thread issue at once
    case 2: HY_CUDA_TRY(hy_launch(ks_apply_kernel<2>, dim3(blocks), dim3(256), 0, s, 1, a)); break;
    case 3: HY_CUDA_TRY(hy_launch(ks_apply_kernel<3>, dim3(blocks), dim3(256), 0, s, 1, a)); break;
    case 5: HY_CUDA_TRY(hy_launch(ks_apply_kernel<5>, dim3(blocks), dim3(256), 0, s, 1, a)); break;
    default: HY_CUDA_TRY(hy_launch(ks_apply_kernel<0>, dim3(blocks), dim3(256), 0, s, 1, a)); break;
  }
  HY_LAUNCH_CHECK();
  return HY_OK;
}

// no-hoisting ablation (Fig. 4 (b)): digit dd (limb i, sub-digit v) of the ROTATED c1,
// [sigma_g(c1)]_{q_i}[k] = +/- c1_i[k g^{-1} mod 2N] (mod q_i), NTT'd into limb l: D [c][ND][L][N]
struct DirectDecompJob {
  const u64* ct;   // [c][2][L][N] coefficient form
  u64* D;
  int L, N, ND, V, wd;
  QArr qa;
  QArr osh{};  // floor(2^64 / q_l) per limb (onesh_arr)
  uint32_t ginv;   // g^{-1} mod 2N
  int limb;
  const u64* s;
  u64* d;
  u64 qi, qd;
  int sh;
  bool red;
  __device__ void bind(int b) {
    const int c = b / (ND * L), r = b % (ND * L);
    const int dd = r / L, i = dd / V;
    limb = r % L;
    s = ct + ((size_t)c * 2 * L + L + i) * N;
    d = D + ((size_t)(c * ND + dd) * L + limb) * N;
    qi = qa.q[i];
    qd = qa.q[limb];
    sh = V > 1 ? wd * (dd % V) : -1;
    red = V > 1 ? false : qa.q[i] / 4 >= qa.q[limb];
  }
  __device__ u64 load(int k) const {
    const uint32_t k0 = (uint32_t)(((uint64_t)k * ginv) % (2 * (uint64_t)N));
    u64 x = k0 < (uint32_t)N ? s[k0] : s[k0 - N];
    if (k0 >= (uint32_t)N) x = x ? qi - x : 0;
    if (sh >= 0) return (x >> sh) & ((1ull << wd) - 1);
    return red ? reduce_2q(x, osh.q[limb], qd) : x;  // [0, 2 q_l): inside the NTT's [0, 4q) input
  }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// plain INTT of an NTT-form ct array [o][cn'][2][L][N] picking diagonal 0 -> ct_out [o][2][L][N]
struct OutInvJob {
  const u64* P;
  size_t o_stride;
  u64* out;
  int L, N;
  int limb;
  const u64* s;
  u64* d;
  __device__ void bind(int b) {
    const int o = b / (2 * L);
    const int cl = b % (2 * L);  // comp*L + limb
    limb = cl % L;
    s = P + (size_t)o * o_stride + (size_t)cl * N;
    d = out + ((size_t)o * 2 * L + cl) * N;
  }
  __device__ u64 load(int k) const { return s[k]; }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// INTT of X [o][2][L][N] plus a coefficient-form addend [o] at add + o * add_stride -> out
// (the coefficient-domain row-swap alignment: Out = P_0 + INTT(KeySwitch(P_1)))
struct OutInvAddJob {
  const u64* X;
  const u64* add;
  size_t add_stride;
  u64* out;
  int L, N;
  QArr qa;
  int limb;
  const u64* s;
  const u64* ad;
  u64* d;
  u64 qd;
  __device__ void bind(int b) {
    const int o = b / (2 * L);
    const int cl = b % (2 * L);
    limb = cl % L;
    qd = qa.q[limb];
    s = X + ((size_t)o * 2 * L + cl) * N;
    ad = add + (size_t)o * add_stride + (size_t)cl * N;
    d = out + ((size_t)o * 2 * L + cl) * N;
  }
  __device__ u64 load(int k) const { return s[k]; }
  __device__ void store(int k, u64 v) const { d[k] = csub(v + ad[k], qd); }
};

// c = INTT(A .* B) where A, B are NTT form [n][L][N] (slow generic product: debug paths only)
struct ProdInvJob {
  const u64* A;
  const u64* B;
  u64* C;
  int L, N;
  QArr qa;
  int limb;
  size_t off;
  __device__ void bind(int b) {
    limb = b % L;
    off = (size_t)b * N;
  }
  __device__ u64 load(int k) const { return mulmod_slow(A[off + k], B[off + k], qa.q[limb]); }
  __device__ void store(int k, u64 v) const { C[off + k] = v; }
};

// decrypt phase: x = c0 + INTT(NTT(c1) .* NTT(s))  per limb
struct C1FwdJob {
  const u64* ct;
  u64* dst;
  int L, N;
  int limb;
  const u64* s;
  u64* d;
  __device__ void bind(int b) {
    const int o = b / L;
    limb = b % L;
    s = ct + ((size_t)(2 * o + 1) * L + limb) * N;
    d = dst + (size_t)b * N;
  }
  __device__ u64 load(int k) const { return s[k]; }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

struct PhaseInvJob {
  const u64* C1n;  // [o][L][N] NTT(c1)
  const u64* Sn;   // [L][N] NTT(s)
  const u64* Snsh;
  const u64* ct;
  u64* out;  // [o][L][N]
  int L, N;
  QArr qa;
  int limb, o;
  __device__ void bind(int b) {
    o = b / L;
    limb = b % L;
  }
  __device__ u64 load(int k) const {
    const u64 q = qa.q[limb];
    const u64 x = shoup_mul(C1n[((size_t)o * L + limb) * N + k], Sn[(size_t)limb * N + k], Snsh[(size_t)limb * N + k], q);
    return csub(x, 2 * q) < 2 * q ? csub(x, 2 * q) : x;  // already < 2q
  }
  __device__ void store(int k, u64 v) const {
    const u64 q = qa.q[limb];
    out[((size_t)o * L + limb) * N + k] = csub(v + ct[((size_t)(2 * o) * L + limb) * N + k], q);
  }
};

template <int LOGN, class Job>
hy_status launch_fwd_t(const hy_params* p, const Job& job, size_t npoly, cudaStream_t s) {
  if (npoly == 0) return HY_OK;
  using C = NttCfg<LOGN>;
  const size_t sm = ntt_smem_bytes<LOGN>();
  HY_CUDA_TRY(hy_smem_attr((const void*)ntt_fwd_kernel<LOGN, Job>, sm));
  HY_CUDA_TRY(hy_launch(ntt_fwd_kernel<LOGN, Job>, dim3((unsigned)(npoly * C::S)), dim3(C::T), sm, s, 1, job, p->tab,
                        limb_consts(p)));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LOGN, class Job>
hy_status launch_inv_t(const hy_params* p, const Job& job, size_t npoly, cudaStream_t s) {
  if (npoly == 0) return HY_OK;
  using C = NttCfg<LOGN>;
  const size_t sm = ntt_smem_bytes<LOGN>();
  HY_CUDA_TRY(hy_smem_attr((const void*)ntt_inv_kernel<LOGN, Job>, sm));
  HY_CUDA_TRY(hy_launch(ntt_inv_kernel<LOGN, Job>, dim3((unsigned)(npoly * C::S)), dim3(C::T), sm, s, C::S, job,
                        p->tab, limb_consts(p)));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

// one-CTA-per-transform NTT (ntt2_*) for N = 4096 / 8192 when the launch has enough transforms to
// fill the GPU (throughput); small launches keep the split kernels (half the latency of one
// transform: the latency-bound small layers).  HY_NTT_V1 forces the split kernels (A/B).
constexpr size_t NTT2_MIN_POLYS = 148 * 4;
static bool ntt_v1() {
  static const bool v = getenv("HY_NTT_V1") != nullptr;
  return v;
}

template <int LOGN, class Job>
hy_status launch_fwd2_t(const hy_params* p, const Job& job, size_t npoly, cudaStream_t s) {
  if (npoly == 0) return HY_OK;
  const size_t sm = ntt2_smem_bytes<LOGN>();
  HY_CUDA_TRY(hy_smem_attr((const void*)ntt2_fwd_kernel<LOGN, Job>, sm));
  HY_CUDA_TRY(hy_launch(ntt2_fwd_kernel<LOGN, Job>, dim3((unsigned)npoly), dim3(Ntt2Cfg<LOGN>::T), sm, s, 1, job,
                        Ntt2Tables{p->tab.psi2, p->tab.kos}, limb_consts(p)));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LOGN, class Job>
hy_status launch_inv2_t(const hy_params* p, const Job& job, size_t npoly, cudaStream_t s) {
  if (npoly == 0) return HY_OK;
  const size_t sm = ntt2_smem_bytes<LOGN>();
  HY_CUDA_TRY(hy_smem_attr((const void*)ntt2_inv_kernel<LOGN, Job>, sm));
  HY_CUDA_TRY(hy_launch(ntt2_inv_kernel<LOGN, Job>, dim3((unsigned)npoly), dim3(Ntt2Cfg<LOGN>::T), sm, s, 1, job,
                        Ntt2Tables{p->tab.ipsi2, p->tab.kos}, limb_consts(p)));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <class Job>
hy_status launch_fwd(const hy_params* p, const Job& job, size_t nblocks, cudaStream_t s) {
  if (!ntt_v1() && nblocks >= NTT2_MIN_POLYS && p->logN == 13) return launch_fwd2_t<13>(p, job, nblocks, s);
  if (!ntt_v1() && nblocks >= NTT2_MIN_POLYS && p->logN == 12) return launch_fwd2_t<12>(p, job, nblocks, s);
  switch (p->logN) {
    case 10: return launch_fwd_t<10>(p, job, nblocks, s);
    case 11: return launch_fwd_t<11>(p, job, nblocks, s);
    case 12: return launch_fwd_t<12>(p, job, nblocks, s);
    case 13: return launch_fwd_t<13>(p, job, nblocks, s);
    case 14: return launch_fwd_t<14>(p, job, nblocks, s);
  }
  hy_set_error("unsupported logN %u", p->logN);
  return HY_EINVAL;
}

template <class Job>
hy_status launch_inv(const hy_params* p, const Job& job, size_t nblocks, cudaStream_t s) {
  if (!ntt_v1() && nblocks >= NTT2_MIN_POLYS && p->logN == 13) return launch_inv2_t<13>(p, job, nblocks, s);
  if (!ntt_v1() && nblocks >= NTT2_MIN_POLYS && p->logN == 12) return launch_inv2_t<12>(p, job, nblocks, s);
  switch (p->logN) {
    case 10: return launch_inv_t<10>(p, job, nblocks, s);
    case 11: return launch_inv_t<11>(p, job, nblocks, s);
    case 12: return launch_inv_t<12>(p, job, nblocks, s);
    case 13: return launch_inv_t<13>(p, job, nblocks, s);
    case 14: return launch_inv_t<14>(p, job, nblocks, s);
  }
  hy_set_error("unsupported logN %u", p->logN);
  return HY_EINVAL;
}

// ------------------------------------------------------------------------------------------
// elementwise kernels
// ------------------------------------------------------------------------------------------
__global__ void shoup_table_kernel(const u64* __restrict__ w, u64* __restrict__ wsh, size_t total, int N, int L,
                                   QArr qa) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)((i / N) % L);
    const u64 q = qa.q[l];
    wsh[i] = (u64)(((u128)w[i] << 64) / q);
  }
}

// w (< 2^60) -> (w mod 2^30) | (w >> 30) << 32: the operand form of the exact 30-bit-split products
__global__ void split30_kernel(const u64* __restrict__ w, u64* __restrict__ out, size_t total) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const u64 x = w[i];
    out[i] = (x & 0x3FFFFFFFull) | ((x >> 30) << 32);
  }
}

// ------------------------------------------------------------------------------------------
// S2 + S3 fused: hoisted PermAuto computed on the fly, lazy MAC of the int weights, Walsh-
// Hadamard butterflies on the accumulators, ONE reduction per output coefficient, PMult by the
// sign plaintext, HAdd (Algorithm :1536-1551 [ign]).
//
// Rotated input R_{c,tau} (never materialised in HBM), for limb l and slot-order position j:
//   R.c0[j] = C0_c[perm(j)] + sum_i D_{c,i}[perm(j)] b_{tau,i}[j],  R.c1[j] = sum_i D_{c,i}[perm(j)] a_{tau,i}[j]
// (identity tap: R = (C0_c, D_{c,l,l})).  perm = cyclic shift (+ half swap) in slot order.
//
// MAC exactness: every canonical R value x < 2^60 is split into 30-bit halves,
// exact as doubles; |w| <= 128 so each product is < 2^37 and sums of up to 2^16 terms stay below
// 2^53: every DFMA is exact, accumulation order is irrelevant, and one reduction per output
// coefficient recovers the residue (lazy reduction).
// ------------------------------------------------------------------------------------------
struct KsMacArgs {
  const u64* D;                // [J][L digit][L limb][N] slot-order NTT
  const u64* C0;               // [J][L][N]
  u64* const* keys;            // [T] key per tap (nullptr = identity)
  const GaloisAct* act;        // [T]
  const double* wt;            // [wblocks][Kpad][Mpad]
  u64* out;                    // [z][M'][2][L][N], M' = M (cn 1) or M/2 (cn 2)
  const u64* sign;             // [L][N] sign plaintext (NTT), then [L][N] Shoup companions
  const int32_t* kt;           // fused tensor-core MAC: K term -> (tap << 16) | ct (-1 = padding)
  u64* out2;                   // coefficient-domain c_n = 2 (tc_coef): [A1] here, [A0] in out; else null
  int coef;                    // 1x1 coefficient-domain MAC: C0 = the input cts [c][2][L][N] (R = ct)
  struct Taps {                // key pointers + automorphisms per tap, by value (no pointer chase)
    const u64* key[HY_MAX_TAPS];
    GaloisAct act[HY_MAX_TAPS];
  } tt;
  int T, Jcb, K, Kpad, M, Mpad, wblocks, L, logN, kscale, cn;
  int dbg;                     // measurement experiments only (HY_DEBUG_KSMAC): 1 = skip the UMMAs
  LimbConsts lcs;
  int ND, wd;                  // gadget digits per ct (D is [ct][ND][L][N]; ND = L: one per limb), base bits
  int hr;                      // c_n = 4: sign holds the 3 dense Hadamard-row plaintexts [3][2][L][N]
};

// NTT_l(c1 limb l) of a ct from its digit block D [ND][L][N] (the identity tap's R.c1): digit l itself
// with one digit per limb, else sum_v 2^{w v} NTT_l(d_{l,v}) (sub-digit base; generic kernels only)
__device__ __forceinline__ u64 ident_c1(const u64* D, int L, int ND, int wd, size_t N, int l, int j, u64 q) {
  if (ND == L) return __ldg(D + ((size_t)l * L + l) * N + j);
  const int V = ND / L;
  u64 acc = 0;
  for (int v = 0; v < V; v++)
    acc = (acc + mulmod_slow(__ldg(D + ((size_t)(l * V + v) * L + l) * N + j), (1ull << (wd * v)) % q, q)) % q;
  return acc;
}

// identity tap of the no-hoisting ablation: R = (NTT(c0), NTT(c1)) with NTT(c1) rebuilt from the
// digits of the (unrotated) c1
__global__ void ident_r_kernel(const u64* __restrict__ C0, const u64* __restrict__ D, u64* __restrict__ R, int nct,
                               int L, int ND, int wd, int logN, QArr qa) {
  const int N = 1 << logN;
  const size_t total = (size_t)nct * L * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx & (N - 1));
    const size_t cl = idx >> logN;
    const int l = (int)(cl % L), c = (int)(cl / L);
    u64* r = R + (size_t)c * 2 * L * N + (size_t)l * N + j;
    r[0] = C0[((size_t)c * L + l) * N + j];
    r[(size_t)L * N] = ident_c1(D + (size_t)c * ND * L * N, L, ND, wd, N, l, j, qa.q[l]);
  }
}

// lazy-reduction-off ablation (Fig. 4 (d)): the MAC over materialised R reducing after EVERY
// product and addition ([acc + w R mod q] mod q), then the Walsh-Hadamard combination and the sign
// PMult for c_n = 2 -- the same residues as the lazy MAC (P10), one Shoup product per coefficient-MAC
__global__ void mac_eager_kernel(KsMacArgs a, const u64* __restrict__ R, const u64* __restrict__ wq, int units) {
  const int N = 1 << a.logN, L = a.L;
  const size_t LN = (size_t)L * N;
  const int outs = a.cn == 2 ? a.M / 2 : a.M;  // P rows per unit
  const size_t total = (size_t)units * outs * 2 * LN;
  const size_t wblk = (size_t)L * a.Kpad * a.Mpad;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % N);
    size_t r = idx / N;
    const int l = (int)(r % L);
    r /= L;
    const int comp = (int)(r % 2);
    r /= 2;
    const int orow = (int)(r % outs), z = (int)(r / outs);
    const LimbConst& c = a.lcs.lc[l];
    const u64 q = c.q;
    const u64* Rz = R + (size_t)z * a.K * 2 * LN + (size_t)comp * LN + (size_t)l * N + j;
    const u64* wl = wq + (size_t)l * a.Kpad * a.Mpad;
    const int nr = a.cn == 2 ? 2 : 1;
    u64 B[2] = {0, 0};
    for (int kk = 0; kk < a.K; kk++) {
      const u64 x = __ldg(Rz + (size_t)kk * 2 * LN);
      for (int rr = 0; rr < nr; rr++) {
        const size_t wi = (size_t)kk * a.Mpad + (size_t)orow * nr + rr;
        const u64 t = csub(shoup_mul(x, __ldg(wl + wi), __ldg(wl + wblk + wi), q), q);
        B[rr] = csub(B[rr] + t, q);
      }
    }
    u64 v = B[0];
    if (a.cn == 2) {
      const u64 a0 = mulmod_slow(csub(B[0] + B[1], q), (u64)a.kscale % q, q);
      const u64 a1 = csub(B[0] + q - B[1], q);
      v = csub(csub(a0 + shoup_mul(a1, __ldg(a.sign + (size_t)l * N + j), __ldg(a.sign + LN + (size_t)l * N + j), q),
                    c.two_q), q);
    }
    a.out[((size_t)(z * outs + orow) * 2 + comp) * LN + (size_t)l * N + j] = v;
  }
}


constexpr uint32_t M30 = 0x3FFFFFFFu;

__device__ __forceinline__ u64 reduce_wide(long long H, long long Lo, const LimbConst& c) {
  // value H * 2^30 + Lo (|H|, |Lo| < 2^59) mod q, canonical: Lo's bits above 30 are folded into H
  // (|H + Lo / 2^30| < 2^60 < off62), so ONE Shoup product by 2^30 mod q reduces the value
  const long long h2 = H + (Lo >> 30);
  const u64 a = shoup_mul((u64)(h2 + (long long)c.off62), c.c30, c.c30_sh, c.q);  // [0, 2q)
  return csub(csub(a + (u64)(Lo & 0x3fffffffll), c.two_q), c.q);                 // < 2q + 2^30
}

// Key words of tap t for limb l at slot position j: digit i, component comp at
// key[((2i + comp) L + l) N + j], Shoup companion one key block (2 L L N words) later.
// Held per thread in registers (KeyRegs) while consecutive K terms use the same tap: the K axis
// is ordered tap-major (kk = tau * Jcb + c), so a thread reloads them once per tap.
template <int LT>
struct KeyRegs {
  static constexpr int NL = LT > 0 ? LT : 1;
  u64 v[2 * NL], sh[2 * NL];
  int tau = -1, pos = -1;
  __device__ __forceinline__ void load(const u64* __restrict__ key, int logN, int l, int j) {
    const size_t N = (size_t)1 << logN, LN = (size_t)LT * N, kblk = 2 * LT * LN;
    const u64* kb = key + (size_t)l * N + j;
#pragma unroll
    for (int x = 0; x < 2 * LT; x++) {
      v[x] = __ldg(kb + x * LN);
      sh[x] = __ldg(kb + x * LN + kblk);
    }
  }
};

// key-switched pair (R.c0, R.c1) of one input ct at limb l, reading slot position jp
template <int LT>
__device__ __forceinline__ void ks_pair_regs(const u64* __restrict__ D, const u64* __restrict__ C0,
                                             const KeyRegs<LT>& k, int logN, int l, int jp, const LimbConst& c,
                                             u64& r0, u64& r1) {
  const size_t N = (size_t)1 << logN;
  const u64 q = c.q;
  u64 dv[LT];
#pragma unroll
  for (int i = 0; i < LT; i++) dv[i] = __ldg(D + ((size_t)i * LT + l) * N + jp);
  u64 a0 = __ldg(C0 + (size_t)l * N + jp), a1 = 0, h0 = 0, h1 = 0;
#pragma unroll
  for (int i = 0; i < LT; i++) {  // lazy: < (2L + 1) q < 2^64, one quotient multiply + reduction each
    a0 += dv[i] * k.v[2 * i];
    h0 += __umul64hi(dv[i], k.sh[2 * i]);
    a1 += dv[i] * k.v[2 * i + 1];
    h1 += __umul64hi(dv[i], k.sh[2 * i + 1]);
  }
  a0 -= h0 * q;
  a1 -= h1 * q;
  r0 = csub(reduce_2q(a0, c.one_sh, q), q);
  r1 = csub(reduce_2q(a1, c.one_sh, q), q);
}

// generic (runtime L, ND digits) version reading the key from global memory
__device__ __forceinline__ void ks_pair_any(const u64* __restrict__ D, const u64* __restrict__ C0,
                                            const u64* __restrict__ key, int L, int logN, int l, int j, int jp,
                                            const LimbConst& c, u64& r0, u64& r1, int ND) {
  const size_t N = (size_t)1 << logN;
  const size_t LN = (size_t)L * N, kblk = 2 * ND * LN;
  const u64 q = c.q, q2 = c.two_q;
  u64 a0 = __ldg(C0 + (size_t)l * N + jp), a1 = 0;
  const u64* kb = key + (size_t)l * N + j;
  for (int i = 0; i < ND; i++) {
    const u64 dv = __ldg(D + ((size_t)i * L + l) * N + jp);
    const u64* k0 = kb + (size_t)(2 * i) * LN;
    const u64* k1 = k0 + LN;
    a0 = csub(a0 + shoup_mul(dv, __ldg(k0), __ldg(k0 + kblk), q), q2);
    a1 = csub(a1 + shoup_mul(dv, __ldg(k1), __ldg(k1 + kblk), q), q2);
  }
  r0 = csub(a0, q);
  r1 = csub(a1, q);
}

// R value pair of K term kk (= tau * Jcb + c) of unit block z at (l, j)
template <int LT>
__device__ __forceinline__ void r_value(const KsMacArgs& a, const u64* const* keys, const GaloisAct* act, int z,
                                        int kk, int l, int j, const LimbConst& c, KeyRegs<LT>& kr, u64& r0,
                                        u64& r1) {
  const int L = LT > 0 ? LT : a.L;
  const int ND = LT > 0 ? LT : a.ND;
  const int N = 1 << a.logN;
  const size_t LN = (size_t)L * N;
  const int t = kk / a.Jcb, cc = kk - t * a.Jcb;
  const size_t ct = (size_t)z * a.Jcb + cc;
  const u64* C0 = a.C0 + ct * LN;
  const u64* D = a.D + ct * ND * LN;
  const u64* key = keys[t];
  if (key == nullptr) {
    r0 = __ldg(C0 + (size_t)l * N + j);
    r1 = ident_c1(D, L, ND, a.wd, N, l, j, c.q);
    return;
  }
  const int jp = galois_perm(j, act[t], N >> 1);
  if constexpr (LT > 0) {
    if (kr.tau != t || kr.pos != j) {
      kr.load(key, a.logN, l, j);
      kr.tau = t;
      kr.pos = j;
    }
    ks_pair_regs<LT>(D, C0, kr, a.logN, l, jp, c, r0, r1);
  } else {
    ks_pair_any(D, C0, key, L, a.logN, l, j, jp, c, r0, r1, ND);
  }
}

// Two-phase R value (prefetch the digit reads, key-switch later) for the tensor-core producers.
template <int LT>
struct RPre {
  u64 c0, d[LT > 0 ? LT : 1];
  int t;  // tap, -1 = padding term (R = 0)
};

template <int LT>
__device__ __forceinline__ void r_finish(const KsMacArgs& a, const u64* const* keys, const RPre<LT>& pr, int l, int j,
                                         const LimbConst& c, KeyRegs<LT>& kr, u64& r0, u64& r1) {
  r0 = r1 = 0;
  if (pr.t < 0) return;
  const u64* key = keys[pr.t];
  if (key == nullptr) {  // identity tap: (C0, D_{l,l})
    r0 = pr.c0;
    r1 = pr.d[0];
    return;
  }
  if (kr.tau != pr.t || kr.pos != j) {
    kr.load(key, a.logN, l, j);
    kr.tau = pr.t;
    kr.pos = j;
  }
  const u64 q = c.q, q2 = c.two_q;
  u64 a0 = pr.c0, a1 = 0;
#pragma unroll
  for (int i = 0; i < LT; i++) {
    a0 = csub(a0 + shoup_mul(pr.d[i], kr.v[2 * i], kr.sh[2 * i], q), q2);
    a1 = csub(a1 + shoup_mul(pr.d[i], kr.v[2 * i + 1], kr.sh[2 * i + 1], q), q2);
  }
  r0 = csub(a0, q);
  r1 = csub(a1, q);
}

__device__ __forceinline__ void store_outputs(const KsMacArgs& a, int z, int row, int comp, int l, int j,
                                              const double* ah, const double* al, int nrows) {
  // rows row .. row+nrows-1 (nrows even for cn = 2) of unit block z at (comp, l, j)
  const int N = 1 << a.logN;
  const size_t LN = (size_t)a.L * N;
  const LimbConst& c = a.lcs.lc[l];
  if (a.cn == 1) {
    for (int r = 0; r < nrows; r++)
      if (row + r < a.M)
        a.out[((size_t)(z * a.M + row + r) * 2 + comp) * LN + (size_t)l * N + j] =
            reduce_wide(__double2ll_rn(ah[r]), __double2ll_rn(al[r]), c);
  } else if (a.cn == 4) {
    // rows (g, d, c): slot group c's accumulator B_c of diagonal d.  Walsh-Hadamard-4 (Sylvester)
    // on the exact accumulators, A_r = sum_c H4[r][c] B_c, ONE reduction each, then the PMults by the
    // Hadamard-row plaintexts (row 0 = 1) and HAdd: P_{g,d} = A_0 + sum_{r >= 1} S_r A_r
    // (PAPER.md:565-572 generalised; ProposedConv, PAPER.md:1536-1551 [ign])
    for (int r0 = 0; r0 + 3 < nrows; r0 += 4) {
      if (row + r0 >= a.M) break;
      long long H[4], Lo[4];
#pragma unroll
      for (int cc = 0; cc < 4; cc++) {
        H[cc] = __double2ll_rn(ah[r0 + cc]);
        Lo[cc] = __double2ll_rn(al[r0 + cc]);
      }
      const long long AH[4] = {H[0] + H[1] + H[2] + H[3], H[0] - H[1] + H[2] - H[3], H[0] + H[1] - H[2] - H[3],
                               H[0] - H[1] - H[2] + H[3]};
      const long long AL[4] = {Lo[0] + Lo[1] + Lo[2] + Lo[3], Lo[0] - Lo[1] + Lo[2] - Lo[3],
                               Lo[0] + Lo[1] - Lo[2] - Lo[3], Lo[0] - Lo[1] - Lo[2] + Lo[3]};
      u64 v = reduce_wide(AH[0], AL[0], c);
#pragma unroll
      for (int r = 1; r < 4; r++) {
        const u64* sr = a.sign + (size_t)(r - 1) * 2 * LN + (size_t)l * N + j;
        v = csub(v + shoup_mul(reduce_wide(AH[r], AL[r], c), __ldg(sr), __ldg(sr + LN), c.q), c.two_q);
      }
      a.out[((size_t)(z * (a.M / 4) + (row + r0) / 4) * 2 + comp) * LN + (size_t)l * N + j] = csub(v, c.q);
    }
  } else {
    const u64 sg = __ldg(a.sign + (size_t)l * N + j), sgs = __ldg(a.sign + LN + (size_t)l * N + j);
    const long long kk = a.kscale;
    for (int r = 0; r < nrows; r += 2) {
      if (row + r < a.M) {
        const long long H0 = __double2ll_rn(ah[r]), L0 = __double2ll_rn(al[r]);
        const long long H1 = __double2ll_rn(ah[r + 1]), L1 = __double2ll_rn(al[r + 1]);
        // Walsh-Hadamard on the accumulators (Eq. 2): A0 = k (B0 + B1), A1 = B0 - B1
        const u64 a0 = reduce_wide(kk * (H0 + H1), kk * (L0 + L1), c);
        const u64 a1 = reduce_wide(H0 - H1, L0 - L1, c);
        // PMult by the [k, -k] plaintext (NTT form, Shoup) and HAdd
        u64 v = a0 + shoup_mul(a1, sg, sgs, c.q);
        v = csub(csub(v, c.two_q), c.q);
        a.out[((size_t)(z * (a.M / 2) + (row + r) / 2) * 2 + comp) * LN + (size_t)l * N + j] = v;
      }
    }
  }
}

// ---- GEMM-shaped variant: C[M][2 x BNP] += W[M][K] x R[K][2 x BNP], K chunked by KC = 2 WM.
// 256 threads = WM row-group warps x PG = 8 / WM position groups; warp (rg, pg) owns rows
// 8 rg .. 8 rg + 7 of the row tile, lane owns position 32 pg + lane (both components).  Every
// thread first produces 2 R items of the next chunk into shared memory (double-buffered), then
// runs its 8 x 2 x 2 DFMAs per k.  <= 128 registers so that two CTAs share an SM: one CTA's
// key switching (INT pipes, L2 loads) overlaps the other's DFMAs.
template <int WM, int LT>
__global__ void __launch_bounds__(256, 2) ksmac_gemm_kernel(KsMacArgs a) {
  pdl_trigger();  // the key staging below reads only uploaded keys: it overlaps the predecessor
  constexpr int BM = 8 * WM, PG = 8 / WM, BNP = 32 * PG, KC = 2 * WM;
  static_assert(KC * BNP == 512, "two R items per thread per chunk");
  constexpr int NL = LT > 0 ? LT : 1;
  extern __shared__ __align__(16) unsigned char smraw[];
  auto Rs = reinterpret_cast<double2(*)[KC][2][BNP]>(smraw);                                // [2][KC][2][BNP]
  auto Ws = reinterpret_cast<double(*)[KC][BM]>(smraw + sizeof(double2) * 2 * KC * 2 * BNP);  // [2][KC][BM]
  // LT > 0: key words of this CTA (limb l, BNP positions) for every tap, staged once:
  // [tap][x = 2 digit + comp][2: value, Shoup][BNP]
  u64* skey = reinterpret_cast<u64*>(smraw + sizeof(double2) * 2 * KC * 2 * BNP + sizeof(double) * 2 * KC * BM);
  __shared__ const u64* s_key[HY_MAX_TAPS];
  __shared__ GaloisAct s_act[HY_MAX_TAPS];

  const int N = 1 << a.logN;
  const size_t LNs = (size_t)(LT > 0 ? LT : a.L) * N;
  const int tiles = N / BNP;
  const int l = blockIdx.x / tiles, j0 = (blockIdx.x % tiles) * BNP;
  const int row0 = blockIdx.y * BM, z = blockIdx.z;
  const double* __restrict__ wt = a.wt + (size_t)(z % a.wblocks) * a.Kpad * a.Mpad;
  const LimbConst cst = a.lcs.lc[l];
  for (int t = threadIdx.x; t < a.T; t += 256) {
    s_key[t] = a.tt.key[t];
    s_act[t] = a.tt.act[t];
  }
  if constexpr (LT > 0) {
    for (int e = threadIdx.x; e < a.T * 4 * LT * (BNP / 2); e += 256) {  // 16-byte loads
      const int p2 = e % (BNP / 2), r = e / (BNP / 2);
      const int sh = r % 2, x = (r / 2) % (2 * LT), tap = r / (4 * LT);
      const u64* key = a.tt.key[tap];
      reinterpret_cast<ulonglong2*>(skey)[e] =
          key ? __ldg(reinterpret_cast<const ulonglong2*>(key + (size_t)sh * 2 * LT * LNs + (size_t)x * LNs +
                                                          (size_t)l * N + j0) + p2)
              : make_ulonglong2(0ull, 0ull);
    }
  }
  __syncthreads();
  pdl_wait();  // D, C0 come from PermDecomp

  // Every thread produces the items (kkl, p) = (tid / BNP + 256 h / BNP, tid % BNP), h = 0, 1:
  // always the same position p.  LT > 0: the digit reads of chunk ch + 1 are issued before the
  // DFMAs of chunk ch (register prefetch) and switched after them, keys come from shared memory.
  constexpr int WPT = (KC * BM + 255) / 256;  // weights staged per thread per chunk
  KeyRegs<LT> kr;
  const int p_own = threadIdx.x % BNP;
  const int jp_own = j0 + p_own;
  const float inv_jc = 1.0f / (float)a.Jcb;
  struct Pre {
    u64 c0, d[NL];
    int tap;
  } pre[2];
  double wpre[WPT];
  auto issue = [&](int chunk) {  // LT > 0: loads of chunk `chunk` into registers
#pragma unroll
    for (int u = 0; u < WPT; u++) {
      const int it = threadIdx.x + 256 * u;
      if (it < KC * BM) wpre[u] = __ldg(wt + (size_t)(chunk * KC + it / BM) * a.Mpad + row0 + it % BM);
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int it = threadIdx.x + 256 * h;
      const int kk = chunk * KC + it / BNP;
      pre[h].tap = -1;
      if (kk >= a.K) continue;
      int tap = (int)((float)kk * inv_jc);  // kk / Jcb (kk < 2^16: off by at most one)
      if (tap * a.Jcb > kk) tap--;
      if ((tap + 1) * a.Jcb <= kk) tap++;
      const int c = kk - tap * a.Jcb;
      pre[h].tap = tap;
      const size_t ct = (size_t)z * a.Jcb + c;
      const u64* C0 = a.C0 + ct * LNs + (size_t)l * N;
      const u64* D = a.D + ct * NL * LNs + (size_t)l * N;
      if (s_key[tap] == nullptr) {
        pre[h].c0 = __ldg(C0 + jp_own);
        pre[h].d[0] = __ldg(D + (size_t)l * LNs + jp_own);
      } else {
        const int jp = galois_perm(jp_own, s_act[tap], N >> 1);
        pre[h].c0 = __ldg(C0 + jp);
#pragma unroll
        for (int i = 0; i < NL; i++) pre[h].d[i] = __ldg(D + (size_t)i * LNs + jp);
      }
    }
  };
  auto finish = [&](int buf) {  // LT > 0: key-switch the prefetched items into Rs[buf], Ws[buf]
    const u64 q = cst.q, q2 = cst.two_q;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int kkl = (threadIdx.x + 256 * h) / BNP;
      u64 r0 = 0, r1 = 0;
      const int tap = pre[h].tap;
      if (tap >= 0) {
        r0 = pre[h].c0;
        if (s_key[tap] == nullptr) {
          r1 = pre[h].d[0];
        } else {
          const u64* kp = skey + (size_t)tap * 4 * NL * BNP + p_own;
          u64 q0 = 0, q1 = 0;  // summed Shoup quotients: one quotient multiply per component
#pragma unroll
          for (int i = 0; i < NL; i++) {  // lazy sums, one canonical reduction each
            r0 += pre[h].d[i] * kp[(4 * i) * BNP];
            q0 += __umul64hi(pre[h].d[i], kp[(4 * i + 1) * BNP]);
            r1 += pre[h].d[i] * kp[(4 * i + 2) * BNP];
            q1 += __umul64hi(pre[h].d[i], kp[(4 * i + 3) * BNP]);
          }
          r0 -= q0 * q;
          r1 -= q1 * q;
          r0 = reduce_lazy_sum<NL>(r0, q);  // canonical: the 30-bit split needs R < 2^60
          r1 = reduce_lazy_sum<NL>(r1, q);
        }
      }
      Rs[buf][kkl][0][p_own] = make_double2((double)(uint32_t)(r0 >> 30), (double)(uint32_t)(r0 & M30));
      Rs[buf][kkl][1][p_own] = make_double2((double)(uint32_t)(r1 >> 30), (double)(uint32_t)(r1 & M30));
    }
#pragma unroll
    for (int u = 0; u < WPT; u++) {
      const int it = threadIdx.x + 256 * u;
      if (it < KC * BM) Ws[buf][it / BM][it % BM] = wpre[u];
    }
  };
  auto produce = [&](int chunk, int buf) {  // LT == 0: generic L, loads + switching in one go
    double wv[WPT];
#pragma unroll
    for (int u = 0; u < WPT; u++) {
      const int it = threadIdx.x + 256 * u;
      if (it < KC * BM) wv[u] = __ldg(wt + (size_t)(chunk * KC + it / BM) * a.Mpad + row0 + it % BM);
    }
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int it = threadIdx.x + 256 * h;
      const int kkl = it / BNP, p = it % BNP, kk = chunk * KC + kkl;
      u64 r0 = 0, r1 = 0;
      if (kk < a.K) r_value<LT>(a, s_key, s_act, z, kk, l, j0 + p, cst, kr, r0, r1);
      Rs[buf][kkl][0][p] = make_double2((double)(uint32_t)(r0 >> 30), (double)(uint32_t)(r0 & M30));
      Rs[buf][kkl][1][p] = make_double2((double)(uint32_t)(r1 >> 30), (double)(uint32_t)(r1 & M30));
    }
#pragma unroll
    for (int u = 0; u < WPT; u++) {
      const int it = threadIdx.x + 256 * u;
      if (it < KC * BM) Ws[buf][it / BM][it % BM] = wv[u];
    }
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = warp % WM, pg = warp / WM;
  const int pos = pg * 32 + lane;
  double acc_h[8][2], acc_l[8][2];
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int n = 0; n < 2; n++) acc_h[r][n] = acc_l[r][n] = 0.0;

  const int nchunks = a.Kpad / KC;
  if constexpr (LT > 0) {
    issue(0);
    finish(0);
    if (nchunks > 1) issue(1);
  } else {
    produce(0, 0);
  }
  __syncthreads();
  for (int ch = 0; ch < nchunks; ch++) {
    const int buf = ch & 1;
    if constexpr (LT == 0) {
      if (ch + 1 < nchunks) produce(ch + 1, buf ^ 1);
    }
#pragma unroll
    for (int kkl = 0; kkl < KC; kkl++) {
      const double2* wp = reinterpret_cast<const double2*>(&Ws[buf][kkl][rg * 8]);
      double w[8];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const double2 t2 = wp[r];
        w[2 * r] = t2.x;
        w[2 * r + 1] = t2.y;
      }
      const double2 x0 = Rs[buf][kkl][0][pos], x1 = Rs[buf][kkl][1][pos];
#pragma unroll
      for (int r = 0; r < 8; r++) {
        acc_h[r][0] = fma(w[r], x0.x, acc_h[r][0]);
        acc_l[r][0] = fma(w[r], x0.y, acc_l[r][0]);
        acc_h[r][1] = fma(w[r], x1.x, acc_h[r][1]);
        acc_l[r][1] = fma(w[r], x1.y, acc_l[r][1]);
      }
    }
    if constexpr (LT > 0) {
      if (ch + 1 < nchunks) {
        finish(buf ^ 1);                     // chunk ch + 1 (its reads were in flight)
        if (ch + 2 < nchunks) issue(ch + 2);
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int n = 0; n < 2; n++) {
    double ah[8], al[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      ah[r] = acc_h[r][n];
      al[r] = acc_l[r][n];
    }
    store_outputs(a, z, row0 + rg * 8, n, l, j0 + pos, ah, al, 8);
  }
}

// ---- thin variant (M <= 2 rows: depthwise): one thread per (limb, position) and CPT units
// (input cts with their own weight block), all K = T taps in registers, no shared memory.  The
// tap's key words are loaded once per tap and reused for the CPT units (the key traffic, 4L words
// per (ct, tap) before, dominated the loads); digit reads are issued for all CPT units before the
// key switching of the first.
template <int MR, int LT, int CPT>
__global__ void __launch_bounds__(256) ksmac_thin_kernel(KsMacArgs a, int units) {
  pdl_begin();
  const int N = 1 << a.logN;
  const int idx = blockIdx.x * 256 + threadIdx.x;
  const int l = idx >> a.logN, j = idx & (N - 1);
  if (l >= a.L) return;
  const int z0 = blockIdx.z * CPT;
  const LimbConst cst = a.lcs.lc[l];
  double ah[CPT][2][MR], al[CPT][2][MR];
#pragma unroll
  for (int u = 0; u < CPT; u++)
#pragma unroll
    for (int c = 0; c < 2; c++)
#pragma unroll
      for (int r = 0; r < MR; r++) ah[u][c][r] = al[u][c][r] = 0.0;
  const size_t LN = (size_t)(LT > 0 ? LT : a.L) * N;
  for (int kk = 0; kk < a.K; kk++) {  // depthwise: one term per tap
    const u64* key = a.tt.key[kk];
    KeyRegs<LT> kr;
    int jp = j;
    if (key != nullptr) {
      jp = galois_perm(j, a.tt.act[kk], N >> 1);
      if constexpr (LT > 0) kr.load(key, a.logN, l, j);
    }
    u64 c0v[CPT], dv[CPT][LT > 0 ? LT : 1];
#pragma unroll
    for (int u = 0; u < CPT; u++) {
      const int z = z0 + u < units ? z0 + u : units - 1;  // clamp: the tail's extra work is discarded
      const u64* C0 = a.C0 + (size_t)z * LN;
      const u64* D = a.D + (size_t)z * (LT > 0 ? LT : a.ND) * LN;
      c0v[u] = __ldg(C0 + (size_t)l * N + jp);
      if constexpr (LT > 0) {
        if (key == nullptr) {
          dv[u][0] = __ldg(D + ((size_t)l * LT + l) * N + jp);
        } else {
#pragma unroll
          for (int i = 0; i < LT; i++) dv[u][i] = __ldg(D + ((size_t)i * LT + l) * N + jp);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CPT; u++) {
      const int z = z0 + u < units ? z0 + u : units - 1;
      u64 r0, r1;
      if constexpr (LT > 0) {
        if (key == nullptr) {
          r0 = c0v[u];
          r1 = dv[u][0];
        } else {
          const u64 q = cst.q, q2 = cst.two_q;
          u64 x0 = c0v[u], x1 = 0, g0 = 0, g1 = 0;
#pragma unroll
          for (int i = 0; i < LT; i++) {  // lazy sums (summed quotients), one canonical reduction each
            x0 += dv[u][i] * kr.v[2 * i];
            g0 += __umul64hi(dv[u][i], kr.sh[2 * i]);
            x1 += dv[u][i] * kr.v[2 * i + 1];
            g1 += __umul64hi(dv[u][i], kr.sh[2 * i + 1]);
          }
          x0 -= g0 * q;
          x1 -= g1 * q;
          r0 = reduce_lazy_sum<LT>(x0, q);  // canonical: the 30-bit split needs R < 2^60
          r1 = reduce_lazy_sum<LT>(x1, q);
        }
      } else {
        const u64* C0 = a.C0 + (size_t)z * LN;
        const u64* D = a.D + (size_t)z * a.ND * LN;
        if (key == nullptr) {
          r0 = c0v[u];
          r1 = ident_c1(D, a.L, a.ND, a.wd, N, l, j, cst.q);
        } else {
          ks_pair_any(D, C0, key, a.L, a.logN, l, j, jp, cst, r0, r1, a.ND);
        }
      }
      const double x0h = (double)(uint32_t)(r0 >> 30), x0l = (double)(uint32_t)(r0 & M30);
      const double x1h = (double)(uint32_t)(r1 >> 30), x1l = (double)(uint32_t)(r1 & M30);
      const double* __restrict__ wt = a.wt + (size_t)(z % a.wblocks) * a.Kpad * a.Mpad;
#pragma unroll
      for (int r = 0; r < MR; r++) {
        const double w = __ldg(wt + (size_t)kk * a.Mpad + r);
        ah[u][0][r] = fma(w, x0h, ah[u][0][r]);
        al[u][0][r] = fma(w, x0l, al[u][0][r]);
        ah[u][1][r] = fma(w, x1h, ah[u][1][r]);
        al[u][1][r] = fma(w, x1l, al[u][1][r]);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < CPT; u++)
    if (z0 + u < units)
#pragma unroll
      for (int c = 0; c < 2; c++) store_outputs(a, z0 + u, 0, c, l, j, ah[u][c], al[u][c], MR);
}

// ------------------------------------------------------------------------------------------
// Split variant of S2 + S3 for dense layers (the default): PermAuto materialises the rotated
// inputs R[unit][kk][2][L][N] (kk = tau * Jc + c, slot-order NTT form), then a pure MAC GEMM
// consumes them.  Keeping the key switching (INT pipes) out of the MAC kernel leaves the FP64
// pipe's issue slots to the DFMAs (fused 42 %, split MAC ~70 % of the FP64 peak).
// ------------------------------------------------------------------------------------------
// PermAuto: one thread per (limb, position) of one tap and unit; the tap's key words for the
// position stay in registers while the thread walks the unit's input ciphertexts.
template <int LT>
__global__ void __launch_bounds__(256) permauto_kernel(KsMacArgs a, u64* __restrict__ R) {
  const int N = 1 << a.logN, L = LT > 0 ? LT : a.L;
  const int idx = blockIdx.x * 256 + threadIdx.x;
  const int l = idx >> a.logN, j = idx & (N - 1);
  if (l >= L) return;
  const int t = blockIdx.y, z = blockIdx.z;
  const LimbConst cst = a.lcs.lc[l];
  const size_t LN = (size_t)L * N;
  const u64* key = a.keys[t];
  u64* out = R + ((size_t)z * a.K + (size_t)t * a.Jcb) * 2 * LN + (size_t)l * N + j;
  const int ND = LT > 0 ? LT : a.ND;
  const u64* C0b = a.C0 + (size_t)z * a.Jcb * LN;
  const u64* Db = a.D + (size_t)z * a.Jcb * ND * LN;
  if (key == nullptr) {  // identity tap: R = (C0, D_{l,l})
    for (int c = 0; c < a.Jcb; c++) {
      const u64 r0 = __ldg(C0b + (size_t)c * LN + (size_t)l * N + j);
      const u64 r1 = ident_c1(Db + (size_t)c * ND * LN, L, ND, a.wd, N, l, j, cst.q);
      __stcs(out + (size_t)c * 2 * LN, r0);
      __stcs(out + (size_t)c * 2 * LN + LN, r1);
    }
    return;
  }
  const int jp = galois_perm(j, a.act[t], N >> 1);
  if constexpr (LT > 0) {
    KeyRegs<LT> kr;
    kr.load(key, a.logN, l, j);
    const u64* C0p = C0b + (size_t)l * N + jp;
    const u64* Dp = Db + (size_t)l * N + jp;
    // software pipeline: the reads of ciphertext c + 1 are in flight while c is key-switched
    u64 c0n = __ldg(C0p), dn[LT];
#pragma unroll
    for (int i = 0; i < LT; i++) dn[i] = __ldg(Dp + (size_t)i * LN);
    for (int c = 0; c < a.Jcb; c++) {
      const u64 c0 = c0n;
      u64 d[LT];
#pragma unroll
      for (int i = 0; i < LT; i++) d[i] = dn[i];
      if (c + 1 < a.Jcb) {
        c0n = __ldg(C0p + (size_t)(c + 1) * LN);
#pragma unroll
        for (int i = 0; i < LT; i++) dn[i] = __ldg(Dp + (size_t)(c + 1) * L * LN + (size_t)i * LN);
      }
      // lazy: each Shoup product is in [0, 2q); c0 + sum < (2L + 1) q < 2^64 for q < 2^60, L <= 7;
      // one reduction per component
      const u64 q = cst.q;
      u64 a0 = c0, a1 = 0, g0 = 0, g1 = 0;
#pragma unroll
      for (int i = 0; i < LT; i++) {  // summed Shoup quotients: one quotient multiply per component
        a0 += d[i] * kr.v[2 * i];
        g0 += __umul64hi(d[i], kr.sh[2 * i]);
        a1 += d[i] * kr.v[2 * i + 1];
        g1 += __umul64hi(d[i], kr.sh[2 * i + 1]);
      }
      a0 -= g0 * q;
      a1 -= g1 * q;
      __stcs(out + (size_t)c * 2 * LN, csub(reduce_2q(a0, cst.one_sh, q), q));
      __stcs(out + (size_t)c * 2 * LN + LN, csub(reduce_2q(a1, cst.one_sh, q), q));
    }
  } else {
    for (int c = 0; c < a.Jcb; c++) {
      u64 r0, r1;
      ks_pair_any(Db + (size_t)c * ND * LN, C0b + (size_t)c * LN, key, L, a.logN, l, j, jp, cst, r0, r1, ND);
      __stcs(out + (size_t)c * 2 * LN, r0);
      __stcs(out + (size_t)c * 2 * LN + LN, r1);
    }
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

// MAC GEMM: C[M][2 x BNP] = W[M][K] x R[K][2 x BNP].  256 threads = WM row-group warps x PG
// position groups; lane owns positions (pg*64 + lane, pg*64 + lane + 32) of both components
// (8 rows x 4 columns of exact FP64 accumulators).  R (u64) and W chunks of KC = 16 terms stream
// in through a 3-stage cp.async ring; each chunk is split once into (hi, lo) doubles in shared
// memory and consumed by every row-group warp.
constexpr int MG_STAGES = 3;

template <int WM>
struct MgTile {
  static constexpr int BM = 8 * WM, PG = 8 / WM, BNP = 64 * PG, KC = WM >= 8 ? 16 : 8;
  static constexpr size_t RAW = sizeof(u64) * KC * 2 * BNP;        // per stage
  static constexpr size_t WSZ = sizeof(double) * KC * BM;           // per stage
  static constexpr size_t RD = sizeof(double2) * KC * 2 * BNP;      // converted chunk
  static constexpr size_t SMEM = MG_STAGES * (RAW + WSZ) + 2 * RD;  // Rd double-buffered
};

template <int WM>
__global__ void __launch_bounds__(256, 1) mac_gemm_kernel(KsMacArgs a, const u64* __restrict__ R) {
  using TL = MgTile<WM>;
  constexpr int BM = TL::BM, BNP = TL::BNP, KC = TL::KC;
  extern __shared__ __align__(16) unsigned char smraw[];
  auto raw = [&](int st) { return reinterpret_cast<u64*>(smraw + st * (TL::RAW + TL::WSZ)); };  // [KC][2][BNP]
  auto wsm = [&](int st) { return reinterpret_cast<double*>(smraw + st * (TL::RAW + TL::WSZ) + TL::RAW); };
  double2* Rd = reinterpret_cast<double2*>(smraw + MG_STAGES * (TL::RAW + TL::WSZ));  // [KC][2][BNP]

  const int N = 1 << a.logN;
  const size_t LN = (size_t)a.L * N;
  const int tiles = N / BNP;
  const int l = blockIdx.x / tiles, j0 = (blockIdx.x % tiles) * BNP;
  const int row0 = blockIdx.y * BM, z = blockIdx.z;
  const double* __restrict__ wt = a.wt + (size_t)(z % a.wblocks) * a.Kpad * a.Mpad;
  const u64* __restrict__ Rz = R + (size_t)z * a.K * 2 * LN + (size_t)l * N + j0;
  const int nchunks = a.Kpad / KC;

  auto issue = [&](int ch) {
    if (ch < nchunks) {
      const int st = ch % MG_STAGES;
      u64* dst = raw(st);
      // R rows (kk, comp): BNP contiguous u64 = BNP/2 16-byte pieces
      for (int e = threadIdx.x; e < KC * 2 * (BNP / 2); e += 256) {
        const int row = e / (BNP / 2), piece = e % (BNP / 2);
        const int kk = ch * KC + row / 2, comp = row % 2;
        u64* d = dst + (size_t)row * BNP + piece * 2;
        if (kk < a.K)
          cp_async16(d, Rz + ((size_t)kk * 2 + comp) * LN + piece * 2);
        else
          d[0] = d[1] = 0;
      }
      double* wd = wsm(st);
      for (int e = threadIdx.x; e < KC * BM / 2; e += 256) {
        const int kk = e / (BM / 2), r2 = e % (BM / 2);
        cp_async16(wd + kk * BM + 2 * r2, wt + (size_t)(ch * KC + kk) * a.Mpad + row0 + 2 * r2);
      }
    }
    cp_async_commit();
  };

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rg = warp % WM, pg = warp / WM;
  const int p0 = pg * 64 + lane;
  double acc_h[8][4], acc_l[8][4];
#pragma unroll
  for (int r = 0; r < 8; r++)
#pragma unroll
    for (int n = 0; n < 4; n++) acc_h[r][n] = acc_l[r][n] = 0.0;

  auto convert = [&](int ch) {  // raw u64 chunk -> (hi, lo) doubles, split once for all warps
    const u64* src = raw(ch % MG_STAGES);
    double2* dst = Rd + (size_t)(ch & 1) * KC * 2 * BNP;
    for (int e = threadIdx.x; e < KC * 2 * BNP; e += 256) {
      const u64 x = src[e];
      dst[e] = make_double2((double)(uint32_t)(x >> 30), (double)(uint32_t)(x & M30));
    }
  };
#pragma unroll
  for (int st = 0; st < MG_STAGES - 1; st++) issue(st);
  cp_async_wait<MG_STAGES - 2>();
  __syncthreads();
  convert(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ch++) {
    issue(ch + MG_STAGES - 1);
    const double* wd = wsm(ch % MG_STAGES);
    const double2* Rc = Rd + (size_t)(ch & 1) * KC * 2 * BNP;
#pragma unroll 4
    for (int kk = 0; kk < KC; kk++) {
      const double2* wp = reinterpret_cast<const double2*>(wd + kk * BM + rg * 8);
      double w[8];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const double2 t2 = wp[r];
        w[2 * r] = t2.x;
        w[2 * r + 1] = t2.y;
      }
      const double2* rp = Rc + (size_t)kk * 2 * BNP + p0;
      double2 x[4];
      x[0] = rp[0];
      x[1] = rp[32];
      x[2] = rp[BNP];
      x[3] = rp[BNP + 32];
#pragma unroll
      for (int r = 0; r < 8; r++)
#pragma unroll
        for (int n = 0; n < 4; n++) {
          acc_h[r][n] = fma(w[r], x[n].x, acc_h[r][n]);
          acc_l[r][n] = fma(w[r], x[n].y, acc_l[r][n]);
        }
    }
    if (ch + 1 < nchunks) {
      cp_async_wait<MG_STAGES - 2>();  // chunk ch + 1 landed (this thread's copies)
      __syncthreads();                 // ... everyone's; stage ch % S and Rd[(ch+1)&1] are free
      convert(ch + 1);
      __syncthreads();
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int n = 0; n < 4; n++) {
    double ah[8], al[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
      ah[r] = acc_h[r][n];
      al[r] = acc_l[r][n];
    }
    store_outputs(a, z, row0 + rg * 8, n >> 1, l, j0 + p0 + 32 * (n & 1), ah, al, 8);
  }
}

// ------------------------------------------------------------------------------------------
// Tensor-core MAC (tcgen05, kind::i8).  The lazy MAC is an exact integer contraction
// B[m][col] = sum_kk w[m][kk] R[kk][col] with |w| <= 128 and R < 2^60: split every R value into
// its 8 bytes, R = sum_b 2^{8b} R_b, and B = sum_b 2^{8b} (W x R_b) with one s8 x u8 -> s32 MMA per
// byte plane.  |W x R_b| <= 128 * 255 * K < 2^31 for K <= 2^16 (the planner's bound), so every
// accumulator is exact; the epilogue recombines the planes as two int64 halves
// S = S_hi 2^32 + S_lo and reduces once per output coefficient.
// CTA = one unit, one limb, 16 positions x 2 components (32 columns), 128 MAC rows; 4 producer
// warps stream R chunks of 32 terms from HBM and transpose them into the 8 byte planes (K-major
// canonical smem layout), one thread issues 8 UMMAs (M=128, N=32, K=32) per chunk into 8 TMEM
// accumulators (256 columns), and the producer warps run the epilogue from TMEM.
// ------------------------------------------------------------------------------------------
constexpr int TC_STAGES = 3, TC_COLS = 32, TC_POS = 16, TC_THREADS = 160;
constexpr uint32_t TC_TMEM_COLS = 8 * TC_COLS;  // 256

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr) {
  // K-major, no swizzle: core matrices of 8 rows x 16 bytes; LBO (next 16 bytes of K) = 128 B,
  // SBO (next 8 rows) = 256 B; version 1 (sm_100)
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(128 >> 4) << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

__device__ __forceinline__ uint32_t umma_idesc_s8u8(int m, int n) {
  return (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  }
}

template <int LT = 0, int LOGN = 0>
__device__ __forceinline__ void tc_store(const KsMacArgs& a, int z, int row, int comp, int l, int j, long long H,
                                         long long Lo) {
  // this lane holds B = H 2^32 + Lo for MAC row `row` (|H|, |Lo| < 2^56); lanes row^1 pair up
  const int N = LOGN > 0 ? (1 << LOGN) : (1 << a.logN);
  const size_t LN = (size_t)(LT > 0 ? LT : a.L) * N;
  const LimbConst& c = a.lcs.lc[l];
  auto red = [&](long long h, long long lo) -> u64 {  // h 2^32 + lo mod q, |h| < 2^61, |lo| < 2^62
    // fold lo's high word into h: value = (h + lo_hi) 2^32 + lo_lo with lo_lo in [0, 2^32), so ONE
    // Shoup product by 2^32 mod q reduces it (|h + lo_hi| < 2^62 = off62 bound, off62 = 0 mod q)
    const long long h2 = h + (lo >> 32);
    const u64 x = shoup_mul((u64)(h2 + (long long)c.off62), c.c32, c.c32_sh, c.q);  // [0, 2q)
    return csub(csub(x + (u64)(lo & 0xffffffffll), c.two_q), c.q);  // < 2q + 2^32 < 3q
  };
  if (a.cn == 1) {
    if (row < a.M) a.out[((size_t)(z * a.M + row) * 2 + comp) * LN + (size_t)l * N + j] = red(H, Lo);
    return;
  }
  const long long H1 = __shfl_xor_sync(0xffffffffu, H, 1), L1 = __shfl_xor_sync(0xffffffffu, Lo, 1);
  if ((row & 1) || row >= a.M) return;
  const long long k = a.kscale;
  // Walsh-Hadamard on the exact accumulators (Eq. 2): A0 = k (B0 + B1), A1 = B0 - B1
  const u64 a0 = red(k * (H + H1), k * (Lo + L1));
  const u64 a1 = red(H - H1, Lo - L1);
  if (a.out2) {  // coefficient domain: the sign PMult is a negacyclic shift, applied by sign_combine
    const size_t at = ((size_t)(z * (a.M / 2) + row / 2) * 2 + comp) * LN + (size_t)l * N + j;
    a.out[at] = a0;
    a.out2[at] = a1;
    return;
  }
  const u64 sg = __ldg(a.sign + (size_t)l * N + j), sgs = __ldg(a.sign + LN + (size_t)l * N + j);
  u64 v = a0 + shoup_mul(a1, sg, sgs, c.q);
  v = csub(csub(v, c.two_q), c.q);
  a.out[((size_t)(z * (a.M / 2) + row / 2) * 2 + comp) * LN + (size_t)l * N + j] = v;
}

// tc_store for 4 consecutive positions j .. j + 3 (j % 4 == 0) of one component: the same
// arithmetic, written as two 16-byte stores per row instead of four 8-byte ones
template <int LT = 0, int LOGN = 0>
__device__ __forceinline__ void tc_store4(const KsMacArgs& a, int z, int row, int comp, int l, int j,
                                          const long long* H, const long long* Lo) {
  const int N = LOGN > 0 ? (1 << LOGN) : (1 << a.logN);
  const size_t LN = (size_t)(LT > 0 ? LT : a.L) * N;
  const LimbConst& c = a.lcs.lc[l];
  auto red = [&](long long h, long long lo) -> u64 {  // as in tc_store: one Shoup product
    const long long h2 = h + (lo >> 32);
    const u64 x = shoup_mul((u64)(h2 + (long long)c.off62), c.c32, c.c32_sh, c.q);
    return csub(csub(x + (u64)(lo & 0xffffffffll), c.two_q), c.q);
  };
  u64 v[4];
  if (a.cn == 1) {
    if (row >= a.M) return;
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = red(H[i], Lo[i]);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(a.out + ((size_t)(z * a.M + row) * 2 + comp) * LN + (size_t)l * N + j);
    dst[0] = make_ulonglong2(v[0], v[1]);
    dst[1] = make_ulonglong2(v[2], v[3]);
    return;
  }
  long long H1[4], L1[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    H1[i] = __shfl_xor_sync(0xffffffffu, H[i], 1);
    L1[i] = __shfl_xor_sync(0xffffffffu, Lo[i], 1);
  }
  if ((row & 1) || row >= a.M) return;
  const long long k = a.kscale;
  u64 a0[4], a1[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {  // Walsh-Hadamard on the exact accumulators (Eq. 2)
    a0[i] = red(k * (H[i] + H1[i]), k * (Lo[i] + L1[i]));
    a1[i] = red(H[i] - H1[i], Lo[i] - L1[i]);
  }
  const size_t at = ((size_t)(z * (a.M / 2) + row / 2) * 2 + comp) * LN + (size_t)l * N + j;
  if (a.out2) {  // coefficient domain: the sign PMult is applied by sign_combine
    reinterpret_cast<ulonglong2*>(a.out + at)[0] = make_ulonglong2(a0[0], a0[1]);
    reinterpret_cast<ulonglong2*>(a.out + at)[1] = make_ulonglong2(a0[2], a0[3]);
    reinterpret_cast<ulonglong2*>(a.out2 + at)[0] = make_ulonglong2(a1[0], a1[1]);
    reinterpret_cast<ulonglong2*>(a.out2 + at)[1] = make_ulonglong2(a1[2], a1[3]);
    return;
  }
  const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(a.sign + (size_t)l * N + j);
  const ulonglong2* ssp = reinterpret_cast<const ulonglong2*>(a.sign + LN + (size_t)l * N + j);
  const ulonglong2 s01 = __ldg(sp), s23 = __ldg(sp + 1), h01 = __ldg(ssp), h23 = __ldg(ssp + 1);
  const u64 sg[4] = {s01.x, s01.y, s23.x, s23.y}, sgs[4] = {h01.x, h01.y, h23.x, h23.y};
#pragma unroll
  for (int i = 0; i < 4; i++) v[i] = csub(csub(a0[i] + shoup_mul(a1[i], sg[i], sgs[i], c.q), c.two_q), c.q);
  reinterpret_cast<ulonglong2*>(a.out + at)[0] = make_ulonglong2(v[0], v[1]);
  reinterpret_cast<ulonglong2*>(a.out + at)[1] = make_ulonglong2(v[2], v[3]);
}

// 4x4 byte transpose: w[b] = byte b of x[0], x[1], x[2], x[3]
__device__ __forceinline__ void byte_tr4(const uint32_t* x, uint32_t* w) {
  const uint32_t t0 = __byte_perm(x[0], x[1], 0x5140), t1 = __byte_perm(x[0], x[1], 0x7362);
  const uint32_t t2 = __byte_perm(x[2], x[3], 0x5140), t3 = __byte_perm(x[2], x[3], 0x7362);
  w[0] = __byte_perm(t0, t2, 0x5410);
  w[1] = __byte_perm(t0, t2, 0x7632);
  w[2] = __byte_perm(t1, t3, 0x5410);
  w[3] = __byte_perm(t1, t3, 0x7632);
}

__global__ void __launch_bounds__(TC_THREADS, 1) mac_tc_kernel(KsMacArgs a, const u64* __restrict__ R,
                                                               const int8_t* __restrict__ w8) {
  __shared__ __align__(1024) uint8_t sA[TC_STAGES][4096];                 // 128 rows x 32 terms
  __shared__ __align__(1024) uint8_t sB[TC_STAGES][8][TC_COLS * 32];      // 8 planes x 32 cols x 32 terms
  __shared__ __align__(8) uint64_t full_bar[TC_STAGES], empty_bar[TC_STAGES], done_bar;
  __shared__ uint32_t s_tmem;

  const int N = 1 << a.logN;
  const size_t LN = (size_t)a.L * N;
  const int tiles = N / TC_POS;
  // M tile fastest in the grid: the CTAs sharing an R column tile run together, so the tile is
  // read from HBM once and from L2 by the other M tiles
  const int nmt_ = (a.Mpad + 127) / 128;
  const int mt = blockIdx.x % nmt_, ct_ = blockIdx.x / nmt_;
  const int l = ct_ / tiles, j0 = (ct_ % tiles) * TC_POS;
  const int z = blockIdx.z;
  const int nmt = (a.Mpad + 127) / 128;
  const int nchunks = a.Kpad / 32;
  const int tid = threadIdx.x, warp = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < TC_STAGES; s++) {
      mbar_init(&full_bar[s], 4);  // one arrival per producer warp
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;

  if (tid < 128) {
    // ---------------- producers: R chunk -> 8 byte planes; weights tile ----------------
    const int n = tid & 31, kq = tid >> 5;           // column n (comp n/16, position n%16), terms 8kq..8kq+7
    const int comp = n >> 4, pos = n & 15;
    const u64* Rp = R + (size_t)z * a.K * 2 * LN + (size_t)comp * LN + (size_t)l * N + j0 + pos;
    const int8_t* wsrc = w8 + ((size_t)(z % a.wblocks) * nmt + mt) * nchunks * 4096;
    const int boff = (n >> 3) * 256 + (kq >> 1) * 128 + (n & 7) * 16 + (kq & 1) * 8;
    u64 xn[8];  // the next chunk's R values, in flight while the current one is transposed
#pragma unroll
    for (int t = 0; t < 8; t++) {
      const int kk = kq * 8 + t;
      xn[t] = kk < a.K ? __ldcs(Rp + (size_t)kk * 2 * LN) : 0ull;
    }
    for (int ch = 0; ch < nchunks; ch++) {
      const int s = ch % TC_STAGES;
      u64 x[8];
#pragma unroll
      for (int t = 0; t < 8; t++) {
        x[t] = xn[t];
        const int kk = (ch + 1) * 32 + kq * 8 + t;
        xn[t] = kk < a.K ? __ldcs(Rp + (size_t)kk * 2 * LN) : 0ull;
      }
      const uint4 wa = __ldg(reinterpret_cast<const uint4*>(wsrc + (size_t)ch * 4096) + tid);
      const uint4 wb = __ldg(reinterpret_cast<const uint4*>(wsrc + (size_t)ch * 4096) + 128 + tid);
      if (ch >= TC_STAGES) mbar_wait(&empty_bar[s], ((ch / TC_STAGES) - 1) & 1);
      reinterpret_cast<uint4*>(sA[s])[tid] = wa;
      reinterpret_cast<uint4*>(sA[s])[128 + tid] = wb;
      // byte transpose (PRMT): plane b gets byte b of x[0..7] (8 consecutive terms of column n)
      uint32_t pa[8], pb[8];
      {
        const uint32_t l0[4] = {(uint32_t)x[0], (uint32_t)x[1], (uint32_t)x[2], (uint32_t)x[3]};
        const uint32_t h0[4] = {(uint32_t)(x[0] >> 32), (uint32_t)(x[1] >> 32), (uint32_t)(x[2] >> 32),
                                (uint32_t)(x[3] >> 32)};
        const uint32_t l1[4] = {(uint32_t)x[4], (uint32_t)x[5], (uint32_t)x[6], (uint32_t)x[7]};
        const uint32_t h1[4] = {(uint32_t)(x[4] >> 32), (uint32_t)(x[5] >> 32), (uint32_t)(x[6] >> 32),
                                (uint32_t)(x[7] >> 32)};
        byte_tr4(l0, pa);
        byte_tr4(h0, pa + 4);
        byte_tr4(l1, pb);
        byte_tr4(h1, pb + 4);
      }
#pragma unroll
      for (int b = 0; b < 8; b++) *reinterpret_cast<uint2*>(&sB[s][b][boff]) = make_uint2(pa[b], pb[b]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&full_bar[s]);
    }
  } else if (tid == 128) {
    // ---------------- MMA issuer ----------------
    // the 8 byte planes are consecutive 8-column core-matrix groups of ONE B operand (SBO = 256 B
    // throughout), so a single UMMA with N = 8 x 32 = 256 covers all planes: D column = 32 b + col
    const uint32_t idesc = umma_idesc_s8u8(128, 8 * TC_COLS);
    for (int ch = 0; ch < nchunks; ch++) {
      const int s = ch % TC_STAGES;
      mbar_wait(&full_bar[s], (ch / TC_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t da = umma_desc_kmajor(smem_u32(sA[s]));
      {
        const uint64_t db = umma_desc_kmajor(smem_u32(sB[s][0]));
        const uint32_t acc = ch > 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&empty_bar[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&done_bar))
                 : "memory");
  }

  if (tid < 128) {
    // ---------------- epilogue: lane = MAC row ----------------
    mbar_wait(&done_bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int row = mt * 128 + warp * 32 + (tid & 31);
    const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < TC_COLS; c0 += 8) {
      uint32_t v[8][8];  // [plane][column]
#pragma unroll
      for (int b = 0; b < 8; b++) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[b][0]), "=r"(v[b][1]), "=r"(v[b][2]), "=r"(v[b][3]), "=r"(v[b][4]), "=r"(v[b][5]),
                       "=r"(v[b][6]), "=r"(v[b][7])
                     : "r"(lane_base + (uint32_t)(b * TC_COLS + c0)));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int cc = 0; cc < 8; cc++) {
        long long lo = 0, hi = 0;
#pragma unroll
        for (int b = 0; b < 4; b++) lo += (long long)(int32_t)v[b][cc] << (8 * b);
#pragma unroll
        for (int b = 4; b < 8; b++) hi += (long long)(int32_t)v[b][cc] << (8 * (b - 4));
        const int col = c0 + cc;
        tc_store(a, z, row, col >> 4, l, j0 + (col & 15), hi, lo);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 4) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
}

// Fused S2 + S3 on the tensor cores (the default for dense layers with M <= 128 MAC rows): the
// producer warps compute the key-switched R values themselves, so R never touches HBM
// (PAPER.md:373-378 hoisted PermAuto; :718-728 lazy MAC).  CTA = one unit, one limb, 16 positions
// x 2 components (32 columns), one 128-row M tile; 8 warps, 2 CTAs per SM (TMEM 2 x 256 columns),
// so one CTA's epilogue overlaps the other's main loop.  The CTA's key words (every tap, 16
// positions, limb l) are staged in shared memory once.  Chunk = 64 terms (two K = 32 UMMA steps):
// every thread key-switches 4 consecutive terms of one position, byte-transposes the 4 (c0, c1)
// pairs into the 8 byte planes with PRMT and stores one 32-bit word per plane and component; the
// digit reads of chunk ch + 1 are in flight while chunk ch is switched (register double buffer).
// There is no dedicated MMA warp: the LAST warp to finish a chunk (shared-memory ticket) issues
// its 2 x 8 UMMAs (M = 128, N = 32, K = 32, s8 x u8 -> s32) into the 8 TMEM accumulators.  TMEM is
// zeroed first and every UMMA accumulates: integer sums are exact, so the issue order of chunks by
// different warps does not matter.
constexpr int KT_THREADS = 384, KT_WARPS = KT_THREADS / 32, KT_STAGES = 2, KT_KS = 3, KT_CHUNK = 32 * KT_KS;
constexpr int KT_STAGE_A = KT_KS * 4096, KT_STAGE_B = KT_KS * 8 * 1024;
constexpr size_t KT_SMEM_MMA = (size_t)KT_STAGES * (KT_STAGE_A + KT_STAGE_B) + 1024;
inline size_t kt_smem(int T, int L) { return KT_SMEM_MMA + (size_t)T * 4 * L * TC_POS * sizeof(u64); }

// LOGN > 0: compile-time ring degree (address math folds into immediates).  UNI: Jc % 4 == 0, so
// every thread's 4-term group is one tap's consecutive cts, all real or all padding: only the
// fast paths are compiled (fewer registers).
template <int LT, int LOGN, bool UNI>
__global__ void __launch_bounds__(KT_THREADS, 2) ksmac_tc_kernel(KsMacArgs a, const int8_t* __restrict__ w8) {
  pdl_trigger();  // key staging and TMEM setup read only uploaded data: they overlap the predecessor
  extern __shared__ uint8_t kt_dyn[];
  uint8_t* smb = reinterpret_cast<uint8_t*>(((uintptr_t)kt_dyn + 1023) & ~(uintptr_t)1023);
  auto sA = [&](int s, int ks) { return smb + (size_t)s * (KT_STAGE_A + KT_STAGE_B) + ks * 4096; };
  auto sB = [&](int s, int ks, int b) {
    return smb + (size_t)s * (KT_STAGE_A + KT_STAGE_B) + KT_STAGE_A + (ks * 8 + b) * 1024;
  };
  // keys: [tap][x = 2 digit + comp][2: value, Shoup][16 positions]
  u64* skey = reinterpret_cast<u64*>(smb + (size_t)KT_STAGES * (KT_STAGE_A + KT_STAGE_B));
  __shared__ __align__(8) uint64_t empty_bar[KT_STAGES];
  __shared__ int s_ticket[KT_STAGES];
  __shared__ uint32_t s_tmem;
  __shared__ int s_haskey[HY_MAX_TAPS];
  __shared__ GaloisAct s_act[HY_MAX_TAPS];

  constexpr bool CN = LOGN > 0;
  const int N = CN ? (1 << LOGN) : (1 << a.logN);
  const int LN = LT * N;  // < 2^31
  const int tiles = N / TC_POS;
  const int l = blockIdx.x / tiles, j0 = (blockIdx.x % tiles) * TC_POS;
  const int mt = blockIdx.y, z = blockIdx.z;
  const int nmt = (a.Mpad + 127) / 128;
  const int nk32 = a.Kpad / 32;
  const int nchunks = (nk32 + KT_KS - 1) / KT_KS;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  // ---------------- producers (all warps) ----------------
  const int pos = tid & 15, tg = tid >> 4;  // position; terms 4 tg .. 4 tg + 3 of each chunk
  const int ks = tg >> 3, kg = tg & 7;
  const int j = j0 + pos;
  const u64 q = a.lcs.lc[l].q;
  const int8_t* wsrc = w8 + ((size_t)(z % a.wblocks) * nmt + mt) * nk32 * 4096;
  const u64* C0u = a.C0 + (size_t)z * a.Jcb * LN + (size_t)l * N;
  const u64* Du = a.D + (size_t)z * a.Jcb * LT * LN + (size_t)l * N;
  // K-major canonical plane offsets of column pos (c0) and 16 + pos (c1), terms 4kg .. 4kg + 3
  const int off0 = (pos >> 3) * 256 + (kg >> 2) * 128 + (pos & 7) * 16 + (kg & 3) * 4;
  const int off1 = off0 + 2 * 256;
  // (tap, c) of this thread's first term of the current chunk, advanced incrementally (no division)
  int tap0 = 0, c0t = tg * 4;
  while (c0t >= a.Jcb) {
    c0t -= a.Jcb;
    tap0++;
  }
  struct Term {
    u64 c0, d[LT];
    int tap;  // -1 = padding term (R = 0); identity tap: d[0] = D_{c,l}
  };
  Term pre[4];
  int grp = -1;  // >= 0: this chunk's 4 terms are consecutive cts of tap grp, all < K (fast path)
  auto load_chunk = [&](int ch, Term* pr) {
    int tap = tap0, c = c0t;
    // common case: the thread's 4 terms share one tap (no ct wrap) and are all real terms: one
    // permutation and base address, strided loads, no per-term tests
    if constexpr (UNI) {
      grp = ch * KT_CHUNK + tg * 4 < a.K ? tap0 : -2;  // -2: a padding group (R = 0)
      if (grp == -2) {
#pragma unroll
        for (int t = 0; t < 4; t++) pr[t].tap = -1;
        return;
      }
    } else {
      grp = (c0t + 3 < a.Jcb && ch * KT_CHUNK + tg * 4 + 3 < a.K && !a.dbg) ? tap0 : -1;
    }
    if (grp >= 0 && a.coef) {  // 1x1 coefficient domain: R = the 4 input cts themselves
      const u64* ctp = a.C0 + ((size_t)z * a.Jcb + c) * 2 * LN + (size_t)l * N + j;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        pr[t].tap = tap;
        pr[t].c0 = __ldg(ctp + (size_t)t * 2 * LN);
        pr[t].d[0] = __ldg(ctp + (size_t)t * 2 * LN + LN);
      }
      c0t += KT_CHUNK;
      while (c0t >= a.Jcb) {
        c0t -= a.Jcb;
        tap0++;
      }
      return;
    }
    if (UNI || grp >= 0) {
      const u64* C0 = C0u + (size_t)c * LN;
      const u64* D = Du + (size_t)c * (LT * LN);
      const bool ident = a.tt.key[tap] == nullptr;
      const int jp = ident ? j : galois_perm(j, a.tt.act[tap], N >> 1);
#pragma unroll
      for (int t = 0; t < 4; t++) {
        pr[t].tap = tap;
        pr[t].c0 = __ldg(C0 + (size_t)t * LN + jp);
        if (ident) {
          pr[t].d[0] = __ldg(D + (size_t)t * LT * LN + l * LN + j);
        } else {
#pragma unroll
          for (int i = 0; i < LT; i++) pr[t].d[i] = __ldg(D + (size_t)t * LT * LN + i * LN + jp);
        }
      }
      c0t += KT_CHUNK;
      while (c0t >= a.Jcb) {
        c0t -= a.Jcb;
        tap0++;
      }
      return;
    }
    if constexpr (UNI) return;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      if (t > 0 && ++c >= a.Jcb) {
        c = 0;
        tap++;
      }
      const int kk = ch * KT_CHUNK + tg * 4 + t;
      pr[t].tap = -1;
      if (kk >= a.K) continue;
      pr[t].tap = tap;
      const u64* C0 = C0u + (size_t)c * LN;
      const u64* D = Du + (size_t)c * (LT * LN);
      if (a.coef) {  // 1x1 in the coefficient domain: R = the input ct itself (identity tap only)
        const u64* ctp = a.C0 + ((size_t)z * a.Jcb + c) * 2 * LN + (size_t)l * N + j;
        pr[t].c0 = __ldg(ctp);
        pr[t].d[0] = __ldg(ctp + LN);
      } else if (a.dbg & 4) {
        pr[t].c0 = c;
#pragma unroll
        for (int i = 0; i < LT; i++) pr[t].d[i] = c + i;
      } else if (a.tt.key[tap] == nullptr) {  // identity tap: R = (C0_c, D_{c,l}) in limb l
        pr[t].c0 = __ldg(C0 + j);
        pr[t].d[0] = __ldg(D + l * LN + j);
      } else {
        const u64* Dp = D + galois_perm(j, a.tt.act[tap], N >> 1);
        pr[t].c0 = __ldg(C0 + (Dp - D));
#pragma unroll
        for (int i = 0; i < LT; i++) pr[t].d[i] = __ldg(Dp + i * LN);
      }
    }
    c0t += KT_CHUNK;  // advance to the next chunk's first term
    while (c0t >= a.Jcb) {
      c0t -= a.Jcb;
      tap0++;
    }
  };

  for (int t = tid; t < a.T; t += KT_THREADS) {
    s_haskey[t] = a.tt.key[t] != nullptr;
    s_act[t] = a.tt.act[t];
  }
  // stage the key words of this CTA (limb l, positions j0 .. j0 + 15) for every tap
  // 16 consecutive words (128 B) per (tap, digit/component, value/Shoup) row: 16-byte loads
  for (int e = tid; e < ((a.dbg & 16) ? 0 : a.T * 4 * LT * (TC_POS / 2)); e += KT_THREADS) {
    const int p2 = e % (TC_POS / 2), r = e / (TC_POS / 2);
    const int sh = r % 2, x = (r / 2) % (2 * LT), tap = r / (4 * LT);
    const u64* key = a.tt.key[tap];
    const ulonglong2 v = key ? __ldg(reinterpret_cast<const ulonglong2*>(key + (size_t)sh * 2 * LT * LN +
                                                                          (size_t)x * LN + (size_t)l * N + j0) + p2)
                             : make_ulonglong2(0ull, 0ull);
    reinterpret_cast<ulonglong2*>(skey)[e] = v;
  }
  if (tid < KT_STAGES) s_ticket[tid] = 0;
  if (tid == 0) {
    for (int s = 0; s < KT_STAGES; s++) mbar_init(&empty_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  // TMEM work split: warp w owns lane quadrant w % 4 (the tcgen05.ld/st lane restriction) and
  // every KT_WARPS / 4-th group of columns of it, so all 12 warps share the zeroing and the epilogue
  constexpr int KT_PARTS = KT_WARPS / 4;
  static_assert(KT_WARPS % 4 == 0, "whole lane quadrants");
  const int quad = warp & 3, part = warp >> 2;
  const bool rows_live = mt * 128 + quad * 32 < a.M;  // rows >= M are padding: never read back
  if (rows_live) {
    const uint32_t zb = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t z0 = 0;
#pragma unroll 1
    for (int c = part * 8; c < (int)TC_TMEM_COLS; c += 8 * KT_PARTS)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(zb + c), "r"(z0)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pdl_wait();  // D, C0 (or the input cts) come from the predecessor
  load_chunk(0, pre);

  const uint32_t idesc = umma_idesc_s8u8(128, 8 * TC_COLS);  // one UMMA covers the 8 byte planes
  // one register buffer (occupancy first: 2 CTAs x 12 warps per SM): the next chunk's digit
  // reads are issued right after this chunk's key switching
  Term* cur = pre;
#pragma unroll 1
  for (int ch = 0; ch < nchunks; ch++) {
    const int s = ch % KT_STAGES;
    const bool has_ks = KT_KS * ch + ks < nk32;
    // weights: K step ws = tid >> 7 of this chunk, 2 x 16 B per thread
    const int ws = tid >> 7;
    const bool has_w = KT_KS * ch + ws < nk32;
    uint4 wv = make_uint4(0, 0, 0, 0), wv2 = make_uint4(0, 0, 0, 0);
    if (has_w) {
      const uint4* wp = reinterpret_cast<const uint4*>(wsrc + (size_t)(KT_KS * ch + ws) * 4096) + (tid & 127);
      wv = __ldg(wp);
      wv2 = __ldg(wp + 128);
    }
    // key switching, fully lazy: Shoup products are in [0, 2q), so R.c0 < (2L + 1) q and
    // R.c1 < 2L q stay below 2^64 (q < 2^60, L <= 5 -> 11 q).  The MAC is exact for any 64-bit
    // R (byte planes), and the epilogue's single reduction makes the output canonical, so R
    // needs no reduction at all.
    uint32_t lo0[4], hi0[4], lo1[4], hi1[4];
    if (UNI && grp < 0) {  // padding group
#pragma unroll
      for (int t = 0; t < 4; t++) lo0[t] = hi0[t] = lo1[t] = hi1[t] = 0;
    } else if (UNI && !s_haskey[grp]) {  // identity tap
#pragma unroll
      for (int t = 0; t < 4; t++) {
        lo0[t] = (uint32_t)cur[t].c0;
        hi0[t] = (uint32_t)(cur[t].c0 >> 32);
        lo1[t] = (uint32_t)cur[t].d[0];
        hi1[t] = (uint32_t)(cur[t].d[0] >> 32);
      }
    } else if (UNI || (grp >= 0 && s_haskey[grp])) {  // fast path: one tap, 4 real terms, keys at one address
      const u64* kp = skey + (size_t)grp * 4 * LT * TC_POS + pos;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        u64 r0 = cur[t].c0, r1 = 0;
#pragma unroll
        for (int i = 0; i < LT; i++) {
          r0 += shoup_mul(cur[t].d[i], kp[(4 * i) * TC_POS], kp[(4 * i + 1) * TC_POS], q);
          r1 += shoup_mul(cur[t].d[i], kp[(4 * i + 2) * TC_POS], kp[(4 * i + 3) * TC_POS], q);
        }
        lo0[t] = (uint32_t)r0;
        hi0[t] = (uint32_t)(r0 >> 32);
        lo1[t] = (uint32_t)r1;
        hi1[t] = (uint32_t)(r1 >> 32);
      }
    } else if constexpr (!UNI)
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int tap = cur[t].tap;
      u64 r0 = 0, r1 = 0;
      if (tap >= 0) {
        r0 = cur[t].c0;
        if (!s_haskey[tap] || (a.dbg & 2)) {
          r1 = cur[t].d[0];
        } else {
          const u64* kp = skey + (size_t)tap * 4 * LT * TC_POS + pos;
#pragma unroll
          for (int i = 0; i < LT; i++) {
            r0 += shoup_mul(cur[t].d[i], kp[(4 * i) * TC_POS], kp[(4 * i + 1) * TC_POS], q);
            r1 += shoup_mul(cur[t].d[i], kp[(4 * i + 2) * TC_POS], kp[(4 * i + 3) * TC_POS], q);
          }
        }
      }
      lo0[t] = (uint32_t)r0;
      hi0[t] = (uint32_t)(r0 >> 32);
      lo1[t] = (uint32_t)r1;
      hi1[t] = (uint32_t)(r1 >> 32);
    }
    if (ch + 1 < nchunks) load_chunk(ch + 1, pre);
    uint32_t p0[8], p1[8];
    byte_tr4(lo0, p0);
    byte_tr4(hi0, p0 + 4);
    byte_tr4(lo1, p1);
    byte_tr4(hi1, p1 + 4);
    if (ch >= KT_STAGES) mbar_wait(&empty_bar[s], ((ch / KT_STAGES) - 1) & 1);
    if (has_w) {
      reinterpret_cast<uint4*>(sA(s, ws))[tid & 127] = wv;
      reinterpret_cast<uint4*>(sA(s, ws))[128 + (tid & 127)] = wv2;
    }
    if (has_ks) {
#pragma unroll
      for (int b = 0; b < 8; b++) {
        *reinterpret_cast<uint32_t*>(sB(s, ks, b) + off0) = p0[b];
        *reinterpret_cast<uint32_t*>(sB(s, ks, b) + off1) = p1[b];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      // the ticket atomic is the thread synchronisation between successive UMMA issuers: order
      // this thread's earlier tcgen05 ops (its last issue + commit) before it
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __threadfence_block();
      const int prev = atomicAdd(&s_ticket[s], 1);  // monotonic: use u of stage s takes tickets
      if (prev % KT_WARPS == KT_WARPS - 1) {       // 8u .. 8u + 7; the last warp issues the UMMAs
        __threadfence_block();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int k2 = 0; k2 < KT_KS && KT_KS * ch + k2 < nk32 && !(a.dbg & 1); k2++) {
          const uint64_t da = umma_desc_kmajor(smem_u32(sA(s, k2)));
          const uint64_t db = umma_desc_kmajor(smem_u32(sB(s, k2, 0)));  // all 8 planes: N = 256
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(da), "l"(db),
              "r"(idesc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&empty_bar[s]))
                     : "memory");
      }
    }
    __syncwarp();
  }

  // ---------------- epilogue: warp w reads TMEM lanes 32 (w % 4) .., columns of component w / 4
  // every chunk's UMMAs are complete once the last KT_STAGES chunks' commits have arrived (earlier
  // stages were waited for before their reuse)
  for (int ch = nchunks > KT_STAGES ? nchunks - KT_STAGES : 0; ch < nchunks; ch++)
    mbar_wait(&empty_bar[ch % KT_STAGES], (ch / KT_STAGES) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rows_live && !(a.dbg & 8)) {
    const int row = mt * 128 + quad * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
    for (int c0 = part * 4; c0 < TC_COLS; c0 += 4 * KT_PARTS) {  // groups of 4 columns
      uint32_t v[8][4];  // [plane][column]
#pragma unroll
      for (int b = 0; b < 8; b++) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[b][0]), "=r"(v[b][1]), "=r"(v[b][2]), "=r"(v[b][3])
                     : "r"(lane_base + (uint32_t)(b * TC_COLS + c0)));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      long long lo4[4], hi4[4];
#pragma unroll
      for (int cc = 0; cc < 4; cc++) {
        long long lo = 0, hi = 0;
#pragma unroll
        for (int b = 0; b < 4; b++) lo += (long long)(int32_t)v[b][cc] << (8 * b);
#pragma unroll
        for (int b = 4; b < 8; b++) hi += (long long)(int32_t)v[b][cc] << (8 * (b - 4));
        lo4[cc] = lo;
        hi4[cc] = hi;
      }
      tc_store4<LT, LOGN>(a, z, row, c0 >> 4, l, j0 + (c0 & 15), hi4, lo4);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
}

#include "ksmac_v2.cuh"

template <int LT, int LOGN, int EPI>
hy_status launch_ksmac_v2_t(const KsMacArgs& a, const int8_t* w8, int units, const V2Geom& g, cudaStream_t s) {
  int dev = 0, nsm = 148;
  HY_CUDA_TRY(cudaGetDevice(&dev));
  HY_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int ntiles = units * a.L * ((1 << a.logN) / TC_POS);
  HY_CUDA_TRY(hy_smem_attr((const void*)ksmac_v2_kernel<LT, LOGN, EPI>, g.bytes));
  HY_CUDA_TRY(hy_launch(ksmac_v2_kernel<LT, LOGN, EPI>, dim3((unsigned)std::min(ntiles, nsm)),
                        dim3(V2Warps<EPI>::THREADS), g.bytes, s, 1, a, w8, g, units));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

#include "ksmac_v3.cuh"

template <int LT, int LOGN, int EPI>
hy_status launch_ksmac_v3_t(const KsMacArgs& a, const int8_t* w8, int units, const V2Geom& g, cudaStream_t s) {
  int dev = 0, nsm = 148;
  HY_CUDA_TRY(cudaGetDevice(&dev));
  HY_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int ntiles = units * a.L * ((1 << a.logN) / V3_POS);
  HY_CUDA_TRY(hy_smem_attr((const void*)ksmac_v3_kernel<LT, LOGN, EPI>, g.bytes));
  HY_CUDA_TRY(hy_launch(ksmac_v3_kernel<LT, LOGN, EPI>, dim3((unsigned)std::min(ntiles, nsm)),
                        dim3(V3Warps<EPI>::THREADS), g.bytes, s, 1, a, w8, g, units));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LT, int LOGN>
hy_status launch_ksmac_v2(const KsMacArgs& a, const int8_t* w8, int units, const V2Geom& g, cudaStream_t s) {
  return a.M <= 64 ? launch_ksmac_v2_t<LT, LOGN, 2>(a, w8, units, g, s) : launch_ksmac_v2_t<LT, LOGN, 4>(a, w8, units, g, s);
}

template <int LT, int LOGN, bool UNI>
hy_status launch_ksmac_tc_t(const KsMacArgs& a, const int8_t* w8, int units, cudaStream_t s) {
  const int N = 1 << a.logN;
  HY_CUDA_TRY(hy_smem_attr((const void*)ksmac_tc_kernel<LT, LOGN, UNI>, kt_smem(HY_MAX_TAPS, LT)));
  dim3 grid((unsigned)(a.L * (N / TC_POS)), (unsigned)((a.Mpad + 127) / 128), (unsigned)units);
  HY_CUDA_TRY(hy_launch(ksmac_tc_kernel<LT, LOGN, UNI>, grid, dim3(KT_THREADS), kt_smem(a.T, LT), s, 1, a, w8));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

// N = 8192 (the metric's ring degree) gets compile-time address math; other N the generic kernel
template <int LT>
hy_status launch_ksmac_tc(const KsMacArgs& a, const int8_t* w8, int units, cudaStream_t s) {
  const bool uni = a.Jcb % 4 == 0 && a.K % 4 == 0 && !a.dbg;
  // default (2): the persistent Shoup-producer kernel; HY_KSMAC=1: the non-persistent one, 3: the
  // persistent exact-product kernel (A/B measurements: measured slower at C4)
  static const int ver = getenv("HY_KSMAC") ? atoi(getenv("HY_KSMAC")) : 2;
  if (uni && !a.coef && ver == 3 && a.Mpad <= 128 && a.wblocks == 1) {
    const V2Geom g = v3_geom(a.T, LT, a.Kpad, 232448);
    if (g.S >= 2) {
      if (a.logN == 13)
        return a.M <= 64 ? launch_ksmac_v3_t<LT, 13, 2>(a, w8, units, g, s) : launch_ksmac_v3_t<LT, 13, 4>(a, w8, units, g, s);
      return a.M <= 64 ? launch_ksmac_v3_t<LT, 0, 2>(a, w8, units, g, s) : launch_ksmac_v3_t<LT, 0, 4>(a, w8, units, g, s);
    }
  }
  if (uni && !a.coef && ver == 2 && a.Mpad <= 128 && a.wblocks == 1) {
    const V2Geom g = v2_geom(a.T, LT, a.Kpad, 232448, a.M);
    if (g.S >= 2) {
      if (a.logN == 13) return launch_ksmac_v2<LT, 13>(a, w8, units, g, s);
      return launch_ksmac_v2<LT, 0>(a, w8, units, g, s);
    }
  }
  if (a.logN == 13) return uni ? launch_ksmac_tc_t<LT, 13, true>(a, w8, units, s) : launch_ksmac_tc_t<LT, 13, false>(a, w8, units, s);
  return uni ? launch_ksmac_tc_t<LT, 0, true>(a, w8, units, s) : launch_ksmac_tc_t<LT, 0, false>(a, w8, units, s);
}

hy_status launch_mac_tc(const KsMacArgs& a, const u64* R, const int8_t* w8, int units, cudaStream_t s) {
  const int N = 1 << a.logN;
  dim3 grid((unsigned)(a.L * (N / TC_POS) * ((a.Mpad + 127) / 128)), 1, (unsigned)units);
  mac_tc_kernel<<<grid, TC_THREADS, 0, s>>>(a, R, w8);
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int WM>
hy_status launch_mac_gemm(const KsMacArgs& a, const u64* R, int units, cudaStream_t s) {
  using TL = MgTile<WM>;
  const int N = 1 << a.logN;
  HY_CUDA_TRY(hy_smem_attr((const void*)mac_gemm_kernel<WM>, TL::SMEM));
  dim3 grid((unsigned)(a.L * (N / TL::BNP)), (unsigned)(a.Mpad / TL::BM), (unsigned)units);
  mac_gemm_kernel<WM><<<grid, 256, TL::SMEM, s>>>(a, R);
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LT>
hy_status launch_permauto(const KsMacArgs& a, u64* R, int units, cudaStream_t s) {
  const int N = 1 << a.logN;
  dim3 grid((unsigned)((a.L * N + 255) / 256), (unsigned)a.T, (unsigned)units);
  permauto_kernel<LT><<<grid, 256, 0, s>>>(a, R);
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int WM, int LT>
hy_status launch_ksmac_gemm_t(const KsMacArgs& a, int units, cudaStream_t s) {
  const int N = 1 << a.logN, BNP = 256 / WM, KC = 2 * WM;
  const size_t sm0 = sizeof(double2) * 2 * KC * 2 * BNP + sizeof(double) * 2 * KC * 8 * WM;
  const size_t sm = sm0 + (LT > 0 ? (size_t)a.T * 4 * LT * BNP * sizeof(u64) : 0);
  HY_CUDA_TRY(hy_smem_attr((const void*)ksmac_gemm_kernel<WM, LT>, sm));
  dim3 grid((unsigned)(a.L * (N / BNP)), (unsigned)(a.Mpad / (8 * WM)), (unsigned)units);
  HY_CUDA_TRY(hy_launch(ksmac_gemm_kernel<WM, LT>, grid, dim3(256), sm, s, 1, a));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

// the key-staging variant (LT > 0) while its shared memory stays <= 100 KB (2 CTAs per SM), else
// the generic one (keys through L1)
template <int WM, int LT>
hy_status launch_ksmac_gemm(const KsMacArgs& a, int units, cudaStream_t s) {
  const size_t keys = (size_t)a.T * 4 * (LT > 0 ? LT : 1) * (256 / WM) * sizeof(u64);
  if (LT > 0 && keys <= 64 * 1024) return launch_ksmac_gemm_t<WM, LT>(a, units, s);
  return launch_ksmac_gemm_t<WM, 0>(a, units, s);
}

template <int MR, int LT>
hy_status launch_ksmac_thin(const KsMacArgs& a, int units, cudaStream_t s) {
  const int N = 1 << a.logN;
  constexpr int CPT = LT == 5 ? 2 : 4;  // units per thread (registers: CPT x (L + 1) digits + 4 MR sums)
  dim3 grid((unsigned)((a.L * N + 255) / 256), 1, (unsigned)((units + CPT - 1) / CPT));
  HY_CUDA_TRY(hy_launch(ksmac_thin_kernel<MR, LT, CPT>, grid, dim3(256), 0, s, 1, a, units));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LT>
hy_status launch_ksmac(const KsMacArgs& a, int tile, int units, cudaStream_t s) {
  switch (tile) {
    case -1: return launch_ksmac_thin<1, LT>(a, units, s);
    case -2: return launch_ksmac_thin<2, LT>(a, units, s);
    case 1: return launch_ksmac_gemm<1, LT>(a, units, s);
    case 2: return launch_ksmac_gemm<2, LT>(a, units, s);
    case 4: return launch_ksmac_gemm<4, LT>(a, units, s);
    case 8: return launch_ksmac_gemm<8, LT>(a, units, s);
  }
  hy_set_error("ksmac: bad row tile");
  return HY_EINVAL;
}

// ------------------------------------------------------------------------------------------
// Client-side draws on the GPU (hy_secret_key / hy_keygen / hy_encrypt):
// Philox4x32-10 with the counter layout and the value mappings of synth/philox.py, which the
// oracle-side client reimplements in NumPy (bit-identical draws; tests/test_gpu_client.py).
// ------------------------------------------------------------------------------------------
struct Philox4 {
  uint32_t x[4];
};
__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint64_t seed) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return Philox4{{c0, c1, c2, c3}};
}
// floor(X q / 2^128), X = the 128-bit block
__device__ __forceinline__ u64 philox_uniform(const Philox4& b, u64 q) {
  const u64 xlo = (u64)b.x[0] | ((u64)b.x[1] << 32), xhi = (u64)b.x[2] | ((u64)b.x[3] << 32);
  const u64 a1 = __umul64hi(xhi, q), a0 = xhi * q, b1 = __umul64hi(xlo, q);
  const u64 s = a0 + b1;
  return a1 + (s < a0 ? 1ull : 0ull);
}
__device__ __forceinline__ int philox_ternary(const Philox4& b) {
  const u64 y = (u64)b.x[0] | ((u64)b.x[1] << 32);
  return (int)__umul64hi(y, 3ull) - 1;
}
__device__ __forceinline__ int philox_cbd20(const Philox4& b) {
  const u64 y = (u64)b.x[0] | ((u64)b.x[1] << 32);
  return __popcll(y & 0xFFFFFull) - __popcll((y >> 20) & 0xFFFFFull);
}

// secret s (ternary) lifted into every limb: out [L][N]
__global__ void gen_secret_kernel(u64 seed, int L, int logN, QArr qa, u64* __restrict__ s_res, int8_t* __restrict__ s8) {
  const int N = 1 << logN;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < N; k += gridDim.x * blockDim.x) {
    const int v = philox_ternary(philox4x32_10((uint32_t)k, 0u, 0u, 1u, seed));
    if (s8) s8[k] = (int8_t)v;
    for (int l = 0; l < L; l++) s_res[(size_t)l * N + k] = v >= 0 ? (u64)v : qa.q[l] - 1;
  }
}

// masks: uniform residues [n][L][N] with counter (k, c1 = base1 + o, c2 = base2 + l (key: 256 i + l), purpose)
struct MaskArgs {
  u64 seed;
  uint32_t purpose;
  int L, logN;
  size_t n;
  const uint32_t* c1;   // per poly-group o: counter word 1 (encryption index or Galois element)
  uint32_t digits;      // key masks: group o = (element, digit dd) with `digits` digits: c2 = 256 dd + l;
                        // encryption (0): c2 = l
  QArr qa;
};
__global__ void gen_mask_kernel(MaskArgs m, u64* __restrict__ out) {
  const int N = 1 << m.logN;
  const size_t total = m.n * m.L * (size_t)N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx & (N - 1));
    const size_t ol = idx >> m.logN;
    const int l = (int)(ol % m.L);
    const size_t o = ol / m.L;
    uint32_t c1, c2;
    if (m.digits) {  // key: o = element index * digits + digit
      c1 = m.c1[o / m.digits];
      c2 = 256u * (uint32_t)(o % m.digits) + (uint32_t)l;
    } else {
      c1 = m.c1[o];
      c2 = (uint32_t)l;
    }
    out[idx] = philox_uniform(philox4x32_10((uint32_t)k, c1, c2, m.purpose, m.seed), m.qa.q[l]);
  }
}
// errors: centered binomial [n][N] (int32), counter (k, c1, c2 = 256 i for keys / 0, purpose)
__global__ void gen_error_kernel(u64 seed, uint32_t purpose, int logN, size_t n, const uint32_t* __restrict__ c1v,
                                 int digits, int32_t* __restrict__ out) {
  const int N = 1 << logN;
  const size_t total = n * (size_t)N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx & (N - 1));
    const size_t o = idx >> logN;
    const uint32_t c1 = digits ? c1v[o / digits] : c1v[o];
    const uint32_t c2 = digits ? 256u * (uint32_t)(o % digits) : 0u;
    out[idx] = philox_cbd20(philox4x32_10((uint32_t)k, c1, c2, purpose, seed));
  }
}

// c = INTT(NTT(a) .* NTT(s)) and the client's combination, per (poly o, limb):
//   encryption: c0 = [Delta m + a s + e], c1 = [-a]           (symmetric BFV)
//   key digit dd = i V + v: b = [-a s + e_dd + [i == l] 2^{w v} s(X^g)], a kept  (reading R5; sub-digit base)
struct ClientInvJob {
  const u64* An;        // [n][L][N] NTT(a)
  const u64* Sn;        // [L][N] NTT(s), then [L][N] Shoup companions
  const u64* A;         // [n][L][N] a (coefficient form)
  const int32_t* E;     // [n][N] errors
  const u64* M;         // encryption: [n][N] plaintext coefficients (< t); keys: null
  const u64* Sg;        // keys: [n_elts][L][N] s(X^g) lifted per limb; encryption: null
  u64* out;             // [n][2][L][N]
  int L, N, digits;     // digits = ND for keys (o = element * ND + dd), 0 for encryption
  QArr qa, delta;       // delta: Delta mod q_l
  int V, wd;            // sub-digits per limb and base bits (V = 1: one digit per limb)
  int limb, o;
  __device__ void bind(int b) {
    o = b / L;
    limb = b % L;
  }
  __device__ u64 load(int k) const {
    const size_t at = ((size_t)o * L + limb) * N + k;
    const u64 q = qa.q[limb];
    return csub(shoup_mul(An[at], Sn[(size_t)limb * N + k], Sn[(size_t)(L + limb) * N + k], q), q);
  }
  __device__ void store(int k, u64 as) const {
    const u64 q = qa.q[limb];
    const size_t at = ((size_t)o * L + limb) * N + k;
    const int32_t e = E[(size_t)o * N + k];
    const u64 er = e >= 0 ? (u64)e : q - (u64)(-e);
    u64* c = out + (size_t)o * 2 * L * N;
    if (!digits) {
      const u64 dm = mulmod_slow(delta.q[limb], M[(size_t)o * N + k], q);
      c[(size_t)limb * N + k] = csub(csub(csub(dm + as, q) + er, q), q);
      c[(size_t)(L + limb) * N + k] = A[at] ? q - A[at] : 0;
    } else {
      const int dd = o % digits;
      u64 b = csub((as ? q - as : 0) + er, q);
      if (dd / V == limb) {
        const u64 sgv = Sg[((size_t)(o / digits) * L + limb) * N + k];
        b = csub(b + (V > 1 ? mulmod_slow(sgv, (1ull << (wd * (dd % V))) % q, q) : sgv), q);
      }
      c[(size_t)limb * N + k] = b;
      c[(size_t)(L + limb) * N + k] = A[at];
    }
  }
};

// s(X^g) coefficient form, lifted per limb: sg[l][(k g) mod N] = +/- s[k]
__global__ void automorph_secret_kernel(const int8_t* __restrict__ s8, const uint32_t* __restrict__ elts, int n_elts,
                                        int L, int logN, QArr qa, u64* __restrict__ sg) {
  const int N = 1 << logN;
  const size_t total = (size_t)n_elts * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx & (N - 1));
    const int e = (int)(idx >> logN);
    const u64 pos = ((u64)k * elts[e]) % (2 * (u64)N);
    int v = s8[k];
    int at = (int)pos;
    if (pos >= (u64)N) {
      at -= N;
      v = -v;
    }
    for (int l = 0; l < L; l++) sg[((size_t)e * L + l) * N + at] = v >= 0 ? (u64)v : qa.q[l] - (u64)(-v);
  }
}

}  // namespace

// ============================================================================================
// launchers
// ============================================================================================
namespace hyk {

hy_status ntt_poly_fwd(const hy_params* p, const u64* src, u64* dst, size_t npoly, cudaStream_t s) {
  PolyJob j{src, dst, (int)p->L, (int)p->N};
  return launch_fwd(p, j, npoly * p->L, s);
}

hy_status ntt_poly_inv(const hy_params* p, const u64* src, u64* dst, size_t npoly, cudaStream_t s) {
  PolyJob j{src, dst, (int)p->L, (int)p->N};
  return launch_inv(p, j, npoly * p->L, s);
}

hy_status pointwise_mul(const hy_params* p, const u64* A, const u64* B, u64* C, size_t npoly, cudaStream_t s) {
  ProdInvJob j{A, B, C, (int)p->L, (int)p->N, qarr(p)};
  return launch_inv(p, j, npoly * p->L, s);
}

hy_status shoup_table(const hy_params* p, const u64* w, u64* wsh, size_t npoly, cudaStream_t s) {
  const size_t total = npoly * p->L * p->N;
  shoup_table_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 16), 256, 0, s>>>(w, wsh, total, p->N, p->L,
                                                                                                 qarr(p));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

hy_status key_to_ntt(const hy_params* p, const u64* key_coeff, u64* key_ntt, cudaStream_t s) {
  // key [L][2][L][N] -> NTT per (digit, comp, limb); Shoup companions in the following block, then
  // the 30-bit split values (the exact-product MAC producers, ksmac_v3)
  const size_t npoly = 2 * p->ND;  // groups of L limbs
  const size_t words = npoly * p->L * p->N;
  HY_TRY(ntt_poly_fwd(p, key_coeff, key_ntt, npoly, s));
  HY_TRY(shoup_table(p, key_ntt, key_ntt + words, npoly, s));
  split30_kernel<<<(unsigned)std::min<size_t>((words + 255) / 256, 148 * 16), 256, 0, s>>>(key_ntt, key_ntt + 2 * words,
                                                                                           words);
  HY_LAUNCH_CHECK();
  return HY_OK;
}

hy_status c0_only(const hy_params* p, const u64* ct, size_t nct, u64* C0, cudaStream_t s) {
  PermDecompJob j{ct, nullptr, C0, (int)p->L, (int)p->N, qarr(p)};
  j.c0_only = true;
  return launch_fwd(p, j, nct * p->L, s);
}

hy_status permdecomp(const hy_params* p, const u64* ct, size_t nct, u64* D, u64* C0, cudaStream_t s) {
  if (p->ND != p->L) {
    PermDecompSubJob j{ct, D, C0, (int)p->L, (int)p->N, (int)p->ND, (int)p->V, (int)p->w_dcmp, 0};
    return launch_fwd(p, j, nct * (p->ND * p->L + p->L), s);
  }
  PermDecompJob j{ct, D, C0, (int)p->L, (int)p->N, qarr(p)};
  return launch_fwd(p, j, nct * (p->L * p->L + p->L), s);
}

// MAC-kernel timing (bench): record an event before/after each MAC launch when enabled
static hy_status mac_mark(hy_weights* w, cudaStream_t s) {
  if (!w->n_ev) return HY_OK;
  if (!w->mac_ev) w->mac_ev = new std::vector<cudaEvent_t>();
  std::vector<cudaEvent_t>& v = *w->mac_ev;
  if (v.size() <= 2 * w->mac_launches + 1) {
    cudaEvent_t e0, e1;
    HY_CUDA_TRY(cudaEventCreate(&e0));
    HY_CUDA_TRY(cudaEventCreate(&e1));
    v.push_back(e0);
    v.push_back(e1);
  }
  return HY_OK;
}

// no-hoisting ablation: rotated inputs R of units u0 .. u0 + nb - 1 by every tap, each rotation with its
// own decomposition of the rotated c1 (DirectDecompJob) and key inner product (ks_apply, d_rot)
static hy_status direct_rotations(hy_weights* w, const u64* ct_in, int u0, int nb, cudaStream_t s) {
  const hy_params* p = w->p;
  const hy_layout& lay = w->lay;
  const size_t L = p->L, N = p->N, LN = L * N, Jc = lay.Jc, ctw = 2 * LN;
  const u64 M2 = 2 * (u64)N;
  for (int zb = 0; zb < nb; zb++) {
    const size_t z = (size_t)u0 + zb;
    for (uint32_t tau = 0; tau < lay.n_taps; tau++) {
      const int64_t st = (((int64_t)lay.tap_step[tau] % (int64_t)(N / 2)) + N / 2) % (N / 2);
      const u64 g = hyhost::powmod(3, (u64)st, M2), ginv = hyhost::powmod(g, N - 1, M2);  // |Z_2N^*| = N
      DirectDecompJob jd{ct_in + z * Jc * ctw, w->d_D, (int)L, (int)N, (int)p->ND, (int)p->V, (int)p->w_dcmp,
                         qarr(p), onesh_arr(p), (uint32_t)ginv};
      HY_TRY(launch_fwd(p, jd, Jc * p->ND * L, s));
      u64* R = w->d_R + ((size_t)zb * w->K + (size_t)tau * Jc) * ctw;
      if (w->h_tap_keys[tau] == nullptr) {
        ident_r_kernel<<<148 * 4, 256, 0, s>>>(w->d_C0 + z * Jc * LN, w->d_D, R, (int)Jc, (int)L, (int)p->ND,
                                                (int)p->w_dcmp, (int)p->logN, qarr(p));
        HY_LAUNCH_CHECK();
        continue;
      }
      KsApplyArgs ka;
      ka.ND = (int)p->ND;
      ka.d_rot = 1;
      ka.c0 = w->d_C0 + z * Jc * LN;
      ka.c0_stride = LN;
      ka.D = w->d_D;
      ka.D_stride = p->ND * LN;
      ka.diag = nullptr;
      ka.diag_stride = 0;
      ka.add = nullptr;
      ka.add_stride = 0;
      ka.key = w->h_tap_keys[tau];
      ka.act = w->h_tap_act[tau];
      ka.out = R;
      ka.L = (int)L;
      ka.logN = (int)p->logN;
      ka.total = Jc * LN;
      ka.lcs = limb_consts(p);
      HY_TRY(launch_ks_apply(ka, s));
    }
  }
  return HY_OK;
}

hy_status ksmac(hy_weights* w, const u64* ct_in, size_t nunits, cudaStream_t s) {
  w->mac_launches = 0;
  const hy_params* p = w->p;
  const hy_layout& lay = w->lay;
  const bool dw = w->shape.depthwise != 0;
  KsMacArgs a{};
  a.D = w->d_D;
  a.C0 = w->d_C0;
  a.keys = w->d_tap_keys;
  a.act = w->d_tap_act;
  for (uint32_t t = 0; t < lay.n_taps && t < HY_MAX_TAPS; t++) {
    a.tt.key[t] = w->h_tap_keys[t];
    a.tt.act[t] = w->h_tap_act[t];
  }
  a.wt = w->d_wt;
  a.out = w->d_P;
  a.sign = w->d_sign;
  a.kt = w->d_kt;
  static const int dbg = getenv("HY_DEBUG_KSMAC") ? atoi(getenv("HY_DEBUG_KSMAC")) : 0;
  a.dbg = dbg;
  a.T = (int)lay.n_taps;
  a.Jcb = dw ? 1 : (int)lay.Jc;
  a.K = w->K;
  a.Kpad = w->Kpad;
  a.M = w->M;
  a.Mpad = w->Mpad;
  a.wblocks = w->wblocks;
  a.L = (int)p->L;
  a.logN = (int)p->logN;
  a.kscale = (int)lay.k;
  a.cn = (int)lay.cn;
  a.lcs = limb_consts(p);
  a.ND = (int)p->ND;
  a.wd = (int)p->w_dcmp;
  const int units = (int)(dw ? nunits * lay.Jc : nunits);
  const int tile = hy_mac_tile(w->M, dw);
  const int path = w->mac_path;
  const int Lsel = p->ND == p->L ? (int)p->L : 0;  // a sub-digit base takes the generic kernels
  if (path == HY_MAC_THIN || path == HY_MAC_FP64_FUSED) {  // key switching fused into the FP64 MAC
    HY_TRY(mac_mark(w, s));
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[0], s));
    hy_status st;
    switch (Lsel) {  // compile-time digit count for the common L
      case 2: st = launch_ksmac<2>(a, tile, units, s); break;
      case 3: st = launch_ksmac<3>(a, tile, units, s); break;
      case 5: st = launch_ksmac<5>(a, tile, units, s); break;
      default: st = launch_ksmac<0>(a, tile, units, s); break;
    }
    HY_TRY(st);
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[1], s));
    w->mac_launches = 1;
    return HY_OK;
  }
  if (path == HY_MAC_TC_FUSED) {  // key switching in the producers of the tensor-core MAC
    HY_TRY(mac_mark(w, s));
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[0], s));
    hy_status st = p->L == 2 ? launch_ksmac_tc<2>(a, w->d_w8, units, s)
                 : p->L == 3 ? launch_ksmac_tc<3>(a, w->d_w8, units, s)
                             : launch_ksmac_tc<5>(a, w->d_w8, units, s);
    HY_TRY(st);
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[1], s));
    w->mac_launches = 1;
    return HY_OK;
  }
  const bool fp64_mac = path == HY_MAC_FP64_SPLIT;
  // dense: PermAuto materialises R for a batch of units, the MAC GEMM consumes it
  const size_t LN = (size_t)p->L * p->N;
  const int mrows = lay.cn == 4 ? w->M / 4 : lay.cn == 2 ? w->M / 2 : w->M;  // output P rows per unit
  for (int u0 = 0; u0 < units; u0 += w->r_units) {
    const int nb = std::min(w->r_units, units - u0);
    KsMacArgs b = a;
    b.D = a.D + (size_t)u0 * a.Jcb * p->ND * LN;
    b.C0 = a.C0 + (size_t)u0 * a.Jcb * LN;
    b.out = a.out + (size_t)u0 * mrows * 2 * LN;
    if (path == HY_MAC_DIRECT) {
      HY_TRY(direct_rotations(w, ct_in, u0, nb, s));
    } else {
      switch (Lsel) {
        case 2: HY_TRY(launch_permauto<2>(b, w->d_R, nb, s)); break;
        case 3: HY_TRY(launch_permauto<3>(b, w->d_R, nb, s)); break;
        case 5: HY_TRY(launch_permauto<5>(b, w->d_R, nb, s)); break;
        default: HY_TRY(launch_permauto<0>(b, w->d_R, nb, s)); break;
      }
    }
    HY_TRY(mac_mark(w, s));
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[2 * w->mac_launches], s));
    if (path == HY_MAC_EAGER) {
      mac_eager_kernel<<<148 * 16, 256, 0, s>>>(b, w->d_R, w->d_wq, nb);
      HY_LAUNCH_CHECK();
    } else if (fp64_mac) {
      HY_TRY(launch_mac_gemm<8>(b, w->d_R, nb, s));
    } else {
      HY_TRY(launch_mac_tc(b, w->d_R, w->d_w8, nb, s));
    }
    if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[2 * w->mac_launches + 1], s));
    w->mac_launches++;
  }
  return HY_OK;
}

// P = [A0] + S * [A1] in the coefficient domain, S = s (X^{N/4} + X^{3N/4}) (the [k, -k] sign
// plaintext): (S * A1)[j] = s (+/- A1[j - N/4] +/- A1[j - 3N/4]) with the
// negacyclic sign for wrapped indices.  In place over P (= A0) [n][2][L][N]; canonical output.
__global__ void sign_combine_kernel(u64* __restrict__ P, const u64* __restrict__ A1, size_t total, int logN, int L,
                                    LimbConsts lcs, QArr sv, QArr svsh) {
  pdl_begin();
  const int N = 1 << logN;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(i & (N - 1));
    const int l = (int)((i >> logN) % L);
    const u64 q = lcs.lc[l].q;
    const size_t row = i - j;
    const u64 t1 = A1[row + ((j - N / 4) & (N - 1))], t3 = A1[row + ((j - 3 * N / 4) & (N - 1))];
    const u64 u = (j >= N / 4 ? t1 : q - t1) + (j >= 3 * N / 4 ? t3 : q - t3);  // < 2q
    u64 v = P[i] + shoup_mul(u, sv.q[l], svsh.q[l], q);
    v = csub(v, 2 * q);
    P[i] = csub(v, q);
  }
}

// 1x1 convolution with c_n = 1 (SURVEY §8(a) special case): the only tap is
// the identity, so the hoisted rotation is the input itself and the MAC is linear: computing
// Out_o = sum_c W[o][c] ct_c on the coefficient-form inputs and reducing once gives the same
// canonical residues as NTT -> MAC -> INTT, with no NTT at all.  The tensor-core MAC reads the
// input ciphertexts [unit][c][2][L][N] as its R operand and writes ct_out [unit][o][2][L][N].
hy_status mac_coef(hy_weights* w, const u64* ct_in, size_t nunits, u64* ct_out, cudaStream_t s) {
  w->mac_launches = 0;
  const hy_params* p = w->p;
  KsMacArgs a{};
  a.out = ct_out;
  a.sign = nullptr;
  a.T = 1;
  a.Jcb = (int)w->lay.Jc;
  a.K = w->K;
  a.Kpad = w->Kpad;
  a.M = w->M;
  a.Mpad = w->Mpad;
  a.wblocks = w->wblocks;
  a.L = (int)p->L;
  a.logN = (int)p->logN;
  a.kscale = (int)w->lay.k;
  a.cn = (int)w->lay.cn;
  a.lcs = limb_consts(p);
  a.out2 = nullptr;
  if (a.cn == 2) {  // [A0] -> P, [A1] -> A1 buffer; the sign PMult and the row swap follow
    a.out = w->d_P;
    a.out2 = w->d_A1;
  }
  // the fused kernel's producers read the inputs directly (identity tap, no key switching): 12
  // warps per CTA and 8 epilogue warps (the epilogue, one reduction per output coefficient,
  // dominates a 1x1 layer)
  a.coef = 1;
  static const int dbg = getenv("HY_DEBUG_KSMAC") ? atoi(getenv("HY_DEBUG_KSMAC")) : 0;
  a.dbg = dbg;
  a.C0 = ct_in;
  a.D = ct_in;
  a.kt = w->d_kt;
  a.tt.key[0] = nullptr;
  a.tt.act[0] = GaloisAct{0u, 0u};
  HY_TRY(mac_mark(w, s));
  if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[0], s));
  if (p->L == 2 || p->L == 3) {  // (L = 5 spills at 12 warps x 80 registers: the older MAC kernel)
    HY_TRY(p->L == 2 ? launch_ksmac_tc<2>(a, w->d_w8, (int)nunits, s) : launch_ksmac_tc<3>(a, w->d_w8, (int)nunits, s));
  } else {
    HY_TRY(launch_mac_tc(a, ct_in, w->d_w8, (int)nunits, s));
  }
  if (w->n_ev) HY_CUDA_TRY(cudaEventRecord((*w->mac_ev)[1], s));
  w->mac_launches = 1;
  return HY_OK;
}

// c_n = 2 coefficient-domain 1x1 layer after mac_coef: P_d = [A0] + S * [A1]; Out_g = P_0 +
// RowSwap(P_1) with RowSwap = the hoisted HRot by 2N - 1 (R15), whose digits are
// the coefficient-form P_1.c1 limbs themselves (PermDecomp: L^2 + L NTTs per output ct).
hy_status finish_coef2(const hy_weights* w, size_t nunits, u64* ct_out, cudaStream_t s) {
  const hy_params* p = w->p;
  const size_t L = p->L, N = p->N, ctw = 2 * L * N;
  const size_t nout = nunits * w->lay.Jo;
  QArr sv, svsh;
  for (size_t l = 0; l < L; l++) {
    const int64_t sc = w->lay.sign_coeff;
    const u64 q = p->q[l];
    sv.q[l] = sc >= 0 ? (u64)sc % q : q - ((u64)(-sc) % q);
    svsh.q[l] = (u64)(((u128)sv.q[l] << 64) / q);
  }
  const size_t total = nout * 2 * ctw;  // P [o][d][2][L][N]
  HY_CUDA_TRY(hy_launch(sign_combine_kernel, dim3((unsigned)std::min<size_t>((total + 255) / 256, 148 * 16)),
                        dim3(256), 0, s, 1, w->d_P, (const u64*)w->d_A1, total, (int)p->logN, (int)L,
                        limb_consts(p), sv, svsh));
  HY_LAUNCH_CHECK();
  if (p->ND != L) {  // P_1 of every output
    PermDecompSubJob jd{w->d_P + ctw, w->d_D, w->d_C0, (int)L, (int)N, (int)p->ND, (int)p->V, (int)p->w_dcmp,
                        2 * ctw};
    HY_TRY(launch_fwd(p, jd, nout * (p->ND * L + L), s));
  } else {
    PermDecompJob jd{w->d_P + ctw, w->d_D, w->d_C0, (int)L, (int)N, qarr(p), 2 * ctw};
    HY_TRY(launch_fwd(p, jd, nout * (L * L + L), s));
  }
  KsApplyArgs ka;
  ka.ND = (int)p->ND;
  ka.c0 = w->d_C0;
  ka.c0_stride = L * N;
  ka.D = w->d_D;
  ka.D_stride = p->ND * L * N;
  ka.diag = nullptr;
  ka.diag_stride = 0;
  ka.add = nullptr;
  ka.add_stride = 0;
  ka.key = w->d_swap_key;
  ka.act = GaloisAct{0u, 1u};  // X -> X^{2N-1}: exchange the two slot rows
  ka.out = w->d_X;
  ka.L = (int)L;
  ka.logN = (int)p->logN;
  ka.total = nout * L * N;
  ka.lcs = limb_consts(p);
  HY_TRY(launch_ks_apply(ka, s));
  OutInvAddJob jx{w->d_X, w->d_P, 2 * ctw, ct_out, (int)L, (int)N, qarr(p)};
  return launch_inv(p, jx, nout * 2 * L, s);
}

// HRot of the partial sums P_d (NTT form) of every output by the Galois element with key `key` /
// action `act`, added to `add` (hoisted HRot of PAPER.md:373-378 applied to one ct): digits of
// P_d.c1 need coefficient form (INTT), then NTT into every limb (with one digit per limb, digit i in
// limb i is P_d.c1 limb i itself)
static hy_status rotate_partials(const hy_weights* w, size_t nout, const u64* Pd, size_t pstride, const u64* add,
                                 size_t add_stride, const u64* key, GaloisAct act, cudaStream_t s) {
  const hy_params* p = w->p;
  const size_t L = p->L, N = p->N, ND = p->ND;
  const bool sub = ND != L;
  u64* dig = w->d_D2 + nout * ND * L * N;  // [o][L][N] scratch after the digit NTTs
  StridedInvJob ja{Pd + L * N, pstride, dig, (int)L, (int)N};
  HY_TRY(launch_inv(p, ja, nout * L, s));
  DigitLiftJob jb{dig, w->d_D2, (int)L, (int)N, qarr(p), onesh_arr(p)};
  if (sub) {
    jb.ND = (int)ND;
    jb.V = (int)p->V;
    jb.wd = (int)p->w_dcmp;
    HY_TRY(launch_fwd(p, jb, nout * ND * L, s));
  } else if (L > 1) {
    HY_TRY(launch_fwd(p, jb, nout * L * (L - 1), s));
  }
  KsApplyArgs ka;
  ka.ND = (int)ND;
  ka.c0 = Pd;
  ka.c0_stride = pstride;
  ka.D = w->d_D2;
  ka.D_stride = ND * L * N;
  ka.diag = sub ? nullptr : Pd + L * N;
  ka.diag_stride = pstride;
  ka.add = add;
  ka.add_stride = add_stride;
  ka.key = key;
  ka.act = act;
  ka.out = w->d_X;
  ka.L = (int)L;
  ka.logN = (int)p->logN;
  ka.total = nout * L * N;
  ka.lcs = limb_consts(p);
  return launch_ks_apply(ka, s);
}

hy_status finish_outputs(const hy_weights* w, size_t nunits, u64* ct_out, cudaStream_t s) {
  const hy_params* p = w->p;
  const hy_layout& lay = w->lay;
  const size_t L = p->L, N = p->N;
  const size_t nout = nunits * lay.Jo;
  const size_t ct_words = 2 * L * N;
  if (lay.cn == 2 && !w->shape.depthwise) {
    // S4 alignment: Out_g = P_{g,0} + RowSwap(P_{g,1}); RowSwap = hoisted HRot
    // with g = 2N-1 (exchange of the two slot rows)
    HY_TRY(rotate_partials(w, nout, w->d_P + ct_words, 2 * ct_words, w->d_P, 2 * ct_words, w->d_swap_key,
                           GaloisAct{0u, 1u}, s));
    OutInvJob jx{w->d_X, ct_words, ct_out, (int)L, (int)N};
    return launch_inv(p, jx, nout * 2 * L, s);
  }
  if (lay.cn == 4) {
    // c_n = 4 alignment: Out_g = P_{g,0} + sum_{d=1..3} HRot_{g_d}(P_{g,d}), g_d moving slot group c
    // to c xor d (row swap x half-row rotation; oracle conv.align_elts)
    for (int d = 1; d < 4; d++)
      HY_TRY(rotate_partials(w, nout, w->d_P + d * ct_words, 4 * ct_words, d == 1 ? w->d_P : w->d_X,
                             d == 1 ? 4 * ct_words : ct_words, w->d_align_key[d - 1], w->h_align_act[d - 1], s));
    OutInvJob jx{w->d_X, ct_words, ct_out, (int)L, (int)N};
    return launch_inv(p, jx, nout * 2 * L, s);
  }
  OutInvJob j{w->d_P, ct_words, ct_out, (int)L, (int)N};
  return launch_inv(p, j, nout * 2 * L, s);
}

hy_status rotate_ct(const hy_params* p, const u64* ct_in, GaloisAct act, const u64* key, u64* ct_out, size_t n,
                    u64* work, cudaStream_t s) {
  const size_t L = p->L, N = p->N, ND = p->ND;
  u64* D = work;
  u64* C0 = work + n * ND * L * N;
  HY_TRY(permdecomp(p, ct_in, n, D, C0, s));
  u64* X = work + n * (ND * L + L) * N;  // [n][2][L][N]
  KsApplyArgs ka;
  ka.ND = (int)ND;
  ka.c0 = C0;
  ka.c0_stride = L * N;
  ka.D = D;
  ka.D_stride = ND * L * N;
  ka.diag = nullptr;
  ka.diag_stride = 0;
  ka.add = nullptr;
  ka.add_stride = 0;
  ka.key = key;
  ka.act = act;
  ka.out = X;
  ka.L = (int)L;
  ka.logN = (int)p->logN;
  ka.total = n * L * N;
  ka.lcs = limb_consts(p);
  HY_TRY(launch_ks_apply(ka, s));
  OutInvJob jx{X, 2 * L * N, ct_out, (int)L, (int)N};
  return launch_inv(p, jx, n * 2 * L, s);
}

// secret key from the seed: host int8 [N] (if sk8_host) and, if s_ntt, NTT form + Shoup [2][L][N]
hy_status client_secret(const hy_params* p, u64 seed, int8_t* sk8_dev, u64* s_res, u64* s_ntt, cudaStream_t st) {
  gen_secret_kernel<<<64, 256, 0, st>>>(seed, (int)p->L, (int)p->logN, qarr(p), s_res, sk8_dev);
  HY_LAUNCH_CHECK();
  if (!s_ntt) return HY_OK;
  HY_TRY(ntt_poly_fwd(p, s_res, s_ntt, 1, st));
  return shoup_table(p, s_ntt, s_ntt + (size_t)p->L * p->N, 1, st);
}

// n encryptions (indices idx[o]) of plaintexts m [n][N] (device) under the secret of `seed`
hy_status client_encrypt(const hy_params* p, u64 seed, const u64* s_ntt, const u64* m_dev, const uint32_t* idx_dev,
                         size_t n, const u64* delta_l, u64* ct_out, u64* work, cudaStream_t st) {
  const size_t L = p->L, N = p->N;
  u64* A = work;                          // [n][L][N]
  u64* An = A + n * L * N;                // [n][L][N]
  int32_t* E = reinterpret_cast<int32_t*>(An + n * L * N);  // [n][N]
  MaskArgs ma{seed, 2u, (int)L, (int)p->logN, n, idx_dev, 0u, qarr(p)};
  gen_mask_kernel<<<148 * 8, 256, 0, st>>>(ma, A);
  HY_LAUNCH_CHECK();
  gen_error_kernel<<<148 * 8, 256, 0, st>>>(seed, 3u, (int)p->logN, n, idx_dev, 0, E);
  HY_LAUNCH_CHECK();
  HY_TRY(ntt_poly_fwd(p, A, An, n, st));
  QArr dl;
  for (size_t l = 0; l < L; l++) dl.q[l] = delta_l[l];
  ClientInvJob j{An, s_ntt, A, E, m_dev, nullptr, ct_out, (int)L, (int)N, 0, qarr(p), dl, 1, 0};
  return launch_inv(p, j, n * L, st);
}

// switching keys for n_elts Galois elements (device elts) under the secret of `seed`:
// keys_out [n][L digits][2][L limbs][N] coefficient form
hy_status client_keygen(const hy_params* p, u64 seed, const u64* s_ntt, const int8_t* sk8_dev, const uint32_t* elts_dev,
                        size_t n_elts, u64* keys_out, u64* work, cudaStream_t st) {
  const size_t L = p->L, N = p->N, ND = p->ND, n = n_elts * ND;  // poly groups o = element * ND + digit
  u64* A = work;                          // [n][L][N]
  u64* An = A + n * L * N;
  u64* Sg = An + n * L * N;               // [n_elts][L][N]
  int32_t* E = reinterpret_cast<int32_t*>(Sg + n_elts * L * N);  // [n][N]
  MaskArgs ma{seed, 4u, (int)L, (int)p->logN, n, elts_dev, (uint32_t)ND, qarr(p)};
  gen_mask_kernel<<<148 * 8, 256, 0, st>>>(ma, A);
  HY_LAUNCH_CHECK();
  gen_error_kernel<<<148 * 8, 256, 0, st>>>(seed, 5u, (int)p->logN, n, elts_dev, (int)ND, E);
  HY_LAUNCH_CHECK();
  automorph_secret_kernel<<<148 * 4, 256, 0, st>>>(sk8_dev, elts_dev, (int)n_elts, (int)L, (int)p->logN, qarr(p), Sg);
  HY_LAUNCH_CHECK();
  HY_TRY(ntt_poly_fwd(p, A, An, n, st));
  QArr dl{};
  ClientInvJob j{An, s_ntt, A, E, nullptr, Sg, keys_out, (int)L, (int)N, (int)ND, qarr(p), dl, (int)p->V,
                 (int)p->w_dcmp};
  return launch_inv(p, j, n * L, st);
}

hy_status decrypt_phase(const hy_params* p, const u64* s_ntt, const u64* s_ntt_sh, const u64* ct, size_t n, u64* x_out,
                        u64* work, cudaStream_t st) {
  C1FwdJob a{ct, work, (int)p->L, (int)p->N};
  HY_TRY(launch_fwd(p, a, n * p->L, st));
  PhaseInvJob b{work, s_ntt, s_ntt_sh, ct, x_out, (int)p->L, (int)p->N, qarr(p)};
  return launch_inv(p, b, n * p->L, st);
}

}  // namespace hyk

int hy_mac_path(int M, int L, bool depthwise, bool coef_ok, int cn, bool subdigits) {
  if (depthwise) return HY_MAC_THIN;
  if (cn == 4) return M <= 32 ? HY_MAC_FP64_FUSED : HY_MAC_FP64_SPLIT;  // WHT-4 epilogue: FP64 MAC only
  static const bool fp64 = getenv("HY_MAC_FP64") != nullptr;    // A/B switches
  static const bool split = getenv("HY_SPLIT_TC") != nullptr;
  if (coef_ok && !fp64 && !split) return HY_MAC_TC_COEF;
  if (fp64) return M <= 32 ? HY_MAC_FP64_FUSED : HY_MAC_FP64_SPLIT;
  // M <= 32 (latency-bound small layers, e.g. C1/C2): the FP64 fused kernel is faster (measured,
  // DESIGN.md §4); 32 < M <= 128: key switching fused into the tcgen05 MAC (one digit per limb only)
  if (!split && M <= 32) return HY_MAC_FP64_FUSED;
  if (!split && !subdigits && M <= 128 && (L == 2 || L == 3 || L == 5)) return HY_MAC_TC_FUSED;
  return HY_MAC_TC_SPLIT;
}
