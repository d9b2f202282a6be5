// Device kernels of the Hyena hot path and their launchers.
#include <stdio.h>

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
// every limb l and NTT'd (L*L jobs), plus NTT(c0) per limb (L jobs).
struct PermDecompJob {
  const u64* ct;
  u64* D;
  u64* C0;
  int L, N;
  QArr qa;
  int limb;
  const u64* s;
  u64* d;
  u64 qd;
  bool red;
  __device__ void bind(int b) {
    const int per = L * L + L;
    const int c = b / per, r = b % per;
    if (r < L * L) {
      const int i = r / L;
      limb = r % L;
      s = ct + ((size_t)(2 * c + 1) * L + i) * N;
      d = D + ((size_t)(c * L + i) * L + limb) * N;
      qd = qa.q[limb];
      red = qa.q[i] / 4 >= qa.q[limb];  // digit may exceed the lazy [0, 4 q_l) input range
    } else {
      limb = r - L * L;
      s = ct + ((size_t)(2 * c) * L + limb) * N;
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

// row-swap step (b): NTT_l of digit i (coefficient form, in [0, q_i)) for l != i
struct DigitLiftJob {
  const u64* dig;  // [o][L][N]
  u64* D2;         // [o][L digit][L limb][N]
  int L, N;
  QArr qa;
  int limb;
  const u64* s;
  u64* d;
  u64 qd;
  bool red;
  __device__ void bind(int b) {
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
    return red ? x % qd : x;
  }
  __device__ void store(int k, u64 v) const { d[k] = v; }
};

// PermAuto value (S2): for limb l, NTT slot k,
//   c0' = C0[perm(k)] + sum_i D_i[perm(k)] * b_{i,l}[k],  c1' = sum_i D_i[perm(k)] * a_{i,l}[k]
// key layout [L digit][2][L limb][N] values, then the same block of Shoup companions.
struct KSSrc {
  const u64* c0;      // [L][N] NTT form for this ct (may be null: treated as 0)
  const u64* D;       // [L digit][L limb][N]
  const u64* diag;    // if non-null: digit i in limb i is diag[i*N + .] instead of D
};

__device__ __forceinline__ void ks_eval(const KSSrc& src, const u64* __restrict__ key, int L, int N, int l, int k, int kp,
                                        const LimbConst& c, u64& o0, u64& o1) {
  const u64 q = c.q, q2 = c.two_q;
  const size_t kblk = (size_t)2 * L * L * N;
  u64 a0 = src.c0 ? src.c0[(size_t)l * N + kp] : 0;
  u64 a1 = 0;
#pragma unroll 4
  for (int i = 0; i < L; i++) {
    const u64 dv = (src.diag && i == l) ? src.diag[(size_t)i * N + kp] : src.D[((size_t)i * L + l) * N + kp];
    const size_t ib = ((size_t)(2 * i) * L + l) * N + k;
    const size_t ia = ((size_t)(2 * i + 1) * L + l) * N + k;
    a0 = csub(a0 + shoup_mul(dv, __ldg(key + ib), __ldg(key + kblk + ib), q), q2);
    a1 = csub(a1 + shoup_mul(dv, __ldg(key + ia), __ldg(key + kblk + ia), q), q2);
  }
  o0 = a0;  // [0, 2q)
  o1 = a1;
}

// Inverse transform whose input is a key-switched (rotated) ciphertext, optionally plus an
// addend (the row-swap alignment Out = P_{g,0} + HRot(P_{g,1})), written to
// coefficient form: hy_rotate and S4+S5.
struct KSFinishJob {
  // per output o: c0 source, D source (+ optional diag), addend (NTT form [2][L][N])
  const u64* c0;
  size_t c0_stride;
  const u64* D;
  size_t D_stride;
  const u64* diag;
  size_t diag_stride;
  const u64* add;
  size_t add_stride;
  const u64* key;
  uint32_t g;
  u64* out;  // [o][2][L][N]
  int L, N, logN;
  LimbConsts lcs;
  int limb, comp, o;
  __device__ void bind(int b) {
    o = b / (2 * L);
    comp = (b / L) % 2;
    limb = b % L;
  }
  __device__ u64 load(int k) const {
    const int kp = auto_perm(k, g, logN);
    KSSrc src{c0 + (size_t)o * c0_stride, D + (size_t)o * D_stride, diag ? diag + (size_t)o * diag_stride : nullptr};
    u64 r0, r1;
    ks_eval(src, key, L, N, limb, k, kp, lcs.lc[limb], r0, r1);
    u64 v = comp ? r1 : r0;
    if (add) v = csub(v + add[(size_t)o * add_stride + ((size_t)comp * L + limb) * N + k], lcs.lc[limb].two_q);
    return v;
  }
  __device__ void store(int k, u64 v) const { out[(((size_t)o * 2 + comp) * L + limb) * N + k] = v; }
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
hy_status launch_fwd_t(const hy_params* p, const Job& job, size_t nblocks, cudaStream_t s) {
  if (nblocks == 0) return HY_OK;
  const size_t sm = ntt_smem_bytes<LOGN>();
  static bool attr_done = false;
  if (!attr_done) {
    HY_CUDA_TRY(cudaFuncSetAttribute(ntt_fwd_kernel<LOGN, Job>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr_done = true;
  }
  ntt_fwd_kernel<LOGN, Job><<<(unsigned)nblocks, (1 << LOGN) / 16, sm, s>>>(job, p->tab, limb_consts(p));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <int LOGN, class Job>
hy_status launch_inv_t(const hy_params* p, const Job& job, size_t nblocks, cudaStream_t s) {
  if (nblocks == 0) return HY_OK;
  const size_t sm = ntt_smem_bytes<LOGN>();
  static bool attr_done = false;
  if (!attr_done) {
    HY_CUDA_TRY(cudaFuncSetAttribute(ntt_inv_kernel<LOGN, Job>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr_done = true;
  }
  ntt_inv_kernel<LOGN, Job><<<(unsigned)nblocks, (1 << LOGN) / 16, sm, s>>>(job, p->tab, limb_consts(p));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

template <class Job>
hy_status launch_fwd(const hy_params* p, const Job& job, size_t nblocks, cudaStream_t s) {
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

// S2 PermAuto, materialised: R[ct][tap][2][L][N] (tap without key = identity: (C0, D_ll)).
__global__ void __launch_bounds__(256) permauto_kernel(const u64* __restrict__ D, const u64* __restrict__ C0, int nct,
                                                       int T, const u64* const* __restrict__ tap_keys,
                                                       const uint32_t* __restrict__ tap_g, u64* __restrict__ R, int L,
                                                       int logN, LimbConsts lcs) {
  const int N = 1 << logN;
  const size_t total = (size_t)nct * T * L * N;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(idx & (N - 1));
    size_t rest = idx >> logN;
    const int l = (int)(rest % L);
    rest /= L;
    const int tap = (int)(rest % T);
    const int c = (int)(rest / T);
    const u64* key = tap_keys[tap];
    u64 r0, r1;
    if (key == nullptr) {
      r0 = C0[((size_t)c * L + l) * N + k];
      r1 = D[(((size_t)c * L + l) * L + l) * N + k];
    } else {
      const int kp = auto_perm(k, tap_g[tap], logN);
      KSSrc src{C0 + (size_t)c * L * N, D + (size_t)c * L * L * N, nullptr};
      ks_eval(src, key, L, N, l, k, kp, lcs.lc[l], r0, r1);
      r0 = csub(r0, lcs.lc[l].q);
      r1 = csub(r1, lcs.lc[l].q);
    }
    u64* out = R + ((size_t)(c * T + tap) * 2 * L + l) * N + k;
    out[0] = r0;
    out[(size_t)L * N] = r1;
  }
}

// ------------------------------------------------------------------------------------------
// S3: lazy MAC + WHT + one reduction + sign PMult
//
// Exact integer accumulation on the FP64 pipe: each R coefficient x < 2^60 is split into
// 30-bit halves (exact doubles); products with |w| <= 128 are < 2^37 and sums of up to
// 2^16 of them stay < 2^53, so every DFMA is exact.  One reduction per output coefficient.
// ------------------------------------------------------------------------------------------
struct MacArgs {
  const u64* R;       // [units][K][ncols]
  const int32_t* wm;  // [wblocks][Mpad][K]
  u64* out;           // CN=1: [units][M][ncols]; CN=2: [units][M/2][ncols]
  const u64* sign;    // [L][N], then [L][N] Shoup
  int K, M, Mpad, ncols, wblocks, L, logN, kscale;
  LimbConsts lcs;
};

constexpr int MAC_THREADS = 128;
constexpr int MAC_KC = 32;

__device__ __forceinline__ u64 reduce_wide(long long H, long long Lo, const LimbConst& c) {
  // value H * 2^30 + Lo (|H|, |Lo| < 2^59) mod q, canonical
  const u64 hu = (u64)(H + (long long)c.off);
  const u64 lu = (u64)(Lo + (long long)c.off);
  u64 a = shoup_mul(hu, c.c30, c.c30_sh, c.q);  // [0, 2q)
  u64 b = reduce_2q(lu, c.one_sh, c.q);         // [0, 2q)
  u64 s = csub(a + b, c.two_q);
  return csub(s, c.q);
}

template <int TM, int CN>
__global__ void __launch_bounds__(MAC_THREADS) mac_kernel(MacArgs a) {
  __shared__ double sw[MAC_KC][TM];
  const int col = blockIdx.x * MAC_THREADS + threadIdx.x;
  const int row0 = blockIdx.y * TM;
  const int unit = blockIdx.z;
  const int wb = unit % a.wblocks;
  const u64* __restrict__ Rp = a.R + (size_t)unit * a.K * a.ncols + col;
  const int32_t* __restrict__ W = a.wm + ((size_t)wb * a.Mpad + row0) * a.K;
  double acc_h[TM], acc_l[TM];
#pragma unroll
  for (int r = 0; r < TM; r++) acc_h[r] = acc_l[r] = 0.0;

  for (int kc0 = 0; kc0 < a.K; kc0 += MAC_KC) {
    const int kcn = min(MAC_KC, a.K - kc0);
    __syncthreads();
    for (int e = threadIdx.x; e < MAC_KC * TM; e += MAC_THREADS) {
      const int kk = e / TM, r = e % TM;
      sw[kk][r] = (kk < kcn) ? (double)W[(size_t)r * a.K + kc0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kcn; kk++) {
      const u64 x = __ldg(Rp + (size_t)(kc0 + kk) * a.ncols);
      const double xh = (double)(uint32_t)(x >> 30);
      const double xl = (double)(uint32_t)(x & 0x3FFFFFFFull);
#pragma unroll
      for (int r = 0; r < TM; r++) {
        const double w = sw[kk][r];
        acc_h[r] = fma(w, xh, acc_h[r]);
        acc_l[r] = fma(w, xl, acc_l[r]);
      }
    }
  }

  const int N = 1 << a.logN;
  const int l = (col >> a.logN) % a.L;
  const int kidx = col & (N - 1);
  const LimbConst& c = a.lcs.lc[l];
  if (CN == 1) {
#pragma unroll
    for (int r = 0; r < TM; r++) {
      if (row0 + r < a.M)
        a.out[((size_t)unit * a.M + row0 + r) * a.ncols + col] =
            reduce_wide(__double2ll_rn(acc_h[r]), __double2ll_rn(acc_l[r]), c);
    }
  } else {
    const u64 sg = a.sign[(size_t)l * N + kidx];
    const u64 sgs = a.sign[(size_t)(a.L + l) * N + kidx];
    const long long kk = a.kscale;
#pragma unroll
    for (int r = 0; r < TM; r += 2) {
      if (row0 + r < a.M) {
        const long long H0 = __double2ll_rn(acc_h[r]), L0 = __double2ll_rn(acc_l[r]);
        const long long H1 = __double2ll_rn(acc_h[r + 1]), L1 = __double2ll_rn(acc_l[r + 1]);
        // Walsh-Hadamard on the accumulators (Eq. 2): A0 = k (B0 + B1), A1 = B0 - B1
        const u64 a0 = reduce_wide(kk * (H0 + H1), kk * (L0 + L1), c);
        const u64 a1 = reduce_wide(H0 - H1, L0 - L1, c);
        // PMult by the [k, -k] plaintext (NTT form, Shoup) and HAdd
        u64 v = a0 + shoup_mul(a1, sg, sgs, c.q);
        v = csub(csub(v, c.two_q), c.q);
        a.out[((size_t)unit * (a.M / 2) + (row0 + r) / 2) * a.ncols + col] = v;
      }
    }
  }
}

template <int TM, int CN>
hy_status launch_mac_t(const MacArgs& a, int units, cudaStream_t s) {
  dim3 grid(a.ncols / MAC_THREADS, a.Mpad / TM, units);
  mac_kernel<TM, CN><<<grid, MAC_THREADS, 0, s>>>(a);
  HY_LAUNCH_CHECK();
  return HY_OK;
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
  // key [L][2][L][N] -> NTT per (digit, comp, limb); Shoup companions in the following block
  const size_t npoly = 2 * p->L;  // groups of L limbs
  HY_TRY(ntt_poly_fwd(p, key_coeff, key_ntt, npoly, s));
  return shoup_table(p, key_ntt, key_ntt + npoly * p->L * p->N, npoly, s);
}

hy_status permdecomp(const hy_params* p, const u64* ct, size_t nct, u64* D, u64* C0, cudaStream_t s) {
  PermDecompJob j{ct, D, C0, (int)p->L, (int)p->N, qarr(p)};
  return launch_fwd(p, j, nct * (p->L * p->L + p->L), s);
}

hy_status permauto(const hy_params* p, const u64* D, const u64* C0, size_t nct, int ntap, u64* const* d_tap_keys,
                   const uint32_t* d_tap_g, u64* R, cudaStream_t s) {
  const size_t total = nct * ntap * p->L * p->N;
  if (!total) return HY_OK;
  const unsigned blocks = (unsigned)std::min<size_t>((total + 255) / 256, 148 * 64);
  permauto_kernel<<<blocks, 256, 0, s>>>(D, C0, (int)nct, ntap, d_tap_keys, d_tap_g, R, (int)p->L, (int)p->logN,
                                         limb_consts(p));
  HY_LAUNCH_CHECK();
  return HY_OK;
}

hy_status mac(const hy_weights* w, size_t nunits, cudaStream_t s) {
  const hy_params* p = w->p;
  const hy_layout& lay = w->lay;
  MacArgs a;
  a.R = w->d_R;
  a.wm = w->d_wm;
  a.out = w->d_P;
  a.sign = w->d_sign;
  a.K = w->K;
  a.M = w->M;
  a.ncols = 2 * p->L * p->N;
  a.wblocks = w->wblocks;
  a.L = p->L;
  a.logN = p->logN;
  a.kscale = (int)lay.k;
  a.lcs = limb_consts(p);
  const bool dw = w->shape.depthwise != 0;
  const int units = (int)(dw ? nunits * lay.Jc : nunits);
  const int tm = w->M >= 16 ? 16 : (w->M >= 8 ? 8 : (w->M >= 4 ? 4 : (w->M >= 2 ? 2 : 1)));
  a.Mpad = (w->M + tm - 1) / tm * tm;
  if (lay.cn == 2) {
    switch (tm) {
      case 16: return launch_mac_t<16, 2>(a, units, s);
      case 8: return launch_mac_t<8, 2>(a, units, s);
      case 4: return launch_mac_t<4, 2>(a, units, s);
      case 2: return launch_mac_t<2, 2>(a, units, s);
    }
  } else {
    switch (tm) {
      case 16: return launch_mac_t<16, 1>(a, units, s);
      case 8: return launch_mac_t<8, 1>(a, units, s);
      case 4: return launch_mac_t<4, 1>(a, units, s);
      case 2: return launch_mac_t<2, 1>(a, units, s);
      case 1: return launch_mac_t<1, 1>(a, units, s);
    }
  }
  hy_set_error("mac: bad row tile");
  return HY_EINVAL;
}

hy_status finish_outputs(const hy_weights* w, size_t nunits, u64* ct_out, cudaStream_t s) {
  const hy_params* p = w->p;
  const hy_layout& lay = w->lay;
  const size_t L = p->L, N = p->N;
  const size_t nout = nunits * lay.Jo;
  const size_t ct_words = 2 * L * N;
  if (lay.cn == 2 && !w->shape.depthwise) {
    // S4 alignment: Out_g = P_{g,0} + RowSwap(P_{g,1}); RowSwap = hoisted HRot
    // with g = 2N-1: digits of P_{g,1}.c1 need coefficient form (INTT), then NTT in other limbs.
    u64* dig = w->d_D2 + nout * L * L * N;  // [o][L][N] scratch after D2
    StridedInvJob ja{w->d_P + ct_words + L * N, 2 * ct_words, dig, (int)L, (int)N};
    HY_TRY(launch_inv(p, ja, nout * L, s));
    if (L > 1) {
      DigitLiftJob jb{dig, w->d_D2, (int)L, (int)N, qarr(p)};
      HY_TRY(launch_fwd(p, jb, nout * L * (L - 1), s));
    }
    KSFinishJob jc;
    jc.c0 = w->d_P + ct_words;  // P_{g,1}.c0
    jc.c0_stride = 2 * ct_words;
    jc.D = w->d_D2;
    jc.D_stride = L * L * N;
    jc.diag = w->d_P + ct_words + L * N;  // P_{g,1}.c1: digit i in limb i is already NTT(d_i)
    jc.diag_stride = 2 * ct_words;
    jc.add = w->d_P;  // P_{g,0}
    jc.add_stride = 2 * ct_words;
    jc.key = w->d_swap_key;
    jc.g = 2 * p->N - 1;
    jc.out = ct_out;
    jc.L = (int)L;
    jc.N = (int)N;
    jc.logN = (int)p->logN;
    jc.lcs = limb_consts(p);
    return launch_inv(p, jc, nout * 2 * L, s);
  }
  OutInvJob j{w->d_P, ct_words, ct_out, (int)L, (int)N};
  return launch_inv(p, j, nout * 2 * L, s);
}

hy_status rotate_ct(const hy_params* p, const u64* ct_in, uint32_t g, const u64* key, u64* ct_out, size_t n,
                    u64* work, cudaStream_t s) {
  const size_t L = p->L, N = p->N;
  u64* D = work;
  u64* C0 = work + n * L * L * N;
  HY_TRY(permdecomp(p, ct_in, n, D, C0, s));
  KSFinishJob j;
  j.c0 = C0;
  j.c0_stride = L * N;
  j.D = D;
  j.D_stride = L * L * N;
  j.diag = nullptr;
  j.diag_stride = 0;
  j.add = nullptr;
  j.add_stride = 0;
  j.key = key;
  j.g = g;
  j.out = ct_out;
  j.L = (int)L;
  j.N = (int)N;
  j.logN = (int)p->logN;
  j.lcs = limb_consts(p);
  return launch_inv(p, j, n * 2 * L, s);
}

hy_status decrypt_phase(const hy_params* p, const u64* s_ntt, const u64* s_ntt_sh, const u64* ct, size_t n, u64* x_out,
                        u64* work, cudaStream_t st) {
  C1FwdJob a{ct, work, (int)p->L, (int)p->N};
  HY_TRY(launch_fwd(p, a, n * p->L, st));
  PhaseInvJob b{work, s_ntt, s_ntt_sh, ct, x_out, (int)p->L, (int)p->N, qarr(p)};
  return launch_inv(p, b, n * p->L, st);
}

}  // namespace hyk
