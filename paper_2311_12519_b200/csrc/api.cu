// C-ABI entry points of include/hyena.h and the library's host-side logic (parameter tables,
// layout planner, weight encoding, debug decryption).  Independent of oracle/ by construction:
// every formula is re-derived from PAPER.md here.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "hy_common.cuh"

// ============================================================================================
// errors
// ============================================================================================
static thread_local char g_err[1024] = "";

void hy_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* hy_last_error(void) { return g_err; }

#include <atomic>
#include <mutex>
static std::atomic<uint64_t> g_launches{0};

cudaError_t hy_smem_attr(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (kernel, device) -> bytes set
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[std::make_pair(kernel, dev)];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}
void hy_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" uint64_t hy_kernel_launches(void) { return g_launches.load(); }

#define HY_CHECK(cond, code, ...) \
  do {                            \
    if (!(cond)) {                \
      hy_set_error(__VA_ARGS__);  \
      return code;                \
    }                             \
  } while (0)

// ============================================================================================
// host number theory
// ============================================================================================
namespace hyhost {
u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
u64 powmod(u64 a, u64 e, u64 m) {
  u64 r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}
u64 invmod(u64 a, u64 m) {  // m prime
  return powmod(a, m - 2, m);
}
bool is_prime(u64 n) {
  if (n < 2) return false;
  static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 p : small)
    if (n % p == 0) return n == p;
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    r++;
  }
  for (u64 a : small) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < r; i++) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}
u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
uint32_t bitrev(uint32_t x, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}
// a primitive 2N-th root of unity mod q (q prime, q = 1 mod 2N)
u64 root_2n(u64 q, uint32_t N) {
  for (u64 x = 2; x < q; x++) {
    u64 psi = powmod(x, (q - 1) / (2 * (u64)N), q);
    if (powmod(psi, N, q) == q - 1) return psi;
  }
  return 0;
}
}  // namespace hyhost

using namespace hyhost;

// g = 3^s (swap 0) or -3^s (swap 1) mod 2N with s in [0, N/2): Z_{2N}^* = <3> x <-1>
bool hy_galois_act(uint32_t g, uint32_t N, GaloisAct* out) {
  const u64 two_n = 2 * (u64)N;
  if (!(g & 1) || g >= two_n) return false;
  u64 e = 1;
  for (uint32_t s = 0; s < N / 2; s++) {
    if (e == g || two_n - e == g) {
      out->shift = s;
      out->swap = (e == g) ? 0u : 1u;
      return true;
    }
    e = e * 3 % two_n;
  }
  return false;
}

static uint32_t next_pow2(uint32_t x) {
  uint32_t r = 1;
  while (r < x) r <<= 1;
  return r;
}

static int64_t centered(u64 x, u64 t) { return x > t / 2 ? (int64_t)x - (int64_t)t : (int64_t)x; }

// ============================================================================================
// layout planner (readings R8-R10, R15)
// ============================================================================================
static bool valid_N(uint32_t N) { return N >= 16 && N <= 65536 && (N & (N - 1)) == 0; }

extern "C" hy_status hy_plan_layout(uint32_t N, uint64_t t, const hy_conv_shape* sh, hy_layout* out) {
  HY_CHECK(sh && out, HY_EINVAL, "null argument");
  HY_CHECK(valid_N(N), HY_EINVAL, "N=%u must be a power of two in [16, 65536]", N);
  HY_CHECK(is_prime(t) && (t - 1) % (2 * (u64)N) == 0, HY_EINVAL, "t=%llu must be a prime = 1 mod 2N",
           (unsigned long long)t);
  HY_CHECK(sh->stride == 1, HY_ESHAPE, "only stride 1 is supported (got %u)", sh->stride);
  HY_CHECK(sh->Ci >= 1 && sh->H >= 1 && sh->W >= 1 && sh->kh >= 1 && sh->kw >= 1 && sh->batch >= 1, HY_ESHAPE,
           "empty shape");
  HY_CHECK(sh->depthwise || sh->Co >= 1, HY_ESHAPE, "Co must be >= 1");
  HY_CHECK(!sh->depthwise || sh->Co == sh->Ci || sh->Co == 0, HY_ESHAPE, "depthwise needs Co == Ci");
  HY_CHECK(sh->force_cn == 0 || sh->force_cn == 1 || sh->force_cn == 2 || sh->force_cn == 4, HY_EINVAL,
           "force_cn must be 0, 1, 2 or 4");
  hy_layout L;
  memset(&L, 0, sizeof(L));
  L.N = N;
  const uint32_t row = N / 2;
  const int64_t Hout = (int64_t)sh->H + 2 * sh->pad - sh->kh + 1, Wout = (int64_t)sh->W + 2 * sh->pad - sh->kw + 1;
  HY_CHECK(Hout > 0 && Wout > 0, HY_ESHAPE, "kernel larger than the padded input");
  HY_CHECK(sh->kh * sh->kw <= HY_MAX_TAPS, HY_ESHAPE, "at most %d taps", HY_MAX_TAPS);
  L.Hout = (uint32_t)Hout;
  L.Wout = (uint32_t)Wout;
  L.Wp = next_pow2(sh->W + 2 * sh->pad);
  L.Hp = next_pow2(sh->H + 2 * sh->pad);
  if ((u64)L.Hp * L.Wp <= row) {
    L.mode = 0;
    L.per_row = row / (L.Hp * L.Wp);
    if (sh->force_cn == 4) {  // c_n = 4: a channel's slot group is half a slot row (N/4 slots)
      HY_CHECK((u64)L.Hp * L.Wp <= row / 2, HY_ESHAPE, "c_n = 4 needs an image block within N/4 slots");
      L.per_row = (row / 2) / (L.Hp * L.Wp);
    }
    L.bands = 1;
    L.G = (sh->batch + L.per_row - 1) / L.per_row;
  } else {
    HY_CHECK(L.Wp <= row, HY_ESHAPE, "padded width %u exceeds a slot row (%u)", L.Wp, row);
    L.mode = 1;
    L.Hb = row / L.Wp;
    HY_CHECK(L.Hb > sh->kh - 1, HY_ESHAPE, "band of %u rows too short for kh=%u", L.Hb, sh->kh);
    L.Hv = L.Hb - (sh->kh - 1);
    L.bands = (L.Hout + L.Hv - 1) / L.Hv;
    L.G = sh->batch * L.bands;
  }
  L.cn = sh->force_cn ? (uint32_t)sh->force_cn : (L.G <= 1 ? 2u : 1u);
  const uint32_t C = sh->Ci;
  if (L.cn == 4) {  // NEXT-1: 4 channels per ciphertext in slot groups c = 2 h + r (row r, half h)
    HY_CHECK(L.mode == 0 && L.G == 1, HY_ESHAPE, "c_n = 4 needs the whole batch in one group of N/4 slots");
    HY_CHECK(!sh->depthwise, HY_ESHAPE, "c_n = 4 is not supported for depthwise layers");
    L.U = 1;
    L.Jc = (C + 3) / 4;
    L.Jo = (sh->Co + 3) / 4;
  } else if (L.cn == 2) {
    L.U = L.G;
    L.Jc = (C + 1) / 2;
    L.Jo = sh->depthwise ? L.Jc : (sh->Co + 1) / 2;
  } else {
    L.U = (L.G + 1) / 2;
    L.Jc = C;
    L.Jo = sh->depthwise ? C : sh->Co;
  }
  L.J = L.U * L.Jc;
  L.Jout = L.U * L.Jo;
  L.n_taps = sh->kh * sh->kw;
  for (uint32_t dy = 0; dy < sh->kh; dy++)
    for (uint32_t dx = 0; dx < sh->kw; dx++) {
      const uint32_t tau = dy * sh->kw + dx;
      L.tap_dy[tau] = (int32_t)dy;
      L.tap_dx[tau] = (int32_t)dx;
      L.tap_step[tau] = ((int32_t)dy - (int32_t)sh->pad) * (int32_t)L.Wp + ((int32_t)dx - (int32_t)sh->pad);
    }
  // Hadamard scale: h = -(w + w^3)/2, w = zeta^{N/4}, zeta = least primitive
  // 2N-th root mod t; k = argmin_{1<=k<=32} |[k h]_t|, ties to the smaller k (reading R13).
  u64 zeta = 0;
  for (u64 x = 2; x < t; x++)
    if (powmod(x, N, t) == t - 1) {
      zeta = x;
      break;
    }
  const u64 w = powmod(zeta, N / 4, t);
  const u64 s = (w + powmod(w, 3, t)) % t;
  const u64 h = mulmod((t - s) % t, invmod(2, t), t);
  L.h = (uint32_t)h;
  if (L.cn == 2) {
    uint32_t k = 0;
    if (sh->k > 0) {
      k = (uint32_t)sh->k;
    } else {
      int64_t best = -1;
      for (uint32_t kk = 1; kk <= 32; kk++) {
        int64_t v = centered(mulmod(kk, h, t), t);
        v = v < 0 ? -v : v;
        if (best < 0 || v < best) {
          best = v;
          k = kk;
        }
      }
    }
    HY_CHECK(k >= 1 && k <= 32, HY_EINVAL, "k must be in [1, 32] (got %d)", sh->k);
    L.k = k;
    L.scale = 2 * k;
    L.sign_coeff = (int32_t)centered(mulmod(k, h, t), t);
  } else {
    L.k = 1;
    L.scale = L.cn == 4 ? 4 : 1;  // c_n = 4: H4 H4^T = 4 I (no k: the dense rows have no small multiple)
    L.sign_coeff = 0;
  }
  // Galois elements: left rotation by s <-> X -> X^{3^{s mod N/2}} (reading R7)
  L.n_galois = 0;
  auto add_g = [&](uint32_t g) {
    for (uint32_t i = 0; i < L.n_galois; i++)
      if (L.galois[i] == g) return;
    L.galois[L.n_galois++] = g;
  };
  for (uint32_t tau = 0; tau < L.n_taps; tau++) {
    const int64_t st = ((int64_t)L.tap_step[tau] % (int64_t)row + row) % row;
    if (st != 0) add_g((uint32_t)powmod(3, (u64)st, 2 * (u64)N));
  }
  if (L.cn == 2 && !sh->depthwise) add_g(2 * N - 1);
  if (L.cn == 4) {  // alignment of diagonal d: row swap^(d & 1) x half-row rotation^(d >> 1)
    const u64 M2 = 2 * (u64)N, half_rot = powmod(3, N / 4, M2);
    add_g(2 * N - 1);
    add_g((uint32_t)half_rot);
    add_g((uint32_t)mulmod(2 * N - 1, half_rot, M2));
  }
  // exactness bounds of the FP64-pipe accumulation
  const u64 K = sh->depthwise ? L.n_taps : (u64)L.Jc * L.n_taps;
  HY_CHECK(K <= 65536, HY_ESHAPE, "MAC depth %llu exceeds 2^16", (unsigned long long)K);
  HY_CHECK(L.cn != 2 || K * L.k <= (1u << 21), HY_ESHAPE, "MAC depth x k too large for exact accumulation");
  *out = L;
  return HY_OK;
}

extern "C" hy_status hy_layout_accounting(const hy_layout* lay, const hy_conv_shape* sh, uint32_t L, uint32_t ND,
                                          hy_accounting* out) {
  HY_CHECK(lay && sh && out && L >= 1 && ND >= L, HY_EINVAL, "bad accounting arguments");
  const u64 N = lay->N, ctb = 2 * (u64)L * N * 8;
  const bool dw = sh->depthwise != 0;
  const u64 Co = dw ? sh->Ci : sh->Co, T = lay->n_taps;
  const u64 elems = dw ? (u64)sh->Ci * T : (u64)sh->Ci * Co * T;  // kernel elements
  hy_accounting a;
  memset(&a, 0, sizeof(a));
  a.input_ct_bytes = (u64)lay->J * ctb;
  a.output_ct_bytes = (u64)lay->Jout * ctb;
  a.input_ct_bytes_paper = (((u64)sh->Ci * lay->Wp * lay->Hp + N - 1) / N) * ctb;
  const u64 plaintexts = lay->cn == 4 ? 3 : lay->cn == 2 ? 1 : 0;
  a.model_bytes_paper = elems * 8 + plaintexts * N * 8;
  a.model_bytes_conventional = elems * N * 8;
  // device copy (hy_encode_weights): int8 tiles + FP64 table over the padded MAC geometry, term
  // table, plaintexts in NTT form with Shoup companions
  const u64 M = dw ? (lay->cn == 2 ? 2 : 1) : (lay->cn == 4 ? 16 * (u64)lay->Jo : lay->cn == 2 ? 4 * (u64)lay->Jo : lay->Jo);
  const u64 K = dw ? T : (u64)lay->Jc * T, wblocks = dw ? lay->Jc : 1;
  const u64 Mpad = (u64)hy_mac_mpad((int)M, dw), Kpad = (K + 31) / 32 * 32;
  a.model_bytes_device = wblocks * Kpad * Mpad * 8 + wblocks * ((Mpad + 127) / 128) * Kpad * 128 +
                         (Kpad + 63) / 64 * 64 * 4 + plaintexts * 2 * (u64)L * N * 8;
  a.n_keys = lay->n_galois;
  a.key_bytes = (u64)lay->n_galois * ND * 2 * L * N * 8;
  u64 ntap = 0;
  for (uint32_t t = 0; t < lay->n_taps; t++)
    if (((int64_t)lay->tap_step[t] % (int64_t)(N / 2)) != 0) ntap++;
  a.rotations = (uint32_t)((u64)lay->J * ntap + (dw ? 0 : (lay->cn == 4 ? 3 : lay->cn == 2 ? 1 : 0)) * (u64)lay->Jout);
  a.coef_macs = (dw ? (u64)lay->U * lay->Jc : lay->U) * M * K * 2 * L * N;
  *out = a;
  return HY_OK;
}

// Noise-driven decomposition-base selection (the smaller the
// noise growth of the convolution, the larger the key-switching decomposition base that still
// decrypts, and the fewer digits every HRot costs).  Heuristic infinity-norm model (6 sigma tails,
// independent random-walk growth), calibrated against the oracle's noise meter
// (tests/test_abi.py::test_noise_model_tracks_the_oracle):
//   one rotation:  sigma_rot = sqrt(ND N / 3) B_d sigma_e   (ND digits < B_d = 2^w or q, CBD sigma_e = sqrt(10))
//   lazy MAC:      sigma_mac = sqrt(K) (w_max / sqrt 3) sigma_rot
//   c_n = 1:       sigma_out = sigma_mac
//   c_n = 2:       sigma_out = sqrt 2 max(k, 2 |[k h]_t|) sigma_mac + sigma_rot      ([k, -k] PMult, row swap)
//   c_n = 4:       sigma_out = 2 sqrt 3 sqrt N (t / sqrt 12) sigma_mac + sqrt 3 sigma_rot (dense rows)
//   noise = log2(6 sigma_out),  budget = log2(Delta / 2) ~= log2(Q / t) - 1.
static hy_status noise_model(uint32_t N, const uint64_t* q, uint32_t L, uint64_t t, const hy_conv_shape* sh,
                             uint32_t w_max, uint32_t w, double* noise, double* budget) {
  hy_layout lay;
  HY_TRY(hy_plan_layout(N, t, sh, &lay));
  double qbits = 0, logQ = 0;
  for (uint32_t l = 0; l < L; l++) {
    uint32_t b = 0;
    while (b < 64 && (q[l] >> b)) b++;
    qbits = std::max(qbits, (double)b);
    logQ += std::log2((double)q[l]);
  }
  const double V = w ? std::ceil(qbits / w) : 1.0, ND = L * V;
  const double Bd = std::exp2(w ? (double)w : qbits), sig = std::sqrt(10.0);
  const double s_rot = std::sqrt(ND * N / 3.0) * Bd * sig;
  const double K = sh->depthwise ? (double)lay.n_taps : (double)lay.Jc * lay.n_taps;
  const double s_mac = std::sqrt(K) * (w_max / std::sqrt(3.0)) * s_rot;
  double s_out = s_mac;
  if (lay.cn == 2)
    s_out = std::sqrt(2.0) * std::max((double)lay.k, 2.0 * std::fabs((double)lay.sign_coeff)) * s_mac +
            (sh->depthwise ? 0.0 : s_rot);
  else if (lay.cn == 4)
    s_out = 2 * std::sqrt(3.0) * std::sqrt((double)N) * (t / std::sqrt(12.0)) * s_mac + std::sqrt(3.0) * s_rot;
  *noise = std::log2(6 * s_out);
  *budget = logQ - std::log2((double)t) - 1;
  return HY_OK;
}

extern "C" hy_status hy_noise_estimate(uint32_t N, const uint64_t* q, uint32_t L, uint64_t t, const hy_conv_shape* sh,
                                       uint32_t w_max, uint32_t w_dcmp, double* log2_noise, double* log2_budget) {
  HY_CHECK(q && sh && log2_noise && log2_budget && L >= 1 && L <= HY_MAX_LIMBS, HY_EINVAL, "null argument");
  return noise_model(N, q, L, t, sh, w_max, w_dcmp, log2_noise, log2_budget);
}

extern "C" hy_status hy_select_dcmp_base(uint32_t N, const uint64_t* q, uint32_t L, uint64_t t,
                                         const hy_conv_shape* sh, uint32_t w_max, double margin_bits,
                                         uint32_t* w_dcmp) {
  HY_CHECK(q && sh && w_dcmp && L >= 1 && L <= HY_MAX_LIMBS, HY_EINVAL, "null argument");
  uint32_t qbits = 0, qmin = 64;
  for (uint32_t l = 0; l < L; l++) {
    uint32_t b = 0;
    while (b < 64 && (q[l] >> b)) b++;
    qbits = std::max(qbits, b);
    qmin = std::min(qmin, b);
  }
  // fewest digits first: V = 1 (one digit per limb), then the smallest w with V sub-digits
  for (uint32_t V = 1; V <= 4 * HY_MAX_LIMBS / L; V++) {
    const uint32_t w = V == 1 ? 0 : (qbits + V - 1) / V;
    if (V > 1 && (w < 4 || w >= qmin)) continue;
    double noise, budget;
    HY_TRY(noise_model(N, q, L, t, sh, w_max, w, &noise, &budget));
    if (budget - noise >= margin_bits) {
      *w_dcmp = w;
      return HY_OK;
    }
  }
  hy_set_error("no decomposition base leaves %.1f bits of noise margin", margin_bits);
  return HY_EINVAL;
}

// ============================================================================================
// params
// ============================================================================================
static hy_status upload(void** dst, const void* src, size_t bytes) {
  HY_CUDA_TRY(cudaMalloc(dst, bytes));
  HY_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return HY_OK;
}

extern "C" hy_status hy_params_create(uint32_t N, const uint64_t* q, uint32_t L, uint64_t t, int device,
                                      hy_params** out) {
  return hy_params_create2(N, q, L, t, 0, device, out);
}

extern "C" hy_status hy_params_create2(uint32_t N, const uint64_t* q, uint32_t L, uint64_t t, uint32_t w_dcmp,
                                       int device, hy_params** out) {
  HY_CHECK(out && q, HY_EINVAL, "null argument");
  HY_CHECK(N >= 1024 && N <= 16384 && (N & (N - 1)) == 0, HY_EINVAL, "N=%u must be a power of two in [1024, 16384]",
           N);
  HY_CHECK(L >= 1 && L <= HY_MAX_LIMBS, HY_EINVAL, "L=%u must be in [1, %d]", L, HY_MAX_LIMBS);
  HY_CHECK(is_prime(t) && (t - 1) % (2 * (u64)N) == 0, HY_EINVAL, "t must be a prime = 1 mod 2N");
  for (uint32_t l = 0; l < L; l++) {
    HY_CHECK(q[l] > (1ull << 20) && q[l] < (1ull << 60), HY_EINVAL, "q[%u] must be in (2^20, 2^60)", l);
    HY_CHECK(is_prime(q[l]), HY_EINVAL, "q[%u]=%llu is not prime", l, (unsigned long long)q[l]);
    HY_CHECK((q[l] - 1) % (2 * (u64)N) == 0, HY_EINVAL, "q[%u] != 1 mod 2N", l);
    HY_CHECK(q[l] != t, HY_EINVAL, "q[%u] equals t", l);
    for (uint32_t m = 0; m < l; m++) HY_CHECK(q[m] != q[l], HY_EINVAL, "duplicate prime");
  }
  uint32_t qbits_max = 0, qbits_min = 64;
  for (uint32_t l = 0; l < L; l++) {
    uint32_t b = 0;
    while (b < 64 && (q[l] >> b)) b++;
    qbits_max = std::max(qbits_max, b);
    qbits_min = std::min(qbits_min, b);
  }
  HY_CHECK(w_dcmp == 0 || (w_dcmp >= 4 && w_dcmp < qbits_min), HY_EINVAL,
           "decomposition base 2^%u: w must be 0 or in [4, %u)", w_dcmp, qbits_min);
  const uint32_t V = w_dcmp ? (qbits_max + w_dcmp - 1) / w_dcmp : 1;
  HY_CHECK(L * V <= 4 * HY_MAX_LIMBS, HY_EINVAL, "too many gadget digits (%u)", L * V);
  HY_CUDA_TRY(cudaSetDevice(device));
  hy_params* p = new hy_params();
  p->w_dcmp = w_dcmp;
  p->V = V;
  p->ND = L * V;
  p->N = N;
  p->logN = 0;
  while ((1u << p->logN) < N) p->logN++;
  p->L = L;
  p->t = t;
  p->device = device;
  std::vector<u64> psi_rev((size_t)L * N), psi_rev_sh((size_t)L * N), ipsi_rev((size_t)L * N),
      ipsi_rev_sh((size_t)L * N);
  for (uint32_t l = 0; l < L; l++) {
    const u64 ql = q[l];
    p->q[l] = ql;
    const u64 psi = root_2n(ql, N);
    const u64 ipsi = invmod(psi, ql);
    for (uint32_t k = 0; k < N; k++) {
      const uint32_t br = bitrev(k, p->logN);
      const u64 w = powmod(psi, br, ql), iw = powmod(ipsi, br, ql);
      psi_rev[(size_t)l * N + k] = w;
      psi_rev_sh[(size_t)l * N + k] = shoup(w, ql);
      ipsi_rev[(size_t)l * N + k] = iw;
      ipsi_rev_sh[(size_t)l * N + k] = shoup(iw, ql);
    }
    LimbConst& c = p->lc[l];
    c.q = ql;
    c.two_q = 2 * ql;
    c.ninv = invmod(N % ql, ql);
    c.ninv_sh = shoup(c.ninv, ql);
    c.one_sh = shoup(1, ql);
    c.c30 = (1ull << 30) % ql;
    c.c30_sh = shoup(c.c30, ql);
    c.off = ql * (((1ull << 59) + ql - 1) / ql);
    c.c32 = (1ull << 32) % ql;
    c.c32_sh = shoup(c.c32, ql);
    c.off62 = ql * (((1ull << 62) + ql - 1) / ql);
    c.c64 = (u64)(((u128)1 << 64) % ql);
    c.c64_sh = shoup(c.c64, ql);
  }
  // slot-order position j <-> bit-reversed butterfly position k, split into the
  // NTT blocks of HY_NTT_BLOCK coefficients
  std::vector<int32_t> kos(N), own_j, own_k;
  {
    u64 e = 1;
    for (uint32_t j = 0; j < N / 2; j++) {
      kos[j] = (int32_t)bitrev((uint32_t)((e - 1) / 2), p->logN);
      const u64 en = 2 * (u64)N - e;
      kos[j + N / 2] = (int32_t)bitrev((uint32_t)((en - 1) / 2), p->logN);
      e = e * 3 % (2 * (u64)N);
    }
    const uint32_t B = N < HY_NTT_BLOCK ? N : HY_NTT_BLOCK, S = N / B;
    for (uint32_t h = 0; h < S; h++)
      for (uint32_t j = 0; j < N; j++)
        if ((uint32_t)kos[j] / B == h) {
          own_j.push_back((int32_t)j);
          own_k.push_back((int32_t)(kos[j] - h * B));
        }
  }
  std::vector<u64> psi2((size_t)2 * L * N), ipsi2((size_t)2 * L * N);
  for (uint32_t l = 0; l < L; l++)
    for (uint32_t k = 0; k < N; k++) {
      const size_t i = (size_t)l * N + k;
      psi2[2 * i] = k ? psi_rev[i] : 0;
      psi2[2 * i + 1] = k ? psi_rev_sh[i] : 0;
      const u64 iw = k ? ipsi_rev[i] : mulmod(ipsi_rev[(size_t)l * N + 1], p->lc[l].ninv, q[l]);
      ipsi2[2 * i] = iw;
      ipsi2[2 * i + 1] = shoup(iw, q[l]);
    }
  const size_t bytes = (size_t)L * N * sizeof(u64);
  hy_status st;
  if ((st = upload((void**)&p->tab.psi_rev, psi_rev.data(), bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.psi_rev_sh, psi_rev_sh.data(), bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.ipsi_rev, ipsi_rev.data(), bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.ipsi_rev_sh, ipsi_rev_sh.data(), bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.own_j, own_j.data(), N * sizeof(int32_t))) != HY_OK ||
      (st = upload((void**)&p->tab.own_k, own_k.data(), N * sizeof(int32_t))) != HY_OK ||
      (st = upload((void**)&p->tab.psi2, psi2.data(), 2 * bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.ipsi2, ipsi2.data(), 2 * bytes)) != HY_OK ||
      (st = upload((void**)&p->tab.kos, kos.data(), N * sizeof(int32_t))) != HY_OK) {
    hy_params_destroy(p);
    return st;
  }
  p->zeta_t = 0;
  for (u64 x = 2; x < t; x++)
    if (powmod(x, N, t) == t - 1) {
      p->zeta_t = x;
      break;
    }
  *out = p;
  return HY_OK;
}

extern "C" void hy_params_destroy(hy_params* p) {
  if (!p) return;
  cudaSetDevice(p->device);
  cudaFree(p->tab.psi_rev);
  cudaFree(p->tab.psi_rev_sh);
  cudaFree(p->tab.ipsi_rev);
  cudaFree(p->tab.ipsi_rev_sh);
  cudaFree(p->tab.own_j);
  cudaFree(p->tab.own_k);
  cudaFree(p->tab.psi2);
  cudaFree(p->tab.ipsi2);
  cudaFree(p->tab.kos);
  for (auto& kv : p->keys) cudaFree(kv.second.ntt);
  delete p;
}

extern "C" hy_status hy_keys_upload(hy_params* p, uint32_t n, const uint32_t* elts, const uint64_t* keys,
                                    int keys_on_device) {
  HY_CHECK(p && (n == 0 || (elts && keys)), HY_EINVAL, "null argument");
  HY_CUDA_TRY(cudaSetDevice(p->device));
  const size_t L = p->L, N = p->N;
  const size_t key_words = (size_t)p->ND * 2 * L * N;
  u64* tmp = nullptr;
  HY_CUDA_TRY(cudaMalloc(&tmp, key_words * sizeof(u64)));
  for (uint32_t e = 0; e < n; e++) {
    const uint32_t g = elts[e];
    if (!(g & 1) || g >= 2 * p->N) {
      cudaFree(tmp);
      hy_set_error("Galois element %u must be odd and < 2N", g);
      return HY_EINVAL;
    }
    if (!p->keys.count(g) && p->keys.size() >= 4 * HY_MAX_GALOIS) {
      cudaFree(tmp);
      hy_set_error("too many keys");
      return HY_EINVAL;
    }
    const u64* src = keys + (size_t)e * key_words;
    cudaError_t ce = cudaMemcpy(tmp, src, key_words * sizeof(u64),
                                keys_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
      cudaFree(tmp);
      hy_set_error("key copy: %s", cudaGetErrorString(ce));
      return HY_ECUDA;
    }
    // a replaced key is written into a FRESH buffer and swapped in only after the device is idle:
    // an evaluation already queued on another stream keeps reading the old, complete key
    u64* fresh = nullptr;
    ce = cudaMalloc(&fresh, 3 * key_words * sizeof(u64));
    if (ce != cudaSuccess) {
      cudaFree(tmp);
      p->keys_version++;  // earlier elements of this call may have been replaced
      hy_set_error("key alloc: %s", cudaGetErrorString(ce));
      return HY_ENOMEM;
    }
    hy_status st = hyk::key_to_ntt(p, tmp, fresh, 0);
    if (st == HY_OK) st = cudaDeviceSynchronize() == cudaSuccess ? HY_OK : HY_ECUDA;
    if (st != HY_OK) {
      cudaFree(fresh);
      cudaFree(tmp);
      p->keys_version++;
      return st;
    }
    KeyEntry& ke = p->keys[g];
    ke.g = g;
    cudaFree(ke.ntt);  // device idle (synchronised above): nothing reads the old key any more
    ke.ntt = fresh;
  }
  cudaError_t ce = cudaDeviceSynchronize();
  cudaFree(tmp);
  p->keys_version++;
  HY_CHECK(ce == cudaSuccess, HY_ECUDA, "key upload: %s", cudaGetErrorString(ce));
  return HY_OK;
}

// ============================================================================================
// weights
// ============================================================================================
namespace {
// host negacyclic transforms mod t (t < 2^32): forward out[k] = m(zeta^{2 bitrev(k) + 1}) (Cooley-Tukey),
// inverse = its exact inverse (Gentleman-Sande with zeta^{-1} and the N^{-1} scaling)
void host_ntt_t(std::vector<u64>& a, u64 t, u64 zeta, uint32_t logN);
void host_intt_t(std::vector<u64>& a, u64 t, u64 zeta, uint32_t logN) {
  const uint32_t N = 1u << logN;
  const u64 zi = invmod(zeta, t);
  std::vector<u64> zr(N);
  for (uint32_t k = 0; k < N; k++) zr[k] = powmod(zi, bitrev(k, logN), t);
  for (uint32_t m = N / 2, tt = 1; m >= 1; m /= 2, tt *= 2)
    for (uint32_t i = 0; i < m; i++) {
      const u64 w = zr[m + i];
      for (uint32_t j = 2 * i * tt; j < 2 * i * tt + tt; j++) {
        const u64 U = a[j], V = a[j + tt];
        a[j] = (U + V) % t;
        a[j + tt] = (U + t - V) % t * w % t;
      }
    }
  const u64 ni = invmod(N % t, t);
  for (auto& x : a) x = x * ni % t;
}
}  // namespace

// c_n = 4 (NEXT-1, Sylvester basis, reading R11): the plaintexts of Walsh-Hadamard
// rows r = 1..3, slot group c = 2 h + r' (slot row r', half h of the row) holding H4[r][c] =
// (-1)^{popcount(r & c)}; encoded mod t on the host (inverse transform), self-checked by the forward
// transform, centered-lifted into every limb (R14), NTT'd with Shoup companions: [3][2][L][N].
static hy_status hadamard_rows(hy_params* p, const hy_layout& lay, u64** out) {
  (void)lay;
  const uint32_t N = p->N, L = p->L, half = N / 2;
  const u64 t = p->t;
  std::vector<u64> host((size_t)3 * L * N);
  for (int r = 1; r < 4; r++) {
    std::vector<u64> a(N);
    std::vector<int> pat(N);
    u64 e = 1;
    for (uint32_t i = 0; i < half; i++) {
      for (int row = 0; row < 2; row++) {
        const u64 ex = row ? 2 * (u64)N - e : e;
        const uint32_t k = bitrev((uint32_t)((ex - 1) / 2), p->logN);
        const int c = 2 * (i >= half / 2 ? 1 : 0) + row;
        const int sgn = __builtin_popcount(r & c) & 1 ? -1 : 1;
        a[k] = sgn > 0 ? 1 : t - 1;
        pat[k] = sgn;
      }
      e = e * 3 % (2 * (u64)N);
    }
    std::vector<u64> m = a;
    host_intt_t(m, t, p->zeta_t, p->logN);
    std::vector<u64> chk = m;
    host_ntt_t(chk, t, p->zeta_t, p->logN);
    for (uint32_t k = 0; k < N; k++)
      HY_CHECK(chk[k] == a[k], HY_EINVAL, "Hadamard-row plaintext self-check failed (row %d)", r);
    for (uint32_t l = 0; l < L; l++)
      for (uint32_t k = 0; k < N; k++) {
        const int64_t cen = centered(m[k], t);
        host[((size_t)(r - 1) * L + l) * N + k] = cen >= 0 ? (u64)cen % p->q[l] : p->q[l] - ((u64)(-cen) % p->q[l]);
      }
  }
  u64* tmp = nullptr;
  hy_status st = upload((void**)&tmp, host.data(), host.size() * sizeof(u64));
  if (st != HY_OK) return st;
  if (cudaMalloc(out, (size_t)3 * 2 * L * N * sizeof(u64)) != cudaSuccess) {
    *out = nullptr;
    cudaFree(tmp);
    hy_set_error("Hadamard-row plaintext allocation failed");
    return HY_ENOMEM;
  }
  for (int r = 0; r < 3 && st == HY_OK; r++) {
    u64* dst = *out + (size_t)r * 2 * L * N;
    st = hyk::ntt_poly_fwd(p, tmp + (size_t)r * L * N, dst, 1, 0);
    if (st == HY_OK) st = hyk::shoup_table(p, dst, dst + (size_t)L * N, 1, 0);
  }
  cudaDeviceSynchronize();
  cudaFree(tmp);
  return st;
}
// 1x1 kernel, no padding, dense: the coefficient-domain MAC applies (HY_MAC_TC_COEF)
static bool coef_ok(const hy_weights* w, const hy_layout& lay) {
  return !w->shape.depthwise && lay.cn <= 2 && lay.n_taps == 1 && lay.tap_step[0] == 0;
}

extern "C" hy_status hy_encode_weights(hy_params* p, const hy_conv_shape* sh, const int8_t* Wt, hy_weights** out) {
  HY_CHECK(p && sh && Wt && out, HY_EINVAL, "null argument");
  hy_layout lay;
  HY_TRY(hy_plan_layout(p->N, p->t, sh, &lay));
  lay.L = p->L;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  hy_weights* w = new hy_weights();
  memset((void*)w, 0, sizeof(*w));
  w->p = p;
  w->shape = *sh;
  w->lay = lay;
  const int T = (int)lay.n_taps;
  const bool dw = sh->depthwise != 0;
  if (dw) {
    w->M = lay.cn == 2 ? 2 : 1;
    w->K = T;
    w->wblocks = (int)lay.Jc;
  } else {
    // MAC rows per output ct: c_n = 2: (diagonal d, slot row c); c_n = 4: (diagonal d, slot group c)
    w->M = lay.cn == 4 ? (int)(16 * lay.Jo) : lay.cn == 2 ? (int)(4 * lay.Jo) : (int)lay.Jo;
    w->K = (int)lay.Jc * T;
    w->wblocks = 1;
  }
  w->Mpad = hy_mac_mpad(w->M, dw);
  w->mac_path = hy_mac_path(w->M, (int)p->L, dw, coef_ok(w, lay), (int)lay.cn, p->ND != p->L);
  w->Kpad = (w->K + 31) / 32 * 32;  // multiple of the MAC K chunks (16 FP64 GEMM, 32 tcgen05)
  // weight table (S0), [block][kk][row] as exact doubles; row semantics documented in DESIGN.md §4
  std::vector<double> wt((size_t)w->wblocks * w->Kpad * w->Mpad, 0.0);
  const uint32_t Ci = sh->Ci, Co = dw ? sh->Ci : sh->Co, kw = sh->kw;
  auto Wat = [&](uint32_t o, uint32_t c, int tau) -> int32_t {
    const uint32_t dy = tau / kw, dx = tau % kw;
    if (dw) return (o == c && c < Ci) ? Wt[((size_t)c * sh->kh + dy) * kw + dx] : 0;
    if (o >= Co || c >= Ci) return 0;
    return Wt[(((size_t)o * Ci + c) * sh->kh + dy) * kw + dx];
  };
  for (int b = 0; b < w->wblocks; b++)
    for (int row = 0; row < w->M; row++)
      for (int kk = 0; kk < w->K; kk++) {
        int32_t v;
        if (dw) {
          v = lay.cn == 2 ? Wat(2 * b + row, 2 * b + row, kk) : Wat(b, b, kk);
        } else if (lay.cn == 4) {
          // row = (g*4 + d)*4 + c : slot group c of diagonal d pairs input 4j+c with output 4g+(c^d)
          const int g = row / 16, d = (row / 4) % 4, c = row % 4;
          const int tau = kk / (int)lay.Jc, j = kk % (int)lay.Jc;
          v = Wat(4 * g + (c ^ d), 4 * j + c, tau);
        } else if (lay.cn == 2) {
          // row = (g*2 + d)*2 + c : slot row c of diagonal d pairs input 2j+c with output 2g+(c^d)
          const int g = row / 4, d = (row / 2) % 2, c = row % 2;
          const int tau = kk / (int)lay.Jc, j = kk % (int)lay.Jc;  // K axis tap-major
          v = Wat(2 * g + (c ^ d), 2 * j + c, tau);
        } else {
          v = Wat(row, kk % (int)lay.Jc, kk / (int)lay.Jc);
        }
        wt[((size_t)b * w->Kpad + kk) * w->Mpad + row] = (double)v;
      }
  hy_status st = upload((void**)&w->d_wt, wt.data(), wt.size() * sizeof(double));
  if (st == HY_OK) {
    // the same weights as int8 in the tcgen05 canonical K-major layout, 128-row x 32-term tiles:
    // byte (row r, term k) of a tile at (r/8)*256 + (k/16)*128 + (r%8)*16 + k%16
    const int mt = (w->Mpad + 127) / 128, kt = w->Kpad / 32;
    std::vector<int8_t> w8((size_t)w->wblocks * mt * kt * 4096, 0);
    for (int b = 0; b < w->wblocks; b++)
      for (int row = 0; row < w->M; row++)
        for (int kk = 0; kk < w->K; kk++) {
          const int r = row % 128, k = kk % 32;
          const size_t tile = ((size_t)b * mt + row / 128) * kt + kk / 32;
          w8[tile * 4096 + (r / 8) * 256 + (k / 16) * 128 + (r % 8) * 16 + k % 16] =
              (int8_t)wt[((size_t)b * w->Kpad + kk) * w->Mpad + row];
        }
    st = upload((void**)&w->d_w8, w8.data(), w8.size());
  }
  if (st == HY_OK) {
    std::vector<int32_t> kt((size_t)(w->Kpad + 63) / 64 * 64, -1);
    const int Jcb = dw ? 1 : (int)lay.Jc;
    for (int kk = 0; kk < w->K; kk++) kt[kk] = ((kk / Jcb) << 16) | (kk % Jcb);
    st = upload((void**)&w->d_kt, kt.data(), kt.size() * sizeof(int32_t));
  }
  if (st != HY_OK) {
    hy_weights_destroy(w);
    return st;
  }
  const size_t L = p->L, N = p->N, ctw = 2 * L * N;
  const size_t Jin = (size_t)lay.U * lay.Jc, Jo = (size_t)lay.U * lay.Jo;
  if (lay.cn == 4 && (st = hadamard_rows(p, lay, &w->d_sign)) != HY_OK) {
    hy_weights_destroy(w);
    return st;
  }
  // sign plaintext [k,-k]: [k h]_t at X^{N/4}, X^{3N/4}, centered lift (R14)
  if (lay.cn == 2) {
    std::vector<u64> sp(L * N, 0);
    for (size_t l = 0; l < L; l++) {
      const int64_t sc = lay.sign_coeff;
      const u64 v = sc >= 0 ? (u64)sc % p->q[l] : p->q[l] - ((u64)(-sc) % p->q[l]);
      sp[l * N + N / 4] = v;
      sp[l * N + 3 * N / 4] = v;
    }
    u64* tmp = nullptr;
    if ((st = upload((void**)&tmp, sp.data(), sp.size() * sizeof(u64))) != HY_OK) {
      hy_weights_destroy(w);
      return st;
    }
    if (cudaMalloc(&w->d_sign, 2 * L * N * sizeof(u64)) != cudaSuccess) {
      w->d_sign = nullptr;
      cudaFree(tmp);
      hy_weights_destroy(w);
      hy_set_error("sign plaintext allocation failed");
      return HY_ENOMEM;
    }
    st = hyk::ntt_poly_fwd(p, tmp, w->d_sign, 1, 0);
    if (st == HY_OK) st = hyk::shoup_table(p, w->d_sign, w->d_sign + L * N, 1, 0);
    cudaDeviceSynchronize();
    cudaFree(tmp);
    if (st != HY_OK) {
      hy_weights_destroy(w);
      return st;
    }
  }
  // workspace; the rotated inputs R of the dense path are materialised for r_units units at a
  // time (at most HY_R_BUDGET bytes)
  {
    const size_t per_unit = (size_t)w->K * ctw * sizeof(u64);
    size_t ru = per_unit ? HY_R_BUDGET / per_unit : 1;
    if (ru < 1) ru = 1;
    w->r_units = (int)std::min<size_t>(ru, lay.U);
  }
  const size_t ND = p->ND;
  const bool align = lay.cn >= 2 && !dw;  // partial sums aligned by HRot (S4)
  struct A {
    u64** ptr;
    size_t words;
  } allocs[] = {
      {&w->d_D, std::max(Jin, (lay.cn == 2 && w->mac_path == HY_MAC_TC_COEF) ? Jo : 0) * ND * L * N},
      {&w->d_C0, std::max(Jin, (lay.cn == 2 && w->mac_path == HY_MAC_TC_COEF) ? Jo : 0) * L * N},
      {&w->d_P, Jo * ctw * (lay.cn == 4 ? 4 : (lay.cn == 2 && !dw) ? 2 : 1)},
      {&w->d_D2, align ? Jo * ND * L * N + Jo * L * N : 0},
      {&w->d_X, align ? Jo * ctw : 0},
      {&w->d_A1, (lay.cn == 2 && w->mac_path == HY_MAC_TC_COEF) ? Jo * 2 * ctw : 0},
      {&w->d_R, (w->mac_path == HY_MAC_TC_SPLIT || w->mac_path == HY_MAC_FP64_SPLIT)
                    ? (size_t)w->r_units * w->K * ctw : 0},
  };
  for (auto& a : allocs) {
    if (!a.words) continue;
    cudaError_t ce = cudaMalloc(a.ptr, a.words * sizeof(u64));
    if (ce != cudaSuccess) {
      hy_weights_destroy(w);
      hy_set_error("workspace allocation of %zu MiB failed: %s", a.words * 8 >> 20, cudaGetErrorString(ce));
      return HY_ENOMEM;
    }
  }
  cudaError_t ce = cudaMalloc(&w->d_tap_keys, T * sizeof(u64*));
  if (ce == cudaSuccess) ce = cudaMalloc(&w->d_tap_act, T * sizeof(GaloisAct));
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    hy_weights_destroy(w);
    hy_set_error("hy_encode_weights: %s", cudaGetErrorString(ce));
    return HY_ECUDA;
  }
  w->keys_version = ~0ull;
  *out = w;
  return HY_OK;
}

extern "C" hy_status hy_weights_set_stage_events(hy_weights* w, void* const* events, uint32_t n) {
  HY_CHECK(w && (n == 0 || events) && n <= 4, HY_EINVAL, "bad stage events");
  for (uint32_t i = 0; i < n; i++) w->ev[i] = (cudaEvent_t)events[i];
  w->n_ev = n;
  return HY_OK;
}

extern "C" hy_status hy_weights_mac_time(const hy_weights* w, float* total_ms, uint32_t* launches) {
  HY_CHECK(w && total_ms && launches, HY_EINVAL, "null argument");
  *total_ms = 0.f;
  *launches = 0;
  if (!w->mac_ev || !w->mac_launches) return HY_OK;
  for (uint32_t i = 0; i < w->mac_launches; i++) {
    float ms = 0.f;
    HY_CUDA_TRY(cudaEventSynchronize((*w->mac_ev)[2 * i + 1]));
    HY_CUDA_TRY(cudaEventElapsedTime(&ms, (*w->mac_ev)[2 * i], (*w->mac_ev)[2 * i + 1]));
    *total_ms += ms;
  }
  *launches = w->mac_launches;
  return HY_OK;
}

extern "C" hy_status hy_weights_mac_path(const hy_weights* w, int32_t* path) {
  HY_CHECK(w && path, HY_EINVAL, "null argument");
  *path = w->mac_path;
  return HY_OK;
}

extern "C" hy_status hy_weights_set_mac_path(hy_weights* w, int32_t path) {
  HY_CHECK(w, HY_EINVAL, "null argument");
  const bool dw = w->shape.depthwise != 0;
  const int L = (int)w->p->L;
  bool ok = false;
  const bool cn4 = w->lay.cn == 4, sub = w->p->ND != w->p->L;
  switch (path) {
    case HY_MAC_THIN: ok = dw; break;
    case HY_MAC_TC_FUSED: ok = !dw && !cn4 && !sub && w->M <= 128 && (L == 2 || L == 3 || L == 5); break;
    case HY_MAC_TC_SPLIT: ok = !dw && !cn4; break;
    case HY_MAC_FP64_SPLIT: ok = !dw && w->M > 32; break;  // 64-row FP64 tiles (hy_mac_mpad)
    case HY_MAC_FP64_FUSED: ok = !dw && w->M <= 32; break;
    case HY_MAC_TC_COEF: ok = coef_ok(w, w->lay); break;
    case HY_MAC_EAGER: ok = !dw && !cn4; break;
    case HY_MAC_DIRECT: ok = !dw && !cn4; break;
  }
  HY_CHECK(ok, HY_EINVAL, "MAC path %d is not valid for this layout (M = %d, L = %d, depthwise = %d)", path, w->M, L,
           (int)dw);
  cudaSetDevice(w->p->device);
  if (path == HY_MAC_TC_COEF && w->lay.cn == 2) {  // [A1] buffer and Jo-sized digit workspaces
    const size_t N = w->p->N, ctw = 2 * (size_t)L * N, Jin = (size_t)w->lay.U * w->lay.Jc,
                 Jo = (size_t)w->lay.U * w->lay.Jo;
    if (!w->d_A1 && cudaMalloc(&w->d_A1, Jo * 2 * ctw * sizeof(u64)) != cudaSuccess) {
      w->d_A1 = nullptr;
      hy_set_error("coefficient-domain workspace allocation failed");
      return HY_ENOMEM;
    }
    if (Jo > Jin) {  // allocate the larger digit workspaces first: on failure the old ones stay valid
      u64 *nd = nullptr, *nc = nullptr;
      if (cudaMalloc(&nd, Jo * w->p->ND * L * N * sizeof(u64)) != cudaSuccess ||
          cudaMalloc(&nc, Jo * L * N * sizeof(u64)) != cudaSuccess) {
        cudaFree(nd);
        hy_set_error("coefficient-domain digit workspace allocation failed");
        return HY_ENOMEM;
      }
      cudaDeviceSynchronize();  // no evaluation may still read the old workspaces
      cudaFree(w->d_D);
      cudaFree(w->d_C0);
      w->d_D = nd;
      w->d_C0 = nc;
    }
  }
  const bool split = path == HY_MAC_TC_SPLIT || path == HY_MAC_FP64_SPLIT || path == HY_MAC_EAGER ||
                     path == HY_MAC_DIRECT;
  if (path == HY_MAC_EAGER && !w->d_wq) {  // weights mod q_l with Shoup companions, [L][Kpad][Mpad] x 2
    const size_t Lq = w->p->L, blk = (size_t)w->Kpad * w->Mpad;
    std::vector<double> wt(blk);
    if (cudaMemcpy(wt.data(), w->d_wt, blk * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess) {
      hy_set_error("weight table read-back failed");
      return HY_ECUDA;
    }
    std::vector<u64> wq(2 * Lq * blk);
    for (size_t l = 0; l < Lq; l++) {
      const u64 q = w->p->q[l];
      for (size_t i = 0; i < blk; i++) {
        const int64_t v = (int64_t)wt[i];
        const u64 r = v >= 0 ? (u64)v % q : q - ((u64)(-v) % q);
        wq[l * blk + i] = r;
        wq[Lq * blk + l * blk + i] = shoup(r, q);
      }
    }
    hy_status st = upload((void**)&w->d_wq, wq.data(), wq.size() * sizeof(u64));
    if (st != HY_OK) {
      w->d_wq = nullptr;
      return st;
    }
  }
  if (split && !w->d_R) {
    const size_t words = (size_t)w->r_units * w->K * 2 * L * w->p->N;
    cudaError_t ce = cudaMalloc(&w->d_R, words * sizeof(u64));
    if (ce != cudaSuccess) {
      w->d_R = nullptr;
      hy_set_error("rotated-input workspace of %zu MiB: %s", words * 8 >> 20, cudaGetErrorString(ce));
      return HY_ENOMEM;
    }
  }
  w->mac_path = path;
  return HY_OK;
}

extern "C" hy_status hy_weights_layout(const hy_weights* w, hy_layout* out) {
  HY_CHECK(w && out, HY_EINVAL, "null argument");
  *out = w->lay;
  return HY_OK;
}

extern "C" void hy_weights_destroy(hy_weights* w) {
  if (!w) return;
  cudaSetDevice(w->p->device);
  cudaFree(w->d_wt);
  cudaFree(w->d_w8);
  cudaFree(w->d_kt);
  cudaFree(w->d_sign);
  cudaFree(w->d_D);
  cudaFree(w->d_C0);
  cudaFree(w->d_P);
  cudaFree(w->d_D2);
  cudaFree(w->d_X);
  cudaFree(w->d_A1);
  cudaFree(w->d_R);
  cudaFree(w->d_wq);
  cudaFree(w->d_in);
  cudaFree(w->d_out);
  if (w->s_h2d) {
    cudaStreamDestroy(w->s_h2d);
    cudaStreamDestroy(w->s_d2h);
    cudaEventDestroy(w->ev_h2d);
    cudaEventDestroy(w->ev_comp);
  }
  cudaFree(w->d_tap_keys);
  cudaFree(w->d_tap_act);
  if (w->mac_ev) {
    for (cudaEvent_t e : *w->mac_ev) cudaEventDestroy(e);
    delete w->mac_ev;
  }
  delete w;
}

static hy_status bind_keys(hy_weights* w) {
  hy_params* p = w->p;
  if (w->keys_version == p->keys_version) return HY_OK;
  const hy_layout& lay = w->lay;
  const uint32_t row = p->N / 2;
  std::vector<u64*> ptrs(lay.n_taps, nullptr);
  std::vector<GaloisAct> acts(lay.n_taps, GaloisAct{0u, 0u});
  for (uint32_t tau = 0; tau < lay.n_taps; tau++) {
    const int64_t st = (((int64_t)lay.tap_step[tau] % (int64_t)row) + row) % row;
    if (st == 0) continue;
    const uint32_t g = (uint32_t)powmod(3, (u64)st, 2 * (u64)p->N);
    auto it = p->keys.find(g);
    HY_CHECK(it != p->keys.end(), HY_ENOKEY, "no Galois key for element %u (tap %u, step %d)", g, tau,
             lay.tap_step[tau]);
    ptrs[tau] = it->second.ntt;
    HY_CHECK(hy_galois_act(g, p->N, &acts[tau]), HY_EINVAL, "bad Galois element %u", g);
  }
  w->d_swap_key = nullptr;
  if (lay.cn == 2 && !w->shape.depthwise) {
    auto it = p->keys.find(2 * p->N - 1);
    HY_CHECK(it != p->keys.end(), HY_ENOKEY, "no Galois key for the row swap (element %u)", 2 * p->N - 1);
    w->d_swap_key = it->second.ntt;
  }
  if (lay.cn == 4) {  // the last three layout elements: alignment of diagonals 1, 2, 3
    for (int d = 0; d < 3; d++) {
      const uint32_t g = d == 0 ? 2 * p->N - 1
                                : d == 1 ? (uint32_t)powmod(3, p->N / 4, 2 * (u64)p->N)
                                         : (uint32_t)mulmod(2 * p->N - 1, powmod(3, p->N / 4, 2 * (u64)p->N),
                                                            2 * (u64)p->N);
      auto it = p->keys.find(g);
      HY_CHECK(it != p->keys.end(), HY_ENOKEY, "no Galois key for the c_n = 4 alignment (element %u)", g);
      w->d_align_key[d] = it->second.ntt;
      HY_CHECK(hy_galois_act(g, p->N, &w->h_align_act[d]), HY_EINVAL, "bad Galois element %u", g);
    }
  }
  for (uint32_t tau = 0; tau < lay.n_taps; tau++) {
    w->h_tap_keys[tau] = ptrs[tau];
    w->h_tap_act[tau] = acts[tau];
  }
  HY_CUDA_TRY(cudaMemcpy(w->d_tap_keys, ptrs.data(), ptrs.size() * sizeof(u64*), cudaMemcpyHostToDevice));
  HY_CUDA_TRY(cudaMemcpy(w->d_tap_act, acts.data(), acts.size() * sizeof(GaloisAct), cudaMemcpyHostToDevice));
  w->keys_version = p->keys_version;
  return HY_OK;
}

// ============================================================================================
// evaluation
// ============================================================================================
extern "C" hy_status hy_conv_eval(hy_weights* w, const uint64_t* ct_in, size_t J, uint64_t* ct_out, size_t Jout,
                                  void* stream) {
  HY_CHECK(w, HY_EINVAL, "null weights");
  const hy_layout& lay = w->lay;
  HY_CHECK(J > 0 && J % lay.Jc == 0, HY_ESHAPE, "J=%zu is not a positive multiple of Jc=%u", J, lay.Jc);
  HY_CHECK(ct_in && ct_out, HY_EINVAL, "null argument");
  const size_t nu = J / lay.Jc;
  HY_CHECK(nu <= lay.U, HY_ESHAPE, "J=%zu covers %zu units > U=%u", J, nu, lay.U);
  HY_CHECK(Jout == nu * lay.Jo, HY_ESHAPE, "Jout=%zu, expected %zu", Jout, nu * lay.Jo);
  hy_params* p = w->p;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  HY_TRY(bind_keys(w));
  cudaStream_t s = (cudaStream_t)stream;
  auto mark = [&](uint32_t i) -> hy_status {
    if (i < w->n_ev) HY_CUDA_TRY(cudaEventRecord(w->ev[i], s));
    return HY_OK;
  };
  HY_TRY(mark(0));
  if (w->mac_path == HY_MAC_TC_COEF) {  // 1x1, c_n = 1: one MAC over the coefficient-form inputs
    HY_TRY(mark(1));
    HY_TRY(hyk::mac_coef(w, ct_in, nu, ct_out, s));
    HY_TRY(mark(2));
    if (lay.cn == 2) HY_TRY(hyk::finish_coef2(w, nu, ct_out, s));  // sign PMult + row swap
    HY_TRY(mark(3));
    return HY_OK;
  }
  if (w->mac_path == HY_MAC_DIRECT)  // no-hoisting ablation: only NTT(c0) here, digits per rotation
    HY_TRY(hyk::c0_only(p, ct_in, J, w->d_C0, s));
  else
    HY_TRY(hyk::permdecomp(p, ct_in, J, w->d_D, w->d_C0, s));  // S1 PermDecomp
  HY_TRY(mark(1));
  HY_TRY(hyk::ksmac(w, ct_in, nu, s));  // S2 PermAuto fused with S3 lazy MAC + WHT + reduce + sign PMult
  HY_TRY(mark(2));
  HY_TRY(hyk::finish_outputs(w, nu, ct_out, s));  // S4 alignment + S5 INTT
  HY_TRY(mark(3));
  return HY_OK;
}

extern "C" hy_status hy_conv_eval_host(hy_weights* w, const uint64_t* in, size_t J, uint64_t* out, size_t Jout,
                                       void* stream) {
  HY_CHECK(w, HY_EINVAL, "null weights");
  const hy_layout& lay = w->lay;
  const size_t ctw = 2 * (size_t)w->p->L * w->p->N;
  HY_CHECK(J > 0 && J % lay.Jc == 0, HY_ESHAPE, "J=%zu is not a positive multiple of Jc=%u", J, lay.Jc);
  HY_CHECK(in && out, HY_EINVAL, "null argument");
  const size_t nu = J / lay.Jc;
  HY_CHECK(nu <= lay.U && Jout == nu * lay.Jo, HY_ESHAPE, "J=%zu / Jout=%zu do not match the layout", J, Jout);
  HY_CUDA_TRY(cudaSetDevice(w->p->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (!w->d_in) {  // staging buffers of the host path: allocated on first use
    const size_t Jin = (size_t)lay.U * lay.Jc, Jo = (size_t)lay.U * lay.Jo;
    if (cudaMalloc(&w->d_in, Jin * ctw * sizeof(u64)) != cudaSuccess ||
        cudaMalloc(&w->d_out, Jo * ctw * sizeof(u64)) != cudaSuccess) {
      cudaFree(w->d_in);
      w->d_in = w->d_out = nullptr;
      hy_set_error("host-path staging allocation failed");
      return HY_ENOMEM;
    }
  }
  if (!w->s_h2d) {
    HY_CUDA_TRY(cudaStreamCreateWithFlags(&w->s_h2d, cudaStreamNonBlocking));
    HY_CUDA_TRY(cudaStreamCreateWithFlags(&w->s_d2h, cudaStreamNonBlocking));
    HY_CUDA_TRY(cudaEventCreateWithFlags(&w->ev_h2d, cudaEventDisableTiming));
    HY_CUDA_TRY(cudaEventCreateWithFlags(&w->ev_comp, cudaEventDisableTiming));
  }
  // Pipelined over batches of units (units are independent): the upload of batch
  // b + 1 and the download of batch b - 1 overlap the evaluation of batch b on the caller's stream.
  // Batch size: the pipeline's fill and drain cost one batch's upload + evaluation + download, so
  // batches are as small as keeps a copy efficient (>= 32 MiB of input per batch, at most 32 batches;
  // HY_HOST_BATCHES overrides the batch count for measurements).
  size_t nbatch = 32;
  if (const char* e = getenv("HY_HOST_BATCHES")) nbatch = std::max<size_t>(1, strtoull(e, nullptr, 10));
  size_t nb = (nu + nbatch - 1) / nbatch;
  if (!getenv("HY_HOST_BATCHES")) {
    const size_t unit_bytes = (size_t)lay.Jc * ctw * sizeof(u64);
    nb = std::max(nb, ((size_t)32 << 20) / unit_bytes + 1);
  }
  nb = std::min(std::max<size_t>(nb, 1), nu);
  for (size_t u0 = 0; u0 < nu; u0 += nb) {
    const size_t n = std::min(nb, nu - u0);
    const size_t i0 = u0 * lay.Jc, ni = n * lay.Jc, o0 = u0 * lay.Jo, no = n * lay.Jo;
    HY_CUDA_TRY(cudaMemcpyAsync(w->d_in + i0 * ctw, in + i0 * ctw, ni * ctw * sizeof(u64), cudaMemcpyHostToDevice,
                                w->s_h2d));
    HY_CUDA_TRY(cudaEventRecord(w->ev_h2d, w->s_h2d));
    HY_CUDA_TRY(cudaStreamWaitEvent(s, w->ev_h2d, 0));
    HY_TRY(hy_conv_eval(w, w->d_in + i0 * ctw, ni, w->d_out + o0 * ctw, no, stream));
    HY_CUDA_TRY(cudaEventRecord(w->ev_comp, s));
    HY_CUDA_TRY(cudaStreamWaitEvent(w->s_d2h, w->ev_comp, 0));
    HY_CUDA_TRY(cudaMemcpyAsync(out + o0 * ctw, w->d_out + o0 * ctw, no * ctw * sizeof(u64), cudaMemcpyDeviceToHost,
                                w->s_d2h));
  }
  HY_CUDA_TRY(cudaStreamSynchronize(w->s_d2h));
  return HY_OK;
}

// ============================================================================================
// per-stage entry points
// ============================================================================================
extern "C" hy_status hy_poly_mul(const hy_params* p, const uint64_t* a, const uint64_t* b, uint64_t* c, size_t n,
                                 void* stream) {
  HY_CHECK(p && a && b && c, HY_EINVAL, "null argument");
  if (n == 0) return HY_OK;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = (cudaStream_t)stream;
  const size_t words = n * p->L * p->N;
  u64* tmp = nullptr;
  HY_CUDA_TRY(cudaMalloc(&tmp, 2 * words * sizeof(u64)));
  hy_status st = hyk::ntt_poly_fwd(p, a, tmp, n, s);
  if (st == HY_OK) st = hyk::ntt_poly_fwd(p, b, tmp + words, n, s);
  if (st == HY_OK) st = hyk::pointwise_mul(p, tmp, tmp + words, c, n, s);
  cudaError_t ce = cudaStreamSynchronize(s);
  cudaFree(tmp);
  if (st != HY_OK) return st;
  HY_CHECK(ce == cudaSuccess, HY_ECUDA, "%s", cudaGetErrorString(ce));
  return HY_OK;
}

extern "C" hy_status hy_ntt_roundtrip(const hy_params* p, uint64_t* x, size_t n, void* stream) {
  HY_CHECK(p && x, HY_EINVAL, "null argument");
  if (n == 0) return HY_OK;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = (cudaStream_t)stream;
  // the forward transform must not run in place: the CTAs of one split transform read every
  // coefficient of their polynomial (ntt.cuh)
  u64* tmp = nullptr;
  HY_CUDA_TRY(cudaMalloc(&tmp, n * p->L * p->N * sizeof(u64)));
  hy_status st = hyk::ntt_poly_fwd(p, x, tmp, n, s);
  if (st == HY_OK) st = hyk::ntt_poly_inv(p, tmp, x, n, s);
  cudaError_t ce = cudaStreamSynchronize(s);
  cudaFree(tmp);
  if (st != HY_OK) return st;
  HY_CHECK(ce == cudaSuccess, HY_ECUDA, "%s", cudaGetErrorString(ce));
  return HY_OK;
}

extern "C" hy_status hy_rotate(hy_params* p, const uint64_t* ct_in, uint32_t g, uint64_t* ct_out, size_t n,
                               void* stream) {
  HY_CHECK(p && ct_in && ct_out, HY_EINVAL, "null argument");
  if (n == 0) return HY_OK;
  auto it = p->keys.find(g);
  HY_CHECK(it != p->keys.end(), HY_ENOKEY, "no Galois key for element %u", g);
  HY_CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = (cudaStream_t)stream;
  u64* work = nullptr;
  GaloisAct act;
  HY_CHECK(hy_galois_act(g, p->N, &act), HY_EINVAL, "Galois element %u is not odd / < 2N", g);
  HY_CUDA_TRY(cudaMalloc(&work, n * (p->ND * p->L + 3 * p->L) * p->N * sizeof(u64)));
  hy_status st = hyk::rotate_ct(p, ct_in, act, it->second.ntt, ct_out, n, work, s);
  cudaError_t ce = cudaStreamSynchronize(s);
  cudaFree(work);
  if (st != HY_OK) return st;
  HY_CHECK(ce == cudaSuccess, HY_ECUDA, "%s", cudaGetErrorString(ce));
  return HY_OK;
}

// ============================================================================================
// client-side draws on the GPU: Philox4x32-10, counter layout of
// synth/philox.py; the oracle-side client reproduces every draw bit for bit
// ============================================================================================
namespace {
struct DevBuf {  // RAII device allocation for the synchronous client calls
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
};
}  // namespace

extern "C" hy_status hy_secret_key(const hy_params* p, uint64_t seed, int8_t* sk_out) {
  HY_CHECK(p && sk_out, HY_EINVAL, "null argument");
  HY_CUDA_TRY(cudaSetDevice(p->device));
  const size_t L = p->L, N = p->N;
  DevBuf sres, s8;
  HY_CUDA_TRY(cudaMalloc(&sres.p, L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&s8.p, N));
  HY_TRY(hyk::client_secret(p, seed, (int8_t*)s8.p, (u64*)sres.p, nullptr, 0));
  HY_CUDA_TRY(cudaMemcpy(sk_out, s8.p, N, cudaMemcpyDeviceToHost));
  return HY_OK;
}

extern "C" hy_status hy_keygen(hy_params* p, uint64_t seed, uint32_t n, const uint32_t* elts, uint64_t* keys_out,
                               int upload) {
  HY_CHECK(p && (n == 0 || elts), HY_EINVAL, "null argument");
  if (n == 0) return HY_OK;
  for (uint32_t e = 0; e < n; e++)
    HY_CHECK((elts[e] & 1) && elts[e] < 2 * p->N, HY_EINVAL, "Galois element %u must be odd and < 2N", elts[e]);
  HY_CUDA_TRY(cudaSetDevice(p->device));
  const size_t L = p->L, N = p->N, ND = p->ND, kw = ND * 2 * L * N;
  DevBuf sres, s8, sntt, del, work, kout;
  HY_CUDA_TRY(cudaMalloc(&sres.p, L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&s8.p, N));
  HY_CUDA_TRY(cudaMalloc(&sntt.p, 2 * L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&del.p, n * sizeof(uint32_t)));
  HY_CUDA_TRY(cudaMemcpy(del.p, elts, n * sizeof(uint32_t), cudaMemcpyHostToDevice));
  // work: A, NTT(A) [n ND][L][N], s(X^g) [n][L][N], errors [n ND][N] int32
  HY_CUDA_TRY(cudaMalloc(&work.p, (2 * n * ND * L * N + n * L * N) * 8 + n * ND * N * 4));
  u64* out = keys_out;
  if (!out) {
    HY_CUDA_TRY(cudaMalloc(&kout.p, n * kw * 8));
    out = (u64*)kout.p;
  }
  HY_TRY(hyk::client_secret(p, seed, (int8_t*)s8.p, (u64*)sres.p, (u64*)sntt.p, 0));
  HY_TRY(hyk::client_keygen(p, seed, (const u64*)sntt.p, (const int8_t*)s8.p, (const uint32_t*)del.p, n, out,
                            (u64*)work.p, 0));
  HY_CUDA_TRY(cudaDeviceSynchronize());
  if (upload) HY_TRY(hy_keys_upload(p, n, elts, out, 1));
  return HY_OK;
}

extern "C" hy_status hy_encrypt(const hy_params* p, uint64_t seed, const uint64_t* m, size_t n, uint32_t first,
                                uint64_t* ct_out, void* stream) {
  HY_CHECK(p && m && ct_out, HY_EINVAL, "null argument");
  if (n == 0) return HY_OK;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  const size_t L = p->L, N = p->N;
  // Delta = floor(Q / t) mod q_l = -(Q mod t) t^{-1} mod q_l  (Q = 0 mod q_l)
  u64 r = 1;
  for (size_t l = 0; l < L; l++) r = mulmod(r, p->q[l] % p->t, p->t);
  u64 delta[HY_MAX_LIMBS];
  for (size_t l = 0; l < L; l++) {
    const u64 q = p->q[l];
    delta[l] = mulmod((q - r % q) % q, invmod(p->t % q, q), q);
  }
  cudaStream_t st = (cudaStream_t)stream;
  DevBuf sres, s8, sntt, md, idx, work;
  HY_CUDA_TRY(cudaMalloc(&sres.p, L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&s8.p, N));
  HY_CUDA_TRY(cudaMalloc(&sntt.p, 2 * L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&md.p, n * N * 8));
  HY_CUDA_TRY(cudaMalloc(&idx.p, n * sizeof(uint32_t)));
  HY_CUDA_TRY(cudaMalloc(&work.p, 2 * n * L * N * 8 + n * N * 4));
  std::vector<uint32_t> ids(n);
  for (size_t o = 0; o < n; o++) ids[o] = first + (uint32_t)o;
  for (size_t i = 0; i < n * N; i++) HY_CHECK(m[i] < p->t, HY_EINVAL, "plaintext coefficient %zu not < t", i);
  HY_CUDA_TRY(cudaMemcpyAsync(md.p, m, n * N * 8, cudaMemcpyHostToDevice, st));
  HY_CUDA_TRY(cudaMemcpyAsync(idx.p, ids.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  HY_TRY(hyk::client_secret(p, seed, (int8_t*)s8.p, (u64*)sres.p, (u64*)sntt.p, st));
  HY_TRY(hyk::client_encrypt(p, seed, (const u64*)sntt.p, (const u64*)md.p, (const uint32_t*)idx.p, n, delta, ct_out,
                             (u64*)work.p, st));
  HY_CUDA_TRY(cudaStreamSynchronize(st));
  return HY_OK;
}

// ============================================================================================
// debug decryption
// ============================================================================================
namespace {
// minimal unsigned big integer (little-endian 32-bit limbs) for the exact CRT rounding
struct Big {
  std::vector<uint32_t> d;
  void trim() {
    while (!d.empty() && d.back() == 0) d.pop_back();
  }
  static Big from(u64 x) {
    Big b;
    b.d = {(uint32_t)x, (uint32_t)(x >> 32)};
    b.trim();
    return b;
  }
  Big mul(u64 m) const {
    Big r;
    const uint32_t m0 = (uint32_t)m, m1 = (uint32_t)(m >> 32);
    r.d.assign(d.size() + 3, 0);
    for (int pass = 0; pass < 2; pass++) {
      const u64 mm = pass ? m1 : m0;
      u64 carry = 0;
      size_t i = 0;
      for (; i < d.size(); i++) {
        u64 cur = (u64)r.d[i + pass] + (u64)d[i] * mm + carry;
        r.d[i + pass] = (uint32_t)cur;
        carry = cur >> 32;
      }
      for (size_t k = i + pass; carry; k++) {
        u64 cur = (u64)r.d[k] + carry;
        r.d[k] = (uint32_t)cur;
        carry = cur >> 32;
      }
    }
    r.trim();
    return r;
  }
  Big add(const Big& o) const {
    Big r;
    r.d.assign(std::max(d.size(), o.d.size()) + 1, 0);
    u64 carry = 0;
    for (size_t i = 0; i < r.d.size(); i++) {
      u64 cur = carry + (i < d.size() ? d[i] : 0) + (i < o.d.size() ? o.d[i] : 0);
      r.d[i] = (uint32_t)cur;
      carry = cur >> 32;
    }
    r.trim();
    return r;
  }
  Big sub(const Big& o) const {  // requires *this >= o
    Big r = *this;
    int64_t borrow = 0;
    for (size_t i = 0; i < r.d.size(); i++) {
      int64_t cur = (int64_t)r.d[i] - (i < o.d.size() ? o.d[i] : 0) - borrow;
      borrow = cur < 0;
      r.d[i] = (uint32_t)(cur + (borrow ? (1ll << 32) : 0));
    }
    r.trim();
    return r;
  }
  double to_double() const {
    double r = 0;
    for (size_t i = d.size(); i-- > 0;) r = r * 4294967296.0 + (double)d[i];
    return r;
  }
  int cmp(const Big& o) const {
    if (d.size() != o.d.size()) return d.size() < o.d.size() ? -1 : 1;
    for (size_t i = d.size(); i-- > 0;)
      if (d[i] != o.d[i]) return d[i] < o.d[i] ? -1 : 1;
    return 0;
  }
};

// host negacyclic NTT mod t (t < 2^32): out[k] = m(zeta^{2 bitrev(k) + 1})
void host_ntt_t(std::vector<u64>& a, u64 t, u64 zeta, uint32_t logN) {
  const uint32_t N = 1u << logN;
  std::vector<u64> zr(N);
  for (uint32_t k = 0; k < N; k++) zr[k] = powmod(zeta, bitrev(k, logN), t);
  for (uint32_t m = 1, tt = N / 2; m < N; m *= 2, tt /= 2)
    for (uint32_t i = 0; i < m; i++) {
      const u64 w = zr[m + i];
      for (uint32_t j = 2 * i * tt; j < 2 * i * tt + tt; j++) {
        const u64 U = a[j], V = a[j + tt] * w % t;
        a[j] = (U + V) % t;
        a[j + tt] = (U + t - V) % t;
      }
    }
}
}  // namespace

extern "C" hy_status hy_decrypt_debug(const hy_params* p, const int8_t* sk, const uint64_t* ct, size_t n,
                                      uint32_t scale, uint64_t* slots_out) {
  return hy_decrypt_debug_noise(p, sk, ct, n, scale, slots_out, nullptr);
}

extern "C" hy_status hy_decrypt_debug_noise(const hy_params* p, const int8_t* sk, const uint64_t* ct, size_t n,
                                            uint32_t scale, uint64_t* slots_out, double* budget_bits) {
  HY_CHECK(p && sk && ct && slots_out, HY_EINVAL, "null argument");
  HY_CHECK(scale % p->t != 0, HY_EINVAL, "scale must be invertible mod t");
  if (n == 0) return HY_OK;
  HY_CUDA_TRY(cudaSetDevice(p->device));
  const size_t L = p->L, N = p->N;
  std::vector<u64> s_res(L * N);
  for (size_t l = 0; l < L; l++)
    for (size_t k = 0; k < N; k++) {
      const int v = sk[k];
      HY_CHECK(v >= -1 && v <= 1, HY_EINVAL, "secret key must be ternary");
      s_res[l * N + k] = v >= 0 ? (u64)v : p->q[l] - 1;
    }
  u64 *d_s = nullptr, *d_sn = nullptr, *d_x = nullptr, *d_work = nullptr;
  HY_CUDA_TRY(cudaMalloc(&d_s, L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&d_sn, 2 * L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&d_x, n * L * N * 8));
  HY_CUDA_TRY(cudaMalloc(&d_work, n * L * N * 8));
  HY_CUDA_TRY(cudaMemcpy(d_s, s_res.data(), L * N * 8, cudaMemcpyHostToDevice));
  hy_status st = hyk::ntt_poly_fwd(p, d_s, d_sn, 1, 0);
  if (st == HY_OK) st = hyk::shoup_table(p, d_sn, d_sn + L * N, 1, 0);
  if (st == HY_OK) st = hyk::decrypt_phase(p, d_sn, d_sn + L * N, ct, n, d_x, d_work, 0);
  std::vector<u64> x(n * L * N);
  cudaError_t ce = cudaMemcpy(x.data(), d_x, n * L * N * 8, cudaMemcpyDeviceToHost);
  cudaFree(d_s);
  cudaFree(d_sn);
  cudaFree(d_x);
  cudaFree(d_work);
  if (st != HY_OK) return st;
  HY_CHECK(ce == cudaSuccess, HY_ECUDA, "%s", cudaGetErrorString(ce));
  // exact CRT rounding: m = round(sum_l t z_l / q_l) mod t, z_l = x_l [(Q/q_l)^{-1}]_{q_l}
  const u64 t = p->t;
  Big Q = Big::from(1);
  for (size_t l = 0; l < L; l++) Q = Q.mul(p->q[l]);
  std::vector<Big> Ql(L);
  std::vector<u64> inv(L);
  for (size_t l = 0; l < L; l++) {
    Big b = Big::from(1);
    u64 r = 1;
    for (size_t m = 0; m < L; m++)
      if (m != l) {
        b = b.mul(p->q[m]);
        r = mulmod(r, p->q[m] % p->q[l], p->q[l]);
      }
    Ql[l] = b;
    inv[l] = invmod(r, p->q[l]);
  }
  const Big Q2 = Q.mul(2);
  const u64 sinv = invmod(scale % t, t);
  std::vector<u64> m(N);
  const uint32_t half = (uint32_t)N / 2;
  const double Qd = Q.to_double();
  double worst = 1e300;
  for (size_t o = 0; o < n; o++) {
    double bud = 1e300;
    for (size_t k = 0; k < N; k++) {
      u64 isum = 0;
      Big S;
      for (size_t l = 0; l < L; l++) {
        const u64 z = mulmod(x[(o * L + l) * N + k], inv[l], p->q[l]);
        const u128 tz = (u128)t * z;
        isum += (u64)(tz / p->q[l]);
        S = S.add(Ql[l].mul((u64)(tz % p->q[l])));
      }
      Big X = S.mul(2).add(Q);  // round(S/Q) = floor((2S + Q) / 2Q)
      u64 j = 0;
      while (X.cmp(Q2) >= 0) {
        X = X.sub(Q2);
        j++;
      }
      m[k] = (isum + j) % t;
      // invariant noise of coefficient k: t x / Q - round(t x / Q) = (X - Q) / 2Q in [-1/2, 1/2);
      // budget = log2(1 / (2 |.|)) = log2(Q / |X - Q|) bits (0 bits = undecryptable)
      const Big dist = X.cmp(Q) >= 0 ? X.sub(Q) : Q.sub(X);
      const double dd = dist.to_double();
      if (dd > 0) bud = std::min(bud, std::log2(Qd / dd));
    }
    if (budget_bits) budget_bits[o] = bud;
    worst = std::min(worst, bud);
    host_ntt_t(m, t, p->zeta_t, p->logN);
    for (uint32_t r = 0; r < 2; r++)
      for (uint32_t i = 0; i < half; i++) {
        u64 e = powmod(3, i, 2 * (u64)N);
        if (r) e = 2 * (u64)N - e;
        const uint32_t kk = bitrev((uint32_t)((e - 1) / 2), p->logN);
        slots_out[o * N + r * half + i] = mulmod(m[kk], sinv, t);
      }
  }
  HY_CHECK(worst >= 1.0, HY_ENOISE, "noise budget exhausted: %.2f bits left (< 1 bit: the decryption is unreliable)",
           worst);
  return HY_OK;
}
