// Internal definitions shared by the library's translation units (NOT shared with oracle/).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <vector>

#include "../../include/hyena.h"

typedef uint64_t u64;
typedef unsigned __int128 u128;

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
void hy_set_error(const char* fmt, ...);

#define HY_CUDA_TRY(expr)                                                                     \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e != cudaSuccess) {                                                                  \
      hy_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e));        \
      return HY_ECUDA;                                                                        \
    }                                                                                         \
  } while (0)

void hy_count_launch();

#define HY_LAUNCH_CHECK()                                                                     \
  do {                                                                                        \
    hy_count_launch();                                                                        \
    cudaError_t _e = cudaGetLastError();                                                      \
    if (_e != cudaSuccess) {                                                                  \
      hy_set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e));    \
      return HY_ECUDA;                                                                        \
    }                                                                                         \
  } while (0)

#define HY_TRY(expr)                 \
  do {                               \
    hy_status _s = (expr);           \
    if (_s != HY_OK) return _s;      \
  } while (0)

// ------------------------------------------------------------------------------------
// per-limb constants passed to kernels by value
// ------------------------------------------------------------------------------------
struct LimbConst {
  u64 q;
  u64 two_q;
  u64 ninv, ninv_sh;      // N^{-1} mod q and its Shoup companion
  u64 one_sh;             // floor(2^64 / q): Shoup companion of 1
  u64 c30, c30_sh;        // 2^30 mod q and Shoup companion
  u64 off;                // q * ceil(2^59 / q): makes |x| < 2^59 signed values nonnegative
  u64 c32, c32_sh;        // 2^32 mod q and Shoup companion (tensor-core MAC epilogue)
  u64 off62;              // q * ceil(2^62 / q): makes |x| < 2^62 signed values nonnegative
  u64 c64, c64_sh;        // 2^64 mod q and Shoup companion (16-plane MAC epilogue)
};

struct DevTables {
  // [L][N] each, device
  u64* psi_rev;       // psi^{bitrev(k)}
  u64* psi_rev_sh;
  u64* ipsi_rev;      // psi^{-bitrev(k)}
  u64* ipsi_rev_sh;
  // [S][B] (B = min(N, HY_NTT_BLOCK), S = N / B): slot-order positions j owned by NTT block h
  // (ascending) and their butterfly position inside the block.  Slot position j holds the
  // evaluation at psi^{e_j} (e_j = 3^j for j < N/2, -3^{j-N/2} for j >= N/2, mod 2N), which the
  // forward transform leaves at butterfly position bitrev((e_j - 1)/2).
  int32_t* own_j;
  int32_t* own_k;
  // one-CTA NTT (ntt2_*, N = 4096 / 8192): interleaved (w, w') [L][N] for psi / psi^{-1} (entry 0 of
  // the inverse table = psi^{-bitrev(1)} N^{-1}, the last inverse stage with the scaling folded in),
  // and kos[j] = butterfly position of slot j
  ulonglong2* psi2;
  ulonglong2* ipsi2;
  int32_t* kos;
};

// Galois automorphism X -> X^g, g = (+/-) 3^shift mod 2N, acting on slot-ordered NTT vectors:
// out[j] = in[perm(j)] with perm(j) = ((j + shift) mod N/2) + (half of j, exchanged if swap).
struct GaloisAct {
  uint32_t shift;
  uint32_t swap;
};

#define HY_NTT_BLOCK 4096
#define HY_R_BUDGET ((size_t)4 << 30)  // bytes of materialised rotated inputs per hy_weights  // coefficients per NTT CTA (must match NttCfg in ntt.cuh)

struct KeyEntry {
  uint32_t g;
  u64* ntt;  // device [L digits][2][L limbs][N] values, then the same again for Shoup companions, then
            // the same again with each value w split into 30-bit halves (w mod 2^30) | (w >> 30) << 32
};

struct hy_params {
  uint32_t N, logN, L;
  uint32_t w_dcmp = 0;  // sub-digit decomposition base 2^w inside each limb (0: one digit per limb)
  uint32_t V = 1;       // sub-digits per limb
  uint32_t ND = 0;      // gadget digits L V: D is [ct][ND][L][N], a key [ND][2][L][N]
  u64 t;
  u64 q[HY_MAX_LIMBS];
  int device;
  LimbConst lc[HY_MAX_LIMBS];
  DevTables tab;
  u64* d_scratch = nullptr;  // small scratch
  // plaintext side (host)
  u64 zeta_t;
  std::map<uint32_t, KeyEntry> keys;
  u64 keys_version = 0;  // bumped by every hy_keys_upload
};

bool hy_galois_act(uint32_t g, uint32_t N, GaloisAct* out);

// Row tile of the fused S2+S3 kernel for M MAC rows: -MR = thin kernel with MR <= 2 rows,
// else WM warps (8 rows each).  Shared by hy_encode_weights (table padding) and the launcher.
inline int hy_mac_tile(int M, bool depthwise) {
  if (depthwise) return -M;  // M <= 2: thin kernel (one term per tap, one input ct per unit)
  if (M <= 8) return 1;
  if (M <= 16) return 2;
  if (M <= 32) return 4;
  return 8;
}
inline int hy_mac_mpad(int M, bool depthwise) {
  const int t = hy_mac_tile(M, depthwise);
  const int bm = t < 0 ? -t : 8 * t;
  return (M + bm - 1) / bm * bm;
}  // false if g is not odd / not in Z_2N^*

// S2 + S3 kernel choice (hy_mac_path, fixed at hy_encode_weights)
enum HyMacPath {
  HY_MAC_THIN = 0,        // depthwise: key switching fused into a thin FP64 MAC (M <= 2 rows)
  HY_MAC_TC_FUSED = 1,    // dense, M <= 128: key switching in the producers of the tcgen05 MAC
  HY_MAC_TC_SPLIT = 2,    // dense, M > 128: PermAuto materialises R, tcgen05 MAC consumes it
  HY_MAC_FP64_FUSED = 3,  // A/B option HY_MAC_FP64 (M <= 32): key switching + FP64 DFMA MAC
  HY_MAC_FP64_SPLIT = 4,  // A/B option HY_MAC_FP64 (M > 32): PermAuto + FP64 DFMA MAC
  HY_MAC_TC_COEF = 5,     // 1x1: tcgen05 MAC straight on the coefficient-form inputs (c_n = 1: no NTT;
                          // c_n = 2: only the row-swap alignment's NTTs)
  HY_MAC_EAGER = 6,       // ablation "lazy reduction off" (Fig. 4 (d)): PermAuto + a MAC reducing every term
  HY_MAC_DIRECT = 7,      // ablation "hoisting off" (Fig. 4 (b)): every rotation decomposes again, tcgen05 MAC
};
int hy_mac_path(int M, int L, bool depthwise, bool coef_ok, int cn, bool subdigits);

struct hy_weights {
  hy_params* p;
  int mac_path;     // HyMacPath
  hy_conv_shape shape;
  hy_layout lay;
  int M;            // MAC rows per unit
  int K;            // MAC depth per unit (Jc*T dense; T depthwise)
  int wblocks;      // number of distinct weight blocks (1 dense, Jc depthwise)
  int Mpad, Kpad;   // M rounded up to the row tile, K rounded up to the MAC chunk
  double* d_wt;     // [wblocks][Kpad][Mpad] weights (exact small integers), zero padded
  int32_t* d_kt;    // [ceil(Kpad/64)*64] K term -> (tap << 16) | input ct (-1 = padding): the fused
                    // tensor-core MAC's term table (no integer division in its producers)
  int8_t* d_w8;     // [wblocks][Mpad/128][Kpad/32][4096]: weights as int8 in the tcgen05 K-major
                    // no-swizzle canonical layout (tensor-core MAC), zero padded
  u64* d_sign;      // [L][N] NTT form of the [k,-k] plaintext, then [L][N] Shoup companions (c_n = 4:
                    // [3][2][L][N] for the dense Hadamard rows 1..3)
  // workspace (device)
  u64* d_D;         // [U*Jc][L digit][L limb][N] NTT-form digits
  u64* d_C0;        // [U*Jc][L][N]    NTT(c0)
  u64* d_P;         // [U*Jo][cn'][2][L][N] partial sums (NTT form)
  u64* d_D2;        // [U*Jo][L][L][N] digits of P_{g,1}.c1 for the row swap
  u64* d_X;         // [U*Jo][2][L][N] aligned outputs (NTT form) before the final INTT
  u64* d_A1;        // [U*Jo][2][2][L][N] [A1] of the coefficient-domain c_n = 2 1x1 path
  u64* d_R;         // [r_units][K][2][L][N] rotated inputs of the dense path (slot-order NTT)
  u64* d_wq;        // HY_MAC_EAGER: [L][Kpad][Mpad] weights mod q_l, then the same block of Shoup companions
  int r_units;      // units per PermAuto + MAC batch
  cudaStream_t s_h2d, s_d2h;   // hy_conv_eval_host copy streams (created on first use)
  cudaEvent_t ev_h2d, ev_comp;
  u64* d_in;        // staging for hy_conv_eval_host
  u64* d_out;
  u64** d_tap_keys;            // device array of key pointers per tap (nullptr = identity)
  u64* h_tap_keys[HY_MAX_TAPS];       // the same tables on the host (passed by value to kernels)
  GaloisAct h_tap_act[HY_MAX_TAPS];
  GaloisAct* d_tap_act;        // device array of slot-order automorphism actions per tap
  u64* d_swap_key;
  u64* d_align_key[3];         // c_n = 4: keys of the alignment automorphisms g_1, g_2, g_3
  GaloisAct h_align_act[3];
  u64 keys_version;            // params->keys_version the tap table was built from
  cudaEvent_t ev[4];           // optional stage-boundary events (bench)
  uint32_t n_ev;
  // per-launch timing of the MAC kernel (enabled with the stage events): event pairs around each
  // MAC launch of the last hy_conv_eval
  std::vector<cudaEvent_t>* mac_ev;
  uint32_t mac_launches;
};

// ------------------------------------------------------------------------------------
// programmatic dependent launch: every kernel of the hy_conv_eval chain lets its successor
// launch as soon as all its CTAs are resident, and waits for its predecessor's completion (and
// memory) before touching the predecessor's outputs.  Both are no-ops for a normal launch.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_begin() {
  pdl_trigger();
  pdl_wait();
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device-context attribute: set it once per
// (kernel, device) to at least `bytes` (thread-safe; api.cu keeps the cache behind a mutex)
cudaError_t hy_smem_attr(const void* kernel, size_t bytes);

// launch with cudaLaunchAttributeProgrammaticStreamSerialization (optionally in clusters of cx)
template <typename... KArgs, typename... Args>
inline cudaError_t hy_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cx,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[n].val.programmaticStreamSerializationAllowed = 1;
  n++;
  if (cx > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cx;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    n++;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

// ------------------------------------------------------------------------------------
// device modular arithmetic
// ------------------------------------------------------------------------------------
__device__ __forceinline__ u64 shoup_mul(u64 x, u64 w, u64 w_sh, u64 q) {
  // x * w mod q in [0, 2q) for any 64-bit x (Shoup; w < q, w_sh = floor(w 2^64 / q)).
  u64 hi = __umul64hi(x, w_sh);
  return x * w - hi * q;
}

// hi64(x w) without the x0 w0 partial product and the low halves of the cross products:
// x1 w1 + hi32(x1 w0) + hi32(x0 w1), which is below the exact high word by at most 3 (the dropped
// parts sum to < 3 * 2^64).  In a Shoup product the quotient then undershoots by <= 3, so
// x w - h q lies in [0, 5q) instead of [0, 2q).  One IMAD.WIDE + two IMAD.HI instead of the four
// partial products of __umul64hi (tools/mmbench: +16% key-switching products per clock).
__device__ __forceinline__ u64 umulhi_apx(u64 x, u64 w) {
  const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), w0 = (uint32_t)w, w1 = (uint32_t)(w >> 32);
  return (u64)x1 * w1 + __umulhi(x1, w0) + __umulhi(x0, w1);
}

__device__ __forceinline__ u64 csub(u64 x, u64 m) { return x >= m ? x - m : x; }

// canonical residue of a lazy sum x < (2L + 1) q (c0 + L Shoup products, each in [0, 2q)):
// log2 conditional subtractions instead of one per term (q < 2^60, L <= 7 keeps x < 16 q)
template <int LT>
__device__ __forceinline__ u64 reduce_lazy_sum(u64 x, u64 q) {
  if constexpr (2 * LT + 1 > 8) x = csub(x, 8 * q);
  if constexpr (2 * LT + 1 > 4) x = csub(x, 4 * q);
  x = csub(x, 2 * q);
  return csub(x, q);
}

// x in [0, 2^64): x mod q in [0, 2q)  (Shoup with w = 1)
__device__ __forceinline__ u64 reduce_2q(u64 x, u64 one_sh, u64 q) { return x - __umul64hi(x, one_sh) * q; }

// full 64x64 -> mod q, both operands < 2^64 and w arbitrary (no precomputation): slow path.
__device__ __forceinline__ u64 mulmod_slow(u64 a, u64 b, u64 q) {
  u128 p = (u128)a * b;
  return (u64)(p % q);
}

// ------------------------------------------------------------------------------------
// host helpers (library-internal)
// ------------------------------------------------------------------------------------
namespace hyhost {
u64 mulmod(u64 a, u64 b, u64 m);
u64 powmod(u64 a, u64 e, u64 m);
u64 invmod(u64 a, u64 m);
bool is_prime(u64 n);
u64 shoup(u64 w, u64 q);
uint32_t bitrev(uint32_t x, uint32_t bits);
}  // namespace hyhost

// kernels API (internal)
namespace hyk {
// forward NTT of n jobs; job table decides sources
hy_status ntt_poly_fwd(const hy_params* p, const u64* src, u64* dst, size_t npoly, cudaStream_t s);  // [n][L][N]
hy_status ntt_poly_inv(const hy_params* p, const u64* src, u64* dst, size_t npoly, cudaStream_t s);  // [n][L][N]
hy_status pointwise_mul(const hy_params* p, const u64* a, const u64* b, u64* c, size_t npoly, cudaStream_t s);
hy_status shoup_table(const hy_params* p, const u64* w, u64* w_sh, size_t npoly, cudaStream_t s);  // [n][L][N]
hy_status key_to_ntt(const hy_params* p, const u64* key_coeff, u64* key_ntt, cudaStream_t s);
hy_status permdecomp(const hy_params* p, const u64* ct, size_t nct, u64* D, u64* C0, cudaStream_t s);
hy_status ksmac(hy_weights* w, const u64* ct_in, size_t nunits, cudaStream_t s);  // S2 + S3
hy_status c0_only(const hy_params* p, const u64* ct, size_t nct, u64* C0, cudaStream_t s);  // NTT(c0) per limb
hy_status finish_outputs(const hy_weights* w, size_t nunits, u64* ct_out, cudaStream_t s);
hy_status mac_coef(hy_weights* w, const u64* ct_in, size_t nunits, u64* ct_out, cudaStream_t s);
hy_status finish_coef2(const hy_weights* w, size_t nunits, u64* ct_out, cudaStream_t s);
hy_status rotate_ct(const hy_params* p, const u64* ct_in, GaloisAct act, const u64* key, u64* ct_out, size_t n,
                    u64* work, cudaStream_t s);
hy_status decrypt_phase(const hy_params* p, const u64* s_ntt, const u64* s_ntt_sh, const u64* ct, size_t n,
                        u64* x_out, u64* work, cudaStream_t st);
hy_status client_secret(const hy_params* p, u64 seed, int8_t* sk8_dev, u64* s_res, u64* s_ntt, cudaStream_t st);
hy_status client_encrypt(const hy_params* p, u64 seed, const u64* s_ntt, const u64* m_dev, const uint32_t* idx_dev,
                         size_t n, const u64* delta_l, u64* ct_out, u64* work, cudaStream_t st);
hy_status client_keygen(const hy_params* p, u64 seed, const u64* s_ntt, const int8_t* sk8_dev, const uint32_t* elts_dev,
                        size_t n_elts, u64* keys_out, u64* work, cudaStream_t st);
}  // namespace hyk
