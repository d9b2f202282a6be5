/*
 * hyena.h — C-ABI of the B200 (sm_100a) implementation of the server-side hot path of
 * "Hyena: Optimizing Homomorphically Encrypted Convolution for Private CNN Inference"
 * (arXiv 2311.12519; /root/reference/PAPER.md).
 *
 * The server receives input ciphertexts, holds switching keys for HRot and model weights
 * prepared offline, and returns output ciphertexts packing the output channels
 * (PAPER.md:883-884, 1590-1594).  The calls below follow that problem statement.
 *
 * Conventions for every call:
 *   - Status codes only (hy_status); no C++ exception crosses the ABI.  On failure the
 *     thread-local message hy_last_error() says why.
 *   - Ciphertexts are BFV pairs (c0, c1) over Q = prod q_l (RNS, L limbs), ring
 *     Z_q[X]/(X^N+1) (PAPER.md:276-280 [\ignore]), stored limb-major uint64
 *     [2][L][N] in COEFFICIENT form with canonical residues in [0, q_l)
 *     (reading R18) — both on input and on output.
 *   - Ciphertext buffers are caller-owned device memory (e.g. torch tensors); the library
 *     never frees them.  Handles are opaque and owned by the library.
 *   - Params, keys and weights are immutable after creation, except that a hy_weights
 *     owns the workspace of hy_conv_eval: one evaluation at a time per hy_weights.
 *   - Device calls are stream-ordered on the given cudaStream_t (void*; NULL = legacy
 *     default stream) and do not synchronise the host except where stated.
 */
#ifndef HYENA_H_
#define HYENA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hy_status;
#define HY_OK 0
#define HY_EINVAL (-1)  /* bad argument (non-prime modulus, N not a power of two, ...) */
#define HY_ENOMEM (-2)  /* device or host allocation failed */
#define HY_ECUDA (-3)   /* a CUDA runtime call or kernel launch failed */
#define HY_ENOKEY (-4)  /* a Galois key the layout needs was not uploaded */
#define HY_ESHAPE (-5)  /* ciphertext counts / shapes do not match the layout */
#define HY_ENOISE (-6)  /* hy_decrypt_debug: a coefficient's noise budget is below 1 bit */

#define HY_MAX_LIMBS 8
#define HY_MAX_TAPS 49     /* kernels up to 7x7 */
#define HY_MAX_GALOIS 64

typedef struct hy_params hy_params;
typedef struct hy_weights hy_weights;

/* One convolution layer: stride 1, zero padding `pad`, cross-correlation
 * out[b,o,y,x] = sum_{c,dy,dx} W[o,c,dy,dx] x[b,c,y+dy-pad,x+dx-pad].
 * depthwise != 0: W is [C][kh][kw] and output channel o reads input channel o only.
 * k = 0 selects the paper's k (argmin_{1<=k<=32} |[k h]_t|; reading R13);
 * force_cn = 0 chooses c_n automatically (reading R10), else 1, 2 or 4 (4: four channels per
 * ciphertext, Walsh-Hadamard-4 packing of PAPER.md:565-572; one unit of N/4-slot groups, dense layers,
 * FP64 MAC paths, output scale 4). */
typedef struct {
  uint32_t Ci, Co, H, W, kh, kw, pad, stride, depthwise, batch;
  int32_t k, force_cn;
} hy_conv_shape;

/* Layout chosen for a layer (readings R8-R10, R15):
 *   Wp = next_pow2(W + 2 pad), Hp = next_pow2(H + 2 pad);
 *   mode 0 ("blocks"): per_row images of Hp x Wp per slot row (N/2 slots);
 *   mode 1 ("bands"):  Hb = (N/2)/Wp rows per band, Hv = Hb - (kh-1) valid rows,
 *                      `bands` bands per image (halo rows duplicated by the client);
 *   G slot-row groups per channel; cn channels per ciphertext (1 or 2);
 *   U independent units, each with Jc input and Jo output ciphertexts
 *   (cn = 2: input ct u*Jc + j holds channels 2j (row 0) and 2j+1 (row 1) of group u;
 *    cn = 1: input ct u*Jc + c holds channel c, groups 2u (row 0) and 2u+1 (row 1));
 *   taps (dy, dx) row-major with left-rotation step (dy-pad)*Wp + (dx-pad);
 *   output slots = (c_n k) * conv (scale), remove with scale^{-1} mod t (reading R12);
 *   galois[] = Galois elements whose keys hy_conv_eval needs (taps, then row swap). */
typedef struct {
  uint32_t N, L;
  uint32_t Hout, Wout, Wp, Hp, mode, per_row, Hb, Hv, bands, G, cn, U, Jc, Jo, J, Jout;
  uint32_t n_taps;
  int32_t tap_dy[HY_MAX_TAPS], tap_dx[HY_MAX_TAPS], tap_step[HY_MAX_TAPS];
  uint32_t k, scale, h;
  int32_t sign_coeff;           /* centered [k h]_t: the [k,-k] plaintext's two coefficients */
  uint32_t n_galois;
  uint32_t galois[HY_MAX_GALOIS];
} hy_layout;

/* Storage / communication accounting of a layer (Table 2 :833-872,
 * Table 3 :917-919, storage example :561-562).  Byte counts use 8-byte words and L limbs.
 *   input_ct_bytes / output_ct_bytes: this layout's J / Jout ciphertexts (2 L N words each): what
 *       the client sends and receives;
 *   input_ct_bytes_paper: the paper's count ceil(Ci Wp Hp / (N / ... )) = ceil(Ci Wp^2 / N)
 *       ciphertexts (channels packed back to back, no halo rows);
 *   model_bytes_paper: the proposed method's model, one 64-bit integer per kernel element
 *       (PAPER.md:557-562), plus one N-word sign plaintext when c_n = 2 (the :561 example) or three
 *       dense Hadamard-row plaintexts when c_n = 4;
 *   model_bytes_conventional: one N-word plaintext per kernel element;
 *   model_bytes_device: what hy_encode_weights keeps on the GPU for the weights (int8 + FP64 tables,
 *       sign / Hadamard-row plaintexts in NTT form with Shoup companions);
 *   key_bytes: the n_keys switching keys (ND x 2 x L x N words each, coefficient form);
 *   rotations: hoisted rotations per evaluation (input cts x non-identity taps) plus alignment
 *       rotations (c_n = 2: one per output ct; c_n = 4: three);
 *   coef_macs: coefficient-level multiply-accumulates of the lazy MAC (S3). */
typedef struct {
  uint64_t input_ct_bytes, output_ct_bytes, input_ct_bytes_paper;
  uint64_t model_bytes_paper, model_bytes_conventional, model_bytes_device;
  uint64_t key_bytes;
  uint32_t n_keys, rotations;
  uint64_t coef_macs;
} hy_accounting;

/* Host-only: accounting of a planned layout (hy_plan_layout) for L limbs and ND key digits
 * (ND = L, or L V with a sub-digit base).  Errors: HY_EINVAL. */
hy_status hy_layout_accounting(const hy_layout* lay, const hy_conv_shape* shape, uint32_t L, uint32_t ND,
                               hy_accounting* out);

/* Noise-driven decomposition-base selection (SURVEY §8(f) NEXT-4; PAPER.md:587-617, :1470 [app]).
 * hy_noise_estimate: host-only heuristic estimate of log2 ||v||_inf of one layer's output noise for a
 *   key-switching base 2^w_dcmp (0: one digit per limb) and weights |w| <= w_max, and the budget
 *   log2(Delta / 2); model in api.cu (one HRot, lazy MAC, c_n = 2 [k, -k] / c_n = 4 dense PMults,
 *   alignment), calibrated against the oracle's noise meter.
 * hy_select_dcmp_base: the base with the FEWEST digits (largest base) whose estimate leaves
 *   margin_bits below the budget: w_dcmp = 0 when one digit per limb suffices.
 * Errors: HY_EINVAL (bad shape, no base meets the margin). */
hy_status hy_noise_estimate(uint32_t N, const uint64_t* q_primes, uint32_t L, uint64_t t, const hy_conv_shape* shape,
                            uint32_t w_max, uint32_t w_dcmp, double* log2_noise, double* log2_budget);
hy_status hy_select_dcmp_base(uint32_t N, const uint64_t* q_primes, uint32_t L, uint64_t t,
                              const hy_conv_shape* shape, uint32_t w_max, double margin_bits, uint32_t* w_dcmp);

/* Thread-local message describing the last failing call ("" if none). */
const char* hy_last_error(void);

/* Host-only layout planner (no device needed).  t is the plaintext modulus.
 * Errors: HY_EINVAL (N not a power of two in [16, 65536], t not prime or t != 1 mod 2N),
 * HY_ESHAPE (stride != 1, kernel larger than the padded input, a band shorter than the
 * kernel, too many taps). */
hy_status hy_plan_layout(uint32_t N, uint64_t t, const hy_conv_shape* shape, hy_layout* out);

/* Create ring parameters on CUDA device `device` (PAPER.md:611 step 1: q = p = 1 mod 2N).
 * q_primes[L] (host): distinct primes 2^20 < q_l < 2^60, q_l = 1 mod 2N; t prime, t = 1 mod 2N,
 * t not among q_l; N a power of two in [1024, 16384]; 1 <= L <= HY_MAX_LIMBS.
 * Builds the per-limb Shoup twiddle tables (bit-reversed psi powers), the plaintext slot
 * tables (zeta_t = least primitive 2N-th root mod t; reading A1) and uploads them.
 * Errors: HY_EINVAL, HY_ENOMEM, HY_ECUDA.  *out is set only on success. */
hy_status hy_params_create(uint32_t N, const uint64_t* q_primes, uint32_t L, uint64_t t, int device,
                           hy_params** out);
/* Same, with a decomposition base 2^w_dcmp INSIDE each RNS limb for the switching keys (SURVEY §8(f)
 * NEXT-4; PAPER.md:1470 [app] "decomposition base"; smaller digits = less key-switching noise, e.g.
 * for the dense Hadamard-row plaintexts of c_n = 4): w_dcmp = 0 is hy_params_create (one digit per
 * limb, reading R5); else 4 <= w_dcmp < bit length of the smallest q_l, and every key has
 * ND = L ceil(max bits / w_dcmp) digits, digit i V + v = floor([c1]_{q_i} / 2^{w v}) mod 2^w with
 * gadget residue [i == l] 2^{w v} mod q_l (the oracle's bfv.galois_keygen).  The tensor-core fused
 * MAC (one digit per limb) is not used with a sub-digit base.  Errors as hy_params_create. */
hy_status hy_params_create2(uint32_t N, const uint64_t* q_primes, uint32_t L, uint64_t t, uint32_t w_dcmp, int device,
                            hy_params** out);
void hy_params_destroy(hy_params* p);

/* Upload server-side switching keys generated by the client (PAPER.md:883-884, 1474-1475 [app]).
 * keys: [n_elts][ND digits][2: b, a][L limbs][N] uint64, COEFFICIENT form, canonical residues
 * (ND = L, or L V with a sub-digit base: hy_params_create2);
 * key for element g satisfies b_{i,l} + a_{i,l} s = e_i + [i == l] s(X^g)  (mod q_l)
 * (RNS-digit gadget, reading R5).  keys_on_device != 0: `keys` is a device pointer.
 * The library converts them to NTT form with Shoup companions and keeps its own copy;
 * re-uploading an element replaces it.  Synchronises the device.  Errors: HY_EINVAL
 * (even or out-of-range element, too many elements), HY_ENOMEM, HY_ECUDA. */
hy_status hy_keys_upload(hy_params* p, uint32_t n_elts, const uint32_t* galois_elts, const uint64_t* keys,
                         int keys_on_device);

/* Prepare one layer: plans the layout, picks k, builds the
 * [k, -k] sign plaintext ([k h]_t at X^{N/4} and X^{3N/4}, centered lift)
 * in NTT form, and the int weight tables; allocates the evaluation workspace for U units.
 * W (host, int8): [Co][Ci][kh][kw], or [C][kh][kw] when depthwise.
 * Errors: HY_EINVAL, HY_ESHAPE, HY_ENOMEM, HY_ECUDA.  Synchronises the device. */
hy_status hy_encode_weights(hy_params* p, const hy_conv_shape* shape, const int8_t* W, hy_weights** out);
hy_status hy_weights_layout(const hy_weights* w, hy_layout* out);
void hy_weights_destroy(hy_weights* w);

/* The encrypted convolution (CNNLayer/ProposedConv):
 * hoisted rotations of every input ciphertext by every tap step (PermDecomp + PermAuto),
 * lazy multiply-accumulate of the int weights with one reduction per output
 * (PAPER.md:718-728), Walsh-Hadamard butterflies + [k,-k] PMult for c_n = 2 (Eq. 2,
 * PAPER.md:532-560), alignment of diagonal 1 by the row-swap HRot,
 * and the return to coefficient form.
 * ct_in: device [J][2][L][N] with J = nu * Jc for 1 <= nu <= U units (unit-major, see
 * hy_layout); ct_out: device [Jout][2][L][N], Jout = nu * Jo.  Output slots hold
 * scale * conv (mod t).  Stream-ordered, no host sync.  Errors: HY_ESHAPE, HY_ENOKEY,
 * HY_ECUDA. */
hy_status hy_conv_eval(hy_weights* w, const uint64_t* ct_in, size_t J, uint64_t* ct_out, size_t Jout,
                       void* cuda_stream);

/* Same computation from/to HOST buffers (pinned or pageable): copies ct_in to the device,
 * evaluates, copies ct_out back, and returns when the outputs are in host memory.  Pipelined over
 * batches of whole units (up to 8 batches) on two library-owned copy streams, so uploads and
 * downloads overlap the evaluation (pinned buffers needed for the overlap).  J, Jout as for
 * hy_conv_eval.  Errors: HY_ESHAPE, HY_ENOKEY, HY_ECUDA. */
hy_status hy_conv_eval_host(hy_weights* w, const uint64_t* ct_in_host, size_t J, uint64_t* ct_out_host,
                            size_t Jout, void* cuda_stream);

/* Per-stage entry points (for per-kernel parity tests; same kernels as hy_conv_eval).
 * hy_poly_mul: c = a * b in Z_{q_l}[X]/(X^N+1) for n polynomial pairs, all device
 *   [n][L][N] coefficient form (forward NTT, pointwise Shoup product, inverse NTT).
 * hy_ntt_roundtrip: x -> INTT(NTT(x)) in place, device [n][L][N] (synchronises the stream).
 * hy_rotate: hoisted HRot of n ciphertexts by Galois element g (key must be uploaded):
 *   device [n][2][L][N] -> device [n][2][L][N], coefficient form. */
hy_status hy_poly_mul(const hy_params* p, const uint64_t* a, const uint64_t* b, uint64_t* c, size_t n,
                      void* cuda_stream);
hy_status hy_ntt_roundtrip(const hy_params* p, uint64_t* x, size_t n, void* cuda_stream);
hy_status hy_rotate(hy_params* p, const uint64_t* ct_in, uint32_t galois_elt, uint64_t* ct_out, size_t n,
                    void* cuda_stream);

/* Measurement hooks (bench.py): total number of kernels this library has launched in the
 * process, and optional CUDA events (cudaEvent_t cast to void*, at most 4) that hy_conv_eval
 * records on its stream at the stage boundaries [before S1, after S1, after the fused S2+S3,
 * after S4+S5].  n = 0 clears them.  Errors: HY_EINVAL. */
uint64_t hy_kernel_launches(void);
hy_status hy_weights_set_stage_events(hy_weights* w, void* const* events, uint32_t n);
/* While stage events are set, hy_conv_eval also brackets every launch of its MAC kernel (the
 * fused S2+S3 kernel, or each batch of the MAC GEMM) with library-owned events; this returns the
 * summed device time of those launches in the last evaluation and their count (synchronises on
 * the last one).  Errors: HY_EINVAL, HY_ECUDA. */
hy_status hy_weights_mac_time(const hy_weights* w, float* total_ms, uint32_t* launches);

/* Kernel choice for S2 + S3, fixed by hy_encode_weights from the layout:
 *   0 HY_MAC_THIN        depthwise: key switching fused into a thin FP64 MAC;
 *   1 HY_MAC_TC_FUSED    dense, 32 < M <= 128 MAC rows, L in {2,3,5}: key switching in the producer
 *                        warps of the tcgen05 int8 MAC (rotated inputs never stored);
 *   2 HY_MAC_TC_SPLIT    dense: PermAuto materialises the rotated inputs, tcgen05 MAC reads them;
 *   3 HY_MAC_FP64_FUSED  dense, M <= 32 (default there): key switching + FP64 DFMA MAC (30-bit halves);
 *   4 HY_MAC_FP64_SPLIT  dense, M > 32: PermAuto + FP64 DFMA MAC;
 *   5 HY_MAC_TC_COEF     1x1 kernel, pad 0, c_n = 1: tcgen05 MAC directly on the coefficient-form
 *                        inputs (identity tap, linear MAC), no NTT / INTT at all;
 *   6 HY_MAC_EAGER       ablation "lazy reduction off" (Fig. 4 (d) vs (e), :718-728): PermAuto +
 *                        a MAC that reduces after every product and addition (same residues);
 *   7 HY_MAC_DIRECT      ablation "hoisting off" (Fig. 4 (b), :373-378): every rotation decomposes the
 *                        rotated c1 again (its bits are the direct HRot's, not the hoisted one's:
 *                        oracle bfv.rotate_direct), then the tcgen05 MAC.
 * 6 and 7 are never chosen automatically (c_n <= 2, dense layers).
 * Every path computes the same bits (the MAC is exact integer arithmetic).  set_mac_path selects
 * another valid path for A/B measurement and parity tests (allocates the rotated-input workspace
 * of the split paths).  Errors: HY_EINVAL (path not valid for this layout), HY_ENOMEM. */
hy_status hy_weights_mac_path(const hy_weights* w, int32_t* path);
hy_status hy_weights_set_mac_path(hy_weights* w, int32_t path);

/* Debug decryption (PAPER.md:256-267 [\ignore]): for each of n device ciphertexts
 * [n][2][L][N] computes [c0 + c1 s]_{q_l} on the GPU, then on the host the exact CRT
 * rounding m = [round(t x / Q)]_t, slot decoding and multiplication by
 * scale^{-1} mod t.  sk: host ternary int8 [N].  slots_out: host [n][N] in slot order
 * (row 0 slots 0..N/2-1, then row 1).  Not on the hot path; synchronises the device. */
hy_status hy_decrypt_debug(const hy_params* p, const int8_t* sk, const uint64_t* ct, size_t n, uint32_t scale,
                           uint64_t* slots_out);
/* As hy_decrypt_debug, and reports each ciphertext's invariant noise budget (PAPER.md:266-267
 * [\ignore]: decryption is correct while the noise stays below Delta / 2): budget_bits[o] = min over
 * coefficients of log2(Q / |2 (t x - round(t x / Q) Q)|) = log2(1 / (2 |v|)) with v = t x / Q - m the
 * invariant noise (budget_bits may be NULL).  Both return HY_ENOISE, after writing slots_out, when
 * some coefficient has less than 1 bit left (|v| > 1/4: the decrypted value is not trustworthy). */
hy_status hy_decrypt_debug_noise(const hy_params* p, const int8_t* sk, const uint64_t* ct, size_t n, uint32_t scale,
                                 uint64_t* slots_out, double* budget_bits);

/* Client-side draws on the GPU (symmetric BFV encryption PAPER.md:242-253
 * [\ignore], keys of reading R5).  Every random number comes from Philox4x32-10 keyed by `seed`, with
 * the counter layout and value mappings documented in synth/philox.py (ternary secret, centered
 * binomial eta = 20 errors, uniform masks), so the CPU oracle reproduces each call bit for bit.
 * All three synchronise the device and allocate their own scratch.
 * hy_secret_key: the ternary secret s of `seed`, host int8 [N] (for hy_decrypt_debug).
 * hy_keygen:     switching keys for n Galois elements (odd, < 2N), [n][L digits][2: b, a][L limbs][N]
 *                coefficient form: b_{i,l} = [-a_{i,l} s + e_i + [i == l] s(X^g)]_{q_l}.  keys_out: device
 *                buffer or NULL; upload != 0 also installs them (hy_keys_upload).
 * hy_encrypt:    ct_j = ([Delta m_j + a_j s + e_j]_{q_l}, [-a_j]_{q_l}), Delta = floor(Q/t), for the n
 *                plaintexts m (host [n][N], coefficients in [0, t)) with encryption counters
 *                first .. first + n - 1; ct_out device [n][2][L][N] coefficient form.
 * Errors: HY_EINVAL (bad element / coefficient), HY_ENOMEM, HY_ECUDA. */
hy_status hy_secret_key(const hy_params* p, uint64_t seed, int8_t* sk_out);
hy_status hy_keygen(hy_params* p, uint64_t seed, uint32_t n, const uint32_t* galois_elts, uint64_t* keys_out,
                    int upload);
hy_status hy_encrypt(const hy_params* p, uint64_t seed, const uint64_t* m, size_t n, uint32_t first,
                     uint64_t* ct_out, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* HYENA_H_ */
