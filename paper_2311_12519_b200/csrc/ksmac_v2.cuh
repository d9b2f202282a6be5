// Persistent, warp-specialised fused S2 + S3 on the tensor cores (included by kernels.cu after
// the definitions it uses: KsMacArgs, tc_store4, byte_tr4, umma_*, mbar_*, galois_perm).
//
// What it computes is exactly ksmac_tc_kernel's: for every output row m and
// column (component, limb l, slot position j) of a unit z,
//   B[m][col] = sum_{kk = tau Jc + c} w[m][kk] R_{c,tau}[col],
//   R_{c,tau}.c0[j] = C0_c[perm_tau(j)] + sum_i D_{c,i}[perm_tau(j)] b_{tau,i}[j],
//   R_{c,tau}.c1[j] =                     sum_i D_{c,i}[perm_tau(j)] a_{tau,i}[j]
// (hoisted PermAuto; lazy: Shoup products in [0, 2q), no reduction of R), as an
// exact int8 byte-plane contraction on tcgen05 (s8 weights x u8 planes -> s32 TMEM), then the
// Walsh-Hadamard epilogue with ONE reduction per output coefficient.
//
// Organisation (one CTA per SM, 17 warps):
//   * warps 0-11  producers: per 96-term chunk, each thread key-switches 4 consecutive terms of one
//                 slot position, byte-transposes them into the 8 planes of a shared-memory stage and
//                 arrives on the stage's FULL mbarrier; the next chunk's digit reads are in flight
//                 (register double buffer) while the current one is switched;
//   * warp 12     the ONLY UMMA issuer: waits FULL[s], issues the chunk's 3 UMMAs (M = 128, N = 256,
//                 K = 32) into the tile's TMEM accumulator, commits to EMPTY[s]; after a tile's last
//                 chunk it commits to TFULL[b].  In-order issue from one thread: the first UMMA of a
//                 tile overwrites (no TMEM zeroing), every later one accumulates;
//   * warps 13-16 epilogue: wait TFULL[b], read TMEM (warp w: lanes 32 (w mod 4) ..), recombine the
//                 planes, WHT + one reduction + sign PMult, store P, arrive TEMPTY[b].
//   TMEM holds two 256-column accumulators, so the epilogue of tile i overlaps the main loop of
//   tile i + 1.  Tiles = (unit z, limb l, 16 positions), z-major, dealt round-robin to the
//   persistent CTAs (every resident CTA works on the same unit: its digits stay in L2).  The
//   weights (128 x Kpad int8) stay resident in shared memory when they fit; the key words of the
//   next tile are prefetched with cp.async into the other half of a double buffer.
#pragma once

// A/B switches (tools/abbuild.py builds variants with -D; the defaults are the measured best)
#ifndef V2_PREFETCH
#define V2_PREFETCH 0
#endif
#ifndef V2_BACKOFF
#define V2_BACKOFF 0
#endif
#ifndef V2_PTX
#define V2_PTX 1
#endif
#ifndef V2_PF
#define V2_PF 0
#endif
#ifndef V2_SMAX
#define V2_SMAX 2
#endif
#ifndef V2_KBMAX
#define V2_KBMAX 3
#endif

#ifndef V2_PW
#define V2_PW 16
#endif
#ifndef V2_WRES  // 0: never keep the weights resident (experiment: more L1 for the digit windows)
#define V2_WRES 1
#endif
#ifndef V2_PAD   // extra shared memory requested (experiment: less L1)
#define V2_PAD 0
#endif
#ifndef V2_KBCONST
#define V2_KBCONST 1
#endif
#ifndef V2_SHFL  // warp index through __shfl_sync (provably warp-uniform role branches)
#define V2_SHFL 1
#endif
#ifndef V2_HALF  // M <= 64: resident weights as 64-row half tiles (more L1 for the digit windows)
#define V2_HALF 1
#endif
// producer warps (a multiple of 4): 16 slot positions x 2 PW term groups of 4 per chunk
constexpr int V2_PROD_WARPS = V2_PW, V2_PROD = V2_PROD_WARPS * 32;
constexpr int V2_KS = V2_PW / 4, V2_CHUNK = 32 * V2_KS;     // PW = 12: 96 terms = 3 UMMA K steps per chunk
constexpr uint32_t V2_STAGE_B = V2_KS * 8 * 1024;           // 8 planes x 32 columns x 32 terms per K step
constexpr uint32_t V2_STAGE_A = V2_KS * 4096;               // streamed weights: 128 rows x 32 terms per K step
constexpr uint32_t V2_TMEM_COLS = 512;
// warps: 0-11 producers, 12 .. 12 + EPI - 1 epilogue (TMEM lane quadrant = warp % 4), 12 + EPI the
// UMMA issuer.  EPI = 2 when M <= 64 (two live lane quadrants): 15 warps, 128 registers per thread
// (4 warps per SM sub-partition); EPI = 4: 17 warps, 96 registers.
template <int EPI>
struct V2Warps {
  static constexpr int MMA = V2_PROD_WARPS + EPI;
  static constexpr int THREADS = (V2_PROD_WARPS + EPI + 1) * 32;
};

struct V2Geom {
  int S;                 // pipeline stages
  int wres;              // 1: all weights resident in shared memory
  int half;              // 1: resident weights hold rows 0..63 only (M <= 64), 2048 bytes per K step
  int kb;                // key buffers (3 or 4; keys are prefetched two tiles ahead)
  uint32_t off_b, off_a, off_key, off_bar;
  uint32_t key_bytes;    // one key buffer
  size_t bytes;          // dynamic shared memory to request (incl. 1024-byte alignment slack)
};

// largest configuration that fits, preferring resident weights, then 4 stages, then 4 key buffers
// (with 4, the buffer a tile's keys are copied into was last read two tiles earlier: the producer
// warps, which the stage ring keeps within S < one tile of each other, never wait for it)
// M <= 64 (V2_HALF): only the 64 live weight rows are kept (rows 0..63 of a canonical 128 x 32 tile are
// its first 2048 bytes); the M = 128 UMMA of K step k then reads K step k + 1's rows as its rows
// 64..127 (the last step reads 2 KB of the stage ring): those accumulator lanes are never read
inline V2Geom v2_geom(int T, int L, int Kpad, size_t smem_max, int M = 128) {
  V2Geom g{};
  g.half = V2_HALF && M <= 64;
  const uint32_t wbytes = (g.half ? 64u : 128u) * (uint32_t)Kpad;
  g.key_bytes = (uint32_t)T * 4 * L * TC_POS * 8;
  const uint32_t bar = 256;
  for (int wres = V2_WRES; wres >= 0; wres--) {
    for (int S = V2_SMAX; S >= 2; S--) {
      for (int kb = V2_KBMAX; kb >= V2_KBMAX; kb--) {  // exactly V2_KBMAX buffers (compile-time count in the kernel)
        const uint32_t w = wres ? wbytes : 0;
        const uint32_t per = V2_STAGE_B + (wres ? 0 : V2_STAGE_A);
        const size_t tot = 1024 + (size_t)w + (size_t)S * per + (size_t)kb * g.key_bytes + bar + V2_PAD;
        if (tot <= smem_max) {
          g.S = S;
          g.wres = wres;
          if (!wres) g.half = 0;
          g.kb = kb;
          g.off_b = w;
          g.off_a = w + S * V2_STAGE_B;
          g.off_key = g.off_a + (wres ? 0 : S * V2_STAGE_A);
          g.off_bar = g.off_key + kb * g.key_bytes;
          g.bytes = tot;
          return g;
        }
      }
    }
  }
  g.S = 0;
  return g;
}

__device__ __forceinline__ void v2_cp16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(g) : "memory");
}
// mbarrier wait that SUSPENDS the warp until the phase completes (try_wait with a suspend-time hint)
// instead of polling: the epilogue and UMMA-issuer warps idle most of the time and their polling took
// a quarter of the issue slots (profiled); the producers' waits use it too
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, int /*ns*/) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)
        : "memory");
  }
}

// mbarrier wait with an explicit nanosleep back-off between polls: for the warps that idle most of
// a tile (epilogue, UMMA issuer); the suspend hint of mbar_wait_sleep returns within ~30 ns, so those
// warps polled ~10^8 times per C4 layer (profiled: 17% of all issued instructions were wait loops)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity, uint32_t ns) {
  if (!V2_BACKOFF) return mbar_wait_sleep(b, parity, (int)ns);
  uint32_t done = 0;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (done) return;
    __nanosleep(ns);
  }
}

// one digit of the lazy key switching of one component, on 32-bit halves (inline PTX: the C form
// compiled to ~60% more instructions, moves of zero high words and split products):
//   r += d k  (mod 2^64),   h += d1 s1 + hi32(d1 s0) + hi32(d0 s1)  (= umulhi_apx(d, s), mod 2^64)
__device__ __forceinline__ void v2_ks_acc(u64& r, u64& h, u64 d, u64 k, u64 sh) {
  // r and h stay 64-bit register pairs (the IMAD.WIDE accumulate operands): no pair-building moves
  asm("{\n\t.reg .u32 rl, rh, hl, hh, d0, d1, k0, k1, s0, s1;\n\t"
      "mov.b64 {rl, rh}, %0;\n\tmov.b64 {hl, hh}, %1;\n\t"
      "mov.b64 {d0, d1}, %2;\n\tmov.b64 {k0, k1}, %3;\n\tmov.b64 {s0, s1}, %4;\n\t"
      "mad.lo.cc.u32 rl, d0, k0, rl;\n\t"
      "madc.hi.u32 rh, d0, k0, rh;\n\t"
      "mad.lo.u32 rh, d0, k1, rh;\n\t"
      "mad.lo.u32 rh, d1, k0, rh;\n\t"
      "mad.lo.cc.u32 hl, d1, s1, hl;\n\t"
      "madc.hi.u32 hh, d1, s1, hh;\n\t"
      "mad.hi.cc.u32 hl, d1, s0, hl;\n\t"
      "addc.u32 hh, hh, 0;\n\t"
      "mad.hi.cc.u32 hl, d0, s1, hl;\n\t"
      "addc.u32 hh, hh, 0;\n\t"
      "mov.b64 %0, {rl, rh};\n\tmov.b64 %1, {hl, hh};\n\t}"
      : "+l"(r), "+l"(h)
      : "l"(d), "l"(k), "l"(sh));
}

__device__ __forceinline__ void v2_prefetch_l2(const void* g) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], 128;" ::"l"(g) : "memory");
}

template <int LT, int LOGN, int EPI>
__global__ void __launch_bounds__(V2Warps<EPI>::THREADS, 1)
    ksmac_v2_kernel(KsMacArgs a, const int8_t* __restrict__ w8, V2Geom geo, int units) {
  pdl_trigger();
  constexpr int MMA_WARP = V2Warps<EPI>::MMA;
  constexpr int NTHREADS = V2Warps<EPI>::THREADS;
  extern __shared__ __align__(1024) uint8_t v2_raw[];
  // 1024-aligned base (UMMA descriptors); shared memory is addressed through offsets from this
  // shared-window pointer (32-bit LDS/STS, no generic addressing)
  uint8_t* const sm = v2_raw + ((1024u - (smem_u32(v2_raw) & 1023u)) & 1023u);
  const uint32_t sm_a = smem_u32(sm);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + geo.off_bar);
  uint64_t* const full_bar = bars;            // [S]  producers -> UMMA issuer
  uint64_t* const empty_bar = bars + 4;       // [S]  UMMA completion -> producers
  uint64_t* const tfull = bars + 8;           // [2]  accumulator complete -> epilogue
  uint64_t* const tempty = bars + 10;         // [2]  accumulator read -> UMMA issuer
  uint64_t* const kfull = bars + 12;          // [kb] key buffer landed (cp.async arrivals)
  uint64_t* const kempty = bars + 16;         // [kb] key buffer no longer read
  uint32_t* const s_tmem = reinterpret_cast<uint32_t*>(bars + 20);
#if V2_KBCONST  // v2_geom only ever returns V2_KBMAX key buffers: a compile-time count turns the per-tile
  // `% KB`, `/ KB` (runtime integer divisions: ~150 SASS per tile and thread, 5% of all executed
  // instructions in the ncu SASS view) into multiply-shift pairs
  constexpr int KB = V2_KBMAX;
#else
  const int KB = geo.kb;
#endif

  constexpr bool CN = LOGN > 0;
  const int N = CN ? (1 << LOGN) : (1 << a.logN);
  const int LN = LT * N;
  const int tiles_pl = N / TC_POS;  // position blocks per limb
  const int per_unit = LT * tiles_pl;
  const int ntiles = units * per_unit;
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nk32 = a.Kpad / 32;
  const int nchunks = (nk32 + V2_KS - 1) / V2_KS;
  const int S = geo.S;
  // warp index through a shuffle: ptxas then treats the role branches as warp-uniform (without it
  // every global load in the producers re-materialised its memory descriptor with two R2UR)
#if V2_SHFL
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
#else
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#endif

  // ---- setup (independent of the predecessor kernel: overlaps it under PDL) ----
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full_bar[s], V2_PROD_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EPI);
    }
    for (int b = 0; b < KB; b++) {
      mbar_init(&kfull[b], V2_PROD);
      mbar_init(&kempty[b], V2_PROD_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(V2_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (geo.wres) {  // resident weights: [nk32][4096] canonical K-major tiles (one 128-row M tile)
    const uint4* src = reinterpret_cast<const uint4*>(w8);
    if (geo.half) {
      for (int e = threadIdx.x; e < nk32 * 128; e += NTHREADS)
        *reinterpret_cast<uint4*>(sm + (size_t)e * 16) = __ldg(src + (e >> 7) * 256 + (e & 127));
    } else {
      for (int e = threadIdx.x; e < nk32 * 256; e += NTHREADS)
        *reinterpret_cast<uint4*>(sm + (size_t)e * 16) = __ldg(src + e);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *s_tmem;

  // key words of tile `it` of this CTA (limb l, positions j0 .. j0 + 15, every tap), copied by the
  // producer threads into key buffer it % KB: [tap][x = 2i + comp][val, sh][16]; every producer
  // thread arrives (cp.async.mbarrier.arrive.noinc) on kfull[it % KB] when its copies have landed
  auto issue_keys = [&](int it) {
    const int tile = blockIdx.x + it * gridDim.x;
    const int rem = tile % per_unit;
    const int l = rem / tiles_pl, j0 = (rem % tiles_pl) * TC_POS;
    const uint32_t kb = sm_a + geo.off_key + (uint32_t)(it % KB) * geo.key_bytes;
    const int pieces = a.T * 4 * LT * (TC_POS / 2);
    for (int e = threadIdx.x; e < pieces; e += V2_PROD) {
      const int p2 = e % (TC_POS / 2), r = e / (TC_POS / 2);
      const int sh = r % 2, x = (r / 2) % (2 * LT), tap = r / (4 * LT);
      const u64* key = a.tt.key[tap];
      if (key)
        v2_cp16(kb + (uint32_t)e * 16,
                key + (size_t)sh * 2 * LT * LN + (size_t)x * LN + (size_t)l * N + j0 + 2 * p2);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&kfull[it % KB])) : "memory");
  };
  // L2 prefetch of the input rows of tile `it` at its identity window (C0 and the L digits of every
  // channel, 128 bytes each): the tap windows of a tile are the identity windows of tiles that the
  // other CTAs process at the same time (+-1, +-Wp positions), so each input row reaches L2 once,
  // two tiles before it is read, instead of stalling the first tap that touches it (ncu: 25% L2 misses)
  // (issued by the epilogue warps, which idle most of a tile and have registers to spare)
  auto prefetch_rows = [&](int it) {
    const int tile = blockIdx.x + it * gridDim.x;
    const int z = tile / per_unit, rem = tile % per_unit;
    const int l = rem / tiles_pl, j0 = (rem % tiles_pl) * TC_POS;
    for (int e = (int)threadIdx.x - 32 * V2_PROD_WARPS; e < a.Jcb * (LT + 1); e += 32 * EPI) {
      const int c = e / (LT + 1), k = e % (LT + 1);
      const u64* row = k == 0 ? a.C0 + ((size_t)z * a.Jcb + c) * LN
                              : a.D + (((size_t)z * a.Jcb + c) * LT + (k - 1)) * LN;
      v2_prefetch_l2(row + (size_t)l * N + j0);
    }
  };

  if (warp < V2_PROD_WARPS) {
    // ======================= producers =======================
    if (my_tiles > 0) issue_keys(0);
    if (my_tiles > 1) issue_keys(1);
    uint64_t ident = 0;  // taps without a key (the identity rotation)
    for (int t = 0; t < a.T; t++)
      if (a.tt.key[t] == nullptr) ident |= 1ull << t;
    pdl_wait();  // D, C0 come from PermDecomp
    const int ptid = threadIdx.x;
    const int pos = ptid & 15, tg = ptid >> 4;  // position; terms 4 tg .. 4 tg + 3 of a chunk
    const int ks = tg >> 3, kg = tg & 7;
    const uint32_t off0 = (pos >> 3) * 256 + (kg >> 2) * 128 + (pos & 7) * 16 + (kg & 3) * 4;
    const uint32_t off1 = off0 + 2 * 256;
    struct Term {
      u64 c0, d[LT];
    };
    // ---- load cursor: runs one chunk ahead of the compute, across tile boundaries ----
    int lit = 0, lch = 0, ltap0 = 0, lc0t = 0, ll = 0, lj = 0;
    const u64 *lC0 = nullptr, *lD = nullptr;
    auto cursor_tile = [&](int it) {
      const int tile = blockIdx.x + it * gridDim.x;
      const int z = tile / per_unit, rem = tile % per_unit;
      ll = rem / tiles_pl;
      lj = (rem % tiles_pl) * TC_POS + pos;
      lC0 = a.C0 + (size_t)z * a.Jcb * LN + (size_t)ll * N;
      lD = a.D + (size_t)z * a.Jcb * LT * LN + (size_t)ll * N;
      ltap0 = 0;
      lc0t = tg * 4;
      while (lc0t >= a.Jcb) {
        lc0t -= a.Jcb;
        ltap0++;
      }
    };
    auto load = [&](Term* pr, int& grp) {
      grp = lch * V2_CHUNK + tg * 4 < a.K ? ltap0 : -1;
      if (grp < 0) {  // K padding: zero terms (their weights are zero too), switched as identity
#pragma unroll
        for (int t = 0; t < 4; t++) pr[t].c0 = pr[t].d[0] = 0;
      } else {
        const u64* C0 = lC0 + (size_t)lc0t * LN;
        const u64* D = lD + (size_t)lc0t * (LT * LN);
        if ((ident >> grp) & 1) {  // identity tap: R = (C0, D_{l,l})
#pragma unroll
          for (int t = 0; t < 4; t++) {
            pr[t].c0 = __ldg(C0 + (size_t)t * LN + lj);
            pr[t].d[0] = __ldg(D + (size_t)t * LT * LN + (size_t)ll * LN + lj);
          }
        } else {
          const int jp = galois_perm(lj, a.tt.act[grp], N >> 1);
#pragma unroll
          for (int t = 0; t < 4; t++) {
            pr[t].c0 = __ldg(C0 + (size_t)t * LN + jp);
#pragma unroll
            for (int i = 0; i < LT; i++) pr[t].d[i] = __ldg(D + (size_t)t * LT * LN + (size_t)i * LN + jp);
          }
        }
      }
      lc0t += V2_CHUNK;
      while (lc0t >= a.Jcb) {
        lc0t -= a.Jcb;
        ltap0++;
      }
      if (++lch == nchunks) {
        lch = 0;
        if (++lit < my_tiles) cursor_tile(lit);
      }
    };
    // ---- compute cursor ----
    int cit = 0, cch = 0, gc = 0;
    int st = 0, sround = 0;    // pipeline stage of chunk gc and how often the ring wrapped (no % S)
    uint32_t kbuf = 0;         // sm offset of the current tile's key buffer
    u64 q = 0;
    auto step = [&](Term* cur, int grp, Term* nxt, int& grp_nxt) {
      if (cch == 0) {  // a new tile: its keys must have landed; prefetch those of tile cit + 2
        q = a.lcs.lc[((blockIdx.x + cit * gridDim.x) % per_unit) / tiles_pl].q;
        if (cit + 2 < my_tiles) {  // buffer (cit + 2) % KB was last read by tile cit + 2 - KB
          const int tp = cit + 2 - KB;
          if (tp >= 0) mbar_wait_sleep(&kempty[tp % KB], (tp / KB) & 1, 0);
          issue_keys(cit + 2);
        }
        kbuf = geo.off_key + (uint32_t)(cit % KB) * geo.key_bytes;
        mbar_wait_sleep(&kfull[cit % KB], (cit / KB) & 1, 0);
      }
      if (V2_PF > 0 && gc + V2_PF < my_tiles * nchunks) load(nxt, grp_nxt);
      uint32_t lo0[4], hi0[4], lo1[4], hi1[4];
      if (grp < 0 || ((ident >> grp) & 1)) {  // identity tap (or K padding): R = (C0, D_{l,l})
#pragma unroll
        for (int t = 0; t < 4; t++) {
          lo0[t] = (uint32_t)cur[t].c0;
          hi0[t] = (uint32_t)(cur[t].c0 >> 32);
          lo1[t] = (uint32_t)cur[t].d[0];
          hi1[t] = (uint32_t)(cur[t].d[0] >> 32);
        }
      } else {
        const uint32_t kp = sm_a + kbuf + (uint32_t)pos * 8 + (uint32_t)grp * (4 * LT * TC_POS * 8);
        // lazy Shoup sums with ONE quotient multiply per component: sum_i (d_i w_i - h_i q) =
        // sum_i d_i w_i - (sum_i h_i) q (mod 2^64), h_i = floor(d_i w'_i / 2^64); the true value is
        // c0 + sum of L Shoup products in [0, 2q) < (2L + 1) q < 2^64, so the mod-2^64 result is
        // exact and bit-identical to the per-product form (2 (L - 1) fewer 64-bit products per term).
        // L <= 3: approximate quotients (umulhi_apx, each product in [0, 5q)): the sum stays below
        // (5L + 1) q <= 16 q < 2^64 (hy_params_create enforces q < 2^60); R is any 64-bit value to
        // the byte-plane MAC and congruent mod q, so the outputs are unchanged bit for bit
#if V2_PTX
        if constexpr (LT <= 3) {
          u64 r0[4], r1[4], h0[4], h1[4];
#pragma unroll
          for (int t = 0; t < 4; t++) {
            r0[t] = cur[t].c0;
            r1[t] = h0[t] = h1[t] = 0;
          }
#pragma unroll
          for (int i = 0; i < LT; i++) {
            u64 kv, ksh, av, ash;
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(kv) : "r"(kp + (4 * i) * TC_POS * 8));
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ksh) : "r"(kp + (4 * i + 1) * TC_POS * 8));
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(av) : "r"(kp + (4 * i + 2) * TC_POS * 8));
            asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ash) : "r"(kp + (4 * i + 3) * TC_POS * 8));
#pragma unroll
            for (int t = 0; t < 4; t++) {
              v2_ks_acc(r0[t], h0[t], cur[t].d[i], kv, ksh);
              v2_ks_acc(r1[t], h1[t], cur[t].d[i], av, ash);
            }
          }
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const u64 x0 = r0[t] - h0[t] * q;
            const u64 x1 = r1[t] - h1[t] * q;
            lo0[t] = (uint32_t)x0;
            hi0[t] = (uint32_t)(x0 >> 32);
            lo1[t] = (uint32_t)x1;
            hi1[t] = (uint32_t)(x1 >> 32);
          }
        } else
#endif
        {
        u64 r0[4], r1[4], h0[4], h1[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
          r0[t] = cur[t].c0;
          r1[t] = h0[t] = h1[t] = 0;
        }
#pragma unroll
        for (int i = 0; i < LT; i++) {
          u64 kv, ksh, av, ash;
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(kv) : "r"(kp + (4 * i) * TC_POS * 8));
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ksh) : "r"(kp + (4 * i + 1) * TC_POS * 8));
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(av) : "r"(kp + (4 * i + 2) * TC_POS * 8));
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ash) : "r"(kp + (4 * i + 3) * TC_POS * 8));
#pragma unroll
          for (int t = 0; t < 4; t++) {
            const u64 d = cur[t].d[i];
            r0[t] += d * kv;
            r1[t] += d * av;
            if constexpr (LT <= 3) {
              h0[t] += umulhi_apx(d, ksh);
              h1[t] += umulhi_apx(d, ash);
            } else {
              h0[t] += __umul64hi(d, ksh);
              h1[t] += __umul64hi(d, ash);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
          r0[t] -= h0[t] * q;
          r1[t] -= h1[t] * q;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
          lo0[t] = (uint32_t)r0[t];
          hi0[t] = (uint32_t)(r0[t] >> 32);
          lo1[t] = (uint32_t)r1[t];
          hi1[t] = (uint32_t)(r1[t] >> 32);
        }
        }
      }
      if (cch == nchunks - 1) {  // this warp is done reading the tile's keys
        __syncwarp();
        if (lane == 0) mbar_arrive(&kempty[cit % KB]);
      }
      uint32_t p0[8], p1[8];
      byte_tr4(lo0, p0);
      byte_tr4(hi0, p0 + 4);
      byte_tr4(lo1, p1);
      byte_tr4(hi1, p1 + 4);
      const int s = st;
      if (sround > 0) mbar_wait_sleep(&empty_bar[s], (sround - 1) & 1, 0);
      if (V2_KS * cch + ks < nk32) {
        const uint32_t bb = sm_a + geo.off_b + (uint32_t)s * V2_STAGE_B + (uint32_t)ks * 8192;
#pragma unroll
        for (int b = 0; b < 8; b++) {
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(bb + b * 1024 + off0), "r"(p0[b]) : "memory");
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(bb + b * 1024 + off1), "r"(p1[b]) : "memory");
        }
      }
      if (!geo.wres) {  // streamed weights: K step ws = ptid >> 7 of this chunk, 2 x 16 B per thread
        const int ws = ptid >> 7;
        if (V2_KS * cch + ws < nk32) {
          const uint4* wp = reinterpret_cast<const uint4*>(w8 + (size_t)(V2_KS * cch + ws) * 4096) + (ptid & 127);
          const uint4 wa = __ldg(wp), wb = __ldg(wp + 128);
          const uint32_t ab = sm_a + geo.off_a + (uint32_t)s * V2_STAGE_A + (uint32_t)ws * 4096 + (ptid & 127) * 16;
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ab), "r"(wa.x), "r"(wa.y), "r"(wa.z), "r"(wa.w)
                       : "memory");
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ab + 2048), "r"(wb.x), "r"(wb.y), "r"(wb.z),
                       "r"(wb.w)
                       : "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[s]);
      gc++;
      if (++st == S) {
        st = 0;
        sround++;
      }
      if (++cch == nchunks) {
        cch = 0;
        cit++;
      }
    };
    const int total = my_tiles * nchunks;
#if V2_PF == 0  // no register prefetch: more producer warps fit (latency hidden by warps instead)
    Term buf[4];
    int gb = -1, gdummy = -1;
    if (total > 0) cursor_tile(0);
    for (int g = 0; g < total; g++) {
      load(buf, gb);
      step(buf, gb, buf, gdummy);
    }
#elif V2_PF == 1
    Term bufA[4], bufB[4];
    int gA = -1, gB = -1;
    if (total > 0) {
      cursor_tile(0);
      load(bufA, gA);
    }
    int g = 0;
    for (; g + 1 < total; g += 2) {
      step(bufA, gA, bufB, gB);
      step(bufB, gB, bufA, gA);
    }
    if (g < total) step(bufA, gA, bufB, gB);
#else  // digit loads two chunks ahead (three register buffers)
    Term bufA[4], bufB[4], bufC[4];
    int gA = -1, gB = -1, gC = -1;
    if (total > 0) {
      cursor_tile(0);
      load(bufA, gA);
    }
    if (total > 1) load(bufB, gB);
    int g = 0;
    for (; g + 2 < total; g += 3) {
      step(bufA, gA, bufC, gC);
      step(bufB, gB, bufA, gA);
      step(bufC, gC, bufB, gB);
    }
    if (g < total) step(bufA, gA, bufC, gC);
    if (g + 1 < total) step(bufB, gB, bufA, gA);
#endif
  } else if (warp == MMA_WARP) {
    // ======================= single UMMA issuer =======================
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_s8u8(128, 8 * TC_COLS);
      int s = 0, sround = 0;
      for (int it = 0; it < my_tiles; it++) {
        const int b = it & 1;
        if (it >= 2) mbar_wait_backoff(&tempty[b], ((it >> 1) - 1) & 1, 256);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_t = tmem + (uint32_t)b * 256;
        for (int ch = 0; ch < nchunks; ch++) {
          mbar_wait_backoff(&full_bar[s], sround & 1, 64);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int k2 = 0; k2 < V2_KS && V2_KS * ch + k2 < nk32; k2++) {
            const uint32_t aaddr = geo.wres ? sm_a + (uint32_t)(V2_KS * ch + k2) * (geo.half ? 2048u : 4096u)
                                            : sm_a + geo.off_a + (uint32_t)s * V2_STAGE_A + (uint32_t)k2 * 4096;
            const uint64_t da = umma_desc_kmajor(aaddr);
            const uint64_t db = umma_desc_kmajor(sm_a + geo.off_b + (uint32_t)s * V2_STAGE_B + (uint32_t)k2 * 8192);
            const uint32_t accum = (ch | k2) != 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_t),
                "l"(da), "l"(db), "r"(idesc), "r"(accum));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty_bar[s]))
                       : "memory");
          if (++s == S) {
            s = 0;
            sround++;
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&tfull[b]))
                     : "memory");
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue =======================
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    if (V2_PREFETCH)
      for (int it = 0; it < 3 && it < my_tiles; it++) prefetch_rows(it);
    for (int it = 0; it < my_tiles; it++) {
      if (V2_PREFETCH && it + 3 < my_tiles) prefetch_rows(it + 3);
      const int b = it & 1;
      const int tile = blockIdx.x + it * gridDim.x;
      const int z = tile / per_unit, rem = tile % per_unit;
      const int l = rem / tiles_pl, j0 = (rem % tiles_pl) * TC_POS;
      mbar_wait_backoff(&tfull[b], (it >> 1) & 1, 1000);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (quad * 32 < a.M) {
        const int row = quad * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)b * 256;
#pragma unroll 1
        for (int c0 = 0; c0 < TC_COLS; c0 += 4) {
          uint32_t v[8][4];
#pragma unroll
          for (int pl = 0; pl < 8; pl++)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[pl][0]), "=r"(v[pl][1]), "=r"(v[pl][2]), "=r"(v[pl][3])
                         : "r"(lane_base + (uint32_t)(pl * TC_COLS + c0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          long long lo4[4], hi4[4];
#pragma unroll
          for (int cc = 0; cc < 4; cc++) {
            long long lo = 0, hi = 0;
#pragma unroll
            for (int pl = 0; pl < 4; pl++) lo += (long long)(int32_t)v[pl][cc] << (8 * pl);
#pragma unroll
            for (int pl = 4; pl < 8; pl++) hi += (long long)(int32_t)v[pl][cc] << (8 * (pl - 4));
            lo4[cc] = lo;
            hi4[cc] = hi;
          }
          tc_store4<LT, LOGN>(a, z, row, c0 >> 4, l, j0 + (c0 & 15), hi4, lo4);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(V2_TMEM_COLS));
  }
}
