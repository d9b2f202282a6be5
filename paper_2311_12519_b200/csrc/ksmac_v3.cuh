// Fused S2 + S3 with EXACT key-switching products (the default tensor-core path; included by
// kernels.cu after ksmac_v2.cuh, whose V2Warps / mbar helpers it reuses).
//
// Same result as ksmac_tc_kernel / ksmac_v2_kernel: per unit z, MAC row m, column
// (component, limb l, slot position j)
//   B[m][col] = sum_{kk = tau Jc + c} w[m][kk] R_{c,tau}[col],
//   R.c0 = C0_c[perm(j)] + sum_i D_{c,i}[perm(j)] b_{tau,i}[j],   R.c1 = sum_i D_{c,i}[perm(j)] a_{tau,i}[j]
// (hoisted PermAuto), and the Walsh-Hadamard epilogue with ONE reduction per output
// coefficient.  The difference is HOW R is formed: instead of one Shoup
// product per key word (6 IMAD.WIDE + 4 IMAD on the FMA pipe, the kernel's bound), every product
// d b (d, b < 2^60) is taken exactly from 30-bit halves,
//   d b = d0 b0 + (d0 b1 + d1 b0) 2^30 + d1 b1 2^60,    d = d1 2^30 + d0, b = b1 2^30 + b0,
// accumulated over the L digits in three 64-bit columns P0, P1, P2 (each product < 2^60, so
// P0 < (L + 1) 2^60, P1 < 2L 2^60, P2 < L 2^60: no overflow for L <= 7) with 4 IMAD.WIDE.U32
// multiply-adds per product, and R = P0 + P1 2^30 + P2 2^60 < 2^124 is the exact integer (no
// modular reduction at all: the lazy MAC of PAPER.md:718-728 taken one step further).  R is split
// into 16 byte planes (R mod 2^64 and R div 2^64), so the int8 tensor-core contraction stays exact
// (|W x plane| <= 128 * 255 * K < 2^31) and the epilogue recombines S = G0 + G1 2^32 + G2 2^64 +
// G3 2^96 and reduces it with three Shoup products.  Half the FMA-pipe work of the Shoup producers.
//
// Tile = (unit z, limb l, 8 slot positions): 16 planes x 2 components x 8 positions = 256 UMMA
// columns.  Chunk = 6 UMMA K steps (192 terms): each of the 384 producer threads handles 4
// consecutive terms of one position.  Warp roles, TMEM double buffering, key prefetch and the
// single UMMA issuer are those of ksmac_v2_kernel.
#pragma once

constexpr int V3_PROD_WARPS = 12, V3_PROD = V3_PROD_WARPS * 32;
template <int EPI>
struct V3Warps {
  static constexpr int MMA = V3_PROD_WARPS + EPI;
  static constexpr int THREADS = (V3_PROD_WARPS + EPI + 1) * 32;
};

constexpr int V3_POS = 8, V3_KS = 6, V3_CHUNK = 32 * V3_KS;  // 8 positions, 192 terms per chunk
constexpr uint32_t V3_STAGE_B = V3_KS * 8192;                // 256 columns x 32 terms per K step
constexpr uint32_t V3_STAGE_A = V3_KS * 4096;

inline V2Geom v3_geom(int T, int L, int Kpad, size_t smem_max) {
  V2Geom g{};
  const uint32_t wbytes = 128u * (uint32_t)Kpad;
  g.key_bytes = (uint32_t)T * L * 2 * V3_POS * 8;  // [tap][digit][b, a][8 positions] split words
  const uint32_t bar = 256;
  for (int wres = 1; wres >= 0; wres--) {
    for (int S = 3; S >= 2; S--) {
      const uint32_t w = wres ? wbytes : 0;
      const uint32_t per = V3_STAGE_B + (wres ? 0 : V3_STAGE_A);
      const size_t tot = 1024 + (size_t)w + (size_t)S * per + 3 * (size_t)g.key_bytes + bar;
      if (tot <= smem_max) {
        g.S = S;
        g.wres = wres;
        g.off_b = w;
        g.off_a = w + S * V3_STAGE_B;
        g.off_key = g.off_a + (wres ? 0 : S * V3_STAGE_A);
        g.off_bar = g.off_key + 3 * g.key_bytes;
        g.bytes = tot;
        return g;
      }
    }
  }
  g.S = 0;
  return g;
}

// epilogue for 4 consecutive positions j .. j + 3 of one component: this lane holds, per position,
// the recombined plane groups S = G[0] + G[1] 2^32 + G[2] 2^64 + G[3] 2^96 of MAC row `row` (lanes
// row ^ 1 pair up for the Walsh-Hadamard butterflies)
template <int LT, int LOGN>
__device__ __forceinline__ void tc_store4_g(const KsMacArgs& a, int z, int row, int comp, int l, int j,
                                            long long (*G)[4]) {
  const int N = LOGN > 0 ? (1 << LOGN) : (1 << a.logN);
  const size_t LN = (size_t)(LT > 0 ? LT : a.L) * N;
  const LimbConst& c = a.lcs.lc[l];
  auto red = [&](long long h, long long lo) -> u64 {  // h 2^32 + lo mod q, |h| < 2^61, |lo| < 2^62
    const long long h2 = h + (lo >> 32);
    const u64 x = shoup_mul((u64)(h2 + (long long)c.off62), c.c32, c.c32_sh, c.q);
    return csub(csub(x + (u64)(lo & 0xffffffffll), c.two_q), c.q);
  };
  auto red4 = [&](long long g0, long long g1, long long g2, long long g3) -> u64 {
    const u64 t = red(g1, g0), u = red(g3, g2);  // S = t + u 2^64 (mod q)
    return csub(csub(t + shoup_mul(u, c.c64, c.c64_sh, c.q), c.two_q), c.q);
  };
  u64 v[4];
  if (a.cn == 1) {
    if (row >= a.M) return;
#pragma unroll
    for (int i = 0; i < 4; i++) v[i] = red4(G[i][0], G[i][1], G[i][2], G[i][3]);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(a.out + ((size_t)(z * a.M + row) * 2 + comp) * LN + (size_t)l * N + j);
    dst[0] = make_ulonglong2(v[0], v[1]);
    dst[1] = make_ulonglong2(v[2], v[3]);
    return;
  }
  long long H[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int g = 0; g < 4; g++) H[i][g] = __shfl_xor_sync(0xffffffffu, G[i][g], 1);
  if ((row & 1) || row >= a.M) return;
  const long long k = a.kscale;
  u64 a0[4], a1[4];
#pragma unroll
  for (int i = 0; i < 4; i++) {  // Walsh-Hadamard on the exact accumulators (Eq. 2), per plane group
    a0[i] = red4(k * (G[i][0] + H[i][0]), k * (G[i][1] + H[i][1]), k * (G[i][2] + H[i][2]), k * (G[i][3] + H[i][3]));
    a1[i] = red4(G[i][0] - H[i][0], G[i][1] - H[i][1], G[i][2] - H[i][2], G[i][3] - H[i][3]);
  }
  const size_t at = ((size_t)(z * (a.M / 2) + row / 2) * 2 + comp) * LN + (size_t)l * N + j;
  const ulonglong2* sp = reinterpret_cast<const ulonglong2*>(a.sign + (size_t)l * N + j);
  const ulonglong2* ssp = reinterpret_cast<const ulonglong2*>(a.sign + LN + (size_t)l * N + j);
  const ulonglong2 s01 = __ldg(sp), s23 = __ldg(sp + 1), h01 = __ldg(ssp), h23 = __ldg(ssp + 1);
  const u64 sg[4] = {s01.x, s01.y, s23.x, s23.y}, sgs[4] = {h01.x, h01.y, h23.x, h23.y};
#pragma unroll
  for (int i = 0; i < 4; i++) v[i] = csub(csub(a0[i] + shoup_mul(a1[i], sg[i], sgs[i], c.q), c.two_q), c.q);
  reinterpret_cast<ulonglong2*>(a.out + at)[0] = make_ulonglong2(v[0], v[1]);
  reinterpret_cast<ulonglong2*>(a.out + at)[1] = make_ulonglong2(v[2], v[3]);
}

// 32 x 32 + 64 -> 64-bit multiply-add: one IMAD.WIDE.U32
__device__ __forceinline__ u64 madw(uint32_t a, uint32_t b, u64 c) {
  u64 d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

template <int LT, int LOGN, int EPI>
__global__ void __launch_bounds__(V3Warps<EPI>::THREADS, 1)
    ksmac_v3_kernel(KsMacArgs a, const int8_t* __restrict__ w8, V2Geom geo, int units) {
  pdl_trigger();
  constexpr int MMA_WARP = V3Warps<EPI>::MMA;
  constexpr int NTHREADS = V3Warps<EPI>::THREADS;
  extern __shared__ __align__(1024) uint8_t v3_raw[];
  uint8_t* const sm = v3_raw + ((1024u - (smem_u32(v3_raw) & 1023u)) & 1023u);
  const uint32_t sm_a = smem_u32(sm);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + geo.off_bar);
  uint64_t* const full_bar = bars;            // [S]  producers -> UMMA issuer
  uint64_t* const empty_bar = bars + 4;       // [S]  UMMA completion -> producers
  uint64_t* const tfull = bars + 8;           // [2]  accumulator complete -> epilogue
  uint64_t* const tempty = bars + 10;         // [2]  accumulator read -> UMMA issuer
  uint64_t* const kfull = bars + 12;          // [3]  key buffer landed (cp.async arrivals)
  uint64_t* const kempty = bars + 15;         // [3]  key buffer no longer read
  uint32_t* const s_tmem = reinterpret_cast<uint32_t*>(bars + 18);

  constexpr bool CN = LOGN > 0;
  const int N = CN ? (1 << LOGN) : (1 << a.logN);
  const int LN = LT * N;
  const int tiles_pl = N / V3_POS;
  const int per_unit = LT * tiles_pl;
  const int ntiles = units * per_unit;
  const int my_tiles = (int)blockIdx.x < ntiles ? (ntiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int nk32 = a.Kpad / 32;
  const int nchunks = (nk32 + V3_KS - 1) / V3_KS;
  const int S = geo.S;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // warp-uniform for ptxas (ksmac_v2.cuh)

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) {
      mbar_init(&full_bar[s], V3_PROD_WARPS);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; b++) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], EPI);
    }
    for (int b = 0; b < 3; b++) {
      mbar_init(&kfull[b], V3_PROD);
      mbar_init(&kempty[b], V3_PROD_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(V2_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (geo.wres) {
    const uint4* src = reinterpret_cast<const uint4*>(w8);
    for (int e = threadIdx.x; e < nk32 * 256; e += NTHREADS)
      *reinterpret_cast<uint4*>(sm + (size_t)e * 16) = __ldg(src + e);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *s_tmem;

  // split key words of tile `it` (limb l, positions j0 .. j0 + 7): [tap][digit i][b, a][8] from the
  // key's third block; every producer thread arrives on kfull[it % 3] when its copies landed
  auto issue_keys = [&](int it) {
    const int tile = blockIdx.x + it * gridDim.x;
    const int rem = tile % per_unit;
    const int l = rem / tiles_pl, j0 = (rem % tiles_pl) * V3_POS;
    const uint32_t kb = sm_a + geo.off_key + (uint32_t)(it % 3) * geo.key_bytes;
    const int pieces = a.T * LT * 2 * (V3_POS / 2);
    for (int e = threadIdx.x; e < pieces; e += V3_PROD) {
      const int p2 = e % (V3_POS / 2), r = e / (V3_POS / 2);  // r = (tap L + i) 2 + comp
      const int comp = r % 2, i = (r / 2) % LT, tap = r / (2 * LT);
      const u64* key = a.tt.key[tap];
      if (key)
        v2_cp16(kb + (uint32_t)e * 16,
                key + (size_t)4 * LT * LN + (size_t)(2 * i + comp) * LN + (size_t)l * N + j0 + 2 * p2);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&kfull[it % 3])) : "memory");
  };

  if (warp < V3_PROD_WARPS) {
    // ======================= producers =======================
    if (my_tiles > 0) issue_keys(0);
    if (my_tiles > 1) issue_keys(1);
    uint64_t ident = 0;
    for (int t = 0; t < a.T; t++)
      if (a.tt.key[t] == nullptr) ident |= 1ull << t;
    pdl_wait();  // D, C0 come from PermDecomp
    const int ptid = threadIdx.x;
    const int pos = ptid & 7, tg = ptid >> 3;  // position; terms 4 tg .. 4 tg + 3 of a chunk
    const int ks = tg >> 3, kg = tg & 7;
    // plane b, component c: K-major core-matrix group 2b + c, row pos, 4 bytes at term 4 kg
    const uint32_t offp = (kg >> 2) * 128 + pos * 16 + (kg & 3) * 4;
    struct Term {
      u64 c0, d[LT];
    };
    int lit = 0, lch = 0, ltap0 = 0, lc0t = 0, ll = 0, lj = 0;
    const u64 *lC0 = nullptr, *lD = nullptr;
    auto cursor_tile = [&](int it) {
      const int tile = blockIdx.x + it * gridDim.x;
      const int z = tile / per_unit, rem = tile % per_unit;
      ll = rem / tiles_pl;
      lj = (rem % tiles_pl) * V3_POS + pos;
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
      grp = lch * V3_CHUNK + tg * 4 < a.K ? ltap0 : -1;
      if (grp >= 0) {
        const u64* C0 = lC0 + (size_t)lc0t * LN;
        const u64* D = lD + (size_t)lc0t * (LT * LN);
        if ((ident >> grp) & 1) {
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
      lc0t += V3_CHUNK;
      while (lc0t >= a.Jcb) {
        lc0t -= a.Jcb;
        ltap0++;
      }
      if (++lch == nchunks) {
        lch = 0;
        if (++lit < my_tiles) cursor_tile(lit);
      }
    };
    int cit = 0, cch = 0, gc = 0;
    auto step = [&](Term* cur, int grp, Term* nxt, int& grp_nxt) {
      if (cch == 0) {  // a new tile: prefetch the keys of tile cit + 2, wait for its own
        if (cit + 2 < my_tiles) {  // buffer (cit + 2) % 3 was last read by tile cit - 1
          if (cit >= 1) mbar_wait(&kempty[(cit + 2) % 3], ((cit - 1) / 3) & 1);
          issue_keys(cit + 2);
        }
        mbar_wait(&kfull[cit % 3], (cit / 3) & 1);
      }
      if (gc + 1 < my_tiles * nchunks) load(nxt, grp_nxt);
      // w[t][k]: 32-bit words of term t: k = 0..3 -> R.c0 bits 0-31, 32-63, 64-95, 96-127; 4..7 -> R.c1
      uint32_t w[4][8];
      if (grp < 0) {
#pragma unroll
        for (int t = 0; t < 4; t++)
#pragma unroll
          for (int k = 0; k < 8; k++) w[t][k] = 0;
      } else if ((ident >> grp) & 1) {
#pragma unroll
        for (int t = 0; t < 4; t++) {
          w[t][0] = (uint32_t)cur[t].c0;
          w[t][1] = (uint32_t)(cur[t].c0 >> 32);
          w[t][2] = w[t][3] = 0;
          w[t][4] = (uint32_t)cur[t].d[0];
          w[t][5] = (uint32_t)(cur[t].d[0] >> 32);
          w[t][6] = w[t][7] = 0;
        }
      } else {
        const uint32_t kp = sm_a + geo.off_key + (uint32_t)(cit % 3) * geo.key_bytes + (uint32_t)pos * 8 +
                            (uint32_t)grp * (LT * 2 * V3_POS * 8);
        uint32_t kb0[LT], kb1[LT], ka0[LT], ka1[LT];
#pragma unroll
        for (int i = 0; i < LT; i++) {
          u64 kb, ka;
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(kb) : "r"(kp + (2 * i) * V3_POS * 8));
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(ka) : "r"(kp + (2 * i + 1) * V3_POS * 8));
          kb0[i] = (uint32_t)kb;
          kb1[i] = (uint32_t)(kb >> 32);
          ka0[i] = (uint32_t)ka;
          ka1[i] = (uint32_t)(ka >> 32);
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
          u64 p0 = cur[t].c0, p1 = 0, p2 = 0, r0 = 0, r1 = 0, r2 = 0;
#pragma unroll
          for (int i = 0; i < LT; i++) {
            const uint32_t d0 = (uint32_t)cur[t].d[i] & 0x3FFFFFFFu, d1 = (uint32_t)(cur[t].d[i] >> 30);
            p0 = madw(d0, kb0[i], p0);
            p1 = madw(d0, kb1[i], p1);
            p1 = madw(d1, kb0[i], p1);
            p2 = madw(d1, kb1[i], p2);
            r0 = madw(d0, ka0[i], r0);
            r1 = madw(d0, ka1[i], r1);
            r1 = madw(d1, ka0[i], r1);
            r2 = madw(d1, ka1[i], r2);
          }
          // R = P0 + P1 2^30 + P2 2^60 exactly (< 2^124), as 128 bits
          const u128 R0 = (u128)p0 + ((u128)p1 << 30) + ((u128)p2 << 60);
          const u128 R1 = (u128)r0 + ((u128)r1 << 30) + ((u128)r2 << 60);
          w[t][0] = (uint32_t)R0;
          w[t][1] = (uint32_t)(R0 >> 32);
          w[t][2] = (uint32_t)(R0 >> 64);
          w[t][3] = (uint32_t)(R0 >> 96);
          w[t][4] = (uint32_t)R1;
          w[t][5] = (uint32_t)(R1 >> 32);
          w[t][6] = (uint32_t)(R1 >> 64);
          w[t][7] = (uint32_t)(R1 >> 96);
        }
      }
      if (cch == nchunks - 1) {  // this warp is done reading the tile's keys
        __syncwarp();
        if (lane == 0) mbar_arrive(&kempty[cit % 3]);
      }
      // byte transposes: plane 4k + b of component c gets byte b of word 4c + k of the 4 terms
      uint32_t pl[8][4];
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint32_t x[4] = {w[0][k], w[1][k], w[2][k], w[3][k]};
        byte_tr4(x, pl[k]);
      }
      const int s = gc % S;
      if (gc >= S) mbar_wait(&empty_bar[s], ((gc / S) - 1) & 1);
      if (V3_KS * cch + ks < nk32) {
        const uint32_t bb = sm_a + geo.off_b + (uint32_t)s * V3_STAGE_B + (uint32_t)ks * 8192 + offp;
#pragma unroll
        for (int c = 0; c < 2; c++)
#pragma unroll
          for (int k = 0; k < 4; k++)
#pragma unroll
            for (int b = 0; b < 4; b++)  // plane 4k + b, component c: core group 2 (4k + b) + c
              asm volatile("st.shared.u32 [%0], %1;" ::"r"(bb + (uint32_t)(2 * (4 * k + b) + c) * 256),
                           "r"(pl[4 * c + k][b])
                           : "memory");
      }
      if (!geo.wres) {  // streamed weights: K steps ws = ptid >> 6 of this chunk, 16 + 16 B per thread
        const int ws = ptid >> 6;
        if (V3_KS * cch + ws < nk32) {
          const uint4* wp = reinterpret_cast<const uint4*>(w8 + (size_t)(V3_KS * cch + ws) * 4096) + (ptid & 63) * 4;
          const uint32_t ab = sm_a + geo.off_a + (uint32_t)s * V3_STAGE_A + (uint32_t)ws * 4096 + (ptid & 63) * 64;
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const uint4 wv = __ldg(wp + e);
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ab + e * 16), "r"(wv.x), "r"(wv.y), "r"(wv.z),
                         "r"(wv.w)
                         : "memory");
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[s]);
      gc++;
      if (++cch == nchunks) {
        cch = 0;
        cit++;
      }
    };
    const int total = my_tiles * nchunks;
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
  } else if (warp == MMA_WARP) {
    // ======================= single UMMA issuer =======================
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_s8u8(128, 256);
      int gc = 0;
      for (int it = 0; it < my_tiles; it++) {
        const int b = it & 1;
        if (it >= 2) mbar_wait_sleep(&tempty[b], ((it >> 1) - 1) & 1, 64);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc_t = tmem + (uint32_t)b * 256;
        for (int ch = 0; ch < nchunks; ch++, gc++) {
          const int s = gc % S;
          mbar_wait_sleep(&full_bar[s], (gc / S) & 1, 32);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          for (int k2 = 0; k2 < V3_KS && V3_KS * ch + k2 < nk32; k2++) {
            const uint32_t aaddr = geo.wres ? sm_a + (uint32_t)(V3_KS * ch + k2) * 4096
                                            : sm_a + geo.off_a + (uint32_t)s * V3_STAGE_A + (uint32_t)k2 * 4096;
            const uint64_t da = umma_desc_kmajor(aaddr);
            const uint64_t db = umma_desc_kmajor(sm_a + geo.off_b + (uint32_t)s * V3_STAGE_B + (uint32_t)k2 * 8192);
            const uint32_t accum = (ch | k2) != 0;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_t),
                "l"(da), "l"(db), "r"(idesc), "r"(accum));
          }
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty_bar[s]))
                       : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&tfull[b]))
                     : "memory");
      }
    }
    __syncwarp();
  } else {
    // ======================= epilogue =======================
    const int quad = warp & 3;
    for (int it = 0; it < my_tiles; it++) {
      const int b = it & 1;
      const int tile = blockIdx.x + it * gridDim.x;
      const int z = tile / per_unit, rem = tile % per_unit;
      const int l = rem / tiles_pl, j0 = (rem % tiles_pl) * V3_POS;
      mbar_wait_sleep(&tfull[b], (it >> 1) & 1, 256);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (quad * 32 < a.M) {
        const int row = quad * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)b * 256;
#pragma unroll 1
        for (int grp4 = 0; grp4 < 4; grp4++) {  // (component, 4 positions)
          const int comp = grp4 >> 1, p0 = (grp4 & 1) * 4;
          long long G[4][4];
#pragma unroll
          for (int gq = 0; gq < 4; gq++) {  // plane groups 4 gq .. 4 gq + 3
            uint32_t v[4][4];
#pragma unroll
            for (int pb = 0; pb < 4; pb++) {
              const int plane = 4 * gq + pb;  // TMEM column = 8 (2 plane + comp) + position
              asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[pb][0]), "=r"(v[pb][1]), "=r"(v[pb][2]), "=r"(v[pb][3])
                           : "r"(lane_base + (uint32_t)(8 * (2 * plane + comp) + p0)));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int cc = 0; cc < 4; cc++) {
              long long s = 0;
#pragma unroll
              for (int pb = 0; pb < 4; pb++) s += (long long)(int32_t)v[pb][cc] << (8 * pb);
              G[cc][gq] = s;
            }
          }
          tc_store4_g<LT, LOGN>(a, z, row, comp, l, j0 + p0, G);
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
