/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 *
 * Schoolbook negacyclic product in Z_q[X]/(X^N + 1), written out from the
 * definition of the ring the paper works in (PAPER.md:276-280 [\ignore], the
 * ring R_q = Z_q[x]/(x^n+1) of BFV; PAPER.md:341-350 PMult/CMult):
 *
 *     c_k = sum_{i+j = k} a_i b_j  -  sum_{i+j = k+N} a_i b_j      (mod q)
 *
 * No NTT, no Montgomery/Barrett/Shoup, no lazy tricks beyond the following
 * exactness device: products (< q^2 <= 2^124) are summed in unsigned __int128
 * accumulators that are reduced with the C '%' operator before they can
 * overflow.  Zero coefficients of `a` are skipped (the terms are zero), which
 * makes products with the sparse sign plaintext and with the
 * ternary secret cheap without changing the definition.
 *
 * Inputs must be canonical: 0 <= a_i, b_j < q, 2 <= q < 2^63.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static unsigned bitlen(uint64_t x) {
  unsigned b = 0;
  while (x) { b++; x >>= 1; }
  return b;
}

/* c = a * b mod (X^N + 1, q).  c may not alias a or b.  Returns 0, or -1 on bad args. */
int oracle_nc_mul(const uint64_t* a, const uint64_t* b, uint64_t* c, uint64_t N, uint64_t q) {
  if (N == 0 || q < 2 || bitlen(q) > 63) return -1;
  u128* pos = (u128*)calloc(N, sizeof(u128));
  u128* neg = (u128*)calloc(N, sizeof(u128));
  if (!pos || !neg) { free(pos); free(neg); return -1; }
  /* each product < 2^(2*bits); 2^(127 - 2*bits) of them fit below 2^127 */
  unsigned bits = bitlen(q - 1);
  uint64_t batch = (2 * bits >= 127) ? 1 : ((uint64_t)1 << (127 - 2 * bits));
  if (batch > (1u << 20)) batch = 1u << 20;
  uint64_t since = 0;
  for (uint64_t i = 0; i < N; i++) {
    uint64_t ai = a[i];
    if (ai == 0) continue;
    for (uint64_t j = 0; j < N - i; j++) pos[i + j] += (u128)ai * b[j];       /* i + j <  N */
    for (uint64_t j = N - i; j < N; j++) neg[i + j - N] += (u128)ai * b[j];   /* X^N = -1   */
    if (++since == batch) {
      for (uint64_t k = 0; k < N; k++) { pos[k] %= q; neg[k] %= q; }
      since = 0;
    }
  }
  for (uint64_t k = 0; k < N; k++) {
    uint64_t p = (uint64_t)(pos[k] % q), n = (uint64_t)(neg[k] % q);
    c[k] = (p >= n) ? (p - n) : (p + (q - n));
  }
  free(pos);
  free(neg);
  return 0;
}
