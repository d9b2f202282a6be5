"""ORACLE — test infrastructure, NOT product code.

A plain, slow, obviously correct CPU implementation of what the Hyena
homomorphic-convolution hot path computes (arXiv 2311.12519, /root/reference/PAPER.md).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import, call, link or execute anything under oracle/.  The CUDA library
(paper_2311_12519_b200/) shares no code, header, table or constant generator
with it; the only shared module is synth/ (seeded integer draws, no arithmetic
of the method).

Modules (each function cites the passage it follows):
  ring      schoolbook negacyclic product mod q (plain C, oracle/negacyclic.c),
            automorphisms X -> X^g on integer polynomials.
  params    primality, NTT-friendly primes, zeta_t, h_{p,n} (by encoding), find_k.
  encoding  SIMD slot encode/decode mod t as O(N^2) interpolation/evaluation.
  bfv       symmetric BFV encrypt/decrypt, Galois keys, hoisted rotation, noise meter.
  conv      layout plan, packing, plain convolution, the HE convolution
            (padded conv for c_n = 1; Walsh-Hadamard packing for c_n = 2).

Pins: see tests/test_oracle_*.py and DESIGN.md "Oracle pins".  Functions whose
result has no independent pin are marked "parity unpinned" in their docstring
(none at present; absolute latencies are unpinned by nature).
"""
