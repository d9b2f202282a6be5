"""ORACLE (test infrastructure only) — the paper's storage / communication accounting.

  * ciphertext packing: a C x H x W input occupies ceil(C H W / n) ciphertexts
    (PAPER.md:415-418), each 2 polynomials of n 64-bit words;
  * widths zero-padded to a power of two (reading R8);
  * proposed model storage = one 64-bit integer per kernel element (PAPER.md:557-562,
    :876-877), plus one sign polynomial (n words) for the example of PAPER.md:561;
  * conventional storage = one n-word plaintext per kernel element.
These formulas pin the padding rule against Tables 2 and 3 (tests/test_oracle_costmodel.py).
"""
from __future__ import annotations


def next_pow2(x: int) -> int:
    return 1 << (x - 1).bit_length()


def ct_bytes(n: int) -> int:
    return 2 * n * 8


def input_cts(C: int, Wp: int, n: int) -> int:
    return -(-C * Wp * Wp // n)


def input_ct_bytes(C: int, Wp: int, n: int) -> int:
    return input_cts(C, Wp, n) * ct_bytes(n)


def model_bytes_proposed(Ci: int, Co: int, f: int) -> int:
    return f * f * Ci * Co * 8


def storage_proposed_bytes(kernel_elems: int, n: int) -> int:
    return n * 8 + kernel_elems * 8


def storage_conventional_bytes(kernel_elems: int, n: int) -> int:
    return kernel_elems * n * 8


def comm_bytes(H: int, Ci: int, Co: int, f: int, n: int) -> int:
    """Client->server input cts plus server->client output cts (output channels packed the same
    way as inputs), for a same-padded f x f layer."""
    pad = (f - 1) // 2
    Wp = next_pow2(H + 2 * pad)
    return (input_cts(Ci, Wp, n) + input_cts(Co, Wp, n)) * ct_bytes(n)
