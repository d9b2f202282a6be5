"""ORACLE (test infrastructure only) — SIMD (batch) encoding mod t.

A plaintext m in Z_t[X]/(X^N+1) holds N slots: its values at the N primitive
2N-th roots of unity zeta^e (e odd).  Slot order = params.slot_exponents(N)
(2 rows of N/2; reading A1).  Decode is evaluation by its definition,

    v_s = m(zeta^{e_s}) = sum_j m_j zeta^{e_s j}                (mod t),

encode is interpolation written out from the orthogonality of the odd powers,

    m_j = N^{-1} sum_s v_s zeta^{-e_s j}                         (mod t),

both as O(N^2) sums (numpy int64 is exact: terms < 2^34, sums of <= 2^14 terms).
"""
from __future__ import annotations

import numpy as np

from .params import min_primitive_2n_root, slot_exponents

_CHUNK = 256


def _tables(t: int, N: int):
    z = min_primitive_2n_root(t, N)
    M = 2 * N
    zpow = np.array([pow(z, x, t) for x in range(M)], dtype=np.int64)
    e = np.array(slot_exponents(N), dtype=np.int64)
    return zpow, e


def encode_batch(V, t: int, N: int) -> np.ndarray:
    """V[n][N] slot values (any ints; reduced mod t) -> coefficient polys [n][N] in [0, t)."""
    V = np.mod(np.asarray(V, dtype=np.int64), t)
    single = V.ndim == 1
    V = np.atleast_2d(V)
    zpow, e = _tables(t, N)
    M = 2 * N
    n_inv = pow(N, -1, t)
    out = np.empty((V.shape[0], N), dtype=np.int64)
    for j0 in range(0, N, _CHUNK):
        j = np.arange(j0, min(N, j0 + _CHUNK), dtype=np.int64)
        Z = zpow[np.mod(-np.outer(e, j), M)]          # [N slots][chunk]: zeta^{-e_s j}
        acc = np.zeros((V.shape[0], j.size), dtype=np.int64)
        for s0 in range(0, N, 4096):                  # sum over slots, exact in int64
            acc = np.mod(acc + V[:, s0:s0 + 4096] @ Z[s0:s0 + 4096], t)
        out[:, j0:j0 + j.size] = np.mod(acc * n_inv, t)
    return out[0] if single else out


def decode_batch(Mp, t: int, N: int) -> np.ndarray:
    """Coefficient polys [n][N] (any ints; reduced mod t) -> slot values [n][N] in [0, t)."""
    Mp = np.mod(np.asarray(Mp, dtype=np.int64), t)
    single = Mp.ndim == 1
    Mp = np.atleast_2d(Mp)
    zpow, e = _tables(t, N)
    M = 2 * N
    out = np.empty((Mp.shape[0], N), dtype=np.int64)
    jj = np.arange(N, dtype=np.int64)
    for s0 in range(0, N, _CHUNK):
        es = e[s0:s0 + _CHUNK]
        Z = zpow[np.mod(np.outer(jj, es), M)]          # [N coeffs][chunk]: zeta^{e_s j}
        acc = np.zeros((Mp.shape[0], es.size), dtype=np.int64)
        for j0 in range(0, N, 4096):
            acc = np.mod(acc + Mp[:, j0:j0 + 4096] @ Z[j0:j0 + 4096], t)
        out[:, s0:s0 + es.size] = acc
    return out[0] if single else out


def encode(slots, t: int, N: int) -> np.ndarray:
    return encode_batch(np.asarray(slots, dtype=np.int64), t, N)


def decode(poly, t: int, N: int) -> np.ndarray:
    return decode_batch(np.asarray(poly, dtype=np.int64), t, N)
