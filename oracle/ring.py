"""ORACLE (test infrastructure only) — ring arithmetic in Z_q[X]/(X^N + 1).

PAPER.md:276-280 [\\ignore]: plaintexts in R_p = Z_p[x]/(x^n+1), ciphertexts pairs of
polynomials in R_q = Z_q[x]/(x^n+1).  The only product the oracle has is the
schoolbook negacyclic product (oracle/negacyclic.c); a pure-Python copy exists
for tiny N so the C routine can be pinned against an independent library path
(numpy.polynomial on Python ints) in tests.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "negacyclic.c")
_LIB = os.path.join(_HERE, "_negacyclic.so")
_lock = threading.Lock()
_lib = None


def build_c(force: bool = False) -> str:
    """Compile oracle/negacyclic.c with gcc (plain -O2, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build_c())
            lib.oracle_nc_mul.restype = ctypes.c_int
            lib.oracle_nc_mul.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_uint64, ctypes.c_uint64]
            _lib = lib
    return _lib


def canon(a, q: int) -> np.ndarray:
    """Reduce an integer array (any int dtype or Python ints) to canonical uint64 residues [0, q)."""
    a = np.asarray(a)
    if a.dtype == object:
        return np.array([int(x) % q for x in a], dtype=np.uint64)
    if a.dtype == np.uint64:
        return (a % np.uint64(q)).astype(np.uint64)
    a = a.astype(np.int64)
    return np.mod(a, np.int64(q)).astype(np.uint64) if q < 2**63 else np.array([int(x) % q for x in a],
                                                                                 dtype=np.uint64)


def nc_mul(a, b, q: int) -> np.ndarray:
    """Schoolbook negacyclic product a*b mod (X^N+1, q) (negacyclic.c).  Inputs any integer arrays."""
    a = np.ascontiguousarray(canon(a, q))
    b = np.ascontiguousarray(canon(b, q))
    assert a.shape == b.shape and a.ndim == 1
    c = np.empty_like(a)
    rc = _load().oracle_nc_mul(a.ctypes.data, b.ctypes.data, c.ctypes.data, a.size, q)
    if rc != 0:
        raise ValueError("oracle_nc_mul: bad arguments")
    return c


def nc_mul_py(a, b, q: int) -> list:
    """Pure-Python schoolbook negacyclic product (tiny N only)."""
    a = [int(x) for x in a]
    b = [int(x) for x in b]
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += a[i] * b[j]
            else:
                c[k - n] -= a[i] * b[j]
    return [x % q for x in c]


def automorphism(p, g: int) -> np.ndarray:
    """sigma_g(p)(X) = p(X^g) on a signed integer polynomial (object or int64 array), g odd.

    X^j -> X^{j g mod 2N}; since X^N = -1, an exponent e >= N lands on -X^{e-N}.
    (Rotation via automorphism: PAPER.md:361-371.)"""
    p = np.asarray(p)
    n = p.shape[-1]
    assert g % 2 == 1
    if p.dtype != object:
        assert np.abs(p.astype(np.int64)).max(initial=0) < 2**62
        p = p.astype(np.int64)
    out = np.zeros_like(p)
    for j in range(n):   # written out term by term: X^j -> +-X^{(j g mod 2N) mod N}
        e = (j * g) % (2 * n)
        if e < n:
            out[..., e] = out[..., e] + p[..., j]
        else:
            out[..., e - n] = out[..., e - n] - p[..., j]
    return out


def automorphism_index(n: int, g: int):
    """(dest, sign) arrays so that sigma_g(p)[dest[j]] = sign[j] * p[j] (vectorised helper)."""
    j = np.arange(n, dtype=np.int64)
    e = (j * g) % (2 * n)
    dest = np.where(e < n, e, e - n)
    sign = np.where(e < n, 1, -1)
    return dest, sign


def automorphism_mod(p: np.ndarray, g: int, q: int) -> np.ndarray:
    """sigma_g on a canonical residue polynomial mod q (uint64 in, uint64 out)."""
    n = p.shape[-1]
    dest, sign = automorphism_index(n, g)
    out = np.empty_like(p)
    pos = sign > 0
    out[..., dest[pos]] = p[..., pos]
    negv = p[..., ~pos]
    out[..., dest[~pos]] = np.where(negv == 0, np.uint64(0), np.uint64(q) - negv)
    return out


def add_mod(a, b, q: int) -> np.ndarray:
    return ((a.astype(object) + b.astype(object)) % q).astype(np.uint64)


def sub_mod(a, b, q: int) -> np.ndarray:
    return ((a.astype(object) - b.astype(object)) % q).astype(np.uint64)


def scalar_mul_mod(a, w: int, q: int) -> np.ndarray:
    return ((a.astype(object) * int(w)) % q).astype(np.uint64)
