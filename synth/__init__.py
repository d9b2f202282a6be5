"""Seeded synthetic-input generators shared by the oracle tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no NTT, no encryption, no
modular products): it only draws seeded integers and names the configurations
of BASELINE.json.  Every random number the method draws (secret key s, errors
e, uniform masks a) is drawn here and passed in as an input, so the oracle and
any later GPU-side generator consume identical integers.

Generator: numpy.random.Generator(numpy.random.Philox(key)) with
key = (SEED_BASE + config_index) * 2^32 + TAG[purpose] * 2^24 + stream, a
counter-based generator (SURVEY.md §8(d) "Generation rules").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

SEED_BASE = 2311125190

TAG = {"x": 1, "W": 2, "sk": 3, "e": 4, "a": 5, "keys": 6, "ct": 7, "misc": 8}


def rng(config_index: int, purpose: str, stream: int = 0) -> np.random.Generator:
    """Counter-based generator for (config, purpose, stream)."""
    assert 0 <= stream < (1 << 24)
    key = ((SEED_BASE + config_index) << 32) + (TAG[purpose] << 24) + stream
    return np.random.Generator(np.random.Philox(key=key))


def uniform_int(g: np.random.Generator, lo: int, hi: int, shape) -> np.ndarray:
    """Uniform integers in [lo, hi) as int64."""
    return g.integers(lo, hi, size=shape, dtype=np.int64)


def ternary(g: np.random.Generator, n: int) -> np.ndarray:
    """Uniform ternary vector in {-1, 0, 1}^n (BASELINE.json configs: 'Ternary uniform secret')."""
    return g.integers(-1, 2, size=n, dtype=np.int64)


def cbd(g: np.random.Generator, shape, eta: int = 20) -> np.ndarray:
    """Centered binomial: sum of eta bits minus sum of eta bits; sigma = sqrt(eta/2) (eta=20: 3.16)."""
    bits = g.integers(0, 2, size=tuple(np.atleast_1d(shape)) + (2, eta), dtype=np.int64)
    return bits[..., 0, :].sum(-1) - bits[..., 1, :].sum(-1)


def uniform_residues(g: np.random.Generator, moduli: List[int], shape) -> np.ndarray:
    """Independent uniform residues in [0, q_l) for each modulus: returns uint64 [..., L, N]-shaped
    array with the limb axis at position -2 (shape = (..., N) given; L inserted before N)."""
    shape = tuple(np.atleast_1d(shape))
    out = np.empty(shape[:-1] + (len(moduli), shape[-1]), dtype=np.uint64)
    for l, q in enumerate(moduli):
        out[..., l, :] = g.integers(0, q, size=shape, dtype=np.uint64)
    return out


# --------------------------------------------------------------------------------------
# BASELINE.json configurations (shapes, ring parameters, value ranges).
# Primes: the largest primes below 2^b with q = 1 mod 2^32 (so q = 1 mod 2N for every N <= 2^31),
# descending (reading R4: "NTT-friendly primes <= b bits").  q = 1 mod 2^32
# makes h q mod 2^64 = h + (h q_hi) 2^32 one 32-bit multiply in every Shoup reduction of the library
# (DESIGN.md §4); the library accepts any NTT-friendly prime and uses that form only when all limbs
# have it.  Both the oracle and the library check primality and q = 1 mod 2N independently.
# --------------------------------------------------------------------------------------

_P60 = [0xFFFFFA000000001, 0xFFFFF8800000001, 0xFFFFF7B00000001, 0xFFFFF6100000001, 0xFFFFF5800000001]
PRIMES = {
    (4096, 50): [0x3FFF300000001, 0x3FFED00000001],
    (4096, 60): _P60[:2],
    (8192, 60): _P60[:3],
    (16384, 60): _P60[:5],
}

T_PLAIN = 65537


@dataclass
class ConvConfig:
    name: str
    index: int              # seed index
    N: int
    primes: List[int]
    batch: int
    Ci: int
    Co: int
    H: int
    W: int
    kh: int
    kw: int
    pad: int
    depthwise: bool
    xrange: Tuple[int, int]  # [lo, hi)
    wrange: Tuple[int, int]
    t: int = T_PLAIN
    force_cn: int = 0
    k: int = 0

    def shape_dict(self) -> Dict[str, int]:
        return dict(Ci=self.Ci, Co=self.Co, H=self.H, W=self.W, kh=self.kh, kw=self.kw, pad=self.pad,
                    stride=1, depthwise=int(self.depthwise), batch=self.batch, k=self.k,
                    force_cn=self.force_cn)


def configs() -> Dict[str, ConvConfig]:
    """BASELINE.json configs[0..4] (C5 split into its depthwise and pointwise layers, per N)."""
    c = {}
    c["C1"] = ConvConfig("C1", 1, 4096, PRIMES[(4096, 50)], 1, 4, 4, 8, 8, 3, 3, 1, False, (-8, 8), (-8, 8))
    c["C2"] = ConvConfig("C2", 2, 8192, PRIMES[(8192, 60)], 1, 16, 16, 32, 32, 3, 3, 1, False,
                         (-128, 128), (-128, 128))
    c["C3a"] = ConvConfig("C3a", 3, 8192, PRIMES[(8192, 60)], 16, 64, 64, 8, 8, 3, 3, 1, False,
                          (-128, 128), (-128, 128))
    c["C3b"] = ConvConfig("C3b", 4, 8192, PRIMES[(8192, 60)], 16, 32, 64, 16, 16, 3, 3, 1, False,
                          (-128, 128), (-128, 128))
    c["C4"] = ConvConfig("C4", 5, 8192, PRIMES[(8192, 60)], 8, 64, 64, 224, 224, 3, 3, 1, False,
                         (-128, 128), (-128, 128))
    for N, L in ((4096, 2), (8192, 3), (16384, 5)):
        pr = PRIMES[(N, 60)][:L]
        c[f"C5dw_{N}"] = ConvConfig(f"C5dw_{N}", 6, N, pr, 32, 512, 512, 14, 14, 3, 3, 1, True,
                                    (-128, 128), (-128, 128))
        c[f"C5pw_{N}"] = ConvConfig(f"C5pw_{N}", 7, N, pr, 32, 512, 512, 14, 14, 1, 1, 0, False,
                                    (-128, 128), (-128, 128))
    return c


def gen_image(cfg: ConvConfig, stream: int = 0) -> np.ndarray:
    """x[batch][Ci][H][W] int64 uniform in cfg.xrange."""
    return uniform_int(rng(cfg.index, "x", stream), cfg.xrange[0], cfg.xrange[1],
                       (cfg.batch, cfg.Ci, cfg.H, cfg.W))


def gen_weights(cfg: ConvConfig, stream: int = 0) -> np.ndarray:
    """W[Co][Ci][kh][kw] (or W[C][kh][kw] depthwise) int8 uniform in cfg.wrange."""
    shape = (cfg.Ci, cfg.kh, cfg.kw) if cfg.depthwise else (cfg.Co, cfg.Ci, cfg.kh, cfg.kw)
    return uniform_int(rng(cfg.index, "W", stream), cfg.wrange[0], cfg.wrange[1], shape).astype(np.int8)


def gen_secret(cfg: ConvConfig) -> np.ndarray:
    return ternary(rng(cfg.index, "sk"), cfg.N)


def gen_uniform_cts(moduli: List[int], n_ct: int, N: int, config_index: int, stream: int = 0) -> np.ndarray:
    """n_ct uniformly random ciphertexts [n_ct][2][L][N] uint64, canonical residues.

    Under RLWE a fresh ciphertext is indistinguishable from this distribution, so
    it is the throughput-benchmark input (bench.py never encrypts: it may not run
    the oracle outside its cpu_baseline leg)."""
    g = rng(config_index, "ct", stream)
    return uniform_residues(g, moduli, (n_ct, 2, N))


def gen_uniform_keys(moduli: List[int], n_elts: int, N: int, config_index: int, stream: int = 0) -> np.ndarray:
    """n_elts uniformly random switching keys [n_elts][L digits][2][L limbs][N] uint64."""
    g = rng(config_index, "keys", 100 + stream)
    L = len(moduli)
    return uniform_residues(g, moduli, (n_elts, L, 2, N))
