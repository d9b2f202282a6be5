"""ORACLE (test infrastructure only) — encrypted convolution, step by step.

Follows PAPER.md §2.4 and §3 and the appended Algorithm 1 (CNNLayer / ProposedConv,
PAPER.md:1504-1567 [\\ignore]):
  * packing of a C x H x W input into ciphertexts, zero-padded to a
    power-of-two width (reading R8) — blocks of images in a slot row, or
    row bands with halos when one channel does not fit a slot row (reading R9);
  * padded convolution: f^2 hoisted rotations of each input ciphertext and scalar
    multiply-accumulate; with c_n = 1 this IS the method
    (PAPER.md:784-787);
  * Walsh-Hadamard output-channel packing for c_n = 2: per Eq. (2)
    PMult(ct, [f0, f1]) == CMult(ct, (f0+f1)) + PMult(CMult(ct, (f0-f1)), [1, -1])  (x 2),
    with [k, -k] instead of [1, -1] and the 1/2 dropped (reading R12);
    lazy accumulation then ONE reduction, then PMult by the sign plaintext, then HAdd
    (Algorithm :1545-1550); partial sums of diagonal 1 are aligned by
    HRot (row swap) and added (Algorithm :1556-1567).

The oracle computes each linear combination directly as its value mod q_l (the eager
result).  That lazy accumulation gives the same residues is pinned separately
(tests/test_oracle_conv.py::test_lazy_equals_eager).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import bfv, ring
from .params import (centered, find_k, galois_elt_for_step, h_pn, rowswap_elt)


def next_pow2(x: int) -> int:
    return 1 << (x - 1).bit_length()


@dataclass
class Plan:
    """Layout of one layer (readings R8-R10, R15)."""
    N: int
    batch: int
    Ci: int
    Co: int
    H: int
    W: int
    kh: int
    kw: int
    pad: int
    depthwise: bool
    Hout: int
    Wout: int
    Wp: int
    Hp: int
    mode: str            # "blocks" | "bands"
    per_row: int         # images per slot row (blocks mode)
    Hb: int              # band rows (bands mode)
    Hv: int              # valid output rows per band (bands mode)
    bands: int           # bands per image (bands mode; 1 in blocks mode)
    G: int               # slot-row groups per channel
    cn: int              # channels per ciphertext (1 or 2)
    U: int               # independent units
    Jc: int              # input cts per unit
    Jo: int              # output cts per unit
    taps: List[Tuple[int, int, int]]   # (dy, dx, step)

    @property
    def J(self) -> int:
        return self.U * self.Jc

    @property
    def Jout(self) -> int:
        return self.U * self.Jo


def plan(N: int, batch: int, Ci: int, Co: int, H: int, W: int, kh: int, kw: int, pad: int,
         depthwise: bool = False, force_cn: int = 0) -> Plan:
    row = N // 2
    Hout, Wout = H + 2 * pad - kh + 1, W + 2 * pad - kw + 1
    assert Hout > 0 and Wout > 0
    Wp = next_pow2(W + 2 * pad)
    Hp = next_pow2(H + 2 * pad)
    if Hp * Wp <= row:
        mode, per_row = "blocks", row // (Hp * Wp)
        if force_cn == 4:   # c_n = 4: a channel's group is a quarter of the slots (half a slot row)
            per_row = (row // 2) // (Hp * Wp)
            assert per_row >= 1, "c_n = 4 needs an image block within N/4 slots"
        Hb = Hv = 0
        bands = 1
        G = -(-batch // per_row)
    else:
        assert Wp <= row, "image row wider than a slot row"
        mode, per_row = "bands", 0
        Hb = row // Wp
        Hv = Hb - (kh - 1)
        assert Hv > 0, "band too short for the kernel height"
        bands = -(-Hout // Hv)
        G = batch * bands
    if force_cn:
        cn = force_cn
    else:
        cn = 2 if G <= 1 else 1
    assert cn in (1, 2, 4)
    if depthwise:
        assert Ci == Co
    if cn == 4:   # NEXT-1: Walsh-Hadamard packing of 4 channels, one unit
        assert mode == "blocks" and G == 1 and not depthwise
        U = 1
        Jc = -(-Ci // 4)
        Jo = -(-Co // 4)
    elif cn == 2:
        U = G
        Jc = -(-Ci // 2)
        Jo = Jc if depthwise else -(-Co // 2)
    else:
        U = -(-G // 2)
        Jc = Ci
        Jo = Ci if depthwise else Co
    taps = [(dy, dx, (dy - pad) * Wp + (dx - pad)) for dy in range(kh) for dx in range(kw)]
    return Plan(N, batch, Ci, Co, H, W, kh, kw, pad, depthwise, Hout, Wout, Wp, Hp, mode, per_row,
                Hb, Hv, bands, G, cn, U, Jc, Jo, taps)


def _group_slots(p: Plan, gamma: int):
    """Enumerate (image b, y, x, slot) of the INPUT pixels held by slot-row group gamma."""
    if p.mode == "blocks":
        for bi in range(p.per_row):
            b = gamma * p.per_row + bi
            if b >= p.batch:
                break
            base = bi * p.Hp * p.Wp
            for y in range(p.H):
                for x in range(p.W):
                    yield b, y, x, base + (y + p.pad) * p.Wp + (x + p.pad)
    else:
        b, beta = divmod(gamma, p.bands)
        for r in range(p.Hb):
            y = beta * p.Hv - p.pad + r
            if 0 <= y < p.H:
                for x in range(p.W):
                    yield b, y, x, r * p.Wp + (x + p.pad)


def _group_out_slots(p: Plan, gamma: int):
    """Enumerate (image b, y', x', slot) of the valid OUTPUT pixels of slot-row group gamma."""
    if p.mode == "blocks":
        for bi in range(p.per_row):
            b = gamma * p.per_row + bi
            if b >= p.batch:
                break
            base = bi * p.Hp * p.Wp
            for y in range(p.Hout):
                for x in range(p.Wout):
                    yield b, y, x, base + (y + p.pad) * p.Wp + (x + p.pad)
    else:
        b, beta = divmod(gamma, p.bands)
        for y in range(beta * p.Hv, min((beta + 1) * p.Hv, p.Hout)):
            r = y - beta * p.Hv + p.pad
            for x in range(p.Wout):
                yield b, y, x, r * p.Wp + (x + p.pad)


def _ct_rows_in(p: Plan, ct_index: int):
    """(channel, group) held by the slot groups of input ciphertext ct_index (None = empty): slot
    rows 0 and 1 (c_n <= 2), or for c_n = 4 the four groups c = 2 h + r (slot row r, half h of
    the row) holding channels 4j + c."""
    u, j = divmod(ct_index, p.Jc)
    if p.cn == 4:
        return [(4 * j + c, u) if 4 * j + c < p.Ci else None for c in range(4)]
    if p.cn == 2:
        return [(2 * j + r, u) if 2 * j + r < p.Ci else None for r in range(2)]
    return [(j, 2 * u + r) if 2 * u + r < p.G else None for r in range(2)]


def _ct_rows_out(p: Plan, ct_index: int):
    C = p.Ci if p.depthwise else p.Co
    u, j = divmod(ct_index, p.Jo)
    if p.cn == 4:
        return [(4 * j + c, u) if 4 * j + c < C else None for c in range(4)]
    if p.cn == 2:
        return [(2 * j + r, u) if 2 * j + r < C else None for r in range(2)]
    return [(j, 2 * u + r) if 2 * u + r < p.G else None for r in range(2)]


def _group_base(p: Plan, c: int) -> int:
    """First slot of slot group c (row-major slot vector: row 0 slots, then row 1 slots)."""
    half = p.N // 2
    if p.cn == 4:
        return (c & 1) * half + (c >> 1) * (half // 2)
    return c * half


def pack(p: Plan, x: np.ndarray, t: int) -> np.ndarray:
    """x[batch][Ci][H][W] -> slot vectors [J][N] mod t (row 0 slots, then row 1 slots)."""
    out = np.zeros((p.J, p.N), dtype=np.int64)
    for ci in range(p.J):
        for r, cg in enumerate(_ct_rows_in(p, ci)):
            if cg is None:
                continue
            c, gamma = cg
            base = _group_base(p, r)
            for b, y, xx, s in _group_slots(p, gamma):
                out[ci, base + s] = int(x[b, c, y, xx]) % t
    return out


def unpack(p: Plan, slots: np.ndarray) -> np.ndarray:
    """slot vectors [Jout][N] -> y[batch][Co][Hout][Wout] (raw residues mod t)."""
    C = p.Ci if p.depthwise else p.Co
    y = np.zeros((p.batch, C, p.Hout, p.Wout), dtype=np.int64)
    for ci in range(p.Jout):
        for r, cg in enumerate(_ct_rows_out(p, ci)):
            if cg is None:
                continue
            c, gamma = cg
            base = _group_base(p, r)
            for b, yy, xx, s in _group_out_slots(p, gamma):
                y[b, c, yy, xx] = slots[ci, base + s]
    return y


def plain_conv(x: np.ndarray, Wt: np.ndarray, pad: int, depthwise: bool = False) -> np.ndarray:
    """out[b,o,y,x] = sum_{c,dy,dx} W[o,c,dy,dx] x[b,c,y+dy-pad,x+dx-pad] (cross-correlation,
    zero padding, stride 1; depthwise: c = o) — exact Python-int arithmetic on int64."""
    x = np.asarray(x, dtype=np.int64)
    Wt = np.asarray(Wt, dtype=np.int64)
    B, C, H, Wd = x.shape
    if depthwise:
        kh, kw = Wt.shape[1:]
        Co = C
    else:
        Co, _, kh, kw = Wt.shape
    Hout, Wout = H + 2 * pad - kh + 1, Wd + 2 * pad - kw + 1
    xp = np.zeros((B, C, H + 2 * pad, Wd + 2 * pad), dtype=np.int64)
    xp[:, :, pad:pad + H, pad:pad + Wd] = x
    out = np.zeros((B, Co, Hout, Wout), dtype=np.int64)
    for dy in range(kh):
        for dx in range(kw):
            win = xp[:, :, dy:dy + Hout, dx:dx + Wout]          # [B][C][Hout][Wout]
            if depthwise:
                out += Wt[None, :, dy, dx, None, None] * win
            else:
                out += np.einsum("oc,bchw->bohw", Wt[:, :, dy, dx], win)
    return out


@dataclass
class LayerSetup:
    plan: Plan
    k: int              # Hadamard scale (c_n = 2), 1 for c_n = 1
    scale: int          # output slot scale c_n * k (1 for c_n = 1)
    sign_coeff: int     # centered [k h]_t (c_n = 2)
    h: int
    galois: List[int]   # required Galois elements (taps with step != 0, then row swap)


def hadamard(n: int) -> np.ndarray:
    """Sylvester's Walsh-Hadamard matrix H_n (reading R11): H_1 = [1], H_2m = [[H, H], [H, -H]]."""
    H = np.array([[1]], dtype=np.int64)
    while H.shape[0] < n:
        H = np.block([[H, H], [H, -H]])
    return H


def align_elts(N: int) -> List[int]:
    """c_n = 4 alignment: diagonal d = 2 dh + dr moves slot group c to c xor d by the row swap
    (dr; X -> X^{2N-1}) and the half-row rotation (dh; left rotation by N/4 = X -> X^{3^{N/4}}),
    one automorphism g_d = (2N-1)^dr (3^{N/4})^dh mod 2N for d = 1, 2, 3."""
    gs = []
    for d in (1, 2, 3):
        g = 1
        if d & 1:
            g = g * rowswap_elt(N) % (2 * N)
        if d & 2:
            g = g * galois_elt_for_step(N, N // 4) % (2 * N)
        gs.append(g)
    return gs


def setup(p: Plan, t: int, k: int = 0) -> LayerSetup:
    """S0: h_{t,N} by encoding, k by find_k, sign-plaintext coefficient.
    c_n = 4: no k (the dense Hadamard rows have no small multiple), output scale 4."""
    h = h_pn(t, p.N) if p.cn == 2 else 0
    if p.cn == 2:
        k = k or find_k(t, h)
        sc = centered(k * h, t)
        scale = 2 * k
    elif p.cn == 4:
        k, sc, scale = 1, 0, 4
    else:
        k, sc, scale = 1, 0, 1
    gal = []
    for (_, _, s) in p.taps:
        if s % (p.N // 2) != 0:
            g = galois_elt_for_step(p.N, s)
            if g not in gal:
                gal.append(g)
    if p.cn == 2 and not p.depthwise:
        gal.append(rowswap_elt(p.N))
    if p.cn == 4:
        gal.extend(g for g in align_elts(p.N) if g not in gal)
    return LayerSetup(p, k, scale, sc, h, gal)


def hadamard_row_polys(P: bfv.BFVParams, p: Plan) -> List[List[np.ndarray]]:
    """c_n = 4: the plaintexts of Hadamard rows r = 1..3, slot group c filled with H_4[r][c]
    (Sylvester basis), encoded (oracle/encoding.py) and centered-lifted into every
    limb (reading R14).  Row 0 is the constant 1.  Returns [r - 1][limb] polynomials."""
    from .encoding import encode
    H = hadamard(4)
    half = P.N // 2
    out = []
    for r in (1, 2, 3):
        slots = np.zeros(P.N, dtype=np.int64)
        for c in range(4):
            b = _group_base(p, c)
            slots[b:b + half // 2] = H[r][c] % P.t
        m = encode(slots, P.t, P.N)
        cen = [centered(int(x), P.t) for x in m]
        out.append([np.array([x % q for x in cen], dtype=np.uint64) for q in P.primes])
    return out


def sign_poly(P: bfv.BFVParams, ls: LayerSetup) -> List[np.ndarray]:
    """The [k, -k] plaintext: [k h]_t at X^{N/4} and X^{3N/4},
    centered-lifted into every limb (reading R14)."""
    N = P.N
    out = []
    for q in P.primes:
        s = np.zeros(N, dtype=np.uint64)
        s[N // 4] = ls.sign_coeff % q
        s[3 * N // 4] = ls.sign_coeff % q
        out.append(s)
    return out


def _lincomb(P: bfv.BFVParams, terms) -> np.ndarray:
    """[sum_n w_n * ct_n] mod q_l, per limb (eager: the value lazy accumulation must match)."""
    terms = [(int(w), c) for w, c in terms if int(w) != 0]
    L, N = P.L, P.N
    out = np.zeros((2, L, N), dtype=np.uint64)
    if not terms:
        return out
    for comp in range(2):
        for l, q in enumerate(P.primes):
            hi = np.zeros(N, dtype=np.int64)
            lo = np.zeros(N, dtype=np.int64)
            # exact in int64: |w| <= 2^13 (Hadamard scalars k (w0 + w1), k <= 32), 30-bit digits,
            # <= 2^16 terms (the planner's bound): |sum| < 2^59
            for w, c in terms:
                v = c[comp, l]
                hi += w * (v >> np.uint64(30)).astype(np.int64)
                lo += w * (v & np.uint64((1 << 30) - 1)).astype(np.int64)
            tot = (hi.astype(object) * (1 << 30) + lo.astype(object)) % q
            out[comp, l] = tot.astype(np.uint64)
    return out


def _weight(Wt: np.ndarray, p: Plan, o: int, c: int, tau: int) -> int:
    dy, dx, _ = p.taps[tau]
    if p.depthwise:
        return int(Wt[c, dy, dx]) if o == c and c < p.Ci else 0
    if o >= p.Co or c >= p.Ci:
        return 0
    return int(Wt[o, c, dy, dx])


def rotations(P: bfv.BFVParams, p: Plan, ct_in: np.ndarray, keys: Dict[int, np.ndarray],
              units: Optional[List[int]] = None, cts: Optional[List[int]] = None, hoisted: bool = True
              ) -> Dict[Tuple[int, int], np.ndarray]:
    """R[(ct, tau)]: every input ciphertext (of `units`, or exactly the ciphertexts `cts`) rotated
    by every tap step, hoisted (PermDecomp once per ciphertext, PermAuto per tap;
    PAPER.md:375-377, 1590-1591), or, for the no-hoisting ablation (Fig. 4 (b)), each rotation with
    its own decomposition (bfv.rotate_direct)."""
    R = {}
    units = range(p.U) if units is None else units
    if cts is None:
        cts = [u * p.Jc + j for u in units for j in range(p.Jc)]
    for ci in cts:
        if True:
            digits = bfv.decompose(P, ct_in[ci])
            for tau, (_, _, s) in enumerate(p.taps):
                if s % (p.N // 2) == 0:
                    R[(ci, tau)] = ct_in[ci].copy()
                else:
                    g = galois_elt_for_step(p.N, s)
                    R[(ci, tau)] = (bfv.rotate_hoisted(P, ct_in[ci], digits, g, keys[g]) if hoisted
                                    else bfv.rotate_direct(P, ct_in[ci], g, keys[g]))
    return R


def he_conv(P: bfv.BFVParams, ls: LayerSetup, Wt: np.ndarray, ct_in: np.ndarray,
            keys: Dict[int, np.ndarray], out_cts: Optional[List[int]] = None,
            R: Optional[dict] = None) -> Dict[int, np.ndarray]:
    """CNNLayer(ProposedConv) of Algorithm 1: returns {out ct index: ct}.
    out_cts restricts the computation to a sample of output ciphertexts (only the rotations
    those need are computed)."""
    p = ls.plan
    out_cts = list(range(p.Jout)) if out_cts is None else list(out_cts)
    units = sorted({oc // p.Jo for oc in out_cts})
    if R is None:
        if p.depthwise:     # a depthwise output reads only its own channel's ciphertext
            R = rotations(P, p, ct_in, keys, cts=sorted({oc // p.Jo * p.Jc + oc % p.Jo for oc in out_cts}))
        else:
            R = rotations(P, p, ct_in, keys, units)
    T = len(p.taps)
    res = {}
    S = sign_poly(P, ls) if p.cn == 2 else None
    if p.cn == 4:
        HR = hadamard_row_polys(P, p)
        H4 = hadamard(4)
        G4 = align_elts(P.N)
    for oc in out_cts:
        u, go = divmod(oc, p.Jo)
        if p.cn == 4:
            # ProposedConv of Algorithm 1 with c_n = 4 (PAPER.md:1530-1551 [ign], :565-572): per
            # diagonal d (input group c pairs with output channel 4g + (c xor d)), Hadamard filter
            # scalars s_r = sum_c H_4[r][c] w_c, lazy MAC of s_r R per Hadamard row r, ONE
            # reduction, PMult by the row-r plaintext, HAdd over r; then diagonal d is aligned by
            # HRot with g_d (group c -> c xor d) and added (PAPER.md:574-579 generalised).
            Pd = []
            for d in range(4):
                terms = [[] for _ in range(4)]
                for j in range(p.Jc):
                    for tau in range(T):
                        wc = [_weight(Wt, p, 4 * go + (c ^ d), 4 * j + c, tau) for c in range(4)]
                        Rjt = R[(u * p.Jc + j, tau)]
                        for r in range(4):
                            terms[r].append((int(sum(H4[r][c] * wc[c] for c in range(4))), Rjt))
                A = [_lincomb(P, terms[r]) for r in range(4)]
                part = np.empty((2, P.L, P.N), dtype=np.uint64)
                for comp in range(2):
                    for l, q in enumerate(P.primes):
                        acc = A[0][comp, l].astype(object)
                        for r in (1, 2, 3):
                            acc = acc + ring.nc_mul(HR[r - 1][l], A[r][comp, l], q).astype(object)
                        part[comp, l] = (acc % q).astype(np.uint64)
                Pd.append(part)
            out = Pd[0].copy()
            for d in (1, 2, 3):
                sw = bfv.hrot(P, Pd[d], G4[d - 1], keys[G4[d - 1]])
                for comp in range(2):
                    for l, q in enumerate(P.primes):
                        out[comp, l] = ring.add_mod(out[comp, l], sw[comp, l], q)
            res[oc] = out
            continue
        if p.cn == 1:
            # padded convolution: Out = sum_{c,tau} W[o][c][tau] R_{c,tau}
            terms = []
            chans = [go] if p.depthwise else range(p.Ci)
            for c in chans:
                for tau in range(T):
                    terms.append((_weight(Wt, p, go, c, tau), R[(u * p.Jc + c, tau)]))
            res[oc] = _lincomb(P, terms)
            continue
        # c_n = 2, ProposedConv of Algorithm 1 (PAPER.md:1530-1551 [ign]) per diagonal d (reading
        # R15: slot row r of diagonal d pairs input channel 2j+r with output channel 2g+(r xor d)):
        # the Hadamard filter scalars of (j, tau) are the slot-row weights w_r pushed through the
        # Walsh-Hadamard rows of Eq. (2) ([k, -k] for [1, -1]):
        #   row 0 ([1, 1], the constant plaintext 1):   k (w_0 + w_1)
        #   row 1 ([k, -k], the sign plaintext S):        w_0 - w_1
        # lazily multiplied with the rotated ct and accumulated into partial sum (row, g), then
        # each partial sum is reduced ONCE, multiplied by its Hadamard-row plaintext, and the rows
        # are added (Algorithm).
        diags = [0] if p.depthwise else [0, 1]
        Pd = []
        for d in diags:
            terms = ([], [])
            js = [go] if p.depthwise else range(p.Jc)
            for j in js:
                for tau in range(T):
                    w0 = _weight(Wt, p, 2 * go + (0 ^ d), 2 * j + 0, tau)
                    w1 = _weight(Wt, p, 2 * go + (1 ^ d), 2 * j + 1, tau)
                    Rjt = R[(u * p.Jc + j, tau)]
                    terms[0].append((ls.k * (w0 + w1), Rjt))
                    terms[1].append((w0 - w1, Rjt))
            A0 = _lincomb(P, terms[0])          # reduced partial sum of Hadamard row 0
            A1 = _lincomb(P, terms[1])          # reduced partial sum of Hadamard row 1
            part = np.empty((2, P.L, P.N), dtype=np.uint64)
            for comp in range(2):
                for l, q in enumerate(P.primes):
                    sa1 = ring.nc_mul(S[l], A1[comp, l], q).astype(object)   # PMult by [k, -k]
                    part[comp, l] = ((A0[comp, l].astype(object) + sa1) % q).astype(np.uint64)   # HAdd
            Pd.append(part)
        if p.depthwise:
            res[oc] = Pd[0]
        else:
            g = rowswap_elt(P.N)
            sw = bfv.hrot(P, Pd[1], g, keys[g])
            out = np.empty_like(Pd[0])
            for comp in range(2):
                for l, q in enumerate(P.primes):
                    out[comp, l] = ring.add_mod(Pd[0][comp, l], sw[comp, l], q)
            res[oc] = out
    return res


def decrypt_outputs(P: bfv.BFVParams, ls: LayerSetup, cts: Dict[int, np.ndarray], s) -> Dict[int, np.ndarray]:
    """Decrypt + slot-decode + remove the output scale c_n k (reading R12)."""
    from .encoding import decode_batch
    idx = sorted(cts)
    polys = np.stack([bfv.decrypt(P, cts[i], s) for i in idx])
    slots = decode_batch(polys, P.t, P.N)
    inv = pow(ls.scale, -1, P.t)
    slots = np.mod(slots * inv, P.t)
    return {i: slots[n] for n, i in enumerate(idx)}
