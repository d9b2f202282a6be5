"""The counter-based generator of the client draws (synth/philox.py): pinned to the published
Philox4x32-10 known-answer vectors, and its value mappings checked against their definitions with
exact Python integers (CPU)."""
import json
import os

import numpy as np

from synth import philox

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")))


def test_philox_known_answers():
    for v in KAT["vectors"]:
        c = [int(x, 16) for x in v["ctr"]]
        k = [int(x, 16) for x in v["key"]]
        out = philox.philox4x32(c[0], c[1], c[2], c[3], k[0] | (k[1] << 32))
        assert [int(x) for x in out] == [int(x, 16) for x in v["out"]]


def test_mappings_match_definitions():
    g = np.random.default_rng(5)
    x = [g.integers(0, 2**32, 300, dtype=np.uint64) for _ in range(4)]
    for q in (0xFFFFFFFFFFFC001, 0x3FFFFFFFFC001, 97):
        u = philox.uniform_mod(x, q)
        for n in range(300):
            X = int(x[0][n]) | int(x[1][n]) << 32 | int(x[2][n]) << 64 | int(x[3][n]) << 96
            assert int(u[n]) == X * q >> 128
    t = philox.ternary(x)
    e = philox.cbd20(x)
    for n in range(300):
        Y = int(x[0][n]) | int(x[1][n]) << 32
        assert int(t[n]) == (Y * 3 >> 64) - 1
        assert int(e[n]) == bin(Y & 0xFFFFF).count("1") - bin((Y >> 20) & 0xFFFFF).count("1")


def test_distributions_are_plausible():
    s = philox.secret(11, 1 << 14)
    assert set(np.unique(s)) == {-1, 0, 1} and abs(np.mean(s)) < 0.05
    e = philox.enc_error(11, 3, 1 << 14)
    assert abs(np.std(e) - np.sqrt(10)) < 0.15 and np.abs(e).max() <= 20
    a = philox.enc_mask(11, 0, [0xFFFFFFFFFFFC001], 1 << 14)
    assert a.max() < 0xFFFFFFFFFFFC001 and abs(a.astype(float).mean() / 0xFFFFFFFFFFFC001 - 0.5) < 0.02
