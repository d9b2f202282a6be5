"""GPU client draws: hy_secret_key / hy_keygen / hy_encrypt against the ORACLE
fed with the same Philox draws (synth/philox.py): secret, switching keys and ciphertexts bit for bit,
decryption = the plaintext, and a full-size C4 unit encrypted on the GPU (dense masks and errors)
through hy_conv_eval decrypts to the plain convolution with the noise margin of P12.  Marked gpu."""
import numpy as np
import pytest

import synth
from oracle import bfv, conv
from oracle.params import ntt_primes
from synth import philox

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hy():
    import paper_2311_12519_b200 as pkg
    from paper_2311_12519_b200 import build
    build.build()
    pkg.load_library()
    assert torch.cuda.is_available()
    return pkg


PARAMS = [(1024, ntt_primes(1024, 50, 2)), (4096, synth.PRIMES[(4096, 50)]), (8192, synth.PRIMES[(8192, 60)])]


@pytest.mark.parametrize("N,primes", PARAMS)
def test_secret_keys_and_encryptions_bit_exact(hy, N, primes):
    seed = 0x5EED0000 + N
    P = bfv.BFVParams(N, list(primes), synth.T_PLAIN)
    p = hy.hy_params_create(N, primes, synth.T_PLAIN, 0)
    try:
        s_gpu = hy.hy_secret_key(p, seed, N)
        s = philox.secret(seed, N)
        assert np.array_equal(s_gpu.astype(np.int64), s)
        # switching keys for a tap rotation and the row swap
        elts = [3, 2 * N - 1, pow(3, 17, 2 * N)]
        L = len(primes)
        kd = torch.zeros((len(elts), L, 2, L, N), dtype=torch.uint64, device="cuda")
        hy.hy_keygen(p, seed, elts, kd, upload=True)
        got = kd.cpu().numpy()
        for n, g in enumerate(elts):
            ref = bfv.galois_keygen(P, s, g, philox.key_mask(seed, g, primes, N), philox.key_error(seed, g, L, N))
            assert np.array_equal(got[n], ref), f"key for element {g} differs"
        # encryptions of random plaintexts, counters 5 .. 8
        m = synth.uniform_int(synth.rng(9, "misc", N), 0, synth.T_PLAIN, (4, N)).astype(np.uint64)
        ct = torch.zeros((4, 2, L, N), dtype=torch.uint64, device="cuda")
        hy.hy_encrypt(p, seed, m, ct, first=5)
        got = ct.cpu().numpy()
        for j in range(4):
            ref = bfv.encrypt(P, m[j], s, philox.enc_mask(seed, 5 + j, primes, N), philox.enc_error(seed, 5 + j, N))
            assert np.array_equal(got[j], ref), f"ciphertext {j} differs"
            assert np.array_equal(bfv.decrypt(P, got[j], s), m[j].astype(np.int64))
    finally:
        hy.hy_params_destroy(p)


def test_c4_unit_gpu_encrypted_decrypts(hy):
    """One full C4 unit (64 input cts of the 4096, dense GPU encryptions of the real image bands,
    GPU-generated switching keys) through hy_conv_eval over the whole layer: the unit's 64 outputs
    decrypt (library debug decryption) to 1 * conv mod t at every valid position, and the oracle's
    noise meter shows >= 4 bits of margin on sampled outputs."""
    cfg = synth.configs()["C4"]
    seed = 0xC4C4
    P = bfv.BFVParams(cfg.N, cfg.primes, cfg.t)
    plan = conv.plan(cfg.N, cfg.batch, cfg.Ci, cfg.Co, cfg.H, cfg.W, cfg.kh, cfg.kw, cfg.pad, cfg.depthwise)
    ls = conv.setup(plan, cfg.t)
    x = synth.gen_image(cfg)
    Wt = synth.gen_weights(cfg)
    slots = conv.pack(plan, x, cfg.t)
    from oracle.encoding import encode_batch
    unit = 5
    ins = list(range(unit * plan.Jc, (unit + 1) * plan.Jc))
    m = encode_batch(slots[ins], cfg.t, cfg.N).astype(np.uint64)
    L = len(cfg.primes)
    p = hy.hy_params_create(cfg.N, cfg.primes, cfg.t, 0)
    try:
        hy.hy_keygen(p, seed, ls.galois, None, upload=True)
        s = hy.hy_secret_key(p, seed, cfg.N)
        ct = torch.from_numpy(synth.gen_uniform_cts(cfg.primes, plan.J, cfg.N, cfg.index, stream=21)).cuda()
        enc = torch.zeros((len(ins), 2, L, cfg.N), dtype=torch.uint64, device="cuda")
        hy.hy_encrypt(p, seed, m, enc, first=ins[0])
        ct[ins[0]: ins[-1] + 1] = enc
        w = hy.hy_encode_weights(p, Wt, **cfg.shape_dict())
        try:
            out = torch.zeros((plan.Jout, 2, L, cfg.N), dtype=torch.uint64, device="cuda")
            hy.hy_conv_eval(w, ct, out)
            torch.cuda.synchronize()
            outs = list(range(unit * plan.Jo, (unit + 1) * plan.Jo))
            dec = hy.hy_decrypt_debug(p, s, out[outs[0]: outs[-1] + 1], ls.scale)
        finally:
            hy.hy_weights_destroy(w)
        full = np.zeros((plan.Jout, cfg.N), dtype=np.int64)
        mask = np.zeros((plan.Jout, cfg.N), dtype=np.int64)
        full[outs] = dec.astype(np.int64)
        mask[outs] = 1
        have = conv.unpack(plan, mask).astype(bool)
        got = conv.unpack(plan, full)
        exp = np.mod(conv.plain_conv(x, Wt, plan.pad), cfg.t)
        assert have.sum() > 0
        bad = np.argwhere(have & (got != exp))
        assert bad.size == 0, f"{len(bad)} mismatches, first {bad[:5].tolist()}"
        host = out[outs[0]: outs[0] + 2].cpu().numpy()
        budget = bfv.noise_budget_bits(P)
        for c in host:
            assert budget - bfv.noise_bits(P, c, s.astype(np.int64), bfv.decrypt(P, c, s.astype(np.int64))) >= 4
    finally:
        hy.hy_params_destroy(p)
