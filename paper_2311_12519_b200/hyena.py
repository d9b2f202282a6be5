"""ctypes binding for libhyena.so (include/hyena.h).  Argument marshalling only: every step of
the encrypted convolution runs in the library's CUDA kernels; nothing here computes.

Device buffers are passed as torch CUDA tensors (dtype torch.uint64, contiguous); host buffers
as numpy arrays.  Every failing call raises HyenaError with hy_last_error()'s message.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

__all__ = ["HyenaError", "hy_conv_shape", "hy_layout", "load_library", "library_path", "hy_last_error",
           "hy_plan_layout", "hy_params_create", "hy_params_destroy", "hy_keys_upload", "hy_encode_weights",
           "hy_weights_layout", "hy_weights_destroy", "hy_conv_eval", "hy_conv_eval_host", "hy_poly_mul",
           "hy_ntt_roundtrip", "hy_rotate", "hy_decrypt_debug", "hy_decrypt_debug_noise", "hy_kernel_launches",
           "hy_weights_set_stage_events", "hy_weights_mac_time", "hy_weights_mac_path", "hy_weights_set_mac_path", "hy_secret_key", "hy_keygen",
           "hy_encrypt", "hy_layout_accounting", "hy_accounting", "hy_noise_estimate", "hy_select_dcmp_base",
           "MAC_PATHS", "layout_dict", "EXPORTED"]

_HERE = os.path.dirname(os.path.abspath(__file__))
HY_MAX_TAPS = 49
HY_MAX_GALOIS = 64
HY_ENOISE = -6  # include/hyena.h: noise budget below 1 bit (hy_decrypt_debug)

# every symbol include/hyena.h declares
EXPORTED = ["hy_last_error", "hy_plan_layout", "hy_params_create", "hy_params_create2", "hy_params_destroy",
            "hy_keys_upload",
            "hy_encode_weights", "hy_weights_layout", "hy_weights_destroy", "hy_conv_eval", "hy_conv_eval_host",
            "hy_poly_mul", "hy_ntt_roundtrip", "hy_rotate", "hy_decrypt_debug", "hy_kernel_launches",
            "hy_weights_set_stage_events", "hy_weights_mac_time", "hy_weights_mac_path", "hy_weights_set_mac_path",
            "hy_secret_key", "hy_keygen", "hy_encrypt", "hy_layout_accounting", "hy_noise_estimate",
            "hy_select_dcmp_base", "hy_decrypt_debug_noise"]

# S2 + S3 kernel choices (include/hyena.h hy_weights_mac_path)
MAC_PATHS = {"thin": 0, "tc_fused": 1, "tc_split": 2, "fp64_fused": 3, "fp64_split": 4, "tc_coef": 5,
             "eager": 6, "direct": 7}


class HyenaError(RuntimeError):
    pass


class hy_conv_shape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in ("Ci", "Co", "H", "W", "kh", "kw", "pad", "stride", "depthwise",
                                                "batch")] + [("k", ctypes.c_int32), ("force_cn", ctypes.c_int32)]


class hy_layout(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_uint32) for n in ("N", "L", "Hout", "Wout", "Wp", "Hp", "mode", "per_row", "Hb", "Hv",
                                                 "bands", "G", "cn", "U", "Jc", "Jo", "J", "Jout", "n_taps")]
                + [("tap_dy", ctypes.c_int32 * HY_MAX_TAPS), ("tap_dx", ctypes.c_int32 * HY_MAX_TAPS),
                   ("tap_step", ctypes.c_int32 * HY_MAX_TAPS)]
                + [(n, ctypes.c_uint32) for n in ("k", "scale", "h")]
                + [("sign_coeff", ctypes.c_int32), ("n_galois", ctypes.c_uint32),
                   ("galois", ctypes.c_uint32 * HY_MAX_GALOIS)])


class hy_accounting(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_uint64) for n in ("input_ct_bytes", "output_ct_bytes", "input_ct_bytes_paper",
                                                 "model_bytes_paper", "model_bytes_conventional",
                                                 "model_bytes_device", "key_bytes")]
                + [("n_keys", ctypes.c_uint32), ("rotations", ctypes.c_uint32), ("coef_macs", ctypes.c_uint64)])


def layout_dict(lay: hy_layout) -> dict:
    d = {n: getattr(lay, n) for n, _ in hy_layout._fields_ if n not in ("tap_dy", "tap_dx", "tap_step", "galois")}
    d["tap_step"] = list(lay.tap_step[:lay.n_taps])
    d["galois"] = list(lay.galois[:lay.n_galois])
    return d


_lib = None


def library_path() -> str:
    # HYENA_LIB: an alternative build of the same library (A/B measurements, tools/abbuild.py)
    return os.environ.get("HYENA_LIB") or os.path.join(_HERE, "libhyena.so")


def load_library() -> ctypes.CDLL:
    """Load the in-tree libhyena.so (built by __graft_entry__.build()); raises if missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not os.path.exists(path):
        raise HyenaError(f"{path} not built: run `python -m paper_2311_12519_b200.build` (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    vp, u32, u64, i32, sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32, ctypes.c_size_t
    sig = {
        "hy_last_error": (ctypes.c_char_p, []),
        "hy_plan_layout": (i32, [u32, u64, ctypes.POINTER(hy_conv_shape), ctypes.POINTER(hy_layout)]),
        "hy_params_create": (i32, [u32, vp, u32, u64, ctypes.c_int, ctypes.POINTER(vp)]),
        "hy_params_create2": (i32, [u32, vp, u32, u64, u32, ctypes.c_int, ctypes.POINTER(vp)]),
        "hy_params_destroy": (None, [vp]),
        "hy_keys_upload": (i32, [vp, u32, vp, vp, ctypes.c_int]),
        "hy_encode_weights": (i32, [vp, ctypes.POINTER(hy_conv_shape), vp, ctypes.POINTER(vp)]),
        "hy_weights_layout": (i32, [vp, ctypes.POINTER(hy_layout)]),
        "hy_weights_destroy": (None, [vp]),
        "hy_conv_eval": (i32, [vp, vp, sz, vp, sz, vp]),
        "hy_conv_eval_host": (i32, [vp, vp, sz, vp, sz, vp]),
        "hy_poly_mul": (i32, [vp, vp, vp, vp, sz, vp]),
        "hy_ntt_roundtrip": (i32, [vp, vp, sz, vp]),
        "hy_rotate": (i32, [vp, vp, u32, vp, sz, vp]),
        "hy_decrypt_debug": (i32, [vp, vp, vp, sz, u32, vp]),
        "hy_decrypt_debug_noise": (i32, [vp, vp, vp, sz, u32, vp, vp]),
        "hy_kernel_launches": (u64, []),
        "hy_weights_set_stage_events": (i32, [vp, vp, u32]),
        "hy_weights_mac_time": (i32, [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(u32)]),
        "hy_weights_mac_path": (i32, [vp, ctypes.POINTER(i32)]),
        "hy_weights_set_mac_path": (i32, [vp, i32]),
        "hy_secret_key": (i32, [vp, u64, vp]),
        "hy_noise_estimate": (i32, [u32, vp, u32, u64, ctypes.POINTER(hy_conv_shape), u32, u32,
                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "hy_select_dcmp_base": (i32, [u32, vp, u32, u64, ctypes.POINTER(hy_conv_shape), u32, ctypes.c_double,
                                      ctypes.POINTER(u32)]),
        "hy_layout_accounting": (i32, [ctypes.POINTER(hy_layout), ctypes.POINTER(hy_conv_shape), u32, u32,
                                       ctypes.POINTER(hy_accounting)]),
        "hy_keygen": (i32, [vp, u64, u32, vp, vp, ctypes.c_int]),
        "hy_encrypt": (i32, [vp, u64, vp, sz, u32, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def hy_last_error() -> str:
    return load_library().hy_last_error().decode()


def _check(status: int, what: str):
    if status != 0:
        raise HyenaError(f"{what} failed ({status}): {hy_last_error()}")


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return int(stream)


def _dev_ptr(t, words: Optional[int] = None) -> int:
    """data_ptr of a contiguous CUDA uint64 tensor (checked)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint64 and t.is_contiguous()):
        raise HyenaError("expected a contiguous CUDA torch.uint64 tensor")
    if words is not None and t.numel() < words:
        raise HyenaError(f"tensor has {t.numel()} words, need {words}")
    return t.data_ptr()


def _shape(**kw) -> hy_conv_shape:
    s = hy_conv_shape()
    for k, v in kw.items():
        setattr(s, k, int(v))
    if "stride" not in kw:
        s.stride = 1
    return s


def hy_plan_layout(N: int, t: int, **shape) -> hy_layout:
    lay = hy_layout()
    s = _shape(**shape)
    _check(load_library().hy_plan_layout(N, t, ctypes.byref(s), ctypes.byref(lay)), "hy_plan_layout")
    return lay


def hy_params_create(N: int, primes: Sequence[int], t: int, device: int = 0, w_dcmp: int = 0) -> int:
    """w_dcmp > 0: decomposition base 2^w_dcmp inside each limb (hy_params_create2)."""
    q = (ctypes.c_uint64 * len(primes))(*[int(x) for x in primes])
    out = ctypes.c_void_p()
    _check(load_library().hy_params_create2(N, q, len(primes), t, w_dcmp, device, ctypes.byref(out)),
           "hy_params_create2")
    return out.value


def hy_params_destroy(p: int):
    load_library().hy_params_destroy(p)


def hy_keys_upload(p: int, galois_elts: Sequence[int], keys):
    """keys: numpy uint64 [n][L][2][L][N] (host) or CUDA uint64 tensor of the same shape."""
    g = (ctypes.c_uint32 * len(galois_elts))(*[int(x) for x in galois_elts])
    if isinstance(keys, np.ndarray):
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        _check(load_library().hy_keys_upload(p, len(galois_elts), g, k.ctypes.data, 0), "hy_keys_upload")
    else:
        _check(load_library().hy_keys_upload(p, len(galois_elts), g, _dev_ptr(keys), 1), "hy_keys_upload")


def hy_encode_weights(p: int, weights: np.ndarray, **shape) -> int:
    """weights: int8 [Co][Ci][kh][kw] (or [C][kh][kw] depthwise); shape: hy_conv_shape fields."""
    Wc = np.ascontiguousarray(weights, dtype=np.int8)
    s = _shape(**shape)
    out = ctypes.c_void_p()
    _check(load_library().hy_encode_weights(p, ctypes.byref(s), Wc.ctypes.data, ctypes.byref(out)),
           "hy_encode_weights")
    return out.value


def hy_weights_layout(w: int) -> hy_layout:
    lay = hy_layout()
    _check(load_library().hy_weights_layout(w, ctypes.byref(lay)), "hy_weights_layout")
    return lay


_RING: dict = {}  # weights handle -> (L, N): the shape check of every eval costs no library call


def hy_weights_destroy(w: int):
    _RING.pop(w, None)
    load_library().hy_weights_destroy(w)


def _ct_words(w: int, shape, what: str) -> int:
    """Words of a [n][2][L][N] ciphertext array for the weights' ring (checked shape)."""
    ring = _RING.get(w)
    if ring is None:
        lay = hy_weights_layout(w)
        ring = _RING[w] = (int(lay.L), int(lay.N))
    if len(shape) != 4 or tuple(shape[1:]) != (2,) + ring:
        raise HyenaError(f"{what}: expected shape [n][2][{ring[0]}][{ring[1]}], got {tuple(shape)}")
    return int(shape[0]) * 2 * ring[0] * ring[1]


def hy_conv_eval(w: int, ct_in, ct_out, J: Optional[int] = None, Jout: Optional[int] = None, stream=None):
    J = ct_in.shape[0] if J is None else J
    Jout = ct_out.shape[0] if Jout is None else Jout
    wi, wo = _ct_words(w, ct_in.shape, "ct_in"), _ct_words(w, ct_out.shape, "ct_out")
    if J > ct_in.shape[0] or Jout > ct_out.shape[0]:
        raise HyenaError("J / Jout exceed the buffers")
    _check(load_library().hy_conv_eval(w, _dev_ptr(ct_in, wi), J, _dev_ptr(ct_out, wo), Jout, _stream(stream)),
           "hy_conv_eval")


def hy_conv_eval_host(w: int, ct_in: np.ndarray, ct_out: np.ndarray, stream=None):
    if not (ct_in.dtype == np.uint64 and ct_out.dtype == np.uint64):
        raise HyenaError("host ciphertexts must be uint64")
    if not (ct_in.flags.c_contiguous and ct_out.flags.c_contiguous):
        raise HyenaError("host ciphertexts must be C-contiguous")
    _ct_words(w, ct_in.shape, "ct_in")
    _ct_words(w, ct_out.shape, "ct_out")
    _check(load_library().hy_conv_eval_host(w, ct_in.ctypes.data, ct_in.shape[0], ct_out.ctypes.data,
                                            ct_out.shape[0], _stream(stream)), "hy_conv_eval_host")


def hy_poly_mul(p: int, a, b, c, stream=None):
    _check(load_library().hy_poly_mul(p, _dev_ptr(a), _dev_ptr(b), _dev_ptr(c), a.shape[0], _stream(stream)),
           "hy_poly_mul")


def hy_ntt_roundtrip(p: int, x, stream=None):
    _check(load_library().hy_ntt_roundtrip(p, _dev_ptr(x), x.shape[0], _stream(stream)), "hy_ntt_roundtrip")


def hy_rotate(p: int, ct_in, galois_elt: int, ct_out, stream=None):
    _check(load_library().hy_rotate(p, _dev_ptr(ct_in), galois_elt, _dev_ptr(ct_out), ct_in.shape[0],
                                    _stream(stream)), "hy_rotate")


def hy_decrypt_debug(p: int, sk: np.ndarray, ct, scale: int) -> np.ndarray:
    """Returns uint64 [n][N] slot values (row 0 then row 1) times scale^{-1} mod t."""
    s = np.ascontiguousarray(sk, dtype=np.int8)
    n, N = ct.shape[0], ct.shape[-1]
    out = np.empty((n, N), dtype=np.uint64)
    _check(load_library().hy_decrypt_debug(p, s.ctypes.data, _dev_ptr(ct), n, scale, out.ctypes.data),
           "hy_decrypt_debug")
    return out


def hy_decrypt_debug_noise(p: int, sk: np.ndarray, ct, scale: int, check: bool = True):
    """(slots [n][N], noise budget bits [n]).  check=False returns both even when the library reports
    HY_ENOISE (a budget below 1 bit); check=True raises HyenaError then."""
    s = np.ascontiguousarray(sk, dtype=np.int8)
    n, N = ct.shape[0], ct.shape[-1]
    out = np.empty((n, N), dtype=np.uint64)
    bud = np.empty(n, dtype=np.float64)
    rc = load_library().hy_decrypt_debug_noise(p, s.ctypes.data, _dev_ptr(ct), n, scale, out.ctypes.data,
                                               bud.ctypes.data)
    if check or rc not in (0, HY_ENOISE):
        _check(rc, "hy_decrypt_debug_noise")
    return out, bud


def hy_kernel_launches() -> int:
    return int(load_library().hy_kernel_launches())


def hy_weights_set_stage_events(w: int, events: Sequence) -> None:
    """events: torch.cuda.Event objects (created with enable_timing=True), at most 5."""
    for e in events:            # torch creates the cudaEvent_t lazily, on its first record()
        if int(e.cuda_event) == 0:
            e.record()
    arr = (ctypes.c_void_p * max(1, len(events)))(*[int(e.cuda_event) for e in events])
    _check(load_library().hy_weights_set_stage_events(w, arr, len(events)), "hy_weights_set_stage_events")


def hy_weights_mac_time(w: int):
    """(summed device ms, launches) of the MAC kernel in the last hy_conv_eval (stage events set)."""
    ms, n = ctypes.c_float(), ctypes.c_uint32()
    _check(load_library().hy_weights_mac_time(w, ctypes.byref(ms), ctypes.byref(n)), "hy_weights_mac_time")
    return float(ms.value), int(n.value)


def hy_weights_mac_path(w: int) -> str:
    """Name of the S2 + S3 kernel path hy_conv_eval uses for these weights (MAC_PATHS)."""
    v = ctypes.c_int32()
    _check(load_library().hy_weights_mac_path(w, ctypes.byref(v)), "hy_weights_mac_path")
    return {i: n for n, i in MAC_PATHS.items()}[v.value]


def hy_weights_set_mac_path(w: int, path: str) -> None:
    _check(load_library().hy_weights_set_mac_path(w, MAC_PATHS[path]), "hy_weights_set_mac_path")


def hy_secret_key(p: int, seed: int, N: int) -> np.ndarray:
    """The ternary secret of `seed` (Philox counter stream, synth/philox.py) as int8 [N]."""
    out = np.empty(N, dtype=np.int8)
    _check(load_library().hy_secret_key(p, seed, out.ctypes.data), "hy_secret_key")
    return out


def hy_keygen(p: int, seed: int, galois_elts: Sequence[int], keys_out=None, upload: bool = True):
    """Switching keys on the GPU; keys_out: CUDA uint64 tensor [n][L][2][L][N] or None."""
    g = (ctypes.c_uint32 * max(1, len(galois_elts)))(*[int(x) for x in galois_elts])
    ptr = _dev_ptr(keys_out) if keys_out is not None else None
    _check(load_library().hy_keygen(p, seed, len(galois_elts), g, ptr, int(upload)), "hy_keygen")


def hy_encrypt(p: int, seed: int, m: np.ndarray, ct_out, first: int = 0, stream=None):
    """Encrypt the plaintext polynomials m (host uint64 [n][N], coefficients < t) into ct_out
    (CUDA uint64 [n][2][L][N]) with encryption counters first .. first + n - 1."""
    mm = np.ascontiguousarray(m, dtype=np.uint64)
    _check(load_library().hy_encrypt(p, seed, mm.ctypes.data, mm.shape[0], first, _dev_ptr(ct_out),
                                     _stream(stream)), "hy_encrypt")


def hy_layout_accounting(lay: hy_layout, L: int, ND: int = 0, **shape) -> dict:
    """Storage / communication accounting of a planned layout (host only; include/hyena.h)."""
    out = hy_accounting()
    s = _shape(**shape)
    _check(load_library().hy_layout_accounting(ctypes.byref(lay), ctypes.byref(s), L, ND or L, ctypes.byref(out)),
           "hy_layout_accounting")
    return {n: getattr(out, n) for n, _ in hy_accounting._fields_}


def hy_noise_estimate(N: int, primes: Sequence[int], t: int, w_dcmp: int = 0, w_max: int = 128, **shape):
    """(log2 noise estimate, log2 budget) of one layer (host only; include/hyena.h)."""
    q = (ctypes.c_uint64 * len(primes))(*[int(x) for x in primes])
    s = _shape(**shape)
    nz, bd = ctypes.c_double(), ctypes.c_double()
    _check(load_library().hy_noise_estimate(N, q, len(primes), t, ctypes.byref(s), w_max, w_dcmp, ctypes.byref(nz),
                                            ctypes.byref(bd)), "hy_noise_estimate")
    return nz.value, bd.value


def hy_select_dcmp_base(N: int, primes: Sequence[int], t: int, margin_bits: float = 4.0, w_max: int = 128,
                        **shape) -> int:
    """The largest decomposition base (fewest key digits) leaving margin_bits of noise margin."""
    q = (ctypes.c_uint64 * len(primes))(*[int(x) for x in primes])
    s = _shape(**shape)
    w = ctypes.c_uint32()
    _check(load_library().hy_select_dcmp_base(N, q, len(primes), t, ctypes.byref(s), w_max, margin_bits,
                                              ctypes.byref(w)), "hy_select_dcmp_base")
    return w.value
