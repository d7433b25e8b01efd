"""ctypes bindings for the C ABI in include/hekan.h.

Shared by the product loader (libhekan_gpu.so, device pointers) and the
test-only oracle loader (oracle/libckks_oracle.so, host pointers): both export
the same symbols with the same semantics.
"""

from __future__ import annotations

import ctypes as C

from .errors import DepthExhausted, DeviceError, LengthMismatch, MissingKey

HK_OK, HK_E_ARG, HK_E_DEPTH, HK_E_LENGTH, HK_E_NOKEY, HK_E_CUDA, HK_E_NOMEM = range(7)

u64p = C.POINTER(C.c_uint64)
i32, u32, u64, dbl, vp = C.c_int32, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p


class HkParams(C.Structure):
    _fields_ = [("log_n", C.c_int32), ("n_q", C.c_int32), ("n_p", C.c_int32),
                ("dnum", C.c_int32), ("q", u64p), ("p", u64p),
                ("psi_q", u64p), ("psi_p", u64p)]


# name -> (restype, argtypes); pointers travel as c_void_p (plain addresses)
SIGNATURES = {
    "hk_ctx_create": (C.c_int, [C.POINTER(HkParams), i32, C.POINTER(vp)]),
    "hk_ctx_destroy": (None, [vp]),
    "hk_last_error": (C.c_char_p, [vp]),
    "hk_set_stream": (C.c_int, [vp, vp]),
    "hk_sync": (C.c_int, [vp]),
    "hk_keygen": (C.c_int, [vp, vp]),
    "hk_add_galois_keys": (C.c_int, [vp, vp, vp, i32]),
    "hk_add_galois_keys_level": (C.c_int, [vp, vp, vp, i32, i32]),
    "hk_has_galois_key": (C.c_int, [vp, u32]),
    "hk_export_key": (C.c_int, [vp, i32, u32, vp]),
    "hk_key_words": (C.c_uint64, [vp, i32]),
    "hk_ntt_fwd": (C.c_int, [vp, vp, i32, i32, i32]),
    "hk_ntt_inv": (C.c_int, [vp, vp, i32, i32, i32]),
    "hk_encode": (C.c_int, [vp, vp, i32, i32, dbl, vp]),
    "hk_encode_diagonals": (C.c_int, [vp, vp, i32, i32, i32, i32, i32, i32, i32, dbl, vp]),
    "hk_encode_const": (C.c_int, [vp, dbl, i32, dbl, vp]),
    "hk_encrypt": (C.c_int, [vp, vp, i32, i32, vp, u64, vp]),
    "hk_decrypt": (C.c_int, [vp, vp, i32, i32, dbl, vp]),
    "hk_add": (C.c_int, [vp, vp, i32, vp, i32, vp, i32]),
    "hk_sub": (C.c_int, [vp, vp, i32, vp, i32, vp, i32]),
    "hk_add_plain": (C.c_int, [vp, vp, i32, vp, i32, i32, i32, vp, i32]),
    "hk_add_const": (C.c_int, [vp, vp, i32, vp, vp, i32]),
    "hk_mul_plain": (C.c_int, [vp, vp, i32, vp, i32, i32, vp, i32]),
    "hk_mul_const": (C.c_int, [vp, vp, i32, vp, vp, i32]),
    "hk_mul": (C.c_int, [vp, vp, i32, vp, i32, vp, i32]),
    "hk_mul_lin": (C.c_int, [vp, vp, i32, vp, i32, vp, i32, vp, vp, i32]),
    "hk_mul_affine": (C.c_int, [vp, vp, i32, vp, i32, i32, vp, vp, i32]),
    "hk_mul2": (C.c_int, [vp, vp, i32, vp, i32, vp, i32, vp, i32, vp, i32]),
    "hk_rescale": (C.c_int, [vp, vp, i32, vp, i32]),
    "hk_rotate": (C.c_int, [vp, vp, i32, u32, vp, i32]),
    "hk_rotate_hoisted": (C.c_int, [vp, vp, i32, vp, i32, vp, i32]),
    "hk_mac_plain": (C.c_int, [vp, vp, vp, i32, i32, i32, i32, vp, i32]),
    "hk_mac_plain_blocks": (C.c_int, [vp, vp, i32, i32, vp, i32, i32, i32, vp, vp, i32]),
    "hk_rotate_sum": (C.c_int, [vp, vp, i32, vp, i32, vp, i32]),
    "hk_version": (C.c_int32, []),
    "hk_launch_count": (C.c_uint64, [vp]),
}

EXPORTED = tuple(SIGNATURES)


def bind(lib: C.CDLL) -> C.CDLL:
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def make_params_struct(params):
    """Build an HkParams (plus the arrays it points into, kept alive)."""
    keep = []

    def arr(vals):
        a = (C.c_uint64 * len(vals))(*[int(v) for v in vals])
        keep.append(a)
        return C.cast(a, u64p)

    st = HkParams(params.log_n, len(params.q), len(params.p), params.dnum,
                  arr(params.q), arr(params.p), arr(params.psi_q), arr(params.psi_p))
    return st, keep


def seed_words(key: bytes) -> C.Array:
    """A 256-bit ChaCha20 seed (32 bytes) as the uint64_t[4] the ABI takes."""
    if len(key) != 32:
        raise ValueError("seeds are 32 bytes")
    return (C.c_uint64 * 4)(*[int.from_bytes(key[8 * i:8 * i + 8], "little") for i in range(4)])


def check(lib, ctx, rc: int, what: str) -> None:
    if rc == HK_OK:
        return
    msg = lib.hk_last_error(ctx)
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg}" if msg else what
    if rc == HK_E_DEPTH:
        raise DepthExhausted(text)
    if rc == HK_E_LENGTH:
        raise LengthMismatch(text)
    if rc == HK_E_NOKEY:
        raise MissingKey(text)
    if rc == HK_E_ARG:
        raise ValueError(text)
    if rc == HK_E_NOMEM:
        raise MemoryError(text)
    raise DeviceError(f"{text} (status {rc})")
